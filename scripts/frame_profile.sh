#!/bin/bash
# Launch table of one config-3 frame (view $1, default 2) under ncu -> gpurun_out/frame_v$1.txt
V=${1:-2}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --nvtx --nvtx-include "frame/" \
  --clock-control none --csv --log-file gpurun_out/frame_v$V.csv python scripts/profile_frame.py cfg3 $V > /dev/null 2>&1
python scripts/frame_kernels.py gpurun_out/frame_v$V.csv | tee gpurun_out/frame_v$V.txt
