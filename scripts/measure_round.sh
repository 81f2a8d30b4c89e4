#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), launch lists and full ncu captures.
# Outputs land in gpurun_out/; scripts/summarise_round.py copies the judged summaries to profiles/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -c 300 gpurun_out/bench_ref.json
# launch list of the bench command itself (cold-cache, serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# per-view launch tables with DRAM bytes
for v in 0 1 2; do ./scripts/frame_profile.sh $v > /dev/null 2>&1; done
# full sections: the blend on all three views, the other top kernels on the far view
timeout 900 ncu --set full --import-source on --nvtx --nvtx-include "frame/" -k regex:k_blend -c 3 --clock-control none \
    -o gpurun_out/ncu_blend python scripts/profile_frame.py cfg3 all > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --nvtx --nvtx-include "frame/" \
    -k regex:"k_cull|k_project|k_bentry_emit" -c 4 --clock-control none \
    -o gpurun_out/ncu_top python scripts/profile_frame.py cfg3 2 > /dev/null 2>&1
# the sort: one depth upsweep, the last depth downsweep and both block-list downsweeps
timeout 900 ncu --set full --import-source on --nvtx --nvtx-include "frame/" \
    -k regex:"k_radix_down" --launch-skip 3 -c 3 --clock-control none \
    -o gpurun_out/ncu_sort python scripts/profile_frame.py cfg3 2 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --nvtx --nvtx-include "frame/" \
    -k regex:"k_radix_up" -c 1 --clock-control none \
    -o gpurun_out/ncu_up python scripts/profile_frame.py cfg3 2 > /dev/null 2>&1
ls gpurun_out
