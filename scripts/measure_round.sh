#!/bin/bash
# One GPU session: tests, bench (both arms), launch list and full ncu captures.
# Outputs land in gpurun_out/; the summaries worth keeping are copied to profiles/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv &
CLK=$!
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json
kill $CLK 2>/dev/null
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 400 gpurun_out/bench_ref.json
# launch list of the bench command itself (cold-cache, serialised; shares not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
# full sections for the top kernels (all three views for the blend)
timeout 900 ncu --set full --import-source on --nvtx --nvtx-include "frame/" -k regex:k_blend -c 3 --clock-control none \
    -o gpurun_out/ncu_blend python scripts/profile_frame.py cfg3 all > /dev/null 2>&1
for k in k_cull k_project k_radix_scatter k_bentry_count; do
  timeout 600 ncu --set full --import-source on --nvtx --nvtx-include "frame/" -k regex:$k -c 1 --clock-control none \
      -o gpurun_out/ncu_$k python scripts/profile_frame.py cfg3 2 > /dev/null 2>&1
done
ls gpurun_out
