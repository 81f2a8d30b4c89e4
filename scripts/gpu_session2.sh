# full-size parity (configs 2 and 3), sanitizer, per-view launch tables, ncu on blend/project/cull
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_frame_path_parity.py -q -m gpu -k config2 > gpurun_out/pytest_cfg2.log 2>&1; tail -3 gpurun_out/pytest_cfg2.log
timeout 1500 python scripts/fullsize_parity.py all > gpurun_out/fullsize_parity.json 2> gpurun_out/fullsize_parity.err; tail -c 300 gpurun_out/fullsize_parity.json; tail -3 gpurun_out/fullsize_parity.err
bash scripts/sanitize.sh
for v in 0 1 2; do ./scripts/frame_profile.sh $v > /dev/null 2>&1; done
timeout 900 ncu --set full --import-source on --nvtx --nvtx-include "frame/" -k regex:k_blend -c 3 --clock-control none \
    -o gpurun_out/ncu_blend python scripts/profile_frame.py cfg3 all > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --nvtx --nvtx-include "frame/" \
    -k regex:"k_cull|k_project|k_bentry_emit" -c 4 --clock-control none \
    -o gpurun_out/ncu_top python scripts/profile_frame.py cfg3 2 > /dev/null 2>&1
ls gpurun_out
