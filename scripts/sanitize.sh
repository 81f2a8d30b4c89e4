#!/bin/bash
# compute-sanitizer over scripts/sanitize.py, one tool at a time -> gpurun_out/sanitize_<tool>.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1200 compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 100000 --kernel-name kns=_ZN2sc \
      python scripts/sanitize.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.txt
done
