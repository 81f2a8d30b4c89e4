#!/bin/bash
# concurrency probe per library variant: bash scripts/conc_ab.sh lib1.so lib2.so ...
for lib in "$@"; do
  echo "== $lib"
  SPLATCULL_B200_VARIANT=$lib python scripts/concurrency_probe.py 2 2>&1 | tail -2
done
