#!/bin/bash
# Build library variants on the GPU box and A/B them on config 3 (scripts/ab_variants.py).
#   scripts/ab_run.sh "name:-DFLAG=1 -DX=2" "name2:" ...
set -e
cd "$(dirname "$0")/../paper_2511_19202_b200/csrc"
mkdir -p /tmp/variants
libs=()
for v in "$@"; do
  n=${v%%:*}; f=${v#*:}
  make -s -j8 BUILD=/tmp/variants/build_$n OUT=/tmp/variants/$n.so EXTRA="$f" > /tmp/variants/$n.log 2>&1 || { cat /tmp/variants/$n.log; exit 1; }
  libs+=(/tmp/variants/$n.so)
done
cd ../..
python scripts/ab_variants.py "${libs[@]}"
