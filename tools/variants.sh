#!/bin/bash
# A/B of library builds on one box: for each _variants/<name>.so, install it in-tree, run the
# given test selection and tools/mla_bench.py; the in-tree library is restored afterwards.
# usage: tools/variants.sh "<pytest args>" name1 name2 ...
set -u
LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp $LIB /tmp/irm_lib_orig.so
TESTS="$1"; shift
for v in "$@"; do
  cp _variants/$v.so $LIB
  echo "=== $v"
  if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -x -q 2>&1 | tail -2; fi
  for i in 1 2; do timeout 300 python tools/mla_bench.py --all 2>&1 | tail -3; done
done
cp /tmp/irm_lib_orig.so $LIB
