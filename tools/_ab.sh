LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp $LIB /tmp/orig.so
for round in 1 2 3; do
for v in "$@"; do
  cp _variants/$v.so $LIB
  echo "=== $v"
  timeout 300 python tools/mla_bench.py --all 2>&1 | tail -3
done
done
cp /tmp/orig.so $LIB
