LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp $LIB /tmp/base.so
for v in pt1 pt1w; do
  cp _variants/$v.so $LIB
  echo "== $v"; timeout 200 python tools/k5_stress.py 30 c4,c3,c2 2>&1 | grep -v "differs" | tail -4
  timeout 120 python tools/mla_bench.py --all 2>&1 | tail -3
done
cp /tmp/base.so $LIB; echo "== base"; timeout 120 python tools/mla_bench.py --all 2>&1 | tail -3
