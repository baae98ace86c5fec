LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp $LIB /tmp/base.so
for i in 1 2; do
for v in base ${VARIANTS}; do
  [ $v = base ] && cp /tmp/base.so $LIB || cp _variants/$v.so $LIB
  echo "== $v"; timeout 120 python tools/mla_bench.py --all 2>&1 | tail -3
done
done
for v in ${VARIANTS}; do cp _variants/$v.so $LIB; echo "== checks $v"; timeout 300 python -m pytest tests/test_gpu_mla.py tests/test_gpu_mla_shapes.py -x -q -k "v3" 2>&1 | tail -1; timeout 200 python tools/k5_stress.py 60 c4,c3 2>&1 | tail -2; done
cp /tmp/base.so $LIB
