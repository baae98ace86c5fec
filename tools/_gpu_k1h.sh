LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp $LIB /tmp/base.so
timeout 300 python -m pytest tests/test_gpu_cdc.py -x -q 2>&1 | tail -1
for v in base ${VARIANTS:-lean0} base; do
  [ $v = base ] && cp /tmp/base.so $LIB || cp _variants/$v.so $LIB
  echo "== $v"
  K1_FORMS=v1,v2,v1,v2 timeout 120 python tools/k1_bench.py ${K1_ARGS:-296 32768 592 32768 8 32900} 2>&1 | tail -6
done
cp /tmp/base.so $LIB
