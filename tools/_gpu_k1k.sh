LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp $LIB /tmp/base.so
for v in base ${VARIANTS}; do
  [ $v = base ] && cp /tmp/base.so $LIB || cp _variants/$v.so $LIB
  echo "== $v"
  IRM_CDC_FORM=fused timeout 120 python -m pytest tests/test_gpu_cdc.py -x -q -k "not table" 2>&1 | tail -1
  IRM_CDC_FORM=split timeout 120 python -m pytest tests/test_gpu_cdc.py -x -q -k "not table" 2>&1 | tail -1
  K1_FORMS=v1,v2,v1,v2 timeout 120 python tools/k1_bench.py 8 32900 296 32768 2>&1 | tail -4
done
cp /tmp/base.so $LIB
