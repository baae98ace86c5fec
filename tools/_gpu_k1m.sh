LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp $LIB /tmp/base.so
timeout 300 python -m pytest tests/test_gpu_cdc.py tests/test_gpu_engine.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -3
for v in base ${VARIANTS} base; do
  [ $v = base ] && cp /tmp/base.so $LIB || cp _variants/$v.so $LIB
  echo "== $v"
  K1_FORMS=v1,v2,v1,v2 timeout 120 python tools/k1_bench.py 8 32900 296 32768 592 32768 2>&1 | tail -6
done
cp /tmp/base.so $LIB
IRM_CDC_FORM=split IRM_CDC_DEBUG=1 python tools/cdc_debug.py 2>&1 | grep "region-split 0 " | sort | head -8
