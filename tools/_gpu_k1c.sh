set -x
LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp $LIB /tmp/base.so
timeout 300 python -m pytest tests/test_gpu_cdc.py -x -q 2>&1 | tail -2
K1_FORMS=v1,t1,v2,v1,t1,v2 timeout 120 python tools/k1_bench.py 296 32768 592 32768 148 32768 8 32900 2>&1
for v in ${VARIANTS:-ks walk1}; do
  cp _variants/$v.so $LIB
  echo "== $v"
  K1_FORMS=v1,t1,v1,t1 timeout 120 python tools/k1_bench.py 296 32768 592 32768 148 32768 2>&1 | tail -12
  IRM_CDC_FORM=fused timeout 120 python -m pytest tests/test_gpu_cdc.py -x -q 2>&1 | tail -1
done
cp /tmp/base.so $LIB
