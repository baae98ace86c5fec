set -x
LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp $LIB /tmp/base.so
K1_FORMS=v1,v1,v1 timeout 120 python tools/k1_bench.py 296 32768 592 32768 > gpurun_out/k1b_base.log 2>&1; cat gpurun_out/k1b_base.log
for v in ${VARIANTS:-walk1}; do
  cp _variants/$v.so $LIB
  echo "== $v"
  K1_FORMS=v1,v1,v1 timeout 120 python tools/k1_bench.py 296 32768 592 32768 2>&1 | tail -6
  IRM_CDC_FORM=fused timeout 120 python -m pytest tests/test_gpu_cdc.py -x -q 2>&1 | tail -1
done
cp /tmp/base.so $LIB
K1_REPS=2 K1_FORMS=v1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cdc_region_kernel -s 1 -c 1 \
  -o gpurun_out/k1_wide -f python tools/k1_bench.py 296 32768 > gpurun_out/k1_wide_ncu.log 2>&1; echo "ncu rc=$?"
