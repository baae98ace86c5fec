set -x
K1_FORMS=v1,v1,v1 timeout 120 python tools/k1_bench.py 296 32768 592 32768 2>&1
K1_REPS=2 K1_FORMS=v1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cdc_region_kernel -s 1 -c 1 \
  -o gpurun_out/k1_wide2 -f python tools/k1_bench.py 296 32768 > gpurun_out/k1_wide2_ncu.log 2>&1; echo "ncu rc=$?"
