LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp $LIB /tmp/base.so
timeout 300 python -m pytest tests/test_gpu_cdc.py tests/test_gpu_engine.py -x -q 2>&1 | tail -1
for v in base ${VARIANTS}; do
  [ $v = base ] && cp /tmp/base.so $LIB || cp _variants/$v.so $LIB
  echo "== $v"
  K1_FORMS=v1,v2,v1,v2 timeout 120 python tools/k1_bench.py 8 32900 296 32768 2>&1 | tail -4
  K1_REPS=3 K1_FORMS=v2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k1j_$v.csv python tools/k1_bench.py 8 32900 > /dev/null 2>&1
  python profiles/ncu_summary.py launches gpurun_out/k1j_$v.csv | grep -E "cdc_|gear"
done
cp /tmp/base.so $LIB
