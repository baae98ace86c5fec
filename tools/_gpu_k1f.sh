LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp $LIB /tmp/base.so
timeout 300 python -m pytest tests/test_gpu_cdc.py -x -q 2>&1 | tail -1
for v in base ${VARIANTS:-rolemap0} base; do
  [ $v = base ] && cp /tmp/base.so $LIB || cp _variants/$v.so $LIB
  echo "== $v"
  K1_FORMS=v1,v1,v1 timeout 120 python tools/k1_bench.py ${K1_ARGS:-296 32768 592 32768 148 32768} 2>&1 | tail -9
done
cp /tmp/base.so $LIB
IRM_CDC_DEBUG=1 K1_REPS=1 K1_FORMS=v1 timeout 120 python tools/k1_bench.py 296 32768 > gpurun_out/k1dbg3.log 2>&1
grep "region 7 \|region 201 " gpurun_out/k1dbg3.log | sort
