IRM_CDC_DEBUG=1 K1_REPS=1 K1_FORMS=v1 timeout 120 python tools/k1_bench.py 296 32768 > gpurun_out/k1dbg2.log 2>&1
grep "region 7 \|region 100 \|region 201 " gpurun_out/k1dbg2.log | sort
