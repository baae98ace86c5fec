set -x
timeout 600 python -m pytest tests/test_gpu_cdc.py -x -q > gpurun_out/k1_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/k1_tests.log
K1_FORMS=${K1_FORMS:-t1,v1,t2,v2,t1,v1,t2,v2} timeout 300 python tools/k1_bench.py ${K1_ARGS:-296 32768 592 32768 148 32768 1184 8192 8 32900} > gpurun_out/k1_forms2.log 2>&1
cat gpurun_out/k1_forms2.log
