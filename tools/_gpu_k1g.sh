timeout 300 python -m pytest tests/test_gpu_cdc.py -x -q 2>&1 | tail -1
K1_FORMS=v1,v2,v1,v2 timeout 120 python tools/k1_bench.py 296 32768 592 32768 1184 8192 148 32768 200 4096 2>&1
