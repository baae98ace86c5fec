LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
timeout 600 python -m pytest tests/test_gpu_mla_shapes.py tests/test_gpu_mla.py -q -x 2>&1 | tail -2
echo "== stress (PT=0 default)"; timeout 200 python tools/k5_stress.py 60 c4,c3,c2 2>&1 | tail -3
cp $LIB /tmp/base.so; cp _variants/pt1.so $LIB
echo "== the determinism test on PT=1 (must fail)"; timeout 300 python -m pytest tests/test_gpu_mla_shapes.py -q -x -k "repeat and v3" 2>&1 | tail -2
cp /tmp/base.so $LIB
for i in 1 2; do echo "== timing"; timeout 120 python tools/mla_bench.py --all 2>&1 | tail -3; done
