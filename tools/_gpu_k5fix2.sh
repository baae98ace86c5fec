LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
echo "== PT=0 (default)"; timeout 300 python -m pytest tests/test_gpu_mla_shapes.py -q -k "repeat" 2>&1 | tail -2
cp $LIB /tmp/base.so; cp _variants/pt1.so $LIB
echo "== PT=1 (must fail)"; timeout 300 python -m pytest tests/test_gpu_mla_shapes.py -q -k "repeat and v3" 2>&1 | tail -3
cp /tmp/base.so $LIB
