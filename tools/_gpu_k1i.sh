LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp $LIB /tmp/base.so
for v in base ${VARIANTS:-h2_0}; do
  [ $v = base ] && cp /tmp/base.so $LIB || cp _variants/$v.so $LIB
  K1_REPS=3 K1_FORMS=v2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k1i_$v.csv python tools/k1_bench.py 8 32900 > /dev/null 2>&1
  echo "== $v"; python profiles/ncu_summary.py launches gpurun_out/k1i_$v.csv | head -12
done
cp /tmp/base.so $LIB
