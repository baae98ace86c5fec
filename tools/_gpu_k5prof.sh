LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp _variants/prof.so $LIB
for v in 0 1; do
  echo "== V4=$v"
  if [ $v = 1 ]; then export IRM_MLA_V4=1; else unset IRM_MLA_V4; fi
  IRM_MLA_DEBUG=1 timeout 120 python -c "
import sys; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import mla_bench; mla_bench.main(65536,4096,reps=1)" 2>&1 | tail -8
done
