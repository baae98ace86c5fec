LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
for v in prof_base prof_pt; do
  cp _variants/$v.so $LIB
  echo "=== $v"
  IRM_MLA_DEBUG=1 timeout 300 python -c "
import sys; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import mla_bench; mla_bench.main(65536,4096,reps=1)" 2>&1 | tail -12
done
