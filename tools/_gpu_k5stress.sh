LIB=paper_2605_05696_b200/_lib/libirminsul_b200.so
cp $LIB /tmp/base.so
for v in base pt0; do
  [ $v = base ] && cp /tmp/base.so $LIB || cp _variants/$v.so $LIB
  echo "== $v"; timeout 120 python tools/k5_stress.py 40 c4,c3,c2 2>&1 | grep -v "^  \|Traceback\|File\|return\|\^" | head -8
done
cp /tmp/base.so $LIB
echo "== v2"; IRM_MLA_V2=1 timeout 120 python tools/k5_stress.py 40 c4,c3 2>&1 | grep -v "^  \|Traceback\|File\|return\|\^" | head -6
echo "== 1sm"; IRM_MLA_1SM=1 timeout 120 python tools/k5_stress.py 20 c4 2>&1 | grep -v "^  \|Traceback\|File\|return\|\^" | head -6
