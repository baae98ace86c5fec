# final-code ncu captures: K5 v3 at 64K/4K, K1 split (8 x 32.9K) and fused (296 x 32K)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mla_reattach_2sm_v3 -s 1 -c 1 \
  -o gpurun_out/k5_final -f python -c "
import sys; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import mla_bench; mla_bench.main(65536,4096,reps=1)" > gpurun_out/k5_final.log 2>&1; echo "k5 rc=$?"
K1_REPS=2 K1_FORMS=v2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cdc_region_split -s 1 -c 1 \
  -o gpurun_out/k1_split_final -f python tools/k1_bench.py 8 32900 > gpurun_out/k1s_final.log 2>&1; echo "k1s rc=$?"
K1_REPS=2 K1_FORMS=v1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cdc_region_kernel -s 1 -c 1 \
  -o gpurun_out/k1_fused_final -f python tools/k1_bench.py 296 32768 > gpurun_out/k1f_final.log 2>&1; echo "k1f rc=$?"
