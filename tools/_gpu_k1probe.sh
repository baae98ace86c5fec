set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rotate_gather_ws -s 14 -c 1 \
  -o gpurun_out/r02t_k4c5b -f python bench.py --workload config5 --steps 2 --warmup 3 --no-cpu --no-attn > gpurun_out/r02t_k4c5b.log 2>&1; echo "ncu rc=$?"
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/nccl_same_gpu.py > gpurun_out/nccl_same.log 2>&1; echo "nccl rc=$?"
tail -5 gpurun_out/nccl_same.log
IRM_CDC_DEBUG=1 K1_REPS=1 K1_FORMS=v1 timeout 120 python tools/k1_bench.py 296 32768 > gpurun_out/k1dbg_wide.log 2>&1
K1_FORMS=v1,v2,v1,v2 timeout 300 python tools/k1_bench.py 296 32768 592 32768 148 32768 1184 8192 8 32900 > gpurun_out/k1_forms.log 2>&1
cat gpurun_out/k1_forms.log
