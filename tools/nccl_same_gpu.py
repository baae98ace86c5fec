"""Probe: can two NCCL ranks share one GPU (torchrun --nproc-per-node 2, both on cuda:0)?"""
import os
import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
try:
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    x = torch.full((4,), rank, dtype=torch.int64, device="cuda")
    y = torch.empty_like(x)
    dist.all_to_all_single(y, x)
    torch.cuda.synchronize()
    print(f"rank {rank}: all_to_all ok {y.tolist()}", flush=True)
    dist.destroy_process_group()
except Exception as e:  # noqa: BLE001
    print(f"rank {rank}: FAILED {type(e).__name__}: {str(e)[:300]}", flush=True)
