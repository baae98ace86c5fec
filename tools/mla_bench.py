"""Quick K5 timing: config 3 shape (64K context, last 4096 queries, 16 heads)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_05696_b200 import ops  # noqa: E402


def main(n_kv=65536, n_q=4096, heads=16, reps=5, theta=5e4):
    rng = np.random.default_rng(0)
    q = torch.randn(n_q, heads, 576, device="cuda").to(torch.bfloat16)
    pool = torch.randn(n_kv, 576, device="cuda").to(torch.bfloat16)
    n_chunks = n_kv // 128
    deltas = torch.from_numpy(rng.integers(-4096, 4096, size=n_chunks)).cuda()
    cs = ops.chunk_cossin(deltas, ops.inv_freq_device(np.power(theta, -2.0 * np.arange(32) / 64)))
    kv_chunk = (torch.arange(n_kv, device="cuda") // 128).to(torch.int32)
    out, lse = ops.mla_reattach_prefill(q, pool, n_kv, n_kv - n_q, 192 ** -0.5, kv_chunk=kv_chunk, chunk_cs=cs)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        ops.mla_reattach_prefill(q, pool, n_kv, n_kv - n_q, 192 ** -0.5, kv_chunk=kv_chunk, chunk_cs=cs, out=out,
                                 lse=lse)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    pos = np.arange(n_kv - n_q, n_kv)
    flops = heads * float((pos + 1).sum()) * 2176
    print(f"n_kv {n_kv} n_q {n_q}: {ms:.3f} ms, {flops / ms / 1e9:.1f} TFLOP/s ({flops / 1e12:.2f} TFLOP)")


if __name__ == "__main__":
    main()
    main(32768, 4096)
    if "--all" in sys.argv:  # config 4 shape: 128K context, last 8K queries, theta 3.2e7
        main(131072, 8192, reps=3, theta=3.2e7)
