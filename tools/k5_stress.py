"""K5 stress: the bench's K5 workloads launched many times in one process; every launch is
synchronised, checked for CUDA errors and compared bit for bit with the first launch's output
(a race would show as a fault, a hang or a changed output).
Usage: python tools/k5_stress.py [n_launches] [shapes: c4,c3,c2] [kernel env: v3|v2|1sm]"""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2605_05696_b200 import _native as N, ops  # noqa: E402

SHAPES = {"c4": (131072, 8192, 3.2e7, N.LAYOUT_HALF_SPLIT), "c3": (65536, 4096, 5e4, N.LAYOUT_HALF_SPLIT),
          "c2": (32768, 4096, 1e4, N.LAYOUT_INTERLEAVED)}
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
shapes = (sys.argv[2] if len(sys.argv) > 2 else "c4,c3,c2").split(",")
for name in shapes:
    n_ctx, n_q, theta, layout = SHAPES[name]
    w = bench.attn_workload(n_ctx, n_q, 16, theta, layout)
    run = lambda: ops.mla_reattach_prefill(w["q"], w["pool"], n_ctx, n_ctx - n_q, 192 ** -0.5, kv_rows=w["rows_d"],
                                           kv_chunk=w["chunk_d"], chunk_cs=w["cs"], layout=w["layout"])
    out0, lse0 = run()
    torch.cuda.synchronize()
    ref_o, ref_l = out0.clone(), lse0.clone()
    bad = 0
    t0 = time.time()
    for i in range(n):
        out, lse = run()
        torch.cuda.synchronize()
        if not (torch.equal(out, ref_o) and torch.equal(lse, ref_l)):
            bad += 1
            d = (out.float() - ref_o.float()).abs()
            print(f"{name} launch {i}: output differs from launch 0 (max abs {d.max().item():.3g}, "
                  f"{int((d > 0).sum())} elements)", flush=True)
    print(f"{name}: {n} launches, {bad} differing, {time.time() - t0:.1f} s", flush=True)
