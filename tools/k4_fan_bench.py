"""K4 microbenchmark on a config-2-shaped wave: R requests reattaching the same
~193 body chunks (27 layers, bf16, 576-wide rows) at their own deltas. Times
the one-read-per-hit gather and the fan-out gather (IRM_FAN_VARIANT sweeps its
tile rows x source x output stages) with CUDA events.
  python tools/k4_fan_bench.py [variants...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_05696_b200 import ops  # noqa: E402

L, R, BODY = 27, 8, 32768
rng = np.random.default_rng(0)
lens = []
while sum(lens) < BODY:
    lens.append(int(rng.integers(32, 340)))
lens = np.array(lens, np.int32)
starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
stride = BODY + 512
src = np.tile(starts, R)
ln = np.tile(lens, R)
dst = np.concatenate([r * stride + 100 + starts for r in range(R)]).astype(np.int64)
delta = np.concatenate([np.full(lens.size, 100 + r * 7 - 0, np.int64) for r in range(R)])
pool = torch.randn(L, BODY + 1024, 576, device="cuda").to(torch.bfloat16)
out = torch.empty(L, R * stride, 576, dtype=torch.bfloat16, device="cuda")
inv = ops.inv_freq_device(np.power(1e4, -2.0 * np.arange(32) / 64))
d = lambda a: torch.from_numpy(a).cuda()
S, D, LN, DE = d(src), d(dst), d(ln), d(delta)
groups = ops.SourceGroups.alloc(src.size, "cuda")
ops.group_by_source(S, D, LN, DE, groups)
rows = int(ln.sum()) * L
uniq = int(lens.sum()) * L


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


sms = int(os.environ.get("SMS", "0"))
ms = t(lambda: ops.rotate_gather(pool, out, S, D, LN, DE, inv, layout=1, max_sms=sms))
print(f"plain      {ms:.3f} ms  {rows * 2304 / ms / 1e6:.0f} GB/s (2 x rows)  eff {rows * 1152 / ms / 1e9:.1f} Mrow/ms")
for v in (sys.argv[1:] or ["0"]):
    os.environ["IRM_FAN_VARIANT"] = v
    ms = t(lambda: ops.rotate_gather_fanout(pool, out, groups, inv, layout=1, max_sms=sms))
    print(f"fan v{v:>3}  {ms:.3f} ms  {(rows + uniq) * 1152 / ms / 1e6:.0f} GB/s (unique reads + writes)")
