"""K4 (bf16, config-2 sized) HBM bandwidth vs the number of SMs it spreads over (irm_rotate_gather's max_sms)."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2605_05696_b200 import ops
L, rows = 27, 40000
pool = torch.randn(L, rows, 576, device="cuda").to(torch.bfloat16)
rng = np.random.default_rng(0)
lens = rng.integers(32, 512, size=1600).astype(np.int32)
n_out = int(lens.sum())
out = torch.empty(L, n_out, 576, dtype=torch.bfloat16, device="cuda")
src = torch.from_numpy(rng.integers(0, rows - 512, size=lens.size).astype(np.int64)).cuda()
dst = torch.from_numpy(np.concatenate([[0], np.cumsum(lens[:-1])]).astype(np.int64)).cuda()
ln = torch.from_numpy(lens).cuda()
delta = torch.from_numpy(rng.integers(-5000, 5000, size=lens.size)).cuda()
inv = ops.inv_freq_device(np.power(1e4, -2.0 * np.arange(32) / 64))
for sms in [148, 144, 140, 136, 132, 128, 120, 112]:
    for _ in range(3):
        ops.rotate_gather(pool, out, src, dst, ln, delta, inv, layout=1, max_sms=sms)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        ops.rotate_gather(pool, out, src, dst, ln, delta, inv, layout=1, max_sms=sms)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(sms, f"{ms:.3f} ms", f"{n_out * L * 2304 / ms / 1e6:.0f} GB/s")
