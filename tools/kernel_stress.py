"""Repeat-launch determinism stress for the non-attention hot kernels (the K5 one is
tools/k5_stress.py): every launch is synchronised, checked for CUDA errors and compared bit
for bit with the first launch.

  K1  irm_cdc_xxh64(_seeded), fused and split forms, 296 x 32K and 8 x 32.9K streams with pins
  K4  irm_group_by_source + irm_rotate_gather_fanout, and the plain irm_rotate_gather, on a
      config-2-sized wave (27 layers, 8 members per ~200 source runs of ~160 rows), all SMs
      and a 4-round retiring grid on 140 SMs

Usage: python tools/kernel_stress.py [n_launches]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_05696_b200 import _native as N, ops  # noqa: E402

n_rep = int(sys.argv[1]) if len(sys.argv) > 1 else 30
failures = 0


def repeat(name, fn, outs):
    """fn() launches; outs() returns the tensors to compare."""
    global failures
    fn()
    torch.cuda.synchronize()
    ref = [o.clone() for o in outs()]
    bad = 0
    t0 = time.time()
    for i in range(n_rep):
        fn()
        torch.cuda.synchronize()
        if not all(torch.equal(a, b) for a, b in zip(outs(), ref)):
            bad += 1
            print(f"{name}: launch {i} differs from the first", flush=True)
    failures += bad
    print(f"{name}: {n_rep} launches, {bad} differing, {time.time() - t0:.1f} s", flush=True)


# ---- K1
rng = np.random.default_rng(5)
for n_streams, n_tok, n_pins in [(296, 32768, 0), (8, 32900, 2)]:
    tok = torch.from_numpy(rng.integers(0, 2**32, size=n_streams * n_tok, dtype=np.uint64).astype(np.uint32)
                           .view(np.int32)).cuda()
    off = torch.arange(0, (n_streams + 1) * n_tok, n_tok, dtype=torch.int64, device="cuda")
    if n_pins:
        pins = torch.from_numpy(np.sort(rng.integers(0, n_tok, size=(n_streams, n_pins)), axis=1).reshape(-1)).cuda()
        pin_off = torch.arange(0, (n_streams + 1) * n_pins, n_pins, dtype=torch.int64, device="cuda")
    else:
        pins = pin_off = None
    for form in ("fused", "split"):
        os.environ["IRM_CDC_FORM"] = form
        ws = ops.CdcWorkspace()
        box = {}

        def run(tok=tok, off=off, pins=pins, pin_off=pin_off, ws=ws, box=box):
            box["t"] = ops.cdc_xxh64(tok, off, pin_off, pins, 7, 32, 512, True, ws=ws, n_tokens=tok.numel())

        def outs(box=box):
            t = box["t"]
            n = int(t.chunk_off[-1])
            return [t.start[:n], t.length[:n], t.fp[:n], t.forced[:n], t.chunk_off]

        repeat(f"K1 {form} {n_streams} x {n_tok}", run, outs)
os.environ.pop("IRM_CDC_FORM", None)

# ---- K4
L, rows = 27, 40000
pool = torch.randn(L, rows, 576, device="cuda").to(torch.bfloat16)
n_src, members = 200, 8
lens = rng.integers(32, 300, size=n_src).astype(np.int32)
starts = rng.integers(0, rows - 300, size=n_src).astype(np.int64)
src = np.repeat(starts, members)
ln = np.repeat(lens, members)
perm = rng.permutation(src.size)
src, ln = src[perm], ln[perm]
dst = np.concatenate([[0], np.cumsum(ln)[:-1]]).astype(np.int64)
delta = rng.integers(-(2**17), 2**17, size=src.size).astype(np.int64)
out_rows = int(dst[-1] + ln[-1])
out = torch.zeros(L, out_rows, 576, dtype=torch.bfloat16, device="cuda")
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
src_d, dst_d, ln_d, delta_d = d(src), d(dst), d(ln), d(delta)
inv = ops.inv_freq_device(np.power(1e4, -2.0 * np.arange(32) / 64))
groups = ops.SourceGroups.alloc(src.size, "cuda")
n_dev = torch.tensor([src.size], dtype=torch.int64, device="cuda")
status = torch.zeros(1, dtype=torch.int64, device="cuda")


def run_fan(max_sms=0, rounds=1):
    ops.group_by_source(src_d, dst_d, ln_d, delta_d, groups, n_dev=n_dev)
    ops.rotate_gather_fanout(pool, out, groups, inv, layout=N.LAYOUT_INTERLEAVED, n_members_dev=n_dev,
                             max_sms=max_sms, status=status, cta_rounds=rounds)


repeat("K4 fan-out, all SMs", run_fan, lambda: [out, status])
repeat("K4 group_by_source order (informational: member order inside a group may vary)", run_fan,
       lambda: [groups.g_src[:int(groups.n_groups)], groups.g_len[:int(groups.n_groups)]])
repeat("K4 fan-out, 140 SMs x 4 retiring rounds", lambda: run_fan(140, 4), lambda: [out, status])
fan_out = out.clone()
out.zero_()
repeat("K4 plain gather", lambda: ops.rotate_gather(pool, out, src_d, dst_d, ln_d, delta_d, inv,
                                                    layout=N.LAYOUT_INTERLEAVED, status=status),
       lambda: [out, status])
same = torch.equal(out, fan_out)
print(f"K4 fan-out == plain gather: {same}", flush=True)
failures += 0 if same else 1
print("FAILURES", failures)
sys.exit(1 if failures else 0)
