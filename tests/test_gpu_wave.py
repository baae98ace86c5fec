"""GPU: the warm-serve step glue kernels against their torch statement
(irm_wave_plan: owner request / absolute position / probe / order per slot;
irm_wave_compact: the hit slots in slot order as K4 work, count on the device).
Bit-exact integer work; empty requests, past-the-end slots and all-miss waves."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _case(seed, n_req, cap, empty_every=0):
    rng = np.random.default_rng(seed)
    counts = rng.integers(0, 40, size=n_req)
    if empty_every:
        counts[::empty_every] = 0
    off = np.zeros(n_req + 1, np.int64)
    np.cumsum(counts, out=off[1:])
    assert off[-1] <= cap
    start = rng.integers(0, 5000, size=cap).astype(np.int32)
    meta = rng.integers(0, 100, size=n_req).astype(np.int64)
    return (torch.from_numpy(off).cuda(), torch.from_numpy(start).cuda(), torch.from_numpy(meta).cuda())


@pytest.mark.parametrize("seed,n_req,cap,empty_every", [(0, 8, 400, 0), (1, 5, 300, 2), (2, 1, 64, 0),
                                                        (3, 64, 4000, 3)])
def test_wave_plan_and_compact(seed, n_req, cap, empty_every):
    from paper_2605_05696_b200 import ops

    off, start, meta = _case(seed, n_req, cap, empty_every)
    dev = start.device
    carve, order0 = 32, 1000
    req = torch.empty(cap, dtype=torch.int64, device=dev)
    p_abs = torch.empty_like(req)
    probe = torch.empty(cap, dtype=torch.uint8, device=dev)
    order = torch.empty_like(req)
    ops.wave_plan(off, n_req, start, meta, carve, order0, req, p_abs, probe, order)
    idx = torch.arange(cap, device=dev)
    r_ref = torch.clamp(torch.searchsorted(off[1:], idx, right=True), max=n_req - 1)
    pa_ref = meta[r_ref] + start.to(torch.int64)
    pr_ref = ((idx < off[-1]) & (pa_ref >= carve)).to(torch.uint8)
    assert torch.equal(req, r_ref) and torch.equal(p_abs, pa_ref) and torch.equal(probe, pr_ref)
    assert torch.equal(order, order0 + idx)

    rng = np.random.default_rng(seed + 100)
    for hit_np in (rng.integers(-1, 2, size=cap), np.zeros(cap, np.int64)):  # mixed; all misses
        hit = torch.from_numpy(hit_np.astype(np.int32)).cuda()
        row = torch.from_numpy(rng.integers(0, 1 << 30, size=cap)).cuda()
        p_src = torch.from_numpy(rng.integers(0, 1 << 20, size=cap)).cuda()
        ln = torch.from_numpy(rng.integers(1, 512, size=cap).astype(np.int32)).cuda()
        outs = [torch.full((cap,), -7, dtype=torch.int64, device=dev) for _ in range(2)]
        len_out = torch.full((cap,), -7, dtype=torch.int32, device=dev)
        delta_out = torch.full((cap,), -7, dtype=torch.int64, device=dev)
        n_hit = torch.zeros(1, dtype=torch.int64, device=dev)
        length = torch.empty(cap, dtype=torch.int32, device=dev)
        tokens = torch.full((), 5, dtype=torch.int64, device=dev)
        for stride in (8192, 2048):  # 2048: some hits would spill past their request's rows
            status = torch.zeros(1, dtype=torch.int64, device=dev)
            tokens.fill_(5)
            ops.wave_compact(hit, row, req, p_abs, p_src, ln, stride, outs[0], outs[1], len_out, delta_out, n_hit,
                             length, hit_tokens=tokens, status=status)
            fits = p_abs + ln.to(torch.int64) <= stride
            is_hit = (hit == 1) & fits
            k = int(is_hit.sum())
            assert int(n_hit) == k
            assert torch.equal(outs[0][:k], row[is_hit])
            assert torch.equal(outs[1][:k], (req * stride + p_abs)[is_hit])
            assert torch.equal(len_out[:k], ln[is_hit]) and torch.equal(delta_out[:k], (p_abs - p_src)[is_hit])
            assert torch.equal(length, torch.where(is_hit, ln, torch.zeros_like(ln)))
            assert int(tokens) == 5 + int(ln[is_hit].sum())
            assert int(status) == (4 if bool(((hit == 1) & ~fits).any()) else 0)
