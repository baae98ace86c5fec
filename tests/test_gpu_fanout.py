"""GPU: K4's fan-out form (csrc/fanout.cu) against the oracle.

irm_group_by_source: the work list grouped by source run, checked against a
host statement (every item lands in exactly one group with its own (dst,
delta); groups ordered by their first item; the workspace left zeroed).
irm_rotate_gather_fanout: every member's rows against the oracle's
rotate+gather (oracle/irm_oracle.c, registry.py:146-166 semantics): c_KV
bit-exact, k_r within bf16 rounding, and bit-identical to the one-read-per-hit
gather (irm_rotate_gather) on the same work. Bounds: out-of-range source or
destination runs are skipped and flagged, never read or written."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _work(seed, n_src=40, n_items=300, L=3, pool_rows=6000, max_len=300):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, max_len, size=n_src).astype(np.int32)
    starts = rng.integers(0, pool_rows - max_len, size=n_src).astype(np.int64)
    pick = rng.integers(0, n_src, size=n_items)
    ln = lens[pick]
    dst = np.concatenate([[0], np.cumsum(ln)[:-1]]).astype(np.int64) + 5
    delta = rng.integers(-(2**17), 2**17, size=n_items).astype(np.int64)
    return starts[pick], dst, ln, delta, int(dst[-1] + ln[-1] + 5)


def _d(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("seed,n_items", [(0, 300), (1, 1), (2, 2500), (3, 64)])
def test_group_by_source(seed, n_items):
    from paper_2605_05696_b200 import ops

    src, dst, ln, delta, _ = _work(seed, n_items=n_items, n_src=max(1, n_items // 6))
    cap = n_items + 17
    pad = lambda a, v: np.concatenate([a, np.full(cap - a.size, v, a.dtype)])
    groups = ops.SourceGroups.alloc(cap, "cuda")
    n_dev = torch.tensor([n_items], dtype=torch.int64, device="cuda")
    for _ in range(2):  # the second call reuses the (re-zeroed) workspace
        ops.group_by_source(_d(pad(src, 7)), _d(pad(dst, 7)), _d(pad(ln, 7)), _d(pad(delta, 7)), groups,
                            n_dev=n_dev)
        torch.cuda.synchronize()
        assert int(groups.ws.count_nonzero()) == 0, "workspace must be left zeroed"
    ng = int(groups.n_groups)
    keys = list(dict.fromkeys(zip(src.tolist(), ln.tolist())))  # first-occurrence order
    assert ng == len(keys)
    gs, gl = groups.g_src[:ng].cpu().numpy(), groups.g_len[:ng].cpu().numpy()
    gf, gc = groups.g_first[:ng].cpu().numpy(), groups.g_count[:ng].cpu().numpy()
    md, mde = groups.m_dst.cpu().numpy(), groups.m_delta.cpu().numpy()
    assert [(int(a), int(b)) for a, b in zip(gs, gl)] == keys
    assert gf[0] == 0 and np.array_equal(gf[1:], np.cumsum(gc)[:-1]) and gc.sum() == n_items
    for g, (s, l) in enumerate(keys):
        sel = (src == s) & (ln == l)
        want = sorted(zip(dst[sel].tolist(), delta[sel].tolist()))
        got = sorted(zip(md[gf[g]:gf[g] + gc[g]].tolist(), mde[gf[g]:gf[g] + gc[g]].tolist()))
        assert got == want


@pytest.mark.parametrize("rounds", [1, 4])
@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("seed,max_len", [(5, 300), (6, 40), (7, 513)])
def test_fanout_matches_oracle_and_plain_gather(layout, seed, max_len, rounds):
    from paper_2605_05696_b200 import ops

    L, pool_rows = 3, 6000
    src, dst, ln, delta, out_rows = _work(seed, L=L, pool_rows=pool_rows, max_len=max_len)
    g = torch.Generator(device="cuda").manual_seed(seed)
    pool = torch.randn(L, pool_rows, 576, device="cuda", generator=g).to(torch.bfloat16)
    inv = O.make_inv_freq(1e4)
    invd = ops.inv_freq_device(inv)
    groups = ops.SourceGroups.alloc(src.size, "cuda")
    ops.group_by_source(_d(src), _d(dst), _d(ln), _d(delta), groups)
    status = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = torch.zeros(L, out_rows, 576, dtype=torch.bfloat16, device="cuda")
    ops.rotate_gather_fanout(pool, out, groups, invd, layout=layout, status=status, cta_rounds=rounds,
                             max_sms=0 if rounds > 1 else 17)  # retiring CTA rounds / a partial grid
    plain = torch.zeros_like(out)
    ops.rotate_gather(pool, plain, _d(src), _d(dst), _d(ln), _d(delta), invd, layout=layout)
    torch.cuda.synchronize()
    assert int(status) == 0
    assert torch.equal(out.view(torch.int16), plain.view(torch.int16)), "fan-out != plain gather"
    pu = pool.view(torch.int16).cpu().numpy().view(np.uint16)
    exp = np.zeros((L, out_rows, 576), np.uint16)
    O.rotate_gather_bf16(pu, exp, src, dst, ln, delta, inv, interleaved=bool(layout))
    got = out.view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(got[..., :512], exp[..., :512])
    f = lambda u: (u.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    assert np.abs(f(got[..., 512:]) - f(exp[..., 512:])).max() <= 2.0 ** -7 * np.abs(f(exp[..., 512:])).max()
    # same fp32 rounding sequence as the oracle (common.cuh rot_lo / rot_hi): bit-exact except where
    # the fp64 cos/sin of CUDA and of libm round to different floats (rare)
    assert np.mean(got[..., 512:] == exp[..., 512:]) >= 0.999


def test_fanout_f32_pool():
    from paper_2605_05696_b200 import ops

    L = 2
    src, dst, ln, delta, out_rows = _work(9, L=L, n_items=80)
    pool = torch.randn(L, 6000, 576, device="cuda", dtype=torch.float32)
    inv = O.make_inv_freq(5e4)
    groups = ops.SourceGroups.alloc(src.size, "cuda")
    ops.group_by_source(_d(src), _d(dst), _d(ln), _d(delta), groups)
    out = torch.zeros(L, out_rows, 576, dtype=torch.float32, device="cuda")
    ops.rotate_gather_fanout(pool, out, groups, ops.inv_freq_device(inv))
    torch.cuda.synchronize()
    p = pool.double().cpu().numpy()
    o = out.double().cpu().numpy()
    for c in range(src.size):
        s, d, l = int(src[c]), int(dst[c]), int(ln[c])
        assert np.array_equal(o[:, d:d + l, :512], p[:, s:s + l, :512])
        for layer in range(L):
            ref = O.rotate_rows(p[layer, s:s + l, 512:], np.full(l, delta[c], np.float64), inv)
            assert O.rel_l2(o[layer, d:d + l, 512:], ref) <= 1e-5


def test_fanout_bounds_are_skipped_and_flagged():
    from paper_2605_05696_b200 import ops

    L, pool_rows = 2, 1000
    pool = torch.randn(L, pool_rows, 576, device="cuda").to(torch.bfloat16)
    inv = ops.inv_freq_device(O.make_inv_freq(1e4))
    src = np.array([10, 990, 100], np.int64)   # item 1: 990 + 20 > pool_rows
    dst = np.array([0, 40, 495], np.int64)     # item 2: 495 + 20 > out_rows
    ln = np.array([20, 20, 20], np.int32)
    delta = np.array([3, 4, 5], np.int64)
    out_rows = 500
    for fan in (True, False):
        status = torch.zeros(1, dtype=torch.int64, device="cuda")
        out = torch.zeros(L, out_rows, 576, dtype=torch.bfloat16, device="cuda")
        if fan:
            groups = ops.SourceGroups.alloc(3, "cuda")
            ops.group_by_source(_d(src), _d(dst), _d(ln), _d(delta), groups)
            ops.rotate_gather_fanout(pool, out, groups, inv, status=status)
        else:
            ops.rotate_gather(pool, out, _d(src), _d(dst), _d(ln), _d(delta), inv, status=status)
        torch.cuda.synchronize()
        assert int(status) == 3, (fan, int(status))
        o = out.float().cpu()
        assert torch.equal(o[:, :20, :512], pool[:, 10:30, :512].float().cpu())  # the in-range item ran
        assert o[:, 20:].abs().sum() == 0  # nothing else written
        with pytest.raises(ValueError, match="source run outside"):
            ops.check_status(status)


def test_fanout_repeat_launches_bit_identical():
    """K4 fan-out relaunched back to back on a 27-layer wave (8 members per source run, all SMs
    and the 4-round retiring grid) writes bit-identical rows, equal to the plain gather's."""
    from paper_2605_05696_b200 import _native as N, ops

    rng = np.random.default_rng(11)
    L, rows, n_src, members = 27, 12000, 60, 8
    lens = rng.integers(32, 300, size=n_src).astype(np.int32)
    starts = rng.integers(0, rows - 300, size=n_src).astype(np.int64)
    perm = rng.permutation(n_src * members)
    src, ln = np.repeat(starts, members)[perm], np.repeat(lens, members)[perm]
    dst = np.concatenate([[0], np.cumsum(ln)[:-1]]).astype(np.int64)
    delta = rng.integers(-(2**17), 2**17, size=src.size).astype(np.int64)
    pool = torch.randn(L, rows, 576, device="cuda").to(torch.bfloat16)
    out = torch.zeros(L, int(dst[-1] + ln[-1]), 576, dtype=torch.bfloat16, device="cuda")
    src_d, dst_d, ln_d, delta_d = _d(src), _d(dst), _d(ln), _d(delta)
    inv = ops.inv_freq_device(np.power(1e4, -2.0 * np.arange(32) / 64))
    groups = ops.SourceGroups.alloc(src.size, "cuda")
    n_dev = torch.tensor([src.size], dtype=torch.int64, device="cuda")
    ops.rotate_gather(pool, out, src_d, dst_d, ln_d, delta_d, inv, layout=N.LAYOUT_INTERLEAVED)
    torch.cuda.synchronize()
    ref = out.clone()
    for max_sms, rounds in [(0, 1)] * 4 + [(140, 4)] * 4:
        out.zero_()
        ops.group_by_source(src_d, dst_d, ln_d, delta_d, groups, n_dev=n_dev)
        ops.rotate_gather_fanout(pool, out, groups, inv, layout=N.LAYOUT_INTERLEAVED, n_members_dev=n_dev,
                                 max_sms=max_sms, cta_rounds=rounds)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
