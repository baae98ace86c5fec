"""GPU parity: rotation (rotate_rows / round_bf16) against the reference's
golden outputs, and K4 rotate+gather (f64 / f32 / bf16 pools, half-split and
interleaved layouts) against the oracle.

Tolerances (BASELINE.json north_star): fp32 k_r <= 1e-5 rel-L2; bf16 <= 4.7e-3
rel-L2 vs f64 truth; f64 <= 1e-12 (GPU fp64 trig vs the host libm)."""

import numpy as np
import pytest
import torch

from inputs import ROT_CASES, rot_case_inputs
from oracle import oracle as O

pytestmark = pytest.mark.gpu

F32_TOL = 1e-5
BF16_TOL = 4.7e-3


@pytest.fixture(scope="module")
def R():
    from paper_2605_05696_b200 import _native as N, ops, rotary

    return rotary, ops, N


@pytest.mark.parametrize("name", sorted(ROT_CASES))
def test_rotate_rows_golden(R, name, golden_rotary):
    rotary, _, _ = R
    case = ROT_CASES[name]
    rows, pos = rot_case_inputs(case)
    spec = rotary.make_spec(case["theta"])
    g = golden_rotary[name]
    assert np.array_equal(spec.inv_freq, g["inv_freq"])
    out = rotary.rotate_rows(rows, pos, spec)
    err = np.abs(out - g["out"]).max()
    assert err <= 1e-12, err
    # store rounding is a deterministic function of the f64 value: bit-exact
    assert np.array_equal(rotary.round_bf16(g["out"]), g["out_bf16"])
    assert np.array_equal(rotary._store(g["out"], rotary.Precision.F32), g["out_f32"])


def test_round_bf16_edge_cases(R):
    rotary, _, _ = R
    x = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1.0, 1.00390625, 1.005859375, 2.0**-133,
                  2.0**-134, 3 * 2.0**-135, 3.3961e38, 3.4e38, -1e-40, 1e-45, 65504.0, 1 / 3])
    got = rotary.round_bf16(x)
    ref = O.round_bf16(x)
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    m = ~np.isnan(ref)
    assert np.array_equal(got[m], ref[m])


def _pool(rng, layers, rows, dtype, ckv=512, kr=64):
    p = rng.standard_normal((layers, rows, ckv + kr))
    return p


@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16"])
@pytest.mark.parametrize("layout", [0, 1])
def test_rotate_gather_vs_oracle(R, dtype, layout):
    rotary, ops, N = R
    rng = np.random.default_rng(5 + layout)
    layers, prow = 3, 4000
    pool64 = _pool(rng, layers, prow, dtype)
    lens = rng.integers(1, 300, size=40).astype(np.int32)
    lens[:4] = [1, 7, 32, 512]
    src = rng.integers(0, prow - 512, size=lens.size).astype(np.int64)
    dst = np.concatenate([[0], np.cumsum(lens[:-1])]).astype(np.int64)
    delta = rng.integers(-(2**20), 2**20, size=lens.size).astype(np.int64)
    delta[:3] = [0, 1, -1]
    inv = O.make_inv_freq(1e4)
    tdt = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    pool = torch.from_numpy(pool64).to("cuda", tdt)
    out = torch.full((layers, int(lens.sum()), 576), float("nan"), dtype=tdt, device="cuda")
    d = lambda a: torch.from_numpy(a).cuda()
    ops.rotate_gather(pool, out, d(src), d(dst), d(lens), d(delta), ops.inv_freq_device(inv), layout=layout)
    got = out.to(torch.float64).cpu().numpy()
    pin = pool.to(torch.float64).cpu().numpy()  # exact input values after storage rounding
    for c in range(lens.size):
        for l in range(layers):
            s, t, n = src[c], dst[c], lens[c]
            src_rows = pin[l, s:s + n]
            g = got[l, t:t + n]
            assert np.array_equal(g[:, :512], src_rows[:, :512])  # c_KV verbatim
            truth = O.rotate_rows(src_rows[:, 512:], np.full(n, delta[c]), inv, interleaved=bool(layout))
            err = O.rel_l2(g[:, 512:], truth)
            tol = {"f64": 1e-13, "f32": 1e-6, "bf16": 4e-3}[dtype]
            assert err <= tol, (dtype, layout, c, l, err)


def test_rotate_gather_f64_rounding_modes(R):
    rotary, ops, N = R
    rng = np.random.default_rng(9)
    pool = torch.from_numpy(rng.standard_normal((1, 600, 576))).cuda()
    lens = np.array([100, 37], np.int32)
    src = np.array([0, 300], np.int64)
    dst = np.array([0, 100], np.int64)
    delta = np.array([777, -4096], np.int64)
    inv = O.make_inv_freq(5e4)
    d = lambda a: torch.from_numpy(a).cuda()
    for mode, fn in [(N.ROUND_F32, lambda x: x.astype(np.float32).astype(np.float64)), (N.ROUND_BF16, O.round_bf16)]:
        out = torch.empty(1, 137, 576, dtype=torch.float64, device="cuda")
        ops.rotate_gather(pool, out, d(src), d(dst), d(lens), d(delta), ops.inv_freq_device(inv), out_round=mode)
        exact = torch.empty_like(out)
        ops.rotate_gather(pool, exact, d(src), d(dst), d(lens), d(delta), ops.inv_freq_device(inv))
        e = exact.cpu().numpy()[0, :, 512:]
        assert np.array_equal(out.cpu().numpy()[0, :, 512:], fn(e))


@pytest.mark.parametrize("theta", [1e4, 5e4, 3.2e7])
def test_delta_precision_sweep(R, theta):
    """Config 4: |delta| in 2^0..2^17 (both signs), rel-L2 vs f64 truth of the
    fresh rotation: fp32 within 1e-5, bf16 (bf16 kr_base in, bf16 out) within 4.7e-3."""
    rotary, ops, N = R
    rng = np.random.default_rng(int(theta) % 1000)
    inv = O.make_inv_freq(theta)
    n = 2000
    raw = rng.standard_normal((n, 64))
    raw /= np.linalg.norm(raw, axis=1, keepdims=True)
    p_src = 5000
    base64 = O.rotate_rows(raw, np.full(n, p_src), inv)
    deltas = np.array([s * 2**e for e in range(18) for s in (1, -1)], np.int64)
    deltas = deltas[p_src + deltas >= 0]
    pool = np.zeros((1, n, 576))
    pool[0, :, 512:] = base64
    d = lambda a: torch.from_numpy(a).cuda()
    for dt, tol in [(torch.float32, F32_TOL), (torch.bfloat16, BF16_TOL)]:
        tp = d(pool).to(dt)
        lens = np.full(deltas.size, n, np.int32)
        out = torch.empty(1, n * deltas.size, 576, dtype=dt, device="cuda")
        ops.rotate_gather(tp, out, d(np.zeros(deltas.size, np.int64)),
                          d(np.arange(deltas.size, dtype=np.int64) * n), d(lens), d(deltas), ops.inv_freq_device(inv))
        got = out.to(torch.float64).cpu().numpy()[0, :, 512:].reshape(deltas.size, n, 64)
        worst = 0.0
        for i, dl in enumerate(deltas):
            truth = O.rotate_rows(raw, np.full(n, p_src + dl), inv)
            worst = max(worst, O.rel_l2(got[i], truth))
        assert worst <= tol, (dt, theta, worst)


def test_rotate_rows_uses_the_specs_own_frequencies():
    """A spec carrying its own (e.g. scaled) inv_freq rotates by THOSE frequencies
    on the device paths, as the reference's rotate_rows reads spec.inv_freq
    (rotary.py:98-108) -- not make_spec's frequencies for the same theta."""
    import dataclasses

    from paper_2605_05696_b200 import rotary

    base = rotary.make_spec(1e4)
    scaled = dataclasses.replace(base, inv_freq=base.inv_freq * 0.25)
    rng = np.random.default_rng(3)
    rows = rng.standard_normal((7, 64))
    pos = np.arange(7, dtype=np.float64) * 1000
    got_base = rotary.rotate_rows(rows, pos, base)
    got_scaled = rotary.rotate_rows(rows, pos, scaled)
    assert O.rel_l2(got_base, O.rotate_rows(rows, pos, base.inv_freq)) <= 1e-12
    assert O.rel_l2(got_scaled, O.rotate_rows(rows, pos, scaled.inv_freq)) <= 1e-12
    assert O.rel_l2(got_scaled, got_base) > 1e-3


def _cr_sincos(x: float):
    """Correctly rounded (sin, cos) of a double via 60-digit Decimal arithmetic."""
    from decimal import Decimal, getcontext

    getcontext().prec = 60
    pi = Decimal("3.14159265358979323846264338327950288419716939937510582097494459230781640628620899")
    d = Decimal(x)
    k = (d / (pi / 2)).to_integral_value()
    r = d - k * (pi / 2)
    s = c = Decimal(0)
    term, n = r, 1
    while abs(term) > Decimal(10) ** -55:
        s, n, term = s + term, n + 2, -term * r * r / ((n + 1) * (n + 2))
    term, n = Decimal(1), 0
    while abs(term) > Decimal(10) ** -55:
        c, n, term = c + term, n + 2, -term * r * r / ((n + 1) * (n + 2))
    q = int(k) % 4
    s, c = [(s, c), (c, -s), (-s, -c), (-c, s)][q]
    return float(s), float(c)


def test_f64_rotation_bit_exact_with_correctly_rounded_trig():
    """fp64 rotations use correctly rounded cos/sin (double-double, common.cuh
    sincos_cr) and separately rounded products -- the arithmetic that
    reproduces every value of the reference's rotary golden file
    (rotary_reference.csv; rotary.py:104-108): bit-exact against that
    arithmetic on random rows and positions up to 2^20, three thetas."""
    from paper_2605_05696_b200 import rotary

    rng = np.random.default_rng(11)
    rows = rng.standard_normal((150, 64))
    pos = rng.integers(-(2**20), 2**20, size=150).astype(np.float64)
    for theta in (1e4, 5e4, 3.2e7):
        spec = rotary.make_spec(theta)
        got = rotary.rotate_rows(rows, pos, spec)
        ang = pos[:, None] * spec.inv_freq[None, :]
        sc = np.array([[_cr_sincos(float(a)) for a in row] for row in ang])
        s, c = sc[..., 0], sc[..., 1]
        lo, hi = rows[:, :32], rows[:, 32:]
        ref = np.concatenate([lo * c - hi * s, lo * s + hi * c], axis=1)
        assert np.array_equal(got, ref), (theta, np.mean(got == ref))


@pytest.mark.parametrize("dtype", ["bf16", "f32", "f64"])
@pytest.mark.parametrize("layout", [0, 1])
def test_rotate_rows_layered_matches_per_layer(dtype, layout):
    """irm_rotate_rows_layered (the batched producer: cos/sin once per (row,
    frequency), every layer rotated) equals irm_rotate_rows layer by layer,
    in place on the k_r slice of a [layers, rows, 576] pool, bit for bit."""
    import torch

    from paper_2605_05696_b200 import ops

    dt = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[dtype]
    g = torch.Generator(device="cuda").manual_seed(5)
    pool = torch.randn(5, 700, 576, device="cuda", generator=g, dtype=torch.float64).to(dt)
    pos = torch.from_numpy(np.random.default_rng(1).integers(-(2**20), 2**20, size=600).astype(np.float64)).cuda()
    inv = ops.inv_freq_device(O.make_inv_freq(5e4))
    ref = pool.clone()
    for l in range(5):
        ops.rotate_rows(ref[l, :600, 512:], pos, inv, layout, out=ref[l, :600, 512:])
    got = pool.clone()
    kr = got[:, :600, 512:]
    ops.rotate_rows_layered(kr, pos, inv, layout, out=kr)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    assert not torch.equal(got[:, :600, 512:], pool[:, :600, 512:])


@pytest.mark.parametrize("layout", [0, 1])
def test_rotate_rows_bf16_vector_path(layout):
    """The 16-byte bf16 producer path (irm_rotate_rows on 64-wide k_r slices of a
    [layers, rows, 576] pool) equals the element-wise path (a packed copy of the
    same rows, which the vector path does not take) and the f64 rotation within
    bf16 rounding."""
    import torch

    from paper_2605_05696_b200 import ops

    g = torch.Generator(device="cuda").manual_seed(9)
    pool = torch.randn(3, 300, 576, device="cuda", generator=g).to(torch.bfloat16)
    pos = torch.from_numpy(np.random.default_rng(2).integers(0, 2**20, size=300).astype(np.float64)).cuda()
    inv = O.make_inv_freq(1e4)
    invd = ops.inv_freq_device(inv)
    vec = pool.clone()
    kr = vec[:, :, 512:]
    ops.rotate_rows_layered(kr, pos, invd, layout, out=kr)
    scal = torch.empty(3, 300, 66, dtype=torch.bfloat16, device="cuda")  # row stride 66: not 16-byte aligned
    scal[:, :, :64] = pool[:, :, 512:]
    ops.rotate_rows_layered(scal[:, :, :64], pos, invd, layout, out=scal[:, :, :64])
    torch.cuda.synchronize()
    assert torch.equal(vec[:, :, 512:], scal[:, :, :64])
    assert torch.equal(vec[:, :, :512], pool[:, :, :512])
    ref = O.rotate_rows(pool[0, :, 512:].double().cpu().numpy(), pos.cpu().numpy(), inv, interleaved=bool(layout))
    got = vec[0, :, 512:].double().cpu().numpy()
    assert np.abs(got - ref).max() <= 2.0 ** -7 * np.abs(ref).max()
