"""Seeded inputs for the golden fixtures (no reference import needed).

Both ``make_golden.py`` (reference side, build container) and the parity tests
(GPU box) regenerate the exact same inputs from these case tables.
"""

from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64_fill(seed: int, n: int) -> np.ndarray:
    """Vectorised splitmix64 stream (reference rng.py:17-38)."""
    with np.errstate(over="ignore"):
        state = np.uint64(seed) + np.arange(1, n + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)
        z = state
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


GEAR = splitmix64_fill(0x49524D494E53554C, 65536)


def rand_tokens(seed: int, n: int) -> np.ndarray:
    return np.random.Generator(np.random.PCG64(seed)).integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)


def marker_tokens() -> np.ndarray:
    with np.errstate(over="ignore"):
        s = np.uint64(0x49524D494E53554C) ^ np.uint64(64)
        s2 = splitmix64_fill(int(s), 1)[0]
    return (splitmix64_fill(int(s2), 64) & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def _adversarial(seed: int, n: int) -> np.ndarray:
    """Tokens whose Gear entries sit next to 0 / 2^64: the rolling state then
    hugs the wrap-around, which is where the warp-parallel MSB speculation of
    the CUDA scan is undetermined and must fall back to exact resolution."""
    order = np.argsort(GEAR)
    lo = order[:8].astype(np.uint32)          # gear ~ 0
    hi = order[-8:].astype(np.uint32)         # gear ~ 2^64
    rng = np.random.Generator(np.random.PCG64(seed))
    pick = rng.integers(0, 4, size=n)
    rnd = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    toks = np.where(pick == 0, lo[rng.integers(0, 8, size=n)],
                    np.where(pick == 1, hi[rng.integers(0, 8, size=n)],
                             np.where(pick == 2, hi[0], rnd)))
    # high 16 bits are ignored by the table index; randomise them
    return (toks & np.uint32(0xFFFF)) | (rnd & np.uint32(0xFFFF0000))


def cdc_case_inputs(case: dict):
    kind = case.get("kind", "random")
    n = case["n"]
    if kind == "random":
        tokens = rand_tokens(case["seed"], n)
    elif kind == "marker":
        pre = rand_tokens(case["seed"], case["prefix"])
        body = rand_tokens(case["seed"] + 1, n - case["prefix"] - 64)
        tokens = np.concatenate([pre, marker_tokens(), body])
    elif kind == "const":
        tokens = np.full(n, case["value"], np.uint32)
    elif kind == "adversarial":
        tokens = _adversarial(case["seed"], n)
    elif kind == "hi_const":
        tokens = np.full(n, int(np.argsort(GEAR)[-1 - case.get("rank", 0)]), np.uint32)
    elif kind == "lo_const":
        tokens = np.full(n, int(np.argsort(GEAR)[case.get("rank", 0)]), np.uint32)
    else:
        raise ValueError(kind)
    pins = list(case.get("pins", []))
    if "pin_every" in case:
        pins += list(range(case["pin_every"] - 1, n, case["pin_every"]))
    if kind == "marker":
        s = case["prefix"]
        pins += [s - 1, s + 63] if s > 0 else [63]
    return tokens, set(pins)


CDC_CASES = {
    "empty": dict(n=0, seed=1, k=7, min=32, max=512),
    "short20": dict(n=20, seed=2, k=7, min=32, max=512),
    "exact32": dict(n=32, seed=3, k=7, min=32, max=512),
    "tile5000": dict(n=5000, seed=3, k=7, min=32, max=512),
    "stats100k": dict(n=100_000, seed=77, k=7, min=32, max=512),
    "k20_maxclamp": dict(n=2000, seed=4, k=20, min=32, max=512),
    "k1": dict(n=3000, seed=5, k=1, min=32, max=512),
    "min1_max2": dict(n=777, seed=6, k=1, min=1, max=2),
    "min1_k3": dict(n=2000, seed=7, k=3, min=1, max=40),
    "small_params_pins": dict(n=4000, seed=8, k=3, min=4, max=9, pins=[0, 1, 2, 5, 100, 101, 3999]),
    "marker_pinned": dict(kind="marker", n=1564, prefix=500, seed=21, k=7, min=32, max=512),
    "marker_at_start": dict(kind="marker", n=1064, prefix=0, seed=22, k=7, min=32, max=512),
    "marker_pins_disabled": dict(kind="marker", n=1064, prefix=500, seed=30, k=7, min=32, max=512, pinned=False),
    "pins_edges": dict(n=3000, seed=9, k=7, min=32, max=512, pins=[-5, 0, 10, 11, 12, 511, 512, 2999, 3003]),
    "pin_every_37": dict(n=20_000, seed=10, k=7, min=32, max=512, pin_every=37),
    "pin_every_1000": dict(n=50_000, seed=11, k=7, min=32, max=512, pin_every=1000),
    "long_131k": dict(n=131_072, seed=12, k=7, min=32, max=512, pins=[4095, 4159, 70000]),
    "const_zero": dict(kind="const", n=3000, value=0, k=7, min=32, max=512),
    "adversarial": dict(kind="adversarial", n=50_000, seed=13, k=7, min=32, max=512),
    "adversarial_k2": dict(kind="adversarial", n=20_000, seed=14, k=2, min=2, max=300, pin_every=4321),
    "hi_const": dict(kind="hi_const", n=5000, k=7, min=32, max=512),
    "lo_const": dict(kind="lo_const", n=5000, k=4, min=8, max=200),
}


def rot_case_inputs(case: dict):
    rng = np.random.Generator(np.random.PCG64(case["seed"]))
    rows = rng.standard_normal((case["n"], 64))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    positions = np.concatenate([
        np.array([0, 1, -1, 1024, -1024, 2**20 - 1, -(2**17), 2**17], np.int64),
        rng.integers(-(2**20), 2**20, size=case["n"] - 8),
    ])
    return rows, positions


ROT_CASES = {f"theta_{int(t)}": dict(theta=t, n=512, seed=100 + i)
             for i, t in enumerate((1e4, 5e4, 3.2e7))}


TRACE_CASES = {
    # config 1 of BASELINE.json: ~4K-token agent_meta prompts with shifted CDC chunks
    "agent_meta_cfg1": dict(pattern="agent_meta", n_req=8, body_len=3900, seed=7),
    "agent_meta_nomark": dict(pattern="agent_meta", n_req=6, body_len=2000, seed=3, markers=False),
    "sysvar": dict(pattern="sysvar", n_req=10, body_len=2500, seed=1),
    "compact": dict(pattern="compact", n_req=12, body_len=2000, seed=2),
    "rerank": dict(pattern="rerank", n_req=20, body_len=2500, seed=4),
    "tool_variants": dict(pattern="tool_variants", n_req=12, body_len=2500, seed=5),
    "agent_meta_k5": dict(pattern="agent_meta", n_req=6, body_len=3000, seed=9, k=5),
    # S1 sub-window fallback (engine.py:116-139, 211-226): s1_enabled serve configs
    "compact_s1": dict(pattern="compact", n_req=10, body_len=3000, seed=11, s1=True),
    "compact_s1_k20": dict(pattern="compact", n_req=10, body_len=3000, seed=11, s1=True, k=20),
    "rerank_s1": dict(pattern="rerank", n_req=12, body_len=2500, seed=4, s1=True),
    "tool_variants_s1_k20": dict(pattern="tool_variants", n_req=10, body_len=2500, seed=5, s1=True, k=20),
    # a shared body behind per-request headers whose lengths differ by multiples of the window
    # but not of the 512-token max-clamp chunk (k=20): chunks miss, aligned sub-windows hit
    "s1_shift": dict(custom="s1_shift", n_req=10, body_len=4000, seed=21, s1=True, k=20, window=128),
    "s1_shift_w64": dict(custom="s1_shift", n_req=10, body_len=3000, seed=22, s1=True, k=20, window=64),
    "s1_shift_k7": dict(custom="s1_shift", n_req=8, body_len=3000, seed=23, s1=True, k=7, window=128),
}


def custom_trace(case: dict):
    """Requests (lists of (kind, tokens, shared_id) segments) of the custom trace cases."""
    assert case["custom"] == "s1_shift"
    rng = np.random.default_rng(case["seed"])
    w = case["window"]
    body = [int(t) for t in rng.integers(0, 2**32, size=case["body_len"], dtype=np.uint64)]
    reqs = []
    for i in range(case["n_req"]):
        hdr_len = 100 + w * (i % 5) + 512 * (i // 5)  # i and i + 5: same shift mod 512 -> PIC hits
        hdr = [int(t) for t in rng.integers(0, 2**32, size=hdr_len, dtype=np.uint64)]
        reqs.append([("header", hdr, None), ("body", body, "s1_body")])
    return reqs


# K0 / radix.py: operation sequences (insert or query, with a token sequence each)
RADIX_CASES = {
    # the reference's own randomized test shape (test_radix.py:75-90): alphabet 6, lengths 0..14
    "small_alphabet": dict(kind="small", n_ops=3000, seed=2024),
    # long sequences sharing prefixes that diverge at random depths (u32 tokens)
    "long_shared": dict(kind="long", n_ops=160, seed=77),
    # serve-loop shape: shared header, random metadata, shared body (engine.py:170, 228)
    "agent_meta": dict(kind="agent", n_ops=48, seed=5),
}


def radix_case_inputs(case: dict):
    """-> list of (is_insert, np.uint32 tokens)."""
    rng = np.random.default_rng(case["seed"])
    ops = []
    if case["kind"] == "small":
        for _ in range(case["n_ops"]):
            seq = rng.integers(0, 6, size=int(rng.integers(0, 15))).astype(np.uint32)
            ops.append((bool(rng.random() < 0.5), seq))
    elif case["kind"] == "long":
        bases = [rng.integers(0, 2**32, size=6000, dtype=np.uint64).astype(np.uint32) for _ in range(4)]
        for _ in range(case["n_ops"]):
            b = bases[int(rng.integers(0, 4))].copy()
            n = int(rng.integers(1, 6000))
            cut = int(rng.integers(0, n))
            b[cut:n] = rng.integers(0, 2**32, size=n - cut, dtype=np.uint64).astype(np.uint32)
            ops.append((bool(rng.random() < 0.6), b[:n].copy()))
    else:
        header = rng.integers(0, 2**32, size=200, dtype=np.uint64).astype(np.uint32)
        body = rng.integers(0, 2**32, size=3000, dtype=np.uint64).astype(np.uint32)
        for i in range(case["n_ops"]):
            meta = rng.integers(0, 2**32, size=int(rng.integers(0, 40)), dtype=np.uint64).astype(np.uint32)
            seq = np.concatenate([header[:int(rng.integers(150, 201))], meta, body[:int(rng.integers(0, 3000))]])
            ops.append((i % 3 != 2, seq))  # two of three requests are inserted after matching
    return ops
