"""CPU: pin the oracle (restated reference) to the reference's own outputs.

The fixtures under tests/golden/ were produced by the reference itself
(tests/golden/make_golden.py); the KATs are the reference tests' own
(test_acceptance.py:347-351, test_fingerprint.py:14-15, test_chunker.py:42-54).
"""

import numpy as np
import pytest

from oracle import oracle as O
from oracle import workloads as W
from goldens import load_npz
from inputs import (CDC_CASES, GEAR, RADIX_CASES, ROT_CASES, TRACE_CASES, cdc_case_inputs, custom_trace, marker_tokens,
                    radix_case_inputs, rot_case_inputs)


def test_gear_table_golden(constants):
    g = O.gear_table()
    assert g.size == 65536
    for i, hexv in constants["gear_sample"].items():
        assert f"{int(g[int(i)]):016x}" == hexv
    assert f"{int(np.bitwise_xor.reduce(g)):016x}" == constants["gear_xor_fold"]
    assert f"{int(g.sum(dtype=np.uint64)):016x}" == constants["gear_sum_mod64"]
    assert (GEAR == g).all()
    # reference golden file values (src/data/gear_reference.json:2-11)
    assert f"{int(g[0]):016x}" == "b716d0295a22ecda"


def test_marker_golden(constants):
    assert list(O.canonical_marker()) == constants["marker"]
    assert list(O.canonical_marker(1)) == constants["marker_seed1"]
    assert tuple(int(x) for x in marker_tokens()) == O.canonical_marker()


def test_xxh64_kats(constants):
    # test_acceptance.py:347-351 KATs
    assert O.xxh64(b"") == 0xEF46DB3751D8E999
    assert O.xxh64(b"a") == 0xD24EC4F1A98C6E5B
    assert O.xxh64(b"abc") == 0x44BC2CF5AD770999
    assert O.xxh64(b"Hello, world!") == 0xF58336A78B6F9476
    for s, hexv in constants["xxh64_bytes"].items():
        assert f"{O.xxh64(s.encode()):016x}" == hexv


def test_token_fingerprints(constants):
    for case in constants["fingerprint_tokens"]:
        assert f"{O.fingerprint(case['tokens']):016x}" == case["fp"]


@pytest.mark.parametrize("name", sorted(CDC_CASES))
def test_cdc_golden(name, golden_cdc):
    case = CDC_CASES[name]
    tokens, pins = cdc_case_inputs(case)
    st, ln, fp, fo = O.cdc_chunk(tokens, case["k"], case["min"], case["max"], pins,
                                 marker_pinned=case.get("pinned", True))
    g = golden_cdc[name]
    assert np.array_equal(st, g["start"]) and np.array_equal(ln, g["len"])
    assert np.array_equal(fp, g["fp"]) and np.array_equal(fo, g["forced"])


@pytest.mark.parametrize("name", sorted(ROT_CASES))
def test_rotation_golden(name, golden_rotary):
    case = ROT_CASES[name]
    rows, pos = rot_case_inputs(case)
    g = golden_rotary[name]
    inv = O.make_inv_freq(case["theta"])
    assert np.array_equal(inv, g["inv_freq"])
    out = O.rotate_rows(rows, pos, inv)
    assert np.array_equal(out, g["out"])
    assert np.array_equal(O.round_bf16(g["out"]), g["out_bf16"])


def test_interleaved_is_permutation_conjugate():
    # DSv2-form parity through the de-interleave identity
    rng = np.random.default_rng(3)
    rows = rng.standard_normal((50, 64))
    pos = rng.integers(-5000, 5000, size=50)
    inv = O.make_inv_freq(1e4)
    perm = np.concatenate([np.arange(0, 64, 2), np.arange(1, 64, 2)])  # interleaved -> half-split
    inter = O.rotate_rows(rows, pos, inv, interleaved=True)
    half = O.rotate_rows(rows[:, perm], pos, inv)
    assert np.allclose(inter[:, perm], half, rtol=0, atol=1e-15)


def test_synth_kv_golden(golden_registry):
    g = golden_registry["theta_10000"]
    toks = [int(t) for t in g["tokens"]]
    c = np.stack([O.synth_kv(t)[0] for t in toks])
    assert np.array_equal(c, g["c_kv"])


def test_registry_materialize_oracle(golden_registry):
    # kr_base = R(p_src + i) kr_raw, materialize = R(delta) kr_base, stores rounded
    for name, g in golden_registry.items():
        theta = float(name.split("_")[1])
        inv = O.make_inv_freq(theta)
        toks = [int(t) for t in g["tokens"]]
        kr_raw = np.stack([O.synth_kv(t)[1] for t in toks])
        kr_base = O.rotate_rows(kr_raw, 512 + np.arange(len(toks)), inv)
        assert np.array_equal(kr_base, g["kr_base"])
        for p in (512, 64, 1536, 2048, 70000):
            k = O.rotate_rows(kr_base, np.full(len(toks), p - 512), inv)
            assert np.array_equal(k, g[f"k_r_{p}_f64"])
            assert np.array_equal(k.astype(np.float32).astype(np.float64), g[f"k_r_{p}_f32"])
            assert np.array_equal(O.round_bf16(k), g[f"k_r_{p}_bf16e"])


@pytest.mark.parametrize("name", sorted(TRACE_CASES))
def test_trace_events_golden(name, golden_traces):
    case = dict(TRACE_CASES[name])
    k = case.pop("k", 7)
    s1, window = case.pop("s1", False), case.pop("window", 128)
    reqs = custom_trace(TRACE_CASES[name]) if "custom" in case else W.generate(**case)
    events, n_entries = W.serve_trace(reqs, k=k, s1=s1, window=window)
    g = golden_traces[name]
    assert n_entries == int(g["registry_len"][0])
    assert len(events) == g["req"].size
    for i, (ri, s, l, kl, fp, d) in enumerate(events):
        assert (ri, s, l, kl) == (g["req"][i], g["start"][i], g["length"][i], g["klass"][i])
        if kl == 1:
            assert fp == int(g["fp"][i]) and d == int(g["delta"][i]) and g["has_delta"][i]
        if kl == 2:  # S1 hit: the window's fingerprint, no delta
            assert fp == int(g["fp"][i]) and not g["has_delta"][i]


def test_threaded_batch_matches_single():
    rng = np.random.default_rng(5)
    lens = rng.integers(0, 3000, size=17)
    toks = rng.integers(0, 2**32, size=int(lens.sum()), dtype=np.uint64).astype(np.uint32)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    pins = [sorted(rng.choice(max(int(n), 1), size=min(3, int(n)), replace=False).tolist()) if n else [] for n in lens]
    pin_off = np.concatenate([[0], np.cumsum([len(p) for p in pins])]).astype(np.int64)
    pin_arr = np.array([x for p in pins for x in p], np.int64)
    out_off, counts, st, ln, fp, fo = O.cdc_batch(toks, off, pin_off, pin_arr, n_threads=4)
    for s in range(lens.size):
        a = O.cdc_chunk(toks[off[s]:off[s + 1]], pins=pins[s])
        o, c = out_off[s], counts[s]
        assert np.array_equal(a[0], st[o:o + c]) and np.array_equal(a[2], fp[o:o + c])


@pytest.mark.parametrize("case", sorted(RADIX_CASES))
def test_prefix_match_oracle_golden(case):
    """oracle.prefix_match (brute force) == the reference RadixTree on every query op."""
    g = load_npz("radix")[case]
    want_m, want_w = g["m"], g["witness"]
    inserted = []
    for i, (is_insert, seq) in enumerate(radix_case_inputs(RADIX_CASES[case])):
        if is_insert:
            inserted.append((i, seq))
            continue
        m, w = O.prefix_match(inserted, seq)
        assert m == want_m[i] and (-1 if w is None else w) == want_w[i], (case, i)


def test_mla_oracle_vs_reference_materialize():
    """K5's fp64 restatement (oracle/mla_ref.py), on the bf16 inputs the kernel sees,
    against attention over k_r rotated by the REFERENCE's KvRegistry.materialize
    (tests/golden/mla.npz): within the 4.7e-3 bound (the gap is bf16 input rounding)."""
    import torch

    from oracle.mla_ref import mla_reattach_ref

    c = load_npz("mla")["case"]
    q = torch.from_numpy(c["q_bf16"].view(np.int16)).view(torch.bfloat16)
    kv = torch.from_numpy(c["pool"][c["kv_rows"]]).to(torch.bfloat16)
    out, lse = mla_reattach_ref(q, kv, kv.shape[0] - q.shape[0], 192 ** -0.5, c["deltas"][c["kv_chunk"]],
                                O.make_inv_freq(float(c["theta"])))
    ref = torch.from_numpy(c["out"]).double()
    assert float((out - ref).norm() / ref.norm()) <= 4.7e-3
    assert float((lse - torch.from_numpy(c["lse"])).abs().max()) <= 2e-2


def test_prefix_lengths_sequential_matches_brute_force():
    """The checker's fast phase-1 oracle (bench.py parity) equals the brute force
    the reference pins RadixTree with (tests/test_radix.py:15-23)."""
    rng = np.random.default_rng(3)
    base = rng.integers(0, 4, size=400).astype(np.uint32)
    seqs = []
    for _ in range(250):
        n, cut = int(rng.integers(0, 400)), int(rng.integers(0, 400))
        s = base[:n].copy()
        s[min(cut, n):] = rng.integers(0, 4, size=max(n - cut, 0))
        seqs.append(s)
    fast = O.prefix_lengths_sequential(seqs, probe=16)
    assert fast == [O.prefix_match([(j, seqs[j]) for j in range(i)], seqs[i])[0] for i in range(len(seqs))]
