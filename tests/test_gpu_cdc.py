"""GPU parity: K1 (CDC + xxh64) and K2 (xxh64 spans) against the reference's
golden chunk tables and the oracle. Bit-exact (start, len, fp, forced)."""

import numpy as np
import pytest

from inputs import CDC_CASES, cdc_case_inputs
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["auto", "fused", "split", "fused-table", "split-table"])
def pkg(request):
    """Both K1 forms (IRM_CDC_FORM, read on every call) and the size-based default, with
    the Gear values computed from the seed (default) or read from the device table."""
    import functools
    import os

    from paper_2605_05696_b200 import chunking, fingerprint, ops

    os.environ.pop("IRM_CDC_FORM", None)
    form, _, table = request.param.partition("-")
    if form != "auto":
        os.environ["IRM_CDC_FORM"] = form
    orig = ops.cdc_xxh64
    if table:
        ops.cdc_xxh64 = functools.partial(orig, gear_from_table=True)
    yield chunking, fingerprint, ops
    ops.cdc_xxh64 = orig
    os.environ.pop("IRM_CDC_FORM", None)


def test_gear_table_device(pkg, constants):
    chunking, _, ops = pkg
    g = ops.gear_table_device().cpu().numpy().view(np.uint64)
    assert np.array_equal(g, O.gear_table())
    assert f"{int(g[0]):016x}" == "b716d0295a22ecda"
    assert chunking.gear_table()[:8] == [int(x, 16) for x in [
        "b716d0295a22ecda", "815540ed8113475b", "836c8e91404c3cca", "27c45423b48fceb0",
        "5addf46622021c40", "244085f2e9dc6d8a", "1cb32fd04fa475f3", "59535b192c89249e"]]
    assert list(chunking.canonical_marker()) == constants["marker"]


def test_xxh64_kats(pkg, constants):
    _, fingerprint, _ = pkg
    assert fingerprint.fingerprint([]) == fingerprint.XXH64_EMPTY
    assert fingerprint.fingerprint_bytes(b"a") == 0xD24EC4F1A98C6E5B
    assert fingerprint.fingerprint_bytes(b"abc") == 0x44BC2CF5AD770999
    assert fingerprint.fingerprint_bytes(b"Hello, world!") == 0xF58336A78B6F9476
    for s, hexv in constants["xxh64_bytes"].items():
        assert f"{fingerprint.fingerprint_bytes(s.encode()):016x}" == hexv
    for case in constants["fingerprint_tokens"]:
        assert f"{fingerprint.fingerprint(case['tokens']):016x}" == case["fp"]
    # library oracle on the reference's own vector (test_fingerprint.py:18-24)
    assert fingerprint.fingerprint([1, 2, 3, 0xFFFFFFFF]) == O.fingerprint([1, 2, 3, 0xFFFFFFFF])


def test_sliding_and_fixed_block(pkg):
    chunking, fingerprint, _ = pkg
    rng = np.random.default_rng(1)
    toks = [int(t) for t in rng.integers(0, 2**32, size=300, dtype=np.uint64)]
    sl = fingerprint.sliding_fingerprints(toks, 64)
    assert len(sl) == 237
    for off, fp in sl[::17]:
        assert fp == O.fingerprint(toks[off:off + 64])
    assert fingerprint.sliding_fingerprints(toks[:10], 64) == []
    blocks = chunking.fixed_block_chunk(toks, 128)
    assert [(c.start, c.len) for c in blocks] == [(0, 128), (128, 128), (256, 44)]
    assert blocks[-1].forced == chunking.Forced.STREAM_END
    assert all(c.fingerprint == O.fingerprint(toks[c.start:c.end]) for c in blocks)


@pytest.mark.parametrize("name", sorted(CDC_CASES))
def test_cdc_golden(pkg, name, golden_cdc):
    chunking, _, _ = pkg
    case = CDC_CASES[name]
    tokens, pins = cdc_case_inputs(case)
    params = chunking.ChunkerParams(mask_exponent=case["k"], min_size=case["min"], max_size=case["max"],
                                    marker_pinned=case.get("pinned", True))
    chunks = chunking.cdc_chunk([int(t) for t in tokens], params, pins)
    g = golden_cdc[name]
    assert [c.start for c in chunks] == g["start"].tolist()
    assert [c.len for c in chunks] == g["len"].tolist()
    assert [c.fingerprint for c in chunks] == [int(x) for x in g["fp"]]
    codes = {chunking.Forced.NONE: 0, chunking.Forced.MAX_CLAMP: 1, chunking.Forced.MARKER: 2,
             chunking.Forced.STREAM_END: 3}
    assert [codes[c.forced] for c in chunks] == g["forced"].tolist()


def test_cdc_batched_random_streams(pkg):
    """Many streams of random length with random pins in one launch vs the oracle."""
    chunking, _, _ = pkg
    rng = np.random.default_rng(7)
    for k, mn, mx in [(7, 32, 512), (3, 1, 9), (12, 64, 100), (1, 2, 3)]:
        lens = rng.integers(0, 6000, size=64)
        lens[:3] = [0, 1, 33]
        streams = [rng.integers(0, 2**32, size=int(n), dtype=np.uint64).astype(np.uint32) for n in lens]
        pins = [set(rng.integers(-3, int(n) + 3, size=int(rng.integers(0, 12))).tolist()) for n in lens]
        params = chunking.ChunkerParams(mask_exponent=k, min_size=mn, max_size=mx)
        table = chunking.cdc_chunk_batch(streams, params, pins)
        st, ln, fp, fo, off = table.to_host()
        for s in range(len(streams)):
            a, b = off[s], off[s + 1]
            ost, oln, ofp, ofo = O.cdc_chunk(streams[s], k, mn, mx, pins[s])
            assert np.array_equal(st[a:b], ost) and np.array_equal(ln[a:b], oln)
            assert np.array_equal(fp[a:b], ofp) and np.array_equal(fo[a:b], ofo), (k, mn, mx, s)


def test_cdc_full_size_properties(pkg):
    """128K-token streams (config 4 size): tiling, clamp bounds and a
    checksum of fingerprints against the oracle."""
    chunking, _, _ = pkg
    rng = np.random.default_rng(11)
    streams = [rng.integers(0, 2**32, size=131072, dtype=np.uint64).astype(np.uint32) for _ in range(4)]
    params = chunking.ChunkerParams()
    table = chunking.cdc_chunk_batch(streams, params, [set(), {4095, 4159}, {0, 131071}, set()])
    st, ln, fp, fo, off = table.to_host()
    for s, toks in enumerate(streams):
        a, b = off[s], off[s + 1]
        assert st[a] == 0 and (st[a + 1:b] == st[a:b - 1] + ln[a:b - 1]).all()
        assert st[b - 1] + ln[b - 1] == toks.size
        free = fo[a:b - 1] == 0
        assert (ln[a:b - 1][free] >= 32).all() and (ln[a:b] <= 512).all()
        o = O.cdc_chunk(toks, pins=[set(), {4095, 4159}, {0, 131071}, set()][s])
        assert np.bitwise_xor.reduce(fp[a:b]) == np.bitwise_xor.reduce(o[2])
        assert np.array_equal(fp[a:b], o[2])


def test_cdc_empty_and_validation(pkg):
    chunking, _, _ = pkg
    assert chunking.cdc_chunk([], chunking.ChunkerParams()) == []
    with pytest.raises(ValueError):
        chunking.ChunkerParams(mask_exponent=0)
    with pytest.raises(ValueError):
        chunking.ChunkerParams(min_size=512, max_size=512)
    table = chunking.cdc_chunk_batch([[], [], []], chunking.ChunkerParams())
    assert table.chunk_off.cpu().tolist() == [0, 0, 0, 0]
