"""GPU parity: K3 chunk store and the KvRegistry drop-in.

Mirrors the reference's registry tests (tests/test_registry.py:59-188) on the
device-backed registry, against golden materialize outputs produced by the
reference (tests/golden/registry.npz), plus a randomized check of the batched
first-writer-wins store against a sequential dict model."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def M():
    from paper_2605_05696_b200 import fingerprint, ops, registry, rotary

    return registry, rotary, fingerprint, ops


def make_registry(M, theta=1e4, seed=0):
    registry, rotary, _, _ = M
    p = registry.SyntheticKvParams(seed=seed)
    return registry.KvRegistry(p, rotary.make_spec(theta, p.kr_dim)), p


def test_store_batched_first_writer_wins(M):
    _, _, _, ops = M
    rng = np.random.default_rng(3)
    store = ops.ChunkStore(max_entries=5000)
    model: dict[int, tuple[int, int, int]] = {}  # fp -> (entry, p_src, row)
    rows_used = 0
    order0 = 0
    for batch in range(6):
        n = int(rng.integers(1, 1500))
        pool_fps = rng.integers(0, 2**64, size=400, dtype=np.uint64)
        fps = pool_fps[rng.integers(0, 400, size=n)]
        if batch == 2:
            fps[:3] = np.uint64(0xFFFFFFFFFFFFFFFF)  # the empty-key sentinel is a legal fingerprint
        p = rng.integers(0, 100000, size=n).astype(np.int64)
        ln = rng.integers(1, 513, size=n).astype(np.int32)
        probe = (rng.random(n) > 0.1).astype(np.uint8)
        order = order0 + np.arange(n, dtype=np.int64)
        order0 += n
        d = lambda a: torch.from_numpy(a).cuda()
        hit, entry, p_src, row = (t.cpu().numpy() for t in store.lookup_insert(
            d(fps.view(np.int64)), d(order), d(p), d(ln), d(probe)))
        for i in range(n):
            f = int(fps[i])
            if not probe[i]:
                assert hit[i] == -1
                continue
            if f in model:
                e, ps, r = model[f]
                assert (hit[i], entry[i], p_src[i], row[i]) == (1, e, ps, r), i
            else:
                model[f] = (len(model), int(p[i]), rows_used)
                assert (hit[i], entry[i], p_src[i], row[i]) == (0, len(model) - 1, p[i], rows_used)
                rows_used += int(ln[i])
        ne, nr, flags = store.counts()
        assert (ne, nr, flags) == (len(model), rows_used, 0)
    look = store.lookup(torch.from_numpy(np.array(list(model.keys()), np.uint64).view(np.int64)).cuda())
    assert look.cpu().tolist() == [v[0] for v in model.values()]


def test_insert_lookup_roundtrip(M):
    _, _, fingerprint, _ = M
    reg, _ = make_registry(M)
    tokens = [1, 2, 3] * 20
    fp = fingerprint.fingerprint(tokens)
    entry = reg.insert(fp, tokens, p_src=100)
    assert reg.lookup(fp) is entry
    assert entry.p_src == 100 and entry.chunk_len == len(tokens) and fp in reg


def test_first_writer_wins_and_pool_accounting(M):
    _, _, fingerprint, _ = M
    reg, _ = make_registry(M)
    tokens = list(range(40))
    fp = fingerprint.fingerprint(tokens)
    first = reg.insert(fp, tokens, p_src=10)
    assert reg.insert(fp, tokens, p_src=999) is first
    assert reg.lookup(fp).p_src == 10 and len(reg) == 1
    assert reg.pool_bytes() == 40 * 512 * 8


def test_entries_sorted_by_epoch(M):
    _, _, fingerprint, _ = M
    reg, _ = make_registry(M)
    for i in range(5):
        tokens = [i] * 40
        reg.insert(fingerprint.fingerprint(tokens), tokens, p_src=i)
    assert [e.insert_epoch for e in reg.entries()] == list(range(5))


@pytest.mark.parametrize("theta", [1e4, 5e4, 3.2e7])
def test_materialize_golden(M, theta, golden_registry):
    registry, rotary, fingerprint, _ = M
    g = golden_registry[f"theta_{int(theta)}"]
    reg, _ = make_registry(M, theta)
    tokens = [int(t) for t in g["tokens"]]
    entry = reg.insert(fingerprint.fingerprint(tokens), tokens, p_src=512)
    assert np.array_equal(entry.c_kv, golden_registry["theta_10000"]["c_kv"])
    assert np.abs(entry.kr_base - g["kr_base"]).max() <= 1e-13
    for p in (512, 64, 1536, 2048, 70000):
        for prec in rotary.Precision:
            m = reg.materialize(entry, p, prec)
            ref = g[f"k_r_{p}_{prec.value}"]
            assert m.c_kv is entry.c_kv and m.delta == p - 512 and m.multiplies == 96 * 64
            if prec == rotary.Precision.F64:
                assert np.abs(m.k_r - ref).max() <= 1e-12
            else:
                # rounding of (f64 up to 1 ulp apart) values: equal except at rare ties
                mism = np.mean(m.k_r != ref)
                assert mism <= 0.002, mism
                assert O.rel_l2(m.k_r, ref) <= 1e-6
    assert np.array_equal(reg.materialize(entry, 512).k_r, entry.kr_base)  # delta 0 exact


def test_materialize_vs_fresh_prefill(M):
    registry, rotary, fingerprint, _ = M
    reg, _ = make_registry(M)
    rng = np.random.default_rng(13)
    tokens = [int(t) for t in rng.integers(0, 2**32, size=96)]
    entry = reg.insert(fingerprint.fingerprint(tokens), tokens, p_src=512)
    _, kr_raw = reg.fresh_rows(tokens)
    for p, tol, prec in [(1536, 1e-9, rotary.Precision.F64), (64, 1e-9, rotary.Precision.F64),
                         (2048, 5e-3, rotary.Precision.BF16E), (3000, 1e-6, rotary.Precision.F32)]:
        out = reg.materialize(entry, p, prec)
        fresh = O.rotate_rows(kr_raw, p + np.arange(96), O.make_inv_freq(1e4))
        assert O.rel_l2(out.k_r, fresh) <= tol
    assert reg.materialize(entry, 64).delta == -448
    with pytest.raises(ValueError):
        reg.materialize(entry, -1)


def test_naive_reuse(M):
    _, _, fingerprint, _ = M
    reg, _ = make_registry(M)
    rng = np.random.default_rng(14)
    tokens = [int(t) for t in rng.integers(0, 2**32, size=64)]
    entry = reg.insert(fingerprint.fingerprint(tokens), tokens, p_src=0)
    assert np.array_equal(reg.naive_reuse(entry, 0).k_r, reg.materialize(entry, 0).k_r)
    assert reg.naive_reuse(entry, 100).multiplies == 0


def test_detect_spec(M):
    _, rotary, _, _ = M
    spec = rotary.make_spec(1e4)
    good = rotary.detect_spec(spec, lambda p: rotary.rotate(rotary.KrVector(rotary.probe_base_vector(64)), p, spec))
    assert good.ok
    wrong = rotary.make_spec(5e4)
    bad = rotary.detect_spec(spec, lambda p: rotary.rotate(rotary.KrVector(rotary.probe_base_vector(64)), p, wrong))
    assert not bad.ok and bad.best_fit_theta == 5e4


def test_sharded_store_single_rank_nccl(M):
    """K6 exchange over NCCL (world 1) reproduces the plain device store."""
    import os

    import torch.distributed as dist

    from paper_2605_05696_b200 import shard

    _, _, _, ops = M
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29537")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(8)
        pool_fps = rng.integers(0, 2**64, size=50, dtype=np.uint64)
        fps = pool_fps[rng.integers(0, 50, size=400)].view(np.int64)
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        order = np.arange(400, dtype=np.int64) * 3
        p = rng.integers(0, 9999, size=400).astype(np.int64)
        ln = rng.integers(1, 100, size=400).astype(np.int32)
        plain = ops.ChunkStore(1024)
        hit_a, _, ps_a, row_a = plain.lookup_insert(d(fps), d(order), d(p), d(ln))
        sh = shard.ShardedStore(ops.ChunkStore(1024), novel_rows=1 << 20)
        hit_b, ps_b, row_b, own = sh.lookup_insert(d(fps), d(order), d(p), d(ln))
        assert torch.equal(hit_a.cpu(), hit_b.cpu()) and torch.equal(ps_a.cpu(), ps_b.cpu())
        assert (own == 0).all()
        # world 1: the owner's per-writer bump allocator is the plain store's row scan
        assert torch.equal(row_a.cpu(), row_b.cpu())
        sh.check()
    finally:
        dist.destroy_process_group()


def test_registry_store_grows(M):
    """A registry created with room for 4 entries keeps serving: the device store is
    rebuilt larger (same ids, rows, p_src) and lookups still hit."""
    registry, rotary, _, ops = M
    reg = registry.KvRegistry(registry.SyntheticKvParams(), rotary.make_spec(1e4), max_entries=4)
    entries = [reg.insert(1000 + i, [7 * i + j for j in range(3 + i)], 40 + i) for i in range(11)]
    assert reg.store.max_entries >= 11 and len(reg) == 11
    for i, e in enumerate(entries):
        assert reg.lookup(1000 + i) is e and e.p_src == 40 + i and e.chunk_len == 3 + i
    assert reg.insert(1003, [1, 2, 3], 999) is entries[3]  # first writer still wins
