"""GPU: capacity limits and degenerate sizes fail loudly or do nothing, never
corrupt: a full chunk store / prefix index / first-writer row range / replica
region raise on their host check; zero-chunk gathers, empty prefix batches and
empty query sets are no-ops; the per-chunk device count of K4 bounds its work."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_store_entries_overflow_raises():
    from paper_2605_05696_b200 import ops

    store = ops.ChunkStore(max_entries=8)
    n = 20
    fp = torch.arange(1, n + 1, dtype=torch.int64, device="cuda") * 0x9E3779B97F4A7C15
    hit, entry, p_src, row = store.lookup_insert(fp, torch.arange(n, device="cuda"),
                                                 torch.arange(n, device="cuda") + 100,
                                                 torch.full((n,), 4, dtype=torch.int32, device="cuda"))
    with pytest.raises(RuntimeError, match="overflow"):
        store.counts()


def test_prefix_index_full_raises():
    from paper_2605_05696_b200.radix import DeviceRadixTree

    tree = DeviceRadixTree(max_prefixes=64, max_tokens=1 << 14, max_sequences=16, grow=False)  # 128 slots
    rng = np.random.default_rng(1)
    tree.run_ops([rng.integers(0, 2**32, size=500, dtype=np.uint64).astype(np.uint32)], [True], [False])
    with pytest.raises(RuntimeError, match="full"):
        tree.check()


def test_prefix_index_arena_capacity():
    from paper_2605_05696_b200.radix import DeviceRadixTree

    tree = DeviceRadixTree(max_prefixes=1 << 10, max_tokens=100, max_sequences=4, grow=False)
    with pytest.raises(ValueError, match="arena"):
        tree.insert(list(range(101)), "x")
    assert tree.run_ops([], [], [])[0].numel() == 0  # empty batch: nothing launched, nothing inserted


def test_sharded_rows_overflow_raises():
    import os

    import torch.distributed as dist

    from paper_2605_05696_b200 import ops, shard

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29551")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        sh = shard.ShardedStore(ops.ChunkStore(1024), novel_rows=64)
        n = 10
        fp = torch.arange(1, n + 1, dtype=torch.int64, device="cuda") * 0x51ED2701
        sh.lookup_insert(fp, torch.arange(n, device="cuda"), torch.zeros(n, dtype=torch.int64, device="cuda"),
                         torch.full((n,), 10, dtype=torch.int32, device="cuda"))  # 100 rows > 64
        with pytest.raises(RuntimeError, match="full"):
            sh.check()
    finally:
        dist.destroy_process_group()


def test_replica_region_overflow_raises():
    from paper_2605_05696_b200 import ops, shard

    pools = [torch.zeros(1, 64, 576, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    cache = shard.ReplicaCache(pools[0], 60, pools, 0, ops.ChunkStore(64))  # 4 replica rows
    grow = shard.encode_row(1, torch.tensor([0, 10], device="cuda"))
    cache.localize(grow, torch.tensor([3, 3], dtype=torch.int32, device="cuda"))
    with pytest.raises(RuntimeError, match="full"):
        cache.check()


def test_rotate_gather_zero_and_device_count():
    """n_dev (the device-side hit count) bounds K4's work: rows past it stay untouched."""
    from paper_2605_05696_b200 import ops

    pool = torch.randn(2, 256, 576, device="cuda").to(torch.bfloat16)
    out = torch.zeros(2, 256, 576, dtype=torch.bfloat16, device="cuda")
    src = torch.tensor([0, 100], dtype=torch.int64, device="cuda")
    dst = torch.tensor([0, 100], dtype=torch.int64, device="cuda")
    ln = torch.tensor([50, 50], dtype=torch.int32, device="cuda")
    delta = torch.zeros(2, dtype=torch.int64, device="cuda")
    inv = ops.inv_freq_device(np.power(1e4, -2.0 * np.arange(32) / 64))
    ops.rotate_gather(pool, out, src, dst, ln, delta, inv, n_dev=torch.zeros(1, dtype=torch.int64, device="cuda"))
    torch.cuda.synchronize()
    assert int(out.abs().sum()) == 0
    ops.rotate_gather(pool, out, src, dst, ln, delta, inv, n_dev=torch.ones(1, dtype=torch.int64, device="cuda"))
    torch.cuda.synchronize()
    assert torch.equal(out[:, :50], pool[:, :50]) and int(out[:, 100:].abs().sum()) == 0


def test_mla_degenerate_sizes():
    from paper_2605_05696_b200 import ops

    kv = torch.randn(1, 576, device="cuda").to(torch.bfloat16)
    q = torch.randn(1, 16, 576, device="cuda").to(torch.bfloat16)
    out, lse = ops.mla_reattach_prefill(q, kv, 1, 0, 192 ** -0.5)  # one key: softmax weight 1
    torch.cuda.synchronize()
    ref = kv[0, :512].float().expand(16, 512)
    assert float((out[0].float() - ref).abs().max()) <= 1e-2 * float(ref.abs().max())
    e_out, e_lse = ops.mla_reattach_prefill(q[:0], kv, 1, 0, 192 ** -0.5)  # no queries: nothing launched
    assert e_out.shape[0] == 0


def test_store_pool_rows_bound():
    """An insert whose rows would pass the latent pool is never published: its row
    is -1, later lookups miss it, and the sticky pool-full flag raises."""
    from paper_2605_05696_b200 import ops

    store = ops.ChunkStore(max_entries=64, pool_rows=100)
    n = 4
    fp = torch.arange(1, n + 1, dtype=torch.int64, device="cuda") * 0x9E3779B97F4A7C15
    hit, entry, p_src, row = store.lookup_insert(fp, torch.arange(n, device="cuda"),
                                                 torch.arange(n, device="cuda") + 100,
                                                 torch.full((n,), 40, dtype=torch.int32, device="cuda"))
    assert row.tolist() == [0, 40, -1, -1]  # 80 rows fit, the third chunk would end at 120
    assert store.lookup(fp).tolist()[:2] == [0, 1] and store.lookup(fp).tolist()[2:] == [-1, -1]
    with pytest.raises(RuntimeError, match="pool rows exhausted"):
        store.counts()


def test_frozen_workspaces_refuse_to_grow():
    """A graph-captured workspace is never replaced: a larger call raises."""
    from paper_2605_05696_b200 import ops

    store = ops.ChunkStore(max_entries=1 << 10)
    store.reserve(16)
    fp = torch.arange(1, 1001, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError, match="reserved"):
        store.lookup_insert(fp, torch.arange(1000, device="cuda"), torch.zeros(1000, dtype=torch.int64, device="cuda"),
                            torch.ones(1000, dtype=torch.int32, device="cuda"))
    ws = ops.CdcWorkspace()
    ws.get(1000, 2, 0, 32)
    ws.freeze()
    with pytest.raises(ValueError, match="frozen"):
        ws.get(1 << 20, 2, 0, 32)


def test_pipeline_request_longer_than_stride():
    """A host-loaded wave whose request would spill past req_stride is refused."""
    from paper_2605_05696_b200 import ops
    from paper_2605_05696_b200.pipeline import ReattachPipeline

    pool = torch.zeros(1, 4096, 576, dtype=torch.bfloat16, device="cuda")
    pipe = ReattachPipeline(ops.ChunkStore(1 << 10), pool, ops.inv_freq_device(np.power(1e4, -np.arange(32) / 32)),
                            2, 4096, 4, req_stride=1000)
    tok = torch.zeros(1500, dtype=torch.int32)
    with pytest.raises(ValueError, match="req_stride"):
        pipe.load(tok, torch.tensor([0, 900, 1500]), torch.zeros(3, dtype=torch.int64),
                  torch.zeros(1, dtype=torch.int64), torch.tensor([200, 0]))
