"""CPU, world size 2 over gloo: the hash-sharded store exchange (K6 host logic)
equals one sequential first-writer-wins store over the union of all ranks'
queries in global order (engine.py:197-223), and the replica cache fetches
remote latent rows once with the right contents."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_05696_b200 import shard

WORLD = 2
NOVEL_ROWS = 1 << 30


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _queries(seed, n_total=600):
    g = torch.Generator().manual_seed(seed)
    pool = torch.randint(-(2**62), 2**62, (120,), generator=g, dtype=torch.int64)
    pool[0] = -1  # the all-ones fingerprint (EMPTY sentinel of the device table) is legal
    fp = pool[torch.randint(0, 120, (n_total,), generator=g)]
    order = torch.arange(n_total, dtype=torch.int64) * 7 + 3
    p = torch.randint(0, 100000, (n_total,), generator=g)
    ln = torch.randint(1, 300, (n_total,), generator=g, dtype=torch.int32)
    probe = torch.rand(n_total, generator=g) > 0.1
    rank_of = torch.arange(n_total) % WORLD  # sessions round-robin over ranks
    return fp, order, p, ln, probe, rank_of


def _worker(rank, port, seed, out_q, pools):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from dict_store import DictStore

    try:
        fp, order, p, ln, probe, rank_of = _queries(seed)
        mine = torch.nonzero(rank_of == rank).flatten()
        store = shard.ShardedStore(DictStore(), novel_rows=NOVEL_ROWS)
        res = []
        for wave in range(3):  # three waves hitting the same sharded store
            sl = mine[wave::3]
            h, ps, row, own = store.lookup_insert(fp[sl], order[sl] + wave * 10**7, p[sl], ln[sl], probe[sl])
            res.append((sl, h, ps, row, own))
        store.check()

        # replica cache: pool rows hold (rank, row) stamps; the shared-memory pools of
        # both ranks stand in for the CUDA-IPC peer mappings of shard.map_peer_pools
        pool = pools[rank]
        cache = shard.ReplicaCache(pool, 32, pools, rank, DictStore())
        other = 1 - rank
        grow = shard.encode_row(other, torch.tensor([3, 10, 3, -1], dtype=torch.int64))
        grow[3] = -1
        local = cache.localize(grow, torch.tensor([4, 2, 4, 1]))
        ok = bool(local[0] == local[2]) and int(cache.fetched_rows) == 6 and int(cache.fetched_runs) == 2
        ok = ok and bool((pool[:, local[0]:local[0] + 4, 0] == other).all())
        ok = ok and bool((pool[:, local[0]:local[0] + 4, 1] == torch.arange(3, 7).float()).all())
        ok = ok and bool((pool[:, local[1]:local[1] + 2, 1] == torch.tensor([10.0, 11.0])).all())
        again = cache.localize(grow, torch.tensor([4, 2, 4, 1]))  # cached: no new rows
        ok = ok and int(cache.fetched_rows) == 6 and bool((again == local).all())
        cache.check()
        # plain lists: tensors would travel as shared-memory handles that vanish with this process
        res = [tuple(x.tolist() for x in r) for r in res]
        out_q.put((rank, res, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed", [1, 2])
def test_sharded_store_matches_sequential(seed):
    from dict_store import DictStore

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    pools = []
    for r in range(WORLD):
        pool = torch.zeros(2, 64, 3)
        pool[:, :, 0] = r
        pool[:, :, 1] = torch.arange(64, dtype=torch.float32)
        pools.append(pool.share_memory_())
    procs = [ctx.Process(target=_worker, args=(r, port, seed, q, pools)) for r in range(WORLD)]
    for pr in procs:
        pr.start()
    outs = [q.get(timeout=240) for _ in range(WORLD)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    fp, order, p, ln, probe, rank_of = _queries(seed)
    # sequential reference over the union, in global order (waves are time-ordered)
    rows = []
    for rank, res, ok in outs:
        assert ok, f"replica cache check failed on rank {rank}"
        for wave, (sl, h, ps, row, own) in enumerate(res):
            for k, i in enumerate(sl):
                rows.append((int(order[i]) + wave * 10**7, i, rank, wave, k, int(h[k]), int(ps[k]), int(row[k]),
                             int(own[k])))
    rows.sort()
    ref = DictStore()
    first: dict[int, tuple] = {}  # fp -> (writer rank, wave, position in the writer's wave)
    for ordk, i, rank, wave, k, h, ps, row, own in rows:
        if not probe[i]:
            assert h == -1
            continue
        f = int(fp[i])
        eh, _, eps, _ = ref.lookup_insert(fp[i:i + 1], torch.tensor([ordk]), p[i:i + 1], ln[i:i + 1])
        assert h == int(eh[0]) and ps == int(eps[0]), (i, h, int(eh[0]))
        if h == 0:
            first[f] = (rank, wave, k)
        assert own == int(shard.owner_of(fp[i:i + 1], WORLD)[0])
    # first-writer rows: owner o bump-allocates in [o * region, (o + 1) * region) of the writer's
    # pool, per writer, in the writer's (wave, query) order
    region = NOVEL_ROWS // WORLD
    nxt = {}
    grow = {}
    for rank, res, ok in sorted(outs):
        for wave, (sl, h, ps, row, own) in enumerate(res):
            for k, i in enumerate(sl):
                if h[k] == 0:
                    o = own[k]
                    grow[(rank, wave, k)] = (rank << shard.ROW_SHIFT) | (o * region + nxt.get((o, rank), 0))
                    nxt[(o, rank)] = nxt.get((o, rank), 0) + int(ln[i])
    for ordk, i, rank, wave, k, h, ps, row, own in rows:
        if probe[i]:
            assert row == grow[first[int(fp[i])]], (i, row)  # every query reads its first writer's rows


def _worker_uneven(rank, port, out_q):
    """Ranks with different query counts per call: the exchange pads to a common slot count."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from dict_store import DictStore

    try:
        g = torch.Generator().manual_seed(5)
        fps = torch.randint(-(2**62), 2**62, (40,), generator=g, dtype=torch.int64)
        n = 50 if rank == 0 else 70
        q = fps[torch.randint(0, 40, (n,), generator=torch.Generator().manual_seed(10 + rank))]
        order = torch.arange(n, dtype=torch.int64) * WORLD + rank
        store = shard.ShardedStore(DictStore(), novel_rows=1 << 20, slots=80)
        h, ps, row, own = store.lookup_insert(q, order, torch.arange(n) + 1000 * rank,
                                              torch.full((n,), 4, dtype=torch.int32))
        out_q.put((rank, q.tolist(), order.tolist(), h.tolist(), ps.tolist()))
    finally:
        dist.destroy_process_group()


def test_sharded_store_uneven_batches():
    from dict_store import DictStore

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_uneven, args=(r, port, q)) for r in range(WORLD)]
    for pr in procs:
        pr.start()
    outs = [q.get(timeout=240) for _ in range(WORLD)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    rows = sorted((o, r, i, f, h, ps) for r, fs, orders, hs, pss in outs
                  for i, (f, o, h, ps) in enumerate(zip(fs, orders, hs, pss)))
    ref = DictStore()
    for o, r, i, f, h, ps in rows:
        eh, _, eps, _ = ref.lookup_insert(torch.tensor([f]), torch.tensor([o]), torch.tensor([i + 1000 * r]),
                                          torch.tensor([4], dtype=torch.int32))
        assert (h, ps) == (int(eh[0]), int(eps[0]))


def _worker_fresh(rank, port, out_q, pools):
    """Rank 0 writes fp X first; rank 1 hits X in the SAME exchange (fresh: the
    writer has not produced the rows yet) and again one wave later."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from dict_store import DictStore

    try:
        store = shard.ShardedStore(DictStore(), novel_rows=32)
        cache = shard.ReplicaCache(pools[rank], 32, pools, rank, DictStore(), scratch_rows=8)
        fp = torch.tensor([0x1234567], dtype=torch.int64)
        ln = torch.tensor([3], dtype=torch.int32)
        seen = []
        for wave in range(2):
            order = torch.tensor([(wave * 2 + rank)], dtype=torch.int64)  # rank 0 first in each wave
            h, ps, row, own = store.lookup_insert(fp, order, torch.tensor([100 + rank]), ln)
            fresh = store.fresh
            local = cache.localize(torch.where(h == 1, row, torch.full_like(row, -1)),
                                   torch.where(h == 1, ln, torch.zeros_like(ln)), fresh=fresh & (h == 1))
            seen.append((int(h[0]), bool(fresh[0]), int(local[0]), len(cache.map.map)))
        cache.check()
        store.check()
        out_q.put((rank, seen))
    finally:
        dist.destroy_process_group()


def test_fresh_remote_hits_are_not_cached():
    """a same-exchange hit on another rank's first write is fetched into
    the per-wave scratch and never published in the replica map; one wave later
    (the writer's rows produced) it is fetched once and cached."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    pools = []
    for r in range(WORLD):
        pool = torch.zeros(1, 64, 3)
        pool[:, :, 0] = r
        pools.append(pool.share_memory_())
    procs = [ctx.Process(target=_worker_fresh, args=(r, port, q, pools)) for r in range(WORLD)]
    for pr in procs:
        pr.start()
    outs = dict(q.get(timeout=240) for _ in range(WORLD))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    (h0, f0, _, n0), (h0b, f0b, _, n0b) = outs[0]
    assert (h0, f0, n0) == (0, False, 0) and (h0b, f0b, n0b) == (1, False, 0)  # the writer never fetches
    (h1, f1, l1, n1), (h1b, f1b, l1b, n1b) = outs[1]
    assert (h1, f1, n1) == (1, True, 0), outs[1]  # same exchange: fresh, scratch, not cached
    assert l1 >= 64 - 2 * 8  # a scratch row
    assert (h1b, f1b, n1b) == (1, False, 1) and 32 <= l1b < 64 - 2 * 8  # next wave: cached replica row
    assert bool((pools[1][0, l1b:l1b + 3, 0] == 0).all())  # rank 0's rows
