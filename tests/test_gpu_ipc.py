"""GPU, two processes on cuda:0 (gloo for the handle exchange): the K6 replica
fetch across processes. Each rank maps the other's latent pool through CUDA IPC
(shard.map_peer_pools), and ReplicaCache.localize pulls remote runs with
irm_copy_runs reading peer memory directly. NCCL cannot put two ranks on one
GPU; on an 8-GPU box the same mapping goes over NVLink."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, port, out_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_2605_05696_b200 import ops, shard

        torch.cuda.set_device(0)
        big = torch.full((3, 256, 576), float(rank + 1), dtype=torch.bfloat16, device="cuda")
        pool = big[1:]  # not at its allocation's base: the exported offset is non-zero
        pool[:, :, 1] = torch.arange(256, device="cuda").to(torch.bfloat16)
        peers = shard.map_peer_pools(pool)
        cache = shard.ReplicaCache(pool, 128, peers, rank, ops.ChunkStore(1 << 10))
        other = 1 - rank
        grow = shard.encode_row(other, torch.tensor([5, 40, 5], device="cuda"))
        ln = torch.tensor([3, 7, 3], dtype=torch.int32, device="cuda")
        local = cache.localize(grow, ln).cpu().tolist()
        torch.cuda.synchronize()
        p = pool.float().cpu()
        ok = local[0] == local[2] and local[0] >= 128 and int(cache.fetched_rows) == 10
        ok = ok and bool((p[:, local[0]:local[0] + 3, 0] == other + 1).all())
        ok = ok and bool((p[:, local[0]:local[0] + 3, 1] == torch.arange(5, 8).float()).all())
        ok = ok and bool((p[:, local[1]:local[1] + 7, 1] == torch.arange(40, 47).float()).all())
        ok = ok and torch.equal(peers[other][:, 100:110, :2].float().cpu(),
                                torch.stack([torch.full((2, 10), float(other + 1)),
                                             torch.arange(100, 110).float().expand(2, 10)], -1))
        out_q.put((rank, ok))
        dist.barrier()  # keep both pools alive until both ranks have read
    finally:
        dist.destroy_process_group()


def test_replica_fetch_across_processes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for pr in procs:
        pr.start()
    outs = dict(q.get(timeout=240) for _ in range(WORLD))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert outs == {0: True, 1: True}, outs


def test_peer_export_rejects_host_memory():
    import ctypes

    from paper_2605_05696_b200 import _native as N

    host = torch.zeros(16)
    h = ctypes.create_string_buffer(N.PEER_HANDLE_BYTES)
    off = ctypes.c_int64(0)
    rc = N.lib().irm_peer_export(ctypes.c_void_p(host.data_ptr()), h, ctypes.byref(off))
    with pytest.raises(ValueError, match="not a device allocation"):
        N.check(rc, "irm_peer_export")
