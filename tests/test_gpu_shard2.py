"""GPU, world sizes 2 and 4 on one B200 (processes on cuda:0, gloo carrying the
all-to-alls on CUDA tensors; NCCL cannot put two ranks on one GPU): the
sharded production step (pipeline.ReattachPipeline.run_overlapped_sharded, the
path bench.py times at N > 1) against one sequential first-writer-wins oracle
over all ranks' requests in global order (wave, request, rank), with the
chunks of each request in order (engine.py:181-226).

Checked on every rank and wave: the per-chunk service map (hit / novel /
carve-out) bit-exact, and every hit row of the per-request KV output against
the oracle's bf16 rotate+gather (registry.py:146-166) of the FIRST WRITER's
pool rows, c_KV bit-exact and k_r within bf16 rounding. Hits whose first
writer is another rank read rows fetched peer-to-peer into the replica
region (CUDA IPC mapping of the peer pool, irm_copy_runs)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def global_oracle(all_waves, novel_rows, WORLD):
    """Per rank, per wave: chunk records (code, writer, row, p_src, p, len, request)."""
    from oracle import oracle as O
    from test_gpu_pipeline import CARVE

    n_waves = len(all_waves[0])
    chunks = [[None] * n_waves for _ in range(WORLD)]
    for k in range(WORLD):
        for w, (tok, off, poff, pins, ms) in enumerate(all_waves[k]):
            recs = []
            for r in range(off.size - 1):
                st, ln, fp, _ = O.cdc_chunk(tok[off[r]:off[r + 1]], pins=pins[poff[r]:poff[r + 1]])
                recs += [(int(ms[r]) + s, l, f, r) for s, l, f in zip(st.tolist(), ln.tolist(), fp.tolist())]
            chunks[k][w] = recs
    # 1) novelty in global order: (wave, request, rank), chunks in order
    reg, novel = {}, set()
    for w in range(n_waves):
        n_req = max(all_waves[k][w][1].size - 1 for k in range(WORLD))
        for r in range(n_req):
            for k in range(WORLD):
                for j, (p, l, f, rr) in enumerate(chunks[k][w]):
                    if rr != r or p < CARVE or f in reg:
                        continue
                    reg[f] = (k, w, j, p)
                    novel.add((k, w, j))
    # 2) first-writer rows: owner o bump-allocates in its sub-range of the writer's pool,
    #    per writer, in the writer's (wave, chunk) order
    region = novel_rows // WORLD
    nxt, rows = {}, {}
    for k in range(WORLD):
        for w in range(n_waves):
            for j, (p, l, f, r) in enumerate(chunks[k][w]):
                if (k, w, j) in novel:
                    o = ((f >> 32) * WORLD) >> 32  # shard.owner_of on the unsigned fingerprint
                    rows[(k, w, j)] = o * region + nxt.get((o, k), 0)
                    nxt[(o, k)] = nxt.get((o, k), 0) + l
    out = [[None] * n_waves for _ in range(WORLD)]
    for k in range(WORLD):
        for w in range(n_waves):
            recs = []
            for j, (p, l, f, r) in enumerate(chunks[k][w]):
                if p < CARVE:
                    recs.append((-1, -1, -1, 0, p, l, r))
                    continue
                wk, ww, wj, p_src = reg[f]
                recs.append((0 if (wk, ww, wj) == (k, w, j) else 1, wk, rows[(wk, ww, wj)], p_src, p, l, r))
            out[k][w] = recs
    return out


def _worker(rank, WORLD, port, out_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        torch.cuda.set_device(0)
        from oracle import oracle as O
        from test_gpu_pipeline import LAYERS, R, WAVES, make_waves, to_dev

        from paper_2605_05696_b200 import _native as N, ops, shard
        from paper_2605_05696_b200.pipeline import ReattachPipeline

        all_waves = [make_waves(seed=11 + k) for k in range(WORLD)]
        novel_rows = WORLD * 12000  # 12K first-writer rows per (owner, writer) sub-range
        ref = global_oracle(all_waves, novel_rows, WORLD)
        waves = all_waves[rank]
        gen = torch.Generator(device="cuda").manual_seed(3 + rank)
        # replica region 8192 rows + a 2 x 6000-row scratch: the cold wave's body is fresh for every
        # rank but its first writer (same exchange), so it is fetched into scratch, uncached
        pool = torch.randn(LAYERS, novel_rows + 8192 + 12000, 576, device="cuda", generator=gen).to(torch.bfloat16)
        peers = shard.map_peer_pools(pool)
        inv = O.make_inv_freq(1e4)
        max_tok = max(int(w[1][-1]) for ws in all_waves for w in ws)
        max_pins = max(int(w[2][-1]) for ws in all_waves for w in ws)
        req_stride = max(int(np.diff(w[1]).max()) for ws in all_waves for w in ws) + 96
        store = ops.ChunkStore(max_entries=1 << 12)
        pipe = ReattachPipeline(store, pool, ops.inv_freq_device(inv), R, max_tok, max_pins, req_stride,
                                layout=N.LAYOUT_INTERLEAVED)
        pipe.enable_sharding(shard.ShardedStore(store, novel_rows),
                             shard.ReplicaCache(pool, novel_rows, peers, rank, ops.ChunkStore(1 << 10),
                                                scratch_rows=6000),
                             rank, WORLD)
        dev = [to_dev(w) for w in waves]
        pipe.load(*dev[0])
        pipe.step_sharded(0)  # cold wave: rank 0 writes the body first, the others fetch it
        hits, outs = {}, {}
        pipe.run_overlapped_sharded(WAVES, lambda i: pipe.load(*dev[1 + i]), wave0=1, k4_sms=100,
                                    after_front=lambda i, s: hits.__setitem__(i, pipe.slots[s]["hit"].clone()),
                                    after_k4=lambda i, s: outs.__setitem__(i, pipe.slots[s]["out"].clone()))
        torch.cuda.synchronize()
        pipe.sharded.check()
        pipe.replica.check()
        pools_u16 = [pp.view(torch.int16).cpu().numpy().view(np.uint16) for pp in peers]
        n_remote = 0
        for i in range(WAVES):
            recs = ref[rank][1 + i]
            got = hits[i].cpu().numpy()[:len(recs)].astype(np.int64)
            want = np.array([r[0] for r in recs], np.int64)
            assert np.array_equal(got, want), (rank, i, np.nonzero(got != want)[0][:10])
            out_u16 = outs[i].view(torch.int16).cpu().numpy().view(np.uint16)
            hit_recs = [r for r in recs if r[0] == 1]
            assert hit_recs
            for writer in range(WORLD):
                hw = [r for r in hit_recs if r[1] == writer]
                if not hw:
                    continue
                n_remote += sum(r[5] for r in hw) if writer != rank else 0
                src = np.array([r[2] for r in hw], np.int64)
                dst = np.array([r[6] * req_stride + r[4] for r in hw], np.int64)
                ln = np.array([r[5] for r in hw], np.int32)
                delta = np.array([r[4] - r[3] for r in hw], np.int64)
                exp = np.zeros((LAYERS, out_u16.shape[1], 576), np.uint16)
                O.rotate_gather_bf16(pools_u16[writer], exp, src, dst, ln, delta, inv, interleaved=True)
                rws = np.concatenate([np.arange(d, d + l) for d, l in zip(dst, ln)])
                assert np.array_equal(out_u16[:, rws, :512], exp[:, rws, :512]), (rank, i, writer)
                f = lambda u: (u.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
                g, e = f(out_u16[:, rws, 512:]), f(exp[:, rws, 512:])
                assert np.abs(g - e).max() <= 2.0 ** -7 * np.abs(e).max(), (rank, i, writer)
        # the other ranks' hits on the body were first written by rank 0: they went through the replica
        assert rank == 0 or n_remote > 0
        out_q.put((rank, "ok", int(pipe.replica.fetched_rows)))
    except Exception as e:  # report, then still meet the other rank at the barrier
        import traceback

        out_q.put((rank, traceback.format_exc()[-2000:], -1))
    finally:
        dist.barrier()  # keep every pool mapped until every rank has read
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_pipeline_one_gpu(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    outs = {}
    for _ in range(world):
        rank, msg, fetched = q.get(timeout=600)
        outs[rank] = (msg, fetched)
    for pr in procs:
        pr.join(timeout=120)
    assert all(m == "ok" for m, _ in outs.values()), outs
    assert all(outs[r][1] > 0 for r in range(1, world)), "ranks > 0 must fetch the body from rank 0's pool"
    for pr in procs:
        assert pr.exitcode == 0
