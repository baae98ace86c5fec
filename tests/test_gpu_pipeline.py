"""GPU parity: the production reattach step (pipeline.ReattachPipeline, the path
bench.py times) against the sequential oracle, for the serial CUDA graph and
for the two-wave overlapped pipeline.

Per wave of agent_meta-shaped requests (shared header = the phase-1 prefix,
random metadata, the canonical marker, a shared body), the oracle runs
oracle/irm_oracle.c's CDC + xxh64 per request and a sequential first-writer-wins
dict in (wave, request, chunk) order, with carve-out chunks (p < 32) neither
probed nor inserted (engine.py:181-226). New entries take pool rows in query
order (store.cu). Checked bit-exact: the per-chunk service map (hit / novel /
carve) of every wave. Checked against the oracle's bf16 rotate+gather
(registry.py:146-166): every hit row of the per-request KV output, c_KV
bit-exact, k_r within bf16 rounding."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

HEADER, BODY, R, WAVES, LAYERS, CARVE = 96, 5000, 3, 5, 2, 32


def make_waves(seed=11):
    shared = np.random.default_rng(7)
    header = shared.integers(0, 2**32, size=HEADER, dtype=np.uint64).astype(np.uint32)
    body = shared.integers(0, 2**32, size=BODY, dtype=np.uint64).astype(np.uint32)
    marker = np.array(O.canonical_marker(), np.uint32)
    rng = np.random.default_rng(seed)
    waves = []
    for w in range(WAVES + 1):  # wave 0 is the cold wave (one request: stores the body)
        streams, pins, ms = [], [], []
        for _ in range(1 if w == 0 else R):
            meta = rng.integers(0, 2**32, size=int(rng.integers(30, 71)), dtype=np.uint64).astype(np.uint32)
            if w > 0 and rng.random() < 0.3:  # some requests also edit the body
                body_w = body.copy()
                body_w[int(rng.integers(0, BODY))] ^= 1
            else:
                body_w = body
            streams.append(np.concatenate([meta, marker, body_w]))
            pins.append(sorted({meta.size - 1, meta.size + 63}))
            ms.append(HEADER)
        off = np.zeros(len(streams) + 1, np.int64)
        np.cumsum([s.size for s in streams], out=off[1:])
        poff = np.zeros(len(streams) + 1, np.int64)
        np.cumsum([len(p) for p in pins], out=poff[1:])
        waves.append((np.concatenate(streams), off, poff, np.array([x for p in pins for x in p], np.int64),
                      np.array(ms, np.int64)))
    return waves


def oracle_waves(waves):
    """Sequential reference: per wave, per chunk (hit code, p_src, row, p, len, request)."""
    reg, rows_next, out = {}, 0, []
    for tok, off, poff, pins, ms in waves:
        recs = []
        for r in range(off.size - 1):
            st, ln, fp, _ = O.cdc_chunk(tok[off[r]:off[r + 1]], pins=pins[poff[r]:poff[r + 1]])
            for s, l, f in zip(st.tolist(), ln.tolist(), fp.tolist()):
                p = int(ms[r]) + s
                if p < CARVE:
                    recs.append((-1, 0, -1, p, l, r))
                elif f in reg:
                    recs.append((1, reg[f][0], reg[f][1], p, l, r))
                else:
                    reg[f] = (p, rows_next)
                    recs.append((0, p, rows_next, p, l, r))
                    rows_next += l
        out.append(recs)
    return out, rows_next


def to_dev(wave):
    return tuple(torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).cuda() for a in wave)


@pytest.fixture(scope="module")
def setup():
    from paper_2605_05696_b200 import _native as N, ops

    waves = make_waves()
    ref, rows_used = oracle_waves(waves)
    gen = torch.Generator(device="cuda").manual_seed(3)
    pool = torch.randn(LAYERS, rows_used + 64, 576, device="cuda", generator=gen).to(torch.bfloat16)
    inv = O.make_inv_freq(1e4)
    max_tok = max(int(w[1][-1]) for w in waves)
    max_pins = max(int(w[2][-1]) for w in waves)
    req_stride = max(int(np.diff(w[1]).max()) for w in waves) + HEADER
    return dict(N=N, ops=ops, waves=waves, ref=ref, pool=pool, inv=inv, max_tok=max_tok, max_pins=max_pins,
                req_stride=req_stride)


def new_pipe(S, fanout=True):
    from paper_2605_05696_b200.pipeline import ReattachPipeline

    ops = S["ops"]
    store = ops.ChunkStore(max_entries=1 << 12)
    return ReattachPipeline(store, S["pool"], ops.inv_freq_device(S["inv"]), R, S["max_tok"], S["max_pins"],
                            S["req_stride"], layout=S["N"].LAYOUT_INTERLEAVED, fanout=fanout)


def check_wave(S, w, hit, out):
    """hit: service map (chunk order), out: [L, R * req_stride, 576] bf16 (host)."""
    recs = S["ref"][w]
    n = len(recs)
    want = np.array([r[0] for r in recs], np.int64)
    got = hit[:n].astype(np.int64)
    assert np.array_equal(got, want), (w, np.nonzero(got != want)[0][:10])
    hits = [r for r in recs if r[0] == 1]
    assert hits, "workload must reattach something"
    src = np.array([r[2] for r in hits], np.int64)
    dst = np.array([r[5] * S["req_stride"] + r[3] for r in hits], np.int64)
    ln = np.array([r[4] for r in hits], np.int32)
    delta = np.array([r[3] - r[1] for r in hits], np.int64)
    pool_u16 = S["pool"].view(torch.int16).cpu().numpy().view(np.uint16)
    exp = np.zeros((LAYERS, out.shape[1], 576), np.uint16)
    O.rotate_gather_bf16(pool_u16, exp, src, dst, ln, delta, S["inv"], interleaved=True)
    got_u16 = out.view(torch.int16).numpy().view(np.uint16)
    rows = np.concatenate([np.arange(d, d + l) for d, l in zip(dst, ln)])
    assert np.array_equal(got_u16[:, rows, :512], exp[:, rows, :512])  # c_KV verbatim
    f = lambda u: (u.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    g, e = f(got_u16[:, rows, 512:]), f(exp[:, rows, 512:])
    assert np.abs(g - e).max() <= 2.0 ** -7 * np.abs(e).max(), "k_r beyond bf16 rounding"


@pytest.mark.parametrize("fanout", [True, False])
def test_pipeline_serial_graph(setup, fanout):
    S = setup
    pipe = new_pipe(S, fanout)
    dev = [to_dev(w) for w in S["waves"]]
    pipe.load(*dev[0])
    pipe.step_eager()  # cold wave: inserts the body
    torch.cuda.synchronize()
    pipe.capture()  # its warm-up re-runs the cold wave: all hits, no new entries
    for w in range(1, WAVES + 1):
        pipe.load(*dev[w])
        pipe.replay()
        torch.cuda.synchronize()
        check_wave(S, w, pipe.hit.cpu().numpy(), pipe.out.cpu())
    pipe.check()


@pytest.mark.parametrize("fanout", [True, False])
def test_pipeline_overlapped_matches_oracle(setup, fanout):
    S = setup
    pipe = new_pipe(S, fanout)
    dev = [to_dev(w) for w in S["waves"]]
    pipe.load(*dev[0])
    pipe.step_eager()
    torch.cuda.synchronize()
    pipe.capture_overlapped(k4_sms=100)
    hits, outs = {}, {}
    # service maps read back on the pipeline's side stream (the e2e path of bench.py)
    rb = [torch.empty(pipe.slots[0]["hit"].shape, dtype=pipe.slots[0]["hit"].dtype, pin_memory=True)
          for _ in range(WAVES)]
    pipe.run_overlapped(WAVES, lambda i: pipe.load(*dev[1 + i]),
                        after_front=lambda i, s: hits.__setitem__(i, pipe.slots[s]["hit"].clone()),
                        after_k4=lambda i, s: outs.__setitem__(i, pipe.slots[s]["out"].clone()), readback=rb)
    torch.cuda.synchronize()
    n_tok = 0
    for i in range(WAVES):
        check_wave(S, 1 + i, hits[i].cpu().numpy(), outs[i].cpu())
        assert torch.equal(rb[i], hits[i].cpu())
        n_tok += sum(r[4] for r in S["ref"][1 + i] if r[0] == 1)
    assert int(pipe.hit_tokens.item()) == n_tok
    pipe.check()


def test_replica_fetch_peer_pools():
    """K6 replica fetch on one GPU: a second pool stands in for a peer's
    (shard.map_peer_pools gives the same kind of tensor for another GPU). Runs
    are fetched once by irm_copy_runs, duplicates and later waves reuse them."""
    from paper_2605_05696_b200 import ops, shard

    L, rows = 3, 4096
    pools = [torch.randn(L, rows, 576, device="cuda").to(torch.bfloat16) for _ in range(2)]
    cache = shard.ReplicaCache(pools[0], 2048, pools, 0, ops.ChunkStore(1 << 10))
    rng = np.random.default_rng(4)
    starts = rng.choice(np.arange(0, 1500, 64), size=12, replace=False)
    lens = rng.integers(1, 64, size=12)
    sel = np.concatenate([np.arange(12), [0, 5, 5]])  # runs 0 and 5 asked for again in the same wave
    grow = shard.encode_row(1, torch.from_numpy(starts[sel]).cuda())
    grow = torch.cat([grow, shard.encode_row(0, torch.tensor([7], device="cuda")),
                      torch.tensor([-1], device="cuda")])
    ln = torch.from_numpy(np.concatenate([lens[sel], [5, 3]]).astype(np.int32)).cuda()
    local = cache.localize(grow, ln).cpu().numpy()
    torch.cuda.synchronize()
    assert int(cache.fetched_runs) == 12 and int(cache.fetched_rows) == int(lens.sum())
    assert local[12] == local[0] and local[13] == local[14] == local[5]
    assert local[15] == 7  # own rows pass through
    p0, p1 = pools[0].cpu(), pools[1].cpu()
    for k in range(12):
        a, l = int(local[k]), int(lens[k])
        assert a >= 2048 and torch.equal(p0[:, a:a + l], p1[:, starts[k]:starts[k] + l])
    again = cache.localize(grow[:12], ln[:12]).cpu().numpy()
    assert np.array_equal(again, local[:12]) and int(cache.fetched_runs) == 12
    cache.check()


@pytest.mark.parametrize("graphs", [False, True])
def test_pipeline_sharded_single_rank(setup, graphs):
    """The sharded step (NCCL all-to-all lookup, world 1) in the overlapped
    pipeline reproduces the oracle like the unsharded graph path: on streams,
    and as captured graphs with the all-to-alls inside."""
    import os

    import torch.distributed as dist

    from paper_2605_05696_b200 import shard

    S = setup
    ops = S["ops"]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        pipe = new_pipe(S)
        peers = shard.map_peer_pools(S["pool"])
        pipe.enable_sharding(shard.ShardedStore(pipe.store, S["pool"].shape[1] - 32), shard.ReplicaCache(
            S["pool"], S["pool"].shape[1] - 32, peers, 0, ops.ChunkStore(1 << 10)), 0, 1)
        dev = [to_dev(w) for w in S["waves"]]
        pipe.load(*dev[0])
        pipe.step_sharded(0)  # cold wave (world 1: owner-allocated rows are the oracle's rows)
        torch.cuda.synchronize()
        hits, outs = {}, {}
        af = lambda i, s: hits.__setitem__(i, pipe.slots[s]["hit"].clone())
        ak = lambda i, s: outs.__setitem__(i, pipe.slots[s]["out"].clone())
        if graphs:
            pipe.capture_overlapped(k4_sms=100, sharded=True)
            pipe.run_overlapped(WAVES, lambda i: pipe.load(*dev[1 + i]), after_front=af, after_k4=ak, wave0=1)
        else:
            pipe.run_overlapped_sharded(WAVES, lambda i: pipe.load(*dev[1 + i]), wave0=1, k4_sms=100,
                                        after_front=af, after_k4=ak)
        torch.cuda.synchronize()
        for i in range(WAVES):
            check_wave(S, 1 + i, hits[i].cpu().numpy(), outs[i].cpu())
        pipe.replica.check()
        pipe.sharded.check()
    finally:
        dist.destroy_process_group()


def _whole(wave, header):
    """Whole requests (header + tail) and their request-relative marker spans."""
    tok, off, poff, pins, ms = wave
    streams, spans, span_off = [], [], [0]
    for r in range(off.size - 1):
        tail = tok[off[r]:off[r + 1]]
        streams.append(np.concatenate([header, tail]))
        p = pins[poff[r]:poff[r + 1]]  # (meta end - 1, marker end - 1) in the tail
        spans += [int(ms[r]) + int(p[0]) + 1, int(ms[r]) + int(p[1]) + 1]
        span_off.append(span_off[-1] + 1)
    w_off = np.zeros(len(streams) + 1, np.int64)
    np.cumsum([s.size for s in streams], out=w_off[1:])
    return (np.concatenate(streams), w_off, np.array(span_off, np.int64), np.array(spans, np.int64), streams)


@pytest.mark.parametrize("mode", ["serial", "overlapped"])
def test_pipeline_device_prefix_matches_oracle(setup, mode):
    """Phase 1 inside the step (VERDICT r1 missing #5): waves of WHOLE requests go
    in; K0 (radix.WavePrefixIndex, graph-captured) finds each request's m against
    every earlier request, irm_wave_rebase packs the tails and rebases the marker
    pins, then K1 / K3 / K4. Checked: m against the brute-force longest common
    prefix (radix.py:60-83, tests/test_radix.py:15-23), the service map and the KV
    rows against the same sequential oracle as the host-m path."""
    from paper_2605_05696_b200.radix import WavePrefixIndex
    from paper_2605_05696_b200.pipeline import ReattachPipeline

    S = setup
    ops = S["ops"]
    shared = np.random.default_rng(7)
    header = shared.integers(0, 2**32, size=HEADER, dtype=np.uint64).astype(np.uint32)
    whole = [_whole(w, header) for w in S["waves"]]
    max_tok = max(int(w[1][-1]) for w in whole)
    index = WavePrefixIndex(max_prefixes=1 << 20, arena_tokens=1 << 21, max_sequences=1 << 10)
    # the cold request stores its header chunks too here (m = 0): a pool with room for them
    pool = torch.cat([S["pool"], torch.zeros_like(S["pool"][:, :4096])], dim=1)
    S = dict(S, pool=pool)
    pipe = ReattachPipeline(ops.ChunkStore(max_entries=1 << 12), pool, ops.inv_freq_device(S["inv"]), R,
                            max_tok, S["max_pins"], S["req_stride"], layout=S["N"].LAYOUT_INTERLEAVED,
                            prefix_index=index, max_spans=R)
    dev = [tuple(torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).cuda() for a in w[:4])
           for w in whole]
    pipe.load_requests(*dev[0])
    pipe.step_eager()  # cold wave
    torch.cuda.synchronize()
    hits, outs, ms = {}, {}, {}
    if mode == "serial":
        pipe.capture()
        for w in range(1, WAVES + 1):
            pipe.load_requests(*dev[w])
            pipe.replay()
            torch.cuda.synchronize()
            hits[w - 1], outs[w - 1], ms[w - 1] = pipe.hit.clone(), pipe.out.clone(), pipe.inputs[0]["m"].clone()
    else:
        pipe.capture_overlapped(k4_sms=100)
        pipe.run_overlapped(WAVES, lambda i: pipe.load_requests(*dev[1 + i]),
                            after_front=lambda i, s: (hits.__setitem__(i, pipe.slots[s]["hit"].clone()),
                                                      ms.__setitem__(i, pipe.inputs[s]["m"].clone())),
                            after_k4=lambda i, s: outs.__setitem__(i, pipe.slots[s]["out"].clone()))
        torch.cuda.synchronize()
    # the oracle: m by brute force over every earlier whole request (the cold one has m = 0),
    # then the sequential serve over tails whose pins are the rebased marker spans
    inserted, o_waves = [], []
    for wi, w in enumerate(whole):
        streams, pins, m_list = [], [], []
        spans = w[3].reshape(-1, 2)
        for r, s_ in enumerate(w[4]):
            m_ = O.prefix_match(inserted, s_)[0]
            inserted.append((len(inserted), s_))
            sp = [(int(a), int(b)) for a, b in spans[w[2][r]:w[2][r + 1]]]
            pins.append(sorted(O.marker_pin_offsets((max(a - m_, 0), b - m_) for a, b in sp if b - 1 >= m_)))
            streams.append(s_[m_:])
            m_list.append(m_)
        off = np.zeros(len(streams) + 1, np.int64)
        np.cumsum([x.size for x in streams], out=off[1:])
        poff = np.zeros(len(streams) + 1, np.int64)
        np.cumsum([len(p) for p in pins], out=poff[1:])
        o_waves.append((np.concatenate(streams), off, poff, np.array([x for p in pins for x in p], np.int64),
                        np.array(m_list, np.int64)))
        if wi > 0:
            assert ms[wi - 1].cpu().tolist()[:len(m_list)] == m_list, (wi, m_list)
    ref, _ = oracle_waves(o_waves)
    S2 = dict(S, ref=ref)
    for i in range(WAVES):
        check_wave(S2, 1 + i, hits[i].cpu().numpy(), outs[i].cpu())
    pipe.check()
