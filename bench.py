"""Benchmark of the cache-reattach hot path (BASELINE.json config 2).

A step = one wave of R fresh 32K-token agent_meta requests (shared 50-token
header, per-request 30..70-token metadata, 64-token marker, shared 32,768-token
body) served warm against a store that already holds the body:
    K1  CDC + xxh64 over every request tail            (irm_cdc_xxh64)
    K3  batched first-writer-wins store lookup/insert   (irm_store_lookup_insert)
    K4  rotate+gather of every hit chunk x 27 layers    (irm_rotate_gather)
        bf16 latent pool [27, rows, 576] -> per-request KV [27, R*33K, 576]
DeepSeek-V2-Lite shape (27 layers, kv_lora_rank 512, rope 64, theta 1e4,
DSv2 interleaved rotary). Synthetic tokens and random-init latent rows.

value = reattached KV tokens / s / GPU (PIC-hit tokens, each gathered and
rotated for all 27 layers) with inputs resident in HBM; e2e adds the H2D of
the wave's tokens/pins from pinned host memory and the D2H of the per-chunk
service result. Components: CDC+hash tokens/s (K1 alone) and, when built,
fused reattach-attention TFLOPS (K5).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "reattached KV tokens/s/GPU (rotate+gather); CDC+hash tokens/s; fused-attn TFLOPS"
UNIT = "tokens/s"
LAYERS, CKV, KR, THETA = 27, 512, 64, 1e4
# SMs the gather of wave i spreads over while K0 + K1 + K3 of wave i + 1 run beside it; 0 = all of them, in 4
# retiring CTA rounds, with the front on a high-priority stream (swept: profiles/r02_k4_sms.md)
K4_SMS = int(os.environ.get("IRM_K4_SMS", "0"))
# the sharded path's front launches NCCL kernels (the lookup all-to-alls), which need SMs that K4
# does not hold: there K4 keeps to 112 SMs (N = 1 sweep, profiles/r02_k4_sms.md: config 5 113.0 M
# tok/s vs 90.0 with all SMs in rounds; config 2 sharded 159.7 at 120 SMs vs 117.2)
K4_SMS_SHARDED = int(os.environ.get("IRM_K4_SMS", "140"))


def k4_placement(sms):
    return ("K4 of wave i on all SMs in 4 retiring CTA rounds, wave i+1's front on a high-priority stream"
            if sms == 0 else "K4 of wave i on %d SMs" % sms)


K4_PLACEMENT = k4_placement(K4_SMS)
BODY, HEADER, R_PER_WAVE = 32768, 50, 8
CARVE = 32


_FLUSH = None


def timed_flushed(fn, reps):
    """Mean device time of ``fn`` over ``reps`` launches, each timed alone with CUDA
    events and preceded (outside its events) by a 256 MB write that evicts the 126 MB
    L2: component inputs smaller than L2 never start warm."""
    import torch

    global _FLUSH
    if _FLUSH is None:
        _FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda.synchronize()
    for a, b in ev:
        _FLUSH.fill_(1)
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / reps


_JSON_OUT = None


def emit(line: dict):
    """The one JSON line on stdout (see ``main``: everything else written to fd 1 goes to stderr)."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def nccl_logs_to_stderr(world):
    """N > 1: NCCL's communicator lines (ranks, NVLink / NVLS paths) stay visible, on stderr,
    so stdout keeps exactly one JSON line."""
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,COLL")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def ncu_traffic(kernel_prefix: str, workload: str = "config2"):
    """dram__bytes_read.sum + dram__bytes_write.sum per K4 launch, from the committed
    ncu --set full capture of this same workload (profiles/ncu_traffic.json), when
    that capture is of the kernel this run's roofline names."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)[workload]
        return float(d["dram_bytes_per_launch"]) if d["kernel"].startswith(kernel_prefix) else None
    except Exception:
        return None


# ----------------------------------------------------------------- workload
def make_requests(rng, header, marker, body, n_req):
    """One wave of whole agent_meta requests (workloads.py:85-100 shape): the shared
    header, 30..70 random metadata tokens, the marker, the shared body. Returns
    the token arrays and each request's marker span [start, end)."""
    reqs, spans = [], []
    for _ in range(n_req):
        meta = rng.integers(0, 2**32, size=int(rng.integers(30, 71)), dtype=np.uint64).astype(np.uint32)
        reqs.append(np.concatenate([header, meta, marker, body]))
        spans.append([(HEADER + meta.size, HEADER + meta.size + marker.size)])
    return reqs, spans


def pack_requests(reqs, spans):
    """-> (tokens u32, off [n+1], span_off [n+1], spans [2 x n_spans] request-relative)."""
    off = np.zeros(len(reqs) + 1, np.int64)
    np.cumsum([r.size for r in reqs], out=off[1:])
    soff = np.zeros(len(reqs) + 1, np.int64)
    np.cumsum([len(s) for s in spans], out=soff[1:])
    flat = np.array([x for s in spans for sp in s for x in sp], np.int64)
    return np.concatenate(reqs), off, soff, flat


def pack_tails(wave):
    """make_wave's (tails, pins, m) -> (tokens u32, off, pin_off, pins, m) arrays."""
    streams, pins, ms = wave
    off = np.zeros(len(streams) + 1, np.int64)
    np.cumsum([x.size for x in streams], out=off[1:])
    poff = np.zeros(len(streams) + 1, np.int64)
    np.cumsum([len(p) for p in pins], out=poff[1:])
    return (np.concatenate(streams), off, poff, np.array([x for p in pins for x in p], np.int64),
            np.array(ms, np.int64))


def make_wave(rng, header, marker, body, n_req):
    """Token streams of one wave plus the host-side phase-1 prefix length m
    (the shared header; exact-prefix matching is host radix work, §8(f))."""
    streams, pins, ms = [], [], []
    for _ in range(n_req):
        meta = rng.integers(0, 2**32, size=int(rng.integers(30, 71)), dtype=np.uint64).astype(np.uint32)
        full = np.concatenate([header, meta, marker, body])
        m = HEADER  # the metadata diverges right after the shared header
        tail = full[m:]
        ms_ = meta.size
        pins.append(sorted({ms_ - 1, ms_ + 63}))  # marker_pin_offsets rebased to the tail
        streams.append(tail)
        ms.append(m)
    return streams, pins, ms


class Clocks:
    """nvidia-smi sampler during the timed region (recipe clocks line)."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()  # nvidia-smi takes ~0.5 s to start: wait for its first sample
            while not self.rows and time.time() - t0 < 5:
                time.sleep(0.02)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2605_05696_b200 import _native as N, ops
    from paper_2605_05696_b200.chunking import canonical_marker

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # IRM_BENCH_ONE_DEVICE=1 + IRM_BENCH_BACKEND=gloo: every rank on cuda:0, a check of the
    # N-rank code path on a one-GPU box (NCCL cannot put two ranks on one GPU; timings are not valid)
    if os.environ.get("IRM_BENCH_ONE_DEVICE") == "1":
        local = 0
    backend = os.environ.get("IRM_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1 or args.sharded:
        if world == 1:  # single-rank group for the K6 path at N=1
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29531")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        if backend == "nccl":
            nccl_logs_to_stderr(world)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    hbm, tf_burst, tf_sust, peak_kind = peaks()

    # -------- inputs (seeded, per rank: sessions s mod G). Every serve takes a FRESH wave:
    # phase 1 runs on the device (K0) against every request served before, so a re-served
    # wave would match whole. Serve order: cold, serial warm-up (graph path), overlapped
    # warm-up, timed, component probe, e2e (pinned host), parity check.
    rng = np.random.default_rng(1000 + rank)
    shared = np.random.default_rng(7)
    header = shared.integers(0, 2**32, size=HEADER, dtype=np.uint64).astype(np.uint32)
    body = shared.integers(0, 2**32, size=BODY, dtype=np.uint64).astype(np.uint32)
    marker = np.array(canonical_marker(), np.uint32)
    R = args.requests
    overlapped = not args.serial
    sharded = world > 1 or args.sharded
    W, K = args.warmup, args.steps
    n_serial_warm = W if not sharded else 0
    n_ovl_warm = W if overlapped else 0
    plan = dict(cold=1, serial_warm=n_serial_warm, ovl_warm=n_ovl_warm, timed=K, comp=1, e2e=K, check=1)
    waves = {k: [pack_requests(*make_requests(rng, header, marker, body, R)) for _ in range(n)]
             for k, n in plan.items()}
    all_waves = [w for k in plan for w in waves[k]]
    max_tok = max(int(w[1][-1]) for w in all_waves)
    max_spans = max(int(w[2][-1]) for w in all_waves)
    req_stride = max(int(np.diff(w[1]).max()) for w in all_waves)  # rows per request in the KV out
    tok_per_wave = int(waves["timed"][0][1][-1]) - R * HEADER  # the tails K1 scans (m = the shared header)
    to_dev = lambda p: tuple(torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).to(dev) for a in p)
    to_pin = lambda p: tuple(torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).pin_memory()
                             for a in p)
    dev_in = {k: [to_dev(w) for w in waves[k]] for k in plan if k != "e2e"}
    host_in = [to_pin(w) for w in waves["e2e"]]
    served = []  # whole-request waves in serve order (the parity oracle replays them)

    # -------- store, prefix index + latent pool, populated by the cold request (untimed)
    from paper_2605_05696_b200.pipeline import ReattachPipeline
    from paper_2605_05696_b200.radix import WavePrefixIndex

    store = ops.ChunkStore(max_entries=1 << 16)
    n_served = sum(plan.values())
    pool_rows = BODY + HEADER + 2048 * (n_served + 2)  # body + the novel meta chunks of every wave
    if sharded:
        # rows [0, novel) hold first-writer KV (split among the G owners), [novel, pool_rows) the replicas
        novel_rows = 2 * (BODY + HEADER + 80 * R * (n_served + 4))
        scratch_rows = BODY + 4096  # per half: a cold body first written by another rank in the same wave
        pool_rows = novel_rows + BODY + 80 * R * (n_served + 4) + 4096 + 2 * scratch_rows
    pool = torch.empty(LAYERS, pool_rows, CKV + KR, dtype=torch.bfloat16, device=dev)
    for l in range(LAYERS):  # random-init latents, a layer at a time
        pool[l].normal_()
    inv = ops.inv_freq_device(np.power(THETA, -2.0 * np.arange(KR // 2) / KR))
    n_tok_all = sum(int(w[1][-1]) for w in all_waves)
    index = WavePrefixIndex(max_prefixes=n_tok_all + 4096, arena_tokens=n_tok_all + 4096,
                            max_sequences=R * (n_served + 4) + 64)
    pipe = ReattachPipeline(store, pool, inv, R, max_tok, 2 * max_spans, req_stride, layout=N.LAYOUT_INTERLEAVED,
                            fanout=not args.no_fanout, prefix_index=index, max_spans=max_spans)

    def load(kind, i, host=False):
        w = host_in[i] if host else dev_in[kind][i]
        pipe.load_requests(*w)
        served.append(waves[kind][i])

    fallback = None
    if sharded:  # K6: hash-sharded store (fixed-capacity NCCL all-to-all) + peer replica cache
        from paper_2605_05696_b200 import shard

        ok, peers = 1, None
        try:
            peers = shard.map_peer_pools(pool)
        except Exception as e:  # no peer mapping between these GPUs: run independent replicas instead
            print(f"bench: peer pool mapping failed ({type(e).__name__}: {e})", file=sys.stderr)
            ok = 0
        if world > 1:  # every rank takes the same path
            t = torch.tensor([ok], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            ok = int(t.item())
        if ok:
            cache = shard.ReplicaCache(pool, novel_rows, peers, rank, ops.ChunkStore(max_entries=1 << 16),
                                       scratch_rows=scratch_rows)
            pipe.enable_sharding(shard.ShardedStore(store, novel_rows), cache, rank, world)
        else:
            sharded = False
            fallback = "peer pool mapping (CUDA IPC) unavailable: every GPU runs an independent store (replicas)"
    wave_no = [0]  # global wave counter of the sharded order key

    def step(kind, i, cold=False):  # one wave on the serial path (eager or the serial graph)
        load(kind, i)
        if sharded:
            pipe.step_sharded(wave_no[0])
        elif cold:
            pipe.step_eager()
        else:
            pipe.replay()
        wave_no[0] += 1

    # cold request wave: inserts the body (its pool rows hold the random latents); the
    # library's launch counter around this eager wave = our kernels per wave (the graphs
    # replay the same launches)
    lc0 = ops.launch_count()
    step("cold", 0, cold=True)
    launches_per_wave = ops.launch_count() - lc0
    torch.cuda.synchronize()
    if not sharded:
        pipe.capture()  # one CUDA graph per step (+ K1-only / K4-only graphs for component timing)
    for i in range(n_serial_warm):
        step("serial_warm", i)
    # sharded: the two-wave graphs with the NCCL all-to-alls captured inside the front
    # (eager streams when the backend cannot be captured, e.g. the gloo one-device check)
    graphs = not sharded or backend == "nccl"
    if overlapped and not sharded:  # two-wave pipeline graphs (K4 on 120 SMs || K0 + K1 + K3 of the next wave)
        pipe.capture_overlapped(k4_sms=K4_SMS)
    if overlapped and sharded and graphs:
        try:
            pipe.capture_overlapped(k4_sms=K4_SMS_SHARDED, sharded=True)
        except Exception as e:  # keep the N-rank run alive on the stream pipeline (same results)
            print(f"bench: sharded graph capture failed ({type(e).__name__}: {e}); running on streams",
                  file=sys.stderr)
            graphs = False
            pipe.wave_t = None
            torch.cuda.synchronize()
        if world > 1:  # every rank must take the same path
            ok = torch.tensor([1 if graphs else 0], device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 0 and graphs:
                graphs = False
                pipe.wave_t = None

    def run_waves(kind, n, host=False, **kw):
        if sharded:
            run_sharded(pipe, n, lambda i: load(kind, i, host), wave_no[0], graphs, **kw)
        else:
            pipe.run_overlapped(n, lambda i: load(kind, i, host), **kw)
        wave_no[0] += n

    if overlapped:
        run_waves("ovl_warm", n_ovl_warm)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # -------- timed region (value): inputs resident in HBM, one graph replay per wave
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lens = []
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        if overlapped:
            pipe.hit_tokens.zero_()
            t0.record()
            run_waves("timed", K)
            t1.record()
        else:
            t0.record()
            for i in range(K):
                step("timed", i)
                lens.append(pipe.length.sum())  # device-side reduction, read after the timed region
            t1.record()
        torch.cuda.synchronize()
    ms_total = t0.elapsed_time(t1)
    hit_tok = int(pipe.hit_tokens.item()) if overlapped else int(torch.stack(lens).sum().item())
    if world > 1:
        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        ht = torch.tensor([hit_tok], device=dev, dtype=torch.int64)
        dist.all_reduce(ht)
        hit_tok = int(ht.item())
    value = hit_tok / (ms_total / 1e3)  # whole-job reattached tokens/s
    ms_step = ms_total / K

    # -------- per-launch K1 / K4 durations: graph replays between events (no host gaps)
    def time_graph(g, n=20):  # each replay timed alone after an L2 flush
        return timed_flushed(g.replay, n)

    step("comp", 0)  # a fresh wave through the serial path: its K1 / K3 / K4 are re-timed below
    torch.cuda.synchronize()
    k4_rows = int(pipe.length.sum().item()) * LAYERS  # reattached rows written per launch
    if pipe.fanout:  # each distinct source run is read once per launch (K4 fan-out)
        ng = int(pipe.groups.n_groups.item())
        src_rows = int(pipe.groups.g_len[:ng].to(torch.int64).sum().item()) * LAYERS
    else:
        src_rows = k4_rows
    n_queries = int(pipe.table.chunk_off[-1].item())  # K3 probes per wave (chunks of the wave)
    if sharded:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record()
        pipe.k1()
        ev[1].record()
        ev[2].record()
        pipe.k4()
        ev[3].record()
        ev[4].record()
        pipe.k3_sharded(10**6)  # the same chunks again under fresh order keys: all hits
        ev[5].record()
        torch.cuda.synchronize()
        k1, k4, k3 = ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3]), ev[4].elapsed_time(ev[5])
    else:
        k1 = time_graph(pipe.graph_k1)
        k4 = time_graph(pipe.graph_k4)
        k3 = time_graph(pipe.graph_k3)

    # -------- e2e: the pipeline fed from pinned host buffers (fresh waves), results read back
    bi = sum(t.numel() * t.element_size() for t in host_in[0])
    bo = 0
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    hit_src = pipe.slots[0]["hit"] if overlapped else pipe.hit
    res = [torch.empty(hit_src.shape, dtype=hit_src.dtype, pin_memory=True) for _ in range(K)]
    e_lens = []
    if overlapped:
        pipe.hit_tokens.zero_()
    e0.record()
    if overlapped:
        def d2h(i, slot):  # D2H of wave i's per-chunk service result
            res[i].copy_(pipe.slots[slot]["hit"], non_blocking=True)

        if sharded and not graphs:
            run_waves("e2e", K, host=True, after_front=d2h)
        else:  # the service maps come back on a side stream (readback), off the critical path
            run_waves("e2e", K, host=True, readback=res)
        bo = pipe.slots[0]["hit"].numel() * pipe.slots[0]["hit"].element_size()
    else:
        for i in range(K):
            load("e2e", i, host=True)  # H2D from pinned memory
            pipe.step_sharded(wave_no[0]) if sharded else pipe.replay()
            wave_no[0] += 1
            res[i].copy_(pipe.hit, non_blocking=True)  # D2H of the per-chunk service result
            e_lens.append(pipe.length.sum())
            bo = pipe.hit.numel() * pipe.hit.element_size()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    e2e_tok = int(pipe.hit_tokens.item()) if overlapped else int(torch.stack(e_lens).sum().item())
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        ht = torch.tensor([e2e_tok], device=dev, dtype=torch.int64)
        dist.all_reduce(ht)
        e2e_tok = int(ht.item())
    e2e_value = e2e_tok / (e2e_ms / 1e3)
    if sharded:  # host checks, outside the timed regions: first-writer rows and replicas all fit
        pipe.sharded.check()
        pipe.replica.check()
    pipe.check()
    # -------- in-run parity (the checker, after every timed region): one fresh wave through the
    # production path vs the sequential oracle over every wave this run served
    parity = None
    if world == 1:
        parity = pipeline_parity(pipe, list(served), waves["check"][0], dev_in["check"][0], overlapped, sharded,
                                 graphs if sharded else True, pool, req_stride, wave0=wave_no[0], prefix=True)
    elif sharded and overlapped:  # every rank serves its check wave (the exchange is collective); rank 0 checks
        parity = sharded_parity(pipe, plan, R, header, marker, body, dev_in["check"][0], graphs, peers, novel_rows,
                                req_stride, wave_no[0], rank, world)

    # -------- roofline of the dominant kernel (K4) and K1
    k4_bytes = (src_rows + k4_rows) * (CKV + KR) * 2  # bf16 rows: unique source reads + destination writes
    k4_gbs = k4_bytes / (k4 / 1e3) / 1e9
    k1_bytes = tok_per_wave * 4 + (tok_per_wave // 128) * 24
    k1_gbs = k1_bytes / (k1 / 1e3) / 1e9
    # K1's real bound: the longest pin-delimited region walks its one-bit chain serially
    longest_region = 0  # tail regions between marker pins (span start - 1, span end - 1), after m = HEADER
    _tk, w_off, w_soff, w_spans = waves["comp"][0]
    for r in range(w_off.size - 1):
        sp = w_spans[2 * w_soff[r]:2 * w_soff[r + 1]].reshape(-1, 2) - HEADER
        cuts = [-1] + sorted(int(x) for a, b in sp for x in (a - 1, b - 1)) + [int(w_off[r + 1] - w_off[r]) - HEADER - 1]
        longest_region = max([longest_region] + [b - a for a, b in zip(cuts[:-1], cuts[1:])])
    sm_mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", 1965.0)) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1965.0
    # serial floors of one region, each measured alone on one warp: the shipped chain step
    # (tools/chain_microbench.cu "shipped lean step": 33.8 cycles per 32 tokens) and the walker
    # (tools/walker_microbench.cu: 228 cycles per chunk at this chunk density, stores included)
    chain_floor_us = -(-longest_region // 32) * 33.8 / sm_mhz
    walker_chunks = longest_region * n_queries / max(tok_per_wave, 1)
    walker_floor_us = walker_chunks * 228 / sm_mhz
    serial_floor_us = max(chain_floor_us, walker_floor_us)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "DeepSeek-V2-Lite reattach (config 2): 27 layers, kv_lora 512 + rope 64, "
                               "DSv2 interleaved rotary theta 1e4, 32K-token agent_meta prompts",
                   "requests_per_step": R, "tokens_per_request": tok_per_wave // R + HEADER,
                   "layers": LAYERS, "l2": "inputs larger than L2 (1.0 GB pool, 8 GB KV out per step); "
                                           "components: L2 flushed (256 MB write) before every timed launch",
                   "pipeline": ("two-wave overlap: %s || K0 + K1 + K3 of wave i+1"
                                % k4_placement(K4_SMS_SHARDED if sharded else K4_SMS)
                                + (" (CUDA graphs; sharded lookup: NCCL all-to-alls captured in the graph, peer replica fetch)"
                                   if sharded and graphs else
                                   " (streams; sharded lookup + peer replica fetch)" if sharded else " (CUDA graphs)"))
                               if overlapped else "serial K1 -> K3 -> K4 per wave",
                   "parallelism": f"sessions s mod G over {world} GPU(s)" + (
                       ", store sharded by fp prefix, NCCL all-to-all lookup" if sharded else
                       f", {fallback}" if fallback else "")},
        "roofline": {"bound": "hbm", "kernel": ("irm_rotate_gather_fanout (K4 fan-out)" if pipe.fanout
                                                else "irm_rotate_gather (K4)"), "achieved": k4_gbs,
                     "peak": hbm, "unit": "GB/s", "frac": k4_gbs / hbm, "traffic": ncu_traffic("rotate_gather_ws_kernel" if pipe.fanout
                                                                          else "rotate_gather_tma_kernel"),
                     "peak_kind": peak_kind, "launch_ms": k4, "algorithmic_bytes": k4_bytes,
                     "source_rows_read": src_rows, "rows_written": k4_rows,
                     "bytes_rule": "1152 B per distinct source row read (once per launch) + 1152 B per reattached "
                                   "row written, x 27 layers"},
        "components": {
            "cdc_hash": {"value": tok_per_wave / (k1 / 1e3), "unit": "tokens/s", "kernel": "irm_cdc_xxh64 (K1)",
                         "launch_ms": k1, "tokens_per_launch": tok_per_wave,
                         "note": "bound by the serial work of the longest pin-delimited region: the one-bit "
                                 "carried chain and the boundary walker (DESIGN.md K1), not by HBM",
                         "roofline": {"bound": "serial", "achieved": serial_floor_us / (k1 * 1e3), "peak": 1.0,
                                      "unit": "fraction of the region's serial floor",
                                      "frac": serial_floor_us / (k1 * 1e3), "serial_floor_us": serial_floor_us,
                                      "chain_floor_us": chain_floor_us, "walker_floor_us": walker_floor_us,
                                      "longest_region_tokens": longest_region,
                                      "floor_rule": "max(chain: ceil(tokens / 32) x 33.8 cycles, walker: chunks x 228 "
                                                    "cycles), each the shipped step timed alone on one warp "
                                                    "(tools/chain_microbench.cu, tools/walker_microbench.cu), at "
                                                    "the max SM clock; the launch adds G, hashing and planning",
                                      "hbm_frac": k1_gbs / hbm}},
            "cdc_hash_wide": cdc_wide_component(hbm),
            "producer_rotate": producer_component(hbm),
            "serve_api": serve_api_component(),
            # K3 / K6 are latency-bound: queries/s and the step's ms, no roofline
            "store_lookup": {"value": n_queries / (k3 / 1e3), "unit": "queries/s", "launch_ms": k3,
                             "queries_per_launch": n_queries,
                             "kernel": "irm_store_lookup_insert (K3)" + (
                                 f" + 2 {backend} all-to-alls over {world} rank(s) (K6)" if sharded else ""),
                             "note": "a re-probe of a stored wave (all hits), per-chunk glue included"},
            "fused_attn": fused_attn_component(args, tf_burst, peak_kind,
                                               cpu=rank == 0 and world == 1 and not args.no_cpu)
            if not args.no_attn else None,
            # the north star's "DeepSeek-V2-Lite shapes": config 2's 32K context, DSv2 interleaved rotary
            "fused_attn_dsv2": fused_attn_component(args, tf_burst, peak_kind, n_ctx=32768, n_q=4096, theta=1e4,
                                                    layout=N.LAYOUT_INTERLEAVED, shape="config 2")
            if not args.no_attn else None,
            # config 4 (JoyAI-Flash shape): 128K context, 8K queries, theta 3.2e7; pool > L2
            "fused_attn_config4": fused_attn_component(args, tf_burst, peak_kind, n_ctx=131072, n_q=8192,
                                                       theta=3.2e7, shape="config 4")
            if not args.no_attn else None,
        },
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo},
        "parity": parity if parity is not None else {"checked": False,
                                                     "why": "N > 1 without the sharded overlapped path"},
        # our kernels per wave (ncu launch list, profiles/r01e_launches.csv): K1 plan / offsets /
        # region / compact, K3 claim / decide / blockscan / commit / resolve, K4 cossin + gather;
        # sharded: + the replica map store's 5 and irm_copy_runs
        "gpu_launches": args.steps * launches_per_wave,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu:  # the CPU leg: rank 0 at N = 1 only
        sample = pack_tails(make_wave(np.random.default_rng(1000), header, marker, body, R))
        line["cpu_baseline"] = cpu_baseline(args, sample, sample_requests=R - 1, min_seconds=10.0)
    if rank == 0:
        emit(line)
    if dist.is_initialized():
        dist.destroy_process_group()


def whole_to_tails(waves):
    """Whole-request waves (tokens, off, span_off, spans) in serve order -> the
    (tails, off, pin_off, pins, m) form, with m the exact phase-1 answer of every
    request against all earlier ones (oracle.prefix_lengths_sequential) and the
    pins of its marker spans rebased to the tail (engine.py:170-179)."""
    from oracle import oracle as O

    reqs, spans = [], []
    for tok, off, soff, sp in waves:
        for r in range(off.size - 1):
            reqs.append(tok[off[r]:off[r + 1]])
            spans.append(sp[2 * soff[r]:2 * soff[r + 1]].reshape(-1, 2))
    ms = O.prefix_lengths_sequential(reqs)
    out, k = [], 0
    for tok, off, soff, sp in waves:
        n = off.size - 1
        streams, pins, mm = [], [], []
        for r in range(n):
            m = ms[k]
            streams.append(reqs[k][m:])
            pins.append(sorted(O.marker_pin_offsets((max(int(a) - m, 0), int(b) - m) for a, b in spans[k]
                                                    if int(b) - 1 >= m)))
            mm.append(m)
            k += 1
        out.append(pack_tails((streams, pins, mm)))
    return out


def sharded_parity(pipe, plan, R, header, marker, body, check_dev, graphs, peers, novel_rows, req_stride, wave0,
                   rank, world, chunks_per_request=3):
    """The checker at N > 1 (after every timed region). Every rank serves its
    never-served check wave through the sharded production path; rank 0 then
    rebuilds EVERY rank's waves (each rank's generator is seeded by its rank) and
    replays one global sequential oracle: phase 1 per rank (a rank's sessions are
    its own), then first-writer-wins over all ranks' chunks in the exchange's
    global order (wave, request, rank), with first-writer rows handed out by the
    fingerprint's owner in its sub-range of the writer's pool (shard.py). Checked
    on EVERY rank (results gathered to rank 0): its check wave's service map,
    bit-exact, and a stratified sample of its hit rows against the oracle's
    rotate+gather of the WRITER's pool bytes (peer pools read through their
    CUDA-IPC mappings) -- ranks other than the body's first writer read rows
    fetched from another GPU."""
    # every rank's waves in serve order (the plan's order; the same generator calls as run_ours)
    def waves_of(k):
        rng = np.random.default_rng(1000 + k)
        ws = {kind: [pack_requests(*make_requests(rng, header, marker, body, R)) for _ in range(n)]
              for kind, n in plan.items()}
        return [w for kind in plan for w in ws[kind]]

    return sharded_check(pipe, waves_of, R, check_dev, graphs, peers, novel_rows, req_stride, wave0, rank, world,
                         chunks_per_request)


def sharded_check(pipe, waves_of, R, check_dev, graphs, peers, novel_rows, req_stride, wave0, rank, world,
                  chunks_per_request=3, prefix=True):
    """The common part of the N > 1 checkers: serve this rank's check wave (``check_dev``)
    through the sharded path, then replay one global sequential oracle over ``waves_of(k)``
    (rank k's whole-request waves in serve order, its check wave last) for every rank k:
    phase 1 per rank, first-writer-wins across ranks in the exchange's order (wave, request,
    rank), owner-allocated rows; check this rank's service map and a KV sample against the
    writer's pool bytes; gather every rank's verdict. ``prefix``: the waves are whole
    requests (phase 1 on the device, replayed exactly here) -- else tails with their m."""
    import torch

    from oracle import oracle as O

    grab = {}
    load = (lambda i: pipe.load_requests(*check_dev)) if prefix else (lambda i: pipe.load(*check_dev))
    run_sharded(pipe, 1, load, wave0, graphs,
                after_front=lambda i, s: grab.__setitem__("hit", pipe.slots[s]["hit"].clone()))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    per_rank = [whole_to_tails(waves_of(k)) if prefix else waves_of(k) for k in range(world)]
    n_waves = len(per_rank[0])
    chunks = [[None] * n_waves for _ in range(world)]
    for k in range(world):
        for w, (tok, off, poff, pins, ms) in enumerate(per_rank[k]):
            recs = []
            for r in range(off.size - 1):
                st, ln, fp, _ = O.cdc_chunk(tok[off[r]:off[r + 1]], pins=pins[poff[r]:poff[r + 1]])
                recs += [(int(ms[r]) + s_, l_, f_, r) for s_, l_, f_ in zip(st.tolist(), ln.tolist(), fp.tolist())]
            chunks[k][w] = recs
    reg, novel = {}, set()
    for w in range(n_waves):  # the exchange's global order: (wave, request, rank), chunks in order
        for r in range(R):
            for k in range(world):
                for j, (p, l, f, rr) in enumerate(chunks[k][w]):
                    if rr == r and p >= CARVE and f not in reg:
                        reg[f] = (k, w, j, p)
                        novel.add((k, w, j))
    region, nxt, rows = novel_rows // world, {}, {}
    for k in range(world):  # owner o bump-allocates in its sub-range of writer k's pool, in k's query order
        for w in range(n_waves):
            for j, (p, l, f, r) in enumerate(chunks[k][w]):
                if (k, w, j) in novel:
                    o = ((f >> 32) * world) >> 32
                    rows[(k, w, j)] = o * region + nxt.get((o, k), 0)
                    nxt[(o, k)] = nxt.get((o, k), 0) + l
    recs = []
    for j, (p, l, f, r) in enumerate(chunks[rank][n_waves - 1]):  # this rank's check wave
        if p < CARVE:
            recs.append((-1, -1, -1, 0, p, l, r))
        else:
            wk, ww, wj, p_src = reg[f]
            recs.append((0 if (wk, ww, wj) == (rank, n_waves - 1, j) else 1, wk, rows[(wk, ww, wj)], p_src, p, l,
                         r))
    want = np.array([x[0] for x in recs], np.int64)
    got_hit = grab["hit"].cpu().numpy().astype(np.int64)
    map_ok = bool(np.array_equal(got_hit[:want.size], want) and (got_hit[want.size:] == -1).all())
    out = pipe.slots[0]["out"]
    sample = []
    for r in range(R):
        hr = [x for x in recs if x[0] == 1 and x[6] == r]
        if hr:
            sample += [hr[i] for i in sorted({0, len(hr) // 2, len(hr) - 1})[:chunks_per_request]]
    ckv_ok, kr_err, n_rows, remote = True, 0.0, 0, 0
    inv = np.power(THETA, -2.0 * np.arange(KR // 2) / KR)
    f32 = lambda u: (u.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    for code, wk, row, p_src, p, l, r in sample:
        got = out[:, r * req_stride + p:r * req_stride + p + l].view(torch.int16).cpu().numpy().view(np.uint16)
        src = peers[wk][:, row:row + l].view(torch.int16).cpu().numpy().view(np.uint16)
        exp = np.zeros_like(got)
        O.rotate_gather_bf16(np.ascontiguousarray(src), exp, np.zeros(1, np.int64), np.zeros(1, np.int64),
                             np.array([l], np.int32), np.array([p - p_src], np.int64), inv, interleaved=True)
        ckv_ok &= bool(np.array_equal(got[..., :CKV], exp[..., :CKV]))
        e = f32(exp[..., CKV:])
        kr_err = max(kr_err, float(np.abs(f32(got[..., CKV:]) - e).max() / max(np.abs(e).max(), 1e-30)))
        n_rows += l
        remote += l if wk != rank else 0
    mine = {"ok": bool(map_ok and ckv_ok and kr_err <= 2.0 ** -7 and sample), "service_map_bit_exact": map_ok,
            "chunks": int(want.size), "hits": int((want == 1).sum()), "kv_rows_checked": n_rows,
            "kv_rows_first_written_by_another_gpu": remote, "ckv_bit_exact": ckv_ok, "kr_max_rel": kr_err}
    import torch.distributed as dist

    every = [None] * world
    dist.all_gather_object(every, mine)
    return {"ok": all(x["ok"] for x in every),
            "service_map_bit_exact": all(x["service_map_bit_exact"] for x in every),
            "ckv_bit_exact": all(x["ckv_bit_exact"] for x in every), "kr_max_rel": max(x["kr_max_rel"] for x in every),
            "kv_rows_checked": sum(x["kv_rows_checked"] for x in every),
            "kv_rows_first_written_by_another_gpu": sum(x["kv_rows_first_written_by_another_gpu"] for x in every),
            "per_rank": every,
            "sample": f"every rank's check wave ({R} fresh requests) through the sharded timed path vs one global "
                      f"sequential oracle over {world} ranks x {n_waves} waves ({time.perf_counter() - t0:.1f} s); "
                      f"KV: first/middle/last hit chunk per request x all layers, from the writer's pool"}


def pipeline_parity(pipe, served, check_packed, check_dev, overlapped, sharded, graphs, pool, req_stride, wave0,
                    chunks_per_request=3, theta=THETA, prefix=False):
    """The checker for the timed path. Runs the never-served
    check wave (``check_packed`` / its device copy ``check_dev``) through the same
    production path the timed region used (overlapped graphs / serial graph /
    sharded), then replays the sequential oracle over every wave this process
    served, in serve order (``served``: packed waves; re-served waves insert
    nothing new):
    oracle/irm_oracle.c CDC + xxh64 per request, a first-writer-wins dict with
    the carve-out (engine.py:181-226) and pool rows handed out in query order
    (store.cu). Checked: the check wave's per-chunk service map, bit-exact; and,
    for a stratified sample of hit chunks (first, middle, last of every
    request), every row in all layers against oracle rotate+gather
    (registry.py:146-166) of the GPU pool's own bytes: c_KV bit-exact, k_r
    within bf16 rounding."""
    import torch

    from oracle import oracle as O

    hit_map = {}
    load = lambda i: pipe.load_requests(*check_dev) if prefix else pipe.load(*check_dev)
    if overlapped:
        grab = lambda i, s: hit_map.__setitem__("hit", pipe.slots[s]["hit"].clone())
        if sharded:
            run_sharded(pipe, 1, load, wave0, graphs, after_front=grab)
        else:
            pipe.run_overlapped(1, load, after_front=grab)
        torch.cuda.synchronize()
        out = pipe.slots[0]["out"]
    else:
        load(0)
        pipe.step_sharded(wave0) if sharded else pipe.replay()
        torch.cuda.synchronize()
        hit_map["hit"] = pipe.hit.clone()
        out = pipe.out
    got_hit = hit_map["hit"].cpu().numpy().astype(np.int64)

    t0 = time.perf_counter()
    reg, rows_next = {}, 0
    order = list(served) + [check_packed]
    if prefix:  # whole requests: phase 1 replayed exactly (K0 ran on the device)
        order = whole_to_tails(order)
    for wave in order:
        tok, off, poff, pins, ms = wave
        recs = []
        for r in range(off.size - 1):
            st, ln, fp, _ = O.cdc_chunk(tok[off[r]:off[r + 1]], pins=pins[poff[r]:poff[r + 1]])
            for s_, l_, f_ in zip(st.tolist(), ln.tolist(), fp.tolist()):
                p = int(ms[r]) + s_
                if p < CARVE:
                    recs.append((-1, 0, -1, p, l_, r))
                elif f_ in reg:
                    recs.append((1, reg[f_][0], reg[f_][1], p, l_, r))
                else:
                    reg[f_] = (p, rows_next)
                    recs.append((0, p, rows_next, p, l_, r))
                    rows_next += l_
    want = np.array([x[0] for x in recs], np.int64)
    n = want.size
    map_ok = bool(np.array_equal(got_hit[:n], want) and (got_hit[n:] == -1).all())
    # stratified KV sample: first / middle / last hit chunk of every request, all rows, all layers
    sample = []
    for r in range(pipe.R):
        hr = [x for x in recs if x[0] == 1 and x[5] == r]
        if hr:
            idx = sorted({0, len(hr) // 2, len(hr) - 1})[:chunks_per_request]
            sample += [hr[i] for i in idx]
    src = np.array([x[2] for x in sample], np.int64)
    ln = np.array([x[4] for x in sample], np.int32)
    delta = np.array([x[3] - x[1] for x in sample], np.int64)
    dst_rows = np.concatenate([x[5] * req_stride + x[3] + np.arange(x[4]) for x in sample])
    src_rows = np.concatenate([x[2] + np.arange(x[4]) for x in sample])
    got = out[:, torch.from_numpy(dst_rows).to(out.device)].view(torch.int16).cpu().numpy().view(np.uint16)
    mini = pool[:, torch.from_numpy(src_rows).to(pool.device)].view(torch.int16).cpu().numpy().view(np.uint16)
    mini = np.ascontiguousarray(mini)
    starts = np.concatenate([[0], np.cumsum(ln)[:-1]]).astype(np.int64)
    exp = np.zeros_like(got)
    inv = np.power(theta, -2.0 * np.arange(KR // 2) / KR)
    O.rotate_gather_bf16(mini, exp, starts, starts, ln, delta, inv, interleaved=True)
    ckv_ok = bool(np.array_equal(got[..., :CKV], exp[..., :CKV]))
    f = lambda u: (u.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    g, e = f(got[..., CKV:]), f(exp[..., CKV:])
    kr_err = float(np.abs(g - e).max() / max(np.abs(e).max(), 1e-30))
    rel = O.rel_l2(g, e)
    return {"ok": bool(map_ok and ckv_ok and kr_err <= 2.0 ** -7 and rel <= 4.7e-3 and len(sample) > 0),
            "service_map_bit_exact": map_ok, "chunks": int(n), "hits": int((want == 1).sum()),
            "kv_rows_checked": int(dst_rows.size), "layers": int(got.shape[0]), "ckv_bit_exact": ckv_ok,
            "kr_max_rel": kr_err, "kr_rel_l2": rel, "bound": "c_KV bit-exact; k_r within bf16 rounding (2^-7 of max), "
                                                          "rel-L2 <= 4.7e-3",
            "sample": f"check wave ({pipe.R} fresh requests, never served before) through the timed path; oracle "
                      f"replayed over {len(order)} waves ({time.perf_counter() - t0:.1f} s); KV: first/middle/last "
                      f"hit chunk per request x all layers"}


# ----------------------------------------------------------------- config 5: sharded sessions
C5_SESSIONS_PER_GPU, C5_R, C5_BODY, C5_DOC, C5_HEADER = 64, 16, 16384, 2048, 64


def c5_request(s, t, header, doc, marker):
    """Session s, turn t of the config-5 agent workload (the agent_meta shape of
    workloads.py:85-100 per session): the fleet-wide system header, the turn's
    metadata, the marker, a tool document shared by every session, and the
    session's own 16K-token context. Returns (tail after the header, pins, m)."""
    srng = np.random.default_rng(1_000_003 * (s + 1))
    body = srng.integers(0, 2**32, size=C5_BODY, dtype=np.uint64).astype(np.uint32)
    trng = np.random.default_rng(7_919 * (s + 1) + t)
    meta = trng.integers(0, 2**32, size=int(trng.integers(30, 71)), dtype=np.uint64).astype(np.uint32)
    tail = np.concatenate([meta, marker, doc, body])
    return tail, sorted({meta.size - 1, meta.size + 63}), C5_HEADER


def c5_wave(rank, world, sessions, block, turn, header, doc, marker):
    """R requests of this rank: local sessions [block*R, (block+1)*R) at `turn`
    (global session id = rank + world * local index: sessions s mod G)."""
    streams, pins, ms = [], [], []
    for i in range(block * C5_R, (block + 1) * C5_R):
        tail, p, m = c5_request(rank + world * (i % sessions), turn, header, doc, marker)
        streams.append(tail)
        pins.append(p)
        ms.append(m)
    off = np.zeros(len(streams) + 1, np.int64)
    np.cumsum([x.size for x in streams], out=off[1:])
    poff = np.zeros(len(streams) + 1, np.int64)
    np.cumsum([len(p) for p in pins], out=poff[1:])
    return (np.concatenate(streams), off, poff, np.array([x for p in pins for x in p], np.int64),
            np.array(ms, np.int64))


def run_config5(args):
    """BASELINE.json configs[4]: agent sessions partitioned s mod G over the GPUs
    (64 per GPU: 512 at 8 GPUs, weak scaling), the chunk store sharded by
    fingerprint prefix with the NCCL all-to-all lookup and peer replica fetch
    (shard.py) captured in the two-wave CUDA graphs. A step = one wave of 16
    session turns per GPU (~18.6K tokens each). Turn 0 of every session (cold:
    inserts the contexts) runs untimed; warm-up and timed waves are later turns
    (new metadata, contexts and the shared tool document reattached)."""
    import torch
    import torch.distributed as dist

    from paper_2605_05696_b200 import _native as N, ops, shard
    from paper_2605_05696_b200.chunking import canonical_marker
    from paper_2605_05696_b200.pipeline import ReattachPipeline

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("IRM_BENCH_ONE_DEVICE") == "1":
        local = 0
    backend = os.environ.get("IRM_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    if backend == "nccl":
        nccl_logs_to_stderr(world)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    hbm, _tf, _tfs, peak_kind = peaks()
    sessions = args.sessions_per_gpu
    assert sessions % C5_R == 0, "sessions per GPU must be a multiple of the wave size"
    blocks = sessions // C5_R
    shared = np.random.default_rng(77)
    header = shared.integers(0, 2**32, size=C5_HEADER, dtype=np.uint64).astype(np.uint32)
    doc = shared.integers(0, 2**32, size=C5_DOC, dtype=np.uint64).astype(np.uint32)
    marker = np.array(canonical_marker(), np.uint32)
    # schedule: turn-major over the blocks of R sessions; turn 0 = cold
    n_cold = blocks
    n_steps = args.warmup + args.steps
    sched = [(b % blocks, 1 + b // blocks) for b in range(2 * n_steps + 1)]
    cold = [c5_wave(rank, world, sessions, b, 0, header, doc, marker) for b in range(n_cold)]
    warm = [c5_wave(rank, world, sessions, b, t, header, doc, marker) for b, t in sched]
    to_dev = lambda p: tuple(torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).to(dev) for a in p)
    to_pin = lambda p: tuple(torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).pin_memory()
                             for a in p)
    cold_dev = [to_dev(p) for p in cold]
    warm_dev = [to_dev(p) for p in warm[:n_steps + 1]]
    warm_host = [to_pin(p) for p in warm[n_steps + 1:]]
    check_wave = c5_wave(rank, world, sessions, 0, 10_000, header, doc, marker)  # the in-run checker's wave
    sized = cold + warm + [check_wave]
    max_tok = max(int(p[1][-1]) for p in sized)
    max_pins = max(int(p[2][-1]) for p in sized)
    req_stride = max(int(np.diff(p[1]).max()) for p in sized) + C5_HEADER

    # pool: [0, novel) first-writer rows (one sub-range per owner), then replicas, then scratch
    n_waves_total = n_cold + 2 * n_steps + 4
    novel_est = sessions * C5_BODY + C5_DOC + C5_R * 80 * n_waves_total + 1024  # contexts + every turn's metadata
    sub = (int(1.25 * novel_est / world) + 4096) if world > 1 else novel_est + 4096
    novel_rows = sub * world
    replica_rows = 4 * C5_DOC + 16384
    scratch = 2 * C5_DOC + 4096
    pool_rows = novel_rows + replica_rows + 2 * scratch
    pool = torch.empty(LAYERS, pool_rows, CKV + KR, dtype=torch.bfloat16, device=dev)
    for l in range(LAYERS):  # random-init latents, one layer at a time (no fp32 temporary)
        pool[l].normal_()
    inv = ops.inv_freq_device(np.power(THETA, -2.0 * np.arange(KR // 2) / KR))
    store = ops.ChunkStore(max_entries=1 << 20)
    pipe = ReattachPipeline(store, pool, inv, C5_R, max_tok, max_pins, req_stride, layout=N.LAYOUT_INTERLEAVED)
    peers = shard.map_peer_pools(pool)
    cache = shard.ReplicaCache(pool, novel_rows, peers, rank, ops.ChunkStore(max_entries=1 << 14),
                               scratch_rows=scratch)
    sharded = shard.ShardedStore(store, novel_rows)
    pipe.enable_sharding(sharded, cache, rank, world)

    graphs = backend == "nccl"
    lc0 = ops.launch_count()
    pipe.load(*cold_dev[0])
    pipe.step_sharded(0)  # one eager wave: our kernels per wave (the graphs replay the same launches)
    launches_per_wave = ops.launch_count() - lc0
    if graphs:
        pipe.capture_overlapped(k4_sms=K4_SMS_SHARDED, sharded=True)
    run_sharded(pipe, n_cold - 1, lambda i: pipe.load(*cold_dev[1 + i]), 1, graphs)
    wave = n_cold
    run_sharded(pipe, args.warmup, lambda i: pipe.load(*warm_dev[i]), wave, graphs)
    wave += args.warmup
    torch.cuda.synchronize()
    dist.barrier()

    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        pipe.hit_tokens.zero_()
        t0.record()
        run_sharded(pipe, args.steps, lambda i: pipe.load(*warm_dev[args.warmup + i]), wave, graphs)
        t1.record()
        torch.cuda.synchronize()
    wave += args.steps
    ms_total = t0.elapsed_time(t1)
    hit_tok = int(pipe.hit_tokens.item())
    t = torch.tensor([ms_total], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ht = torch.tensor([hit_tok], device=dev, dtype=torch.int64)
    dist.all_reduce(ht)
    hit_all = int(ht.item())
    value = hit_all / (ms_total / 1e3)

    # e2e: the next turns from pinned host buffers, service maps read back
    n_e2e = min(args.steps, len(warm_host))
    res = [torch.empty(pipe.slots[0]["hit"].shape, dtype=pipe.slots[0]["hit"].dtype, pin_memory=True)
           for _ in range(n_e2e)]
    pipe.hit_tokens.zero_()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if graphs:
        pipe.run_overlapped(n_e2e, lambda i: pipe.load(*warm_host[i]), readback=res, wave0=wave)
    else:
        pipe.run_overlapped_sharded(n_e2e, lambda i: pipe.load(*warm_host[i]), wave0=wave, k4_sms=K4_SMS_SHARDED,
                                    after_front=lambda i, sl: res[i].copy_(pipe.slots[sl]["hit"], non_blocking=True))
    e1.record()
    torch.cuda.synchronize()
    wave += n_e2e
    e2e_ms = e0.elapsed_time(e1)
    t = torch.tensor([e2e_ms], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ht = torch.tensor([int(pipe.hit_tokens.item())], device=dev, dtype=torch.int64)
    dist.all_reduce(ht)
    e2e_value = int(ht.item()) / (float(t.item()) / 1e3)
    bi = sum(x.numel() * x.element_size() for x in warm_host[0])
    bo = res[0].numel() * res[0].element_size() if n_e2e else 0
    sharded.check()
    cache.check()
    pipe.check()
    fetched = torch.stack([cache.fetched_runs, cache.fetched_rows]).to(torch.int64)
    dist.all_reduce(fetched)
    fetched = fetched.tolist()
    # the exchange alone: K1 of a served wave, then its sharded lookup again (all hits), timed per rank
    pipe.load(*warm_dev[0])
    pipe.k1()
    torch.cuda.synchronize()
    dist.barrier()
    for _ in range(2):  # warm (first calls allocate)
        pipe.k3_sharded(10**6)
    torch.cuda.synchronize()
    x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x0.record()
    for _ in range(3):
        pipe.k3_sharded(10**6)
    x1.record()
    torch.cuda.synchronize()
    xt = torch.tensor([x0.elapsed_time(x1) * 1e3 / 3], device=dev)
    every_us = [torch.zeros_like(xt) for _ in range(world)]
    dist.all_gather(every_us, xt)
    exchange_us = [float(x.item()) for x in every_us]
    # the same exchange as the timed step runs it: captured once in a CUDA graph, replayed
    exchange_graph_us = None
    if graphs:
        gx = torch.cuda.CUDAGraph()
        sx = torch.cuda.Stream()
        sx.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(sx):
            pipe.k3_sharded(10**6)
        torch.cuda.current_stream().wait_stream(sx)
        torch.cuda.synchronize()
        with torch.cuda.graph(gx):
            pipe.k3_sharded(10**6)
        gx.replay()
        torch.cuda.synchronize()
        dist.barrier()
        x0.record()
        for _ in range(10):
            gx.replay()
        x1.record()
        torch.cuda.synchronize()
        xt = torch.tensor([x0.elapsed_time(x1) * 1e3 / 10], device=dev)
        every_us = [torch.zeros_like(xt) for _ in range(world)]
        dist.all_gather(every_us, xt)
        exchange_graph_us = [float(x.item()) for x in every_us]
        del gx
    # K4 of that re-probed wave (every chunk a hit), timed alone after an L2 flush: the roofline
    k4_rows = int(pipe.length.sum().item()) * LAYERS
    ng = int(pipe.groups.n_groups.item())
    src_rows = int(pipe.groups.g_len[:ng].to(torch.int64).sum().item()) * LAYERS
    k4_ms = timed_flushed(pipe.k4, 10)
    k4_bytes = (k4_rows + src_rows) * (CKV + KR) * 2
    k4_gbs = k4_bytes / (k4_ms / 1e3) / 1e9

    if world == 1:
        check = check_wave
        served = cold + warm[:n_steps] + warm[n_steps + 1:n_steps + 1 + n_e2e]
        parity = pipeline_parity(pipe, served, check, to_dev(check), True, True, graphs, pool, req_stride, wave0=wave)
    else:  # every rank's check wave vs one global oracle over all ranks' waves (rebuilt per rank k)
        def waves_of(k):
            c = [c5_wave(k, world, sessions, b, 0, header, doc, marker) for b in range(n_cold)]
            wk = [c5_wave(k, world, sessions, b, t, header, doc, marker) for b, t in sched]
            return (c + wk[:n_steps] + wk[n_steps + 1:n_steps + 1 + n_e2e]
                    + [c5_wave(k, world, sessions, 0, 10_000, header, doc, marker)])

        check = check_wave
        parity = sharded_check(pipe, waves_of, C5_R, to_dev(check), graphs, peers, novel_rows, req_stride, wave,
                               rank, world, prefix=False)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"config 5: {sessions * world} agent sessions ({sessions} per GPU, s mod G), "
                               f"27 layers, DSv2 interleaved theta 1e4, ~{C5_BODY // 1024 + 2}K-token turns",
                   "sessions": sessions * world, "sessions_per_gpu": sessions, "requests_per_step": C5_R,
                   "tokens_per_request": int(np.mean(np.diff(warm[0][1]))) + C5_HEADER, "layers": LAYERS,
                   "l2": "inputs larger than L2 (pool of %.0f GB per GPU)" % (pool.numel() * 2 / 1e9),
                   "pipeline": "two-wave overlap (%s); sharded lookup (%s all-to-alls%s) + peer replica fetch"
                               % (k4_placement(K4_SMS_SHARDED), backend,
                                  " captured in the CUDA graphs" if graphs else ", streams"),
                   "parallelism": f"sessions s mod G over {world} GPU(s), store sharded by fingerprint prefix"},
        "exchange": {"lookup_us_per_rank": exchange_us, "lookup_graph_us_per_rank": exchange_graph_us,
                     "lookup_graph_note": "the same exchange captured in one CUDA graph and replayed (10 replays, "
                                          "CUDA events per rank): the form the timed step runs",
                     "lookup_note": "eager (host-launched) exchange of one wave (re-probe, all hits): irm_exchange_pack, "
                                    "all-to-all, split, K3 on the owner's shard, reply, reverse all-to-all, unpack, "
                                    "replica lookup; CUDA events per rank; in the timed step the same work is "
                                    "replayed from the front's CUDA graph",
                     "bytes_per_lookup": sharded.last_exchange_bytes, "owner_slots": sharded.owner_slots or
                     (sharded.slots if world == 1 else min(sharded.slots, (5 * sharded.slots) // (4 * world) + 64)),
                     "query_capacity": sharded.slots, "replica_runs_fetched_all_ranks": fetched[0],
                     "replica_rows_fetched_all_ranks": fetched[1]},
        "roofline": {"bound": "hbm", "kernel": "irm_rotate_gather_fanout (K4 fan-out)", "achieved": k4_gbs,
                     "peak": hbm, "unit": "GB/s", "frac": k4_gbs / hbm,
                     "traffic": ncu_traffic("rotate_gather_ws_kernel" if pipe.fanout else "rotate_gather_tma", "config5"),
                     "peak_kind": peak_kind,
                     "launch_ms": k4_ms, "algorithmic_bytes": k4_bytes, "source_rows_read": src_rows,
                     "rows_written": k4_rows, "wave": "a served wave re-probed (every chunk a hit), rank 0",
                     "peak_note": "the peak is MEASURED_PEAKS.json's torch copy (1:1 read:write); at this wave's "
                                  "~0.9:1 mix K4's bulk TMA streams can move more (frac > 1 is possible)",
                     "bytes_rule": "1152 B per distinct source row read (once per launch) + 1152 B per reattached "
                                   "row written, x 27 layers"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo},
        "parity": parity,
        "gpu_launches": args.steps * launches_per_wave,
        "clocks": clk.summary(),
    }
    if rank == 0:
        emit(line)
    dist.destroy_process_group()


def run_sharded(pipe, n, load, wave0, graphs, after_front=None, readback=None):
    if graphs:
        pipe.run_overlapped(n, load, after_front=after_front, wave0=wave0, readback=readback)
    else:
        assert readback is None, "the stream pipeline reads service maps back in after_front"
        pipe.run_overlapped_sharded(n, load, wave0=wave0, k4_sms=K4_SMS_SHARDED, after_front=after_front)


# ----------------------------------------------------------------- the reference-facing serve API
_REF_SERVE = r"""
import hashlib, json, sys, time
sys.path.insert(0, sys.argv[1])
from irminsul import engine, model
text = open(sys.argv[2]).read()
t0 = time.perf_counter()
import io
trace = model.parse_trace(io.StringIO(text))
state = engine.EngineState(engine.ServeConfig())
results, row = engine.run_trace(state, trace)
dt = time.perf_counter() - t0
h = hashlib.sha256()
for ri, r in enumerate(results):
    for e in r.events:
        h.update(repr((ri, e.start, e.length, e.klass.value, e.fingerprint, e.delta)).encode())
print(json.dumps({"seconds": dt, "digest": h.hexdigest()[:16], "tokens": sum(r.num_tokens for r in results)}))
"""


def serve_api_component(n_warm=8):
    """The drop-in's public serve API end to end (engine.run_trace, engine.py:283-306)
    on a config-2 trace: one cold + ``n_warm`` warm 32.9K-token agent_meta requests
    as JSONL text -> model.parse_trace (native ingest) -> run_trace in one batch:
    K0 prefix match/insert, K1 CDC + xxh64, K3 first-writer-wins store, per-request
    events on the host (observer mode). Tokens served per second, all included.
    When the reference is installed (baseline/_ref, the offline pip install), the
    reference's own parse_trace + run_trace runs the same text on the same host and
    the two event streams are compared by digest."""
    import hashlib
    import io
    import tempfile

    import torch

    from paper_2605_05696_b200 import engine, model
    from paper_2605_05696_b200.chunking import canonical_marker

    shared = np.random.default_rng(7)
    header = tuple(int(t) for t in shared.integers(0, 2**32, size=HEADER, dtype=np.uint64))
    body = tuple(int(t) for t in shared.integers(0, 2**32, size=BODY, dtype=np.uint64))
    marker = tuple(canonical_marker())
    rng = np.random.default_rng(99)
    reqs = []
    for i in range(1 + n_warm):
        meta = tuple(int(t) for t in rng.integers(0, 2**32, size=int(rng.integers(30, 71)), dtype=np.uint64))
        reqs.append(model.Request(f"s{i}", 0, (model.Segment("system", header, "agent_header"),
                                               model.Segment("header", meta), model.Segment("marker", marker),
                                               model.Segment("body", body, "agent_body"))))
    text = model.serialize_trace(model.Trace(tuple(reqs)))
    times = []
    for _ in range(6):  # the first pass pays one-time library / allocator set-up; median of the other 5
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        trace = model.parse_trace(io.StringIO(text))
        ta = time.perf_counter()
        state = engine.EngineState(engine.ServeConfig())
        tb = time.perf_counter()
        results, row = engine.run_trace(state, trace)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        if os.environ.get("IRM_BENCH_SERVE_DEBUG"):
            print(f"serve_api pass: parse {1e3 * (ta - t0):.1f} ms, state {1e3 * (tb - ta):.1f} ms, run_trace "
                  f"{1e3 * (times[-1] - (tb - t0)):.1f} ms", file=sys.stderr)
        # a server keeps one state; here each pass builds its own, so the previous pass's device
        # tables are released first and the caching allocator hands their blocks to the next
        # pass instead of cudaMalloc-ing a second set while the first is still referenced
        del state, trace
    dt = statistics.median(times[1:])  # (a fresh EngineState occasionally meets a ~0.1 s device allocation)
    n_tok = sum(r.num_tokens for r in results)
    pic = sum(r.counts[engine.ServiceClass.PIC_HIT] for r in results)
    h = hashlib.sha256()
    for ri, r in enumerate(results):
        for e in r.events:
            h.update(repr((ri, e.start, e.length, e.klass.value, e.fingerprint, e.delta)).encode())
    out = {"value": n_tok / dt, "unit": "tokens/s", "api": "model.parse_trace + engine.run_trace (observer)",
           "workload": f"{1 + n_warm} x {n_tok // (1 + n_warm)}-token agent_meta requests as JSONL "
                       f"({len(text) / 1e6:.1f} MB), one serve batch; median of 5 timed passes, each with a "
                       f"fresh EngineState", "seconds": dt,
           "pic_hit_tokens": pic, "warm_total_cached": row.warm_total, "events_digest": h.hexdigest()[:16]}
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "irminsul")):
        with tempfile.NamedTemporaryFile("w", suffix=".jsonl", delete=False) as f:
            f.write(text)
        try:
            p = subprocess.run([sys.executable, "-c", _REF_SERVE, ref_dir, f.name], capture_output=True, text=True,
                               timeout=600)
            r = json.loads(p.stdout.strip().splitlines()[-1])
            out["reference"] = {"value": r["tokens"] / r["seconds"], "unit": "tokens/s", "seconds": r["seconds"],
                                "events_digest": r["digest"], "events_identical": r["digest"] == out["events_digest"],
                                "what": "the reference package itself (baseline/_ref: irminsul 0.1.0, pure Python), "
                                        "same JSONL text, same host, one process"}
        except Exception as e:  # the comparison is informational; never fail the bench line on it
            out["reference"] = {"unavailable": f"{type(e).__name__}: {e}"}
        finally:
            os.unlink(f.name)
    return out


# ----------------------------------------------------------------- producer rotation
def producer_component(hbm, n_rows=BODY):
    """The producer side of the store (registry.py:126-140) at the
    config-2 shape: the cold request's 32,768 novel rows, kr_raw of all 27 layers
    rotated in place to p_src + i by ONE irm_rotate_rows_layered launch (cos/sin
    per (row, frequency) once, applied to every layer). HBM-bound: the 128-byte
    k_r slice of each 1,152-byte bf16 row is read and written."""
    import torch

    from paper_2605_05696_b200 import _native as N, ops

    rng = np.random.default_rng(41)
    pool = torch.randn(LAYERS, n_rows + 64, CKV + KR, device="cuda").to(torch.bfloat16)
    kr = pool[:, :n_rows, CKV:]
    lens, pos = [], []
    while sum(lens) < n_rows:
        lens.append(min(int(rng.integers(32, 400)), n_rows - sum(lens)))
    p0 = 50 + 64
    for ln in lens:
        pos.append(np.arange(p0, p0 + ln))
        p0 += ln
    positions = torch.from_numpy(np.concatenate(pos).astype(np.float64)).cuda()
    inv = ops.inv_freq_device(np.power(THETA, -2.0 * np.arange(KR // 2) / KR))
    run = lambda: ops.rotate_rows_layered(kr, positions, inv, N.LAYOUT_INTERLEAVED, out=kr)
    run()
    ms = timed_flushed(run, 20)
    rows = n_rows * LAYERS
    byt = rows * KR * 2 * 2
    return {"value": rows / (ms / 1e3), "unit": "rows/s", "kernel": "irm_rotate_rows_layered (producer)",
            "workload": f"{n_rows} novel rows x {LAYERS} layers, bf16 k_r rotated in place to p_src + i "
                        f"({len(lens)} chunks), DSv2 interleaved theta {THETA:g}",
            "launch_ms": ms, "roofline": {"bound": "hbm", "achieved": byt / (ms / 1e3) / 1e9, "peak": hbm,
                                          "unit": "GB/s", "frac": byt / (ms / 1e3) / 1e9 / hbm,
                                          "bytes_rule": "128 B of k_r read + written per (row, layer)"}}


# ----------------------------------------------------------------- K1 with wide parallelism
def cdc_wide_component(hbm, n_streams=296, n_tok=32768):
    """K1 over a config-5-sized wave: 296 independent 32K-token session tails (2 per SM).
    CDC is sequential within a pin-delimited region (one bit of carried state per
    token, K1), so K1's throughput is regions in flight x per-region rate;
    the config-2 line above has only 8 long regions per wave."""
    import torch

    from paper_2605_05696_b200 import ops

    rng = np.random.default_rng(21)
    tok = torch.from_numpy(rng.integers(0, 2**32, size=n_streams * n_tok, dtype=np.uint64).astype(np.uint32)
                           .view(np.int32)).cuda()
    off = torch.arange(0, (n_streams + 1) * n_tok, n_tok, dtype=torch.int64, device="cuda")
    ws = ops.CdcWorkspace()
    run = lambda: ops.cdc_xxh64(tok, off, None, None, 7, 32, 512, True, ws=ws, n_tokens=tok.numel())
    t = run()
    ms = timed_flushed(run, 10)
    n_chunks = int(t.chunk_off[-1].item())
    byt = tok.numel() * 4 + n_chunks * 24
    return {"value": tok.numel() / (ms / 1e3), "unit": "tokens/s", "kernel": "irm_cdc_xxh64 (K1)",
            "workload": f"{n_streams} streams x {n_tok} tokens (config-5 scale wave)", "launch_ms": ms,
            "roofline": {"bound": "hbm", "achieved": byt / (ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                         "frac": byt / (ms / 1e3) / 1e9 / hbm},
            "note": "nominal HBM bound only: the launch is set by each region's serial chain and walker "
                    "(~1,024 dependent 32-token steps and ~205 dependent chunk decisions per region, 2 regions "
                    "per SM; profiles/r02_k1_wide.md)"}


# ----------------------------------------------------------------- K5 component
def attn_workload(n_ctx=65536, n_q=4096, heads=16, theta=5e4, layout=None, seed=35):
    """The reattached prompt of BASELINE.json configs 2-4 for K5: a
    ``n_ctx``-token prompt = 512-token prefix + marker-wrapped 1K-token documents
    re-permuted relative to the cached order (the rerank shape of
    workloads.py:142-162, scaled) + a novel tail holding the ``n_q`` queries.
    Its KV lives in the latent pool in SOURCE order with k_r entangled at the
    source positions; ``kv_rows`` maps request order -> pool row, ``kv_chunk``
    each key to its document (chunk 0 = delta 0). Shared by bench.py and the
    benchmarked-shape parity tests (tests/test_gpu_mla_shapes.py)."""
    import torch

    from paper_2605_05696_b200 import _native as N, ops

    rng = np.random.default_rng(seed)
    layout = N.LAYOUT_HALF_SPLIT if layout is None else layout
    doc, prefix = 960, 512  # 1K-token documents (960 + 64-token marker) after a 512-token prefix
    n_docs = (n_ctx - prefix - 512) // (doc + 64)  # 63 at 64K (65,024 tokens + a 512-token novel tail)
    seg = doc + 64
    src_start = prefix + np.arange(n_docs) * seg  # cached layout
    perm = rng.permutation(n_docs)
    kv_rows = np.arange(n_ctx, dtype=np.int64)
    chunk_of_key = np.zeros(n_ctx, np.int32)
    deltas = [0]
    for j, d in enumerate(perm):  # request layout: doc d now sits at slot j
        dst = prefix + j * seg
        kv_rows[dst:dst + seg] = src_start[d] + np.arange(seg)
        chunk_of_key[dst:dst + seg] = len(deltas)
        deltas.append(int(dst - src_start[d]))
    tail = prefix + n_docs * seg  # the novel tail holds the queries
    chunk_of_key[tail:] = 0
    dev = torch.device("cuda")
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    pool = torch.randn(n_ctx, 576, device=dev, generator=g).to(torch.bfloat16)
    q = torch.randn(n_q, heads, 576, device=dev, generator=g).to(torch.bfloat16)
    inv_np = np.power(theta, -2.0 * np.arange(32) / 64)
    inv = ops.inv_freq_device(inv_np)
    deltas = np.array(deltas, np.int64)
    cs = ops.chunk_cossin(torch.from_numpy(deltas).to(dev), inv)
    return dict(pool=pool, q=q, cs=cs, rows_d=torch.from_numpy(kv_rows.astype(np.int32)).to(dev),
                chunk_d=torch.from_numpy(chunk_of_key).to(dev), kv_rows=kv_rows, chunk_of_key=chunk_of_key,
                deltas=deltas, inv=inv_np, n_docs=n_docs, layout=layout, n_ctx=n_ctx, n_q=n_q, heads=heads,
                theta=theta)


def attn_parity(w, out, lse, sample=64, device="cuda"):
    """The checker, after the timed region: the first, a middle and the last
    ``sample`` query rows x all heads of the kernel's output against the fp64
    restatement (oracle/mla_ref.py) over their full causal context, on the
    same bf16 inputs. Bound: the north star's 4.7e-3 rel-L2; lse within 2e-2."""
    import torch

    from oracle.mla_ref import mla_reattach_ref

    n_q, n_ctx = w["n_q"], w["n_ctx"]
    mid = n_q // 2 - sample // 2
    idx = np.concatenate([np.arange(sample), np.arange(mid, mid + sample), np.arange(n_q - sample, n_q)])
    kv = w["pool"][torch.from_numpy(w["kv_rows"]).to(w["pool"].device)]  # request order
    ref, ref_lse = mla_reattach_ref(w["q"], kv, n_ctx - n_q, 192 ** -0.5, w["deltas"][w["chunk_of_key"]], w["inv"],
                                    interleaved=bool(w["layout"]), q_index=idx, device=device)
    got = out[torch.from_numpy(idx).to(out.device)].double().cpu()
    rel = float((got - ref).norm() / ref.norm())
    row = float(((got - ref).norm(dim=-1) / ref.norm(dim=-1).clamp_min(1e-30)).max())
    lerr = float((lse[torch.from_numpy(idx).to(lse.device)].double().cpu() - ref_lse).abs().max())
    return {"rel_l2": rel, "max_row_rel_l2": row, "lse_max_abs": lerr, "bound": 4.7e-3,
            "ok": bool(rel <= 4.7e-3 and lerr <= 2e-2),
            "sample": f"query rows [0,{sample}) [{mid},{mid + sample}) [{n_q - sample},{n_q}) x {out.shape[1]} heads, "
                      f"full causal context each, vs the fp64 restatement (oracle/mla_ref.py)"}


def fused_attn_component(args, tf_peak, peak_kind, n_ctx=65536, n_q=4096, heads=16, theta=5e4, layout=None,
                         shape="config 3", cpu=False):
    """BASELINE.json config 3 (Moonlight-16B-A3B shape, DSv3-form half-split
    rotary, theta 5e4) by default: attn_workload's re-permuted 64K prompt. The
    fused kernel gathers the rows (contiguous runs -> tiled TMA, seams ->
    gather4), rotates each document's k_r by its delta in shared memory, and
    runs the absorbed causal prefill of the last 4,096 (novel) query tokens
    over all 64K keys."""
    import torch

    from paper_2605_05696_b200 import _native as N, ops

    w = attn_workload(n_ctx, n_q, heads, theta, layout)
    q, pool, cs, rows_d, chunk_d, layout = w["q"], w["pool"], w["cs"], w["rows_d"], w["chunk_d"], w["layout"]
    # start from an idle GPU (1 s): the power-managed clocks after the HBM-bound step or the
    # previous component otherwise lower the first launches (1246 vs 1395 TFLOP/s measured at
    # 32K right after a 64K run); the peak it is compared with is the burst figure too
    torch.cuda.synchronize()
    time.sleep(1.0)
    out, lse = ops.mla_reattach_prefill(q, pool, n_ctx, n_ctx - n_q, 192 ** -0.5, kv_rows=rows_d,
                                        kv_chunk=chunk_d, chunk_cs=cs, layout=layout)
    torch.cuda.synchronize()
    # each launch timed alone after an L2 flush (the 64K pool, 75 MB, would otherwise stay in L2)
    ms = timed_flushed(lambda: ops.mla_reattach_prefill(q, pool, n_ctx, n_ctx - n_q, 192 ** -0.5, kv_rows=rows_d,
                                                        kv_chunk=chunk_d, chunk_cs=cs, layout=layout, out=out,
                                                        lse=lse), 5)
    pos = np.arange(n_ctx - n_q, n_ctx, dtype=np.float64)
    flops = heads * float((pos + 1).sum()) * 2176  # (2*576 + 2*512) per visible (query, key, head)
    tflops = flops / (ms / 1e3) / 1e12
    extra = {"parity": attn_parity(w, out, lse)}
    if cpu:
        extra["cpu_baseline"] = attn_cpu_baseline(q, pool, w["kv_rows"], w["chunk_of_key"], w["deltas"], theta,
                                                  layout == N.LAYOUT_INTERLEAVED, n_ctx, n_q)
    return {**extra, "value": tflops, "unit": "TFLOP/s", "kernel": "irm_mla_reattach_prefill (K5, tcgen05/TMEM)",
            "workload": f"{shape}: {n_ctx} ctx, last {n_q} queries, {heads} heads, {w['n_docs']} re-permuted docs, "
                        f"{'DSv2 interleaved' if layout == N.LAYOUT_INTERLEAVED else 'DSv3 half-split'} theta {theta:g}, bf16",
            "launch_ms": ms, "flop_per_launch": flops,
            "roofline": {"bound": "tensor", "achieved": tflops, "peak": tf_peak, "unit": "TFLOP/s",
                         "frac": tflops / tf_peak, "peak_kind": f"{peak_kind} bf16 burst",
                         "frac_vs_sustained": tflops / peaks()[2],
                         "note": "a multi-ms launch runs into the 1 kW cap like cuBLAS's sustained loop "
                                 "(profiles/r02_k5_bound.md §3); frac is against the burst figure"}}


# ----------------------------------------------------------------- CPU legs
def attn_cpu_baseline(q, pool, kv_rows, chunk_of_key, deltas, theta, interleaved, n_ctx, n_q, sample_q=64):
    """K5 has no reference CPU path: the restated absorbed MLA
    reattach prefill in torch-CPU fp32 on all host threads, for the last
    `sample_q` queries of the same workload (same bf16 inputs, keys gathered
    from the pool and their k_r rotated by each document's delta). TFLOP/s
    counts the same causally visible FLOPs as the kernel's figure."""
    import torch

    torch.set_num_threads(os.cpu_count() or 1)
    t0 = time.perf_counter()
    kv = pool.float().cpu()[torch.from_numpy(kv_rows)]  # [n_ctx, 576] in request order
    inv = torch.from_numpy(np.power(theta, -2.0 * np.arange(32) / 64))
    ang = (torch.from_numpy(deltas[chunk_of_key]).double()[:, None] * inv[None, :]).float()
    c, s_ = torch.cos(ang), torch.sin(ang)
    kr = kv[:, 512:]
    lo, hi = (kr[:, 0::2], kr[:, 1::2]) if interleaved else (kr[:, :32], kr[:, 32:])
    rlo, rhi = lo * c - hi * s_, lo * s_ + hi * c
    if interleaved:
        kr = torch.stack([rlo, rhi], dim=-1).reshape(-1, 64)
    else:
        kr = torch.cat([rlo, rhi], dim=1)
    k = torch.cat([kv[:, :512], kr], dim=1)
    qs = q[n_q - sample_q:].float().cpu()  # [sample_q, H, 576], positions n_ctx - sample_q ..
    heads = qs.shape[1]
    sc = torch.einsum("qhd,kd->qhk", qs, k) * 192 ** -0.5
    pos = torch.arange(n_ctx - sample_q, n_ctx)
    sc.masked_fill_(torch.arange(n_ctx)[None, None, :] > pos[:, None, None], float("-inf"))
    out = torch.einsum("qhk,kd->qhd", torch.softmax(sc, dim=-1), kv[:, :512])
    dt = time.perf_counter() - t0
    flops = heads * float((pos + 1).sum()) * 2176
    assert torch.isfinite(out).all()
    return {"value": flops / dt / 1e12, "unit": "TFLOP/s", "cores": torch.get_num_threads(), "kind": "restated",
            "sample": f"last {sample_q} of {n_q} queries x {heads} heads over {n_ctx} keys, torch-CPU fp32 "
                      f"(gather, delta rotation, causal softmax; {dt:.2f} s)"}


def cpu_baseline(args, packed, sample_requests=1, n_threads=0, min_seconds=0.0):
    """The oracle port (restated reference, oracle/irm_oracle.c) on host cores:
    CDC + xxh64, dict lookup, bf16 rotate+gather for `sample_requests` requests
    of the same workload, repeated until `min_seconds` of CPU work. Returns
    reattached tokens/s."""
    from oracle import oracle as O

    tok, off, poff, pins, ms = packed
    n_req = off.size - 1
    assert n_req > sample_requests, "need a cold request beyond the sample"
    streams = [tok[off[i]:off[i + 1]] for i in range(n_req)]
    pin_l = [pins[poff[i]:poff[i + 1]] for i in range(n_req)]
    threads = n_threads or O.max_threads()
    rng = np.random.default_rng(5)
    # the store holds the body chunks (cold request), as on the GPU
    cold = O.cdc_chunk(streams[-1], pins=pin_l[-1])  # the cold request populates the store
    registry = {int(f): (int(s) + HEADER, int(s)) for s, f in zip(cold[0], cold[2]) if int(s) + HEADER >= CARVE}
    rows = BODY + 4096
    # bf16 bit patterns of values in [1, 2) with random mantissas (random-init latents)
    pool = (np.uint16(0x3F80) | rng.integers(0, 128, size=(LAYERS, rows, CKV + KR), dtype=np.uint16))
    out = np.zeros((LAYERS, sample_requests * (BODY + 512), CKV + KR), np.uint16)
    out.fill(1)  # fault the pages in before the clock: the port's timing must not include first-touch
    inv = np.power(THETA, -2.0 * np.arange(KR // 2) / KR)
    t0 = time.perf_counter()
    total_hit = 0
    passes = 0
    while passes == 0 or time.perf_counter() - t0 < min_seconds:
        total_hit += _cpu_pass(O, streams, pin_l, ms, registry, pool, out, inv, sample_requests, threads)
        passes += 1
    dt = time.perf_counter() - t0
    return {"value": total_hit / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{passes} pass(es) over {sample_requests} x 32K-token request(s): oracle CDC+xxh64, dict "
                      f"lookup, bf16 rotate+gather of {total_hit} hit tokens x {LAYERS} layers ({dt:.2f} s)"}


def _cpu_pass(O, streams, pin_l, ms, registry, pool, out, inv, sample_requests, threads):
    total_hit = 0
    for i in range(sample_requests):
        st, ln, fp, fo = O.cdc_chunk(streams[i], pins=pin_l[i])
        src, dst, lens, deltas = [], [], [], []
        for s, l, f in zip(st, ln, fp):
            p = int(ms[i]) + int(s)
            if p < CARVE:
                continue
            e = registry.get(int(f))
            if e is None:
                continue
            src.append(e[1]); dst.append(i * (BODY + 512) + int(s)); lens.append(int(l)); deltas.append(p - e[0])
        total_hit += sum(lens)
        O.rotate_gather_bf16(pool, out, np.array(src), np.array(dst), np.array(lens), np.array(deltas),
                             inv, interleaved=True, n_threads=threads)
    return total_hit


def run_reference(args):
    """--impl reference: the reference algorithm's CPU implementation (the
    oracle port; the Python reference cannot travel to the GPU box) on all
    host threads, same metric/config, a bounded sample per step."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2605_05696_b200.rng import SplitMix64  # host constant only

    shared = np.random.default_rng(7)
    header = shared.integers(0, 2**32, size=HEADER, dtype=np.uint64).astype(np.uint32)
    body = shared.integers(0, 2**32, size=BODY, dtype=np.uint64).astype(np.uint32)
    gen = SplitMix64(SplitMix64(0x49524D494E53554C ^ 64).next_u64())
    marker = np.array([v & 0xFFFFFFFF for v in gen.fill(64)], np.uint32)
    rng = np.random.default_rng(1000)
    n_sample = 4
    streams, pins, ms = make_wave(rng, header, marker, body, n_sample + 1)
    off = np.zeros(len(streams) + 1, np.int64)
    np.cumsum([x.size for x in streams], out=off[1:])
    poff = np.zeros(len(streams) + 1, np.int64)
    np.cumsum([len(p) for p in pins], out=poff[1:])
    packed = (np.concatenate(streams), off, poff, np.array([x for p in pins for x in p], np.int64),
              np.array(ms, np.int64))
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(args, packed, n_sample)
        if i >= args.warmup:
            vals.append(r)
    v = statistics.median([r["value"] for r in vals])
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "DeepSeek-V2-Lite reattach (config 2): 27 layers, kv_lora 512 + rope 64, "
                                   "DSv2 interleaved rotary theta 1e4, 32K-token agent_meta prompts (CPU oracle port)",
                       "requests_per_step": n_sample},
            "cpu_baseline": {**vals[-1], "value": v},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=150)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--requests", type=int, default=R_PER_WAVE)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-attn", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="K6 sharded-store path even at N=1")
    ap.add_argument("--workload", default="config2", choices=["config2", "config5"],
                    help="config2: DeepSeek-V2-Lite 8 x 32K wave (default); config5: sharded agent sessions")
    ap.add_argument("--sessions-per-gpu", type=int, default=C5_SESSIONS_PER_GPU)
    ap.add_argument("--no-fanout", action="store_true",
                    help="K4 reads every hit's source rows (default: one read per distinct source run per wave)")
    ap.add_argument("--serial", action="store_true",
                    help="one graph per wave, K1 -> K3 -> K4 in series (default: wave i's K4 overlaps "
                         "K1 + K3 of wave i + 1)")
    args = ap.parse_args()
    # stdout carries exactly one JSON line: libraries that print to fd 1 from C (NCCL's
    # "NCCL version" banner, for one) are sent to stderr, the line goes to a dup of the real stdout
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "config5":
        run_config5(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
