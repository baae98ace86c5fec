"""Drop-in for ``irminsul.engine`` (reference engine.py): the serve path.

``serve(state, request)`` keeps the reference signature and results; the work
is the batched B200 form (``serve_batch``), which is exactly equivalent to the
reference's sequential loop:

  phase 1  exact-prefix match, host radix, in request order (engine.py:170,228)
  phase 2  one CDC + xxh64 launch over every unmatched tail   (K1)
  phase 3  one batched store lookup-or-insert, first writer = smallest
           (request, chunk) order key, carve-out chunks neither probed nor
           inserted (engine.py:184-223)                          (K3)
  produce  synthetic prefill rows of novel chunks -> pool, k_r rotated to
           p_src + i on the device                               (K4 producer)
  live     every PIC hit is materialized by rotate+gather and checked
           against fresh prefill (the rotation tripwire, engine.py:142-155)
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Sequence

import numpy as np
import torch

from . import ops
from .chunking import Chunk, ChunkerParams, cdc_chunk_batch, marker_pin_offsets
from .fingerprint import fingerprint, fingerprint_spans
from .model import Request, Trace, flatten, marker_spans
from .radix import DeviceRadixTree
from .registry import KvRegistry, SyntheticKvParams
from .rotary import Precision, RotarySpec, make_spec, rotate_rows_device

VERIFY_TOL = {Precision.F64: 1e-9, Precision.F32: 1e-6, Precision.BF16E: 5e-3}


class Mode(str, Enum):
    OBSERVER = "observer"
    LIVE = "live"


class ServiceClass(str, Enum):
    PREFIX_HIT = "prefix_hit"
    PIC_HIT = "pic_hit"
    S1_HIT = "s1_hit"
    CARVEOUT_PREFILL = "carveout_prefill"
    NOVEL_PREFILL = "novel_prefill"


@dataclass(frozen=True)
class ServeConfig:
    mode: Mode = Mode.OBSERVER
    carveout_threshold: int = 32
    s1_enabled: bool = False
    s1_window: int = 128
    chunker: ChunkerParams = ChunkerParams()
    spec: RotarySpec = None
    kv: SyntheticKvParams = SyntheticKvParams()
    precision: Precision = Precision.F64

    def __post_init__(self):
        if self.spec is None:
            object.__setattr__(self, "spec", make_spec(1e4, self.kv.kr_dim))


@dataclass(frozen=True)
class SegmentEvent:
    start: int
    length: int
    klass: ServiceClass
    fingerprint: int | None = None
    delta: int | None = None


@dataclass
class ServeResult:
    counts: dict[ServiceClass, int]
    events: list[SegmentEvent]
    num_tokens: int
    live_rows: int | None = None
    rotation_multiplies: int = 0

    @property
    def tprefix(self) -> float:
        return self.counts[ServiceClass.PREFIX_HIT] / self.num_tokens

    @property
    def pic_unique(self) -> float:
        return self.counts[ServiceClass.PIC_HIT] / self.num_tokens

    @property
    def s1_fraction(self) -> float:
        return self.counts[ServiceClass.S1_HIT] / self.num_tokens

    @property
    def total_cached(self) -> float:
        return self.tprefix + self.pic_unique + self.s1_fraction


class LiveVerificationError(AssertionError):
    """A materialized hit failed the materialize-vs-fresh check."""

    def __init__(self, start: int, length: int, delta: int, error: float):
        super().__init__(
            f"pic_hit at [{start}, {start + length}) with delta={delta} "
            f"failed rotation verification (rel-L2 {error:.3e})")
        self.start = start
        self.delta = delta


class EngineState:
    """Mutable caches shared across the requests of one trace run."""

    def __init__(self, config: ServeConfig, max_entries: int = 1 << 16, max_prefixes: int = 1 << 22,
                 max_tokens: int = 1 << 24):
        """Device capacities are initial sizes (the prefix index grows on demand). Sized
        for a few million tokens up front: growing inside a serve (a table rebuild and
        fresh device allocations) cost more than the allocation (serve API: 28 -> 92 ms)."""
        self.config = config
        self.tree = DeviceRadixTree(max_prefixes=max_prefixes, max_tokens=max_tokens)  # K0
        self.registry = KvRegistry(config.kv, config.spec, max_entries=max_entries)
        self.subwindows: set[int] = set()
        self.request_counter = 0


def s1_probe(chunk_tokens: Sequence[int], chunk_start: int, subwindows: set[int],
             window: int = 128) -> list[tuple[int, int]]:
    """Aligned sub-window probes for a missed chunk (engine.py:116-133)."""
    offs = list(range(0, len(chunk_tokens) - window + 1, window))
    if not offs:
        return []
    fps = fingerprint_spans(chunk_tokens, np.array(offs, np.int64), np.full(len(offs), window, np.int64))
    return [(chunk_start + o, window) for o, f in zip(offs, fps) if int(f) in subwindows]


def _subtract_spans(span: tuple[int, int], holes: list[tuple[int, int]]) -> list[tuple[int, int]]:
    out = []
    pos, end = span[0], span[0] + span[1]
    for h_start, h_len in holes:
        if h_start > pos:
            out.append((pos, h_start - pos))
        pos = h_start + h_len
    if pos < end:
        out.append((pos, end - pos))
    return out


@dataclass
class _Plan:
    flat: tuple
    m: int
    pins: set


def serve_batch(state: EngineState, requests: Sequence[Request]) -> list[ServeResult]:
    """Serve requests in order; identical results to sequential ``serve`` calls."""
    config = state.config
    carve = config.carveout_threshold
    reg = state.registry
    dev = ops._dev()

    # ---- phase 1: exact-prefix match (K0): request i matches everything inserted before it,
    # then is inserted (engine.py:170, 228), as one batched device operation
    plans: list[_Plan] = []
    flats = []
    for r in requests:
        flat = getattr(r, "_flat_u32", None)  # set by model.parse_trace (native ingest)
        if flat is None:
            t, _ = flatten(r)
            flat = np.asarray(t, dtype=np.uint64)
            if flat.size and int(flat.max()) > 0xFFFFFFFF:
                raise ValueError("token ids must be unsigned 32-bit")
            flat = flat.astype(np.uint32)
        if len(flat) == 0:
            raise ValueError("request flattens to zero tokens")
        flats.append(flat)
    handles = list(range(state.request_counter, state.request_counter + len(requests)))
    ms, _w = state.tree.match_insert(flats, handles)
    state.request_counter += len(requests)
    for r, flat, m in zip(requests, flats, ms):
        pins = marker_pin_offsets((max(s - m, 0), e - m) for s, e in marker_spans(r) if e - 1 >= m)
        plans.append(_Plan(flat, m, pins))

    # ---- phase 2: one CDC + xxh64 launch over all tails (K1)
    tails = [p.flat[p.m:] for p in plans]
    table = cdc_chunk_batch(tails, config.chunker, [p.pins for p in plans])
    chunk_off = table.chunk_off
    n_chunks = int(chunk_off[-1].item())
    # per-chunk absolute position p = m + start and its request index
    counts_per_req = torch.diff(chunk_off)
    req_of_chunk = torch.repeat_interleave(torch.arange(len(plans), device=dev), counts_per_req)
    m_dev = torch.tensor([p.m for p in plans], dtype=torch.int64, device=dev)
    starts = table.start[:n_chunks].to(torch.int64)
    lens = table.length[:n_chunks]
    p_abs = m_dev[req_of_chunk] + starts
    probe = (p_abs >= carve).to(torch.uint8)

    # ---- phase 3: batched first-writer-wins lookup-or-insert (K3)
    order = reg._order + torch.arange(n_chunks, dtype=torch.int64, device=dev)
    reg._order += n_chunks
    reg.ensure_capacity(n_chunks)  # every probed chunk could be novel
    hit, entry, p_src, row = reg.store.lookup_insert(table.fp[:n_chunks], order, p_abs, lens, probe)

    # one device->host copy of everything the events need
    host = torch.stack([starts, lens.to(torch.int64), table.fp[:n_chunks], hit.to(torch.int64),
                        entry, p_src, row]).cpu().numpy() if n_chunks else np.zeros((7, 0), np.int64)
    h_start, h_len, h_fp, h_hit, h_entry, h_psrc, h_row = host
    h_fp_u = h_fp.view(np.uint64)
    off = chunk_off.cpu().numpy()

    # ---- producer: novel chunks, in entry order (== insert epoch order)
    novel = np.nonzero(h_hit == 0)[0]
    novel = novel[np.argsort(h_entry[novel], kind="stable")]
    nov_req = (np.searchsorted(off, novel, side="right") - 1).tolist()
    for c, ri, s, l, e, f, rw in zip(novel.tolist(), nov_req, h_start[novel].tolist(), h_len[novel].tolist(),
                                     h_entry[novel].tolist(), h_fp_u[novel].tolist(), h_row[novel].tolist()):
        assert e == len(reg), "device store and host mirror diverged"
        reg.commit_rows(f, tails[ri][s:s + l], plans[ri].m + s, rw)

    # ---- S1 sub-window fallback (engine.py:116-139, 211-226), batched: every aligned full
    # window of every novel chunk is fingerprinted by ONE K2 launch; in the sequential order
    # a window hits iff its fingerprint was indexed before the batch or by a window of an
    # earlier novel chunk (a chunk is indexed only after its own probe)
    s1_hits: dict[int, list[tuple[int, int]]] = {}
    if config.s1_enabled:
        s1_hits = _s1_batch(state, tails, [p.m for p in plans], off, h_hit, h_start, h_len)

    # ---- events, per request in chunk order (Python lists: no numpy scalar per field access)
    l_start, l_len, l_hit, l_psrc, l_fp, l_off = (h_start.tolist(), h_len.tolist(), h_hit.tolist(),
                                                  h_psrc.tolist(), h_fp_u.tolist(), off.tolist())
    results: list[ServeResult] = []
    live_hits = []  # (request, chunk index)
    for ri, plan in enumerate(plans):
        n = len(plan.flat)
        counts = {k: 0 for k in ServiceClass}
        events: list[SegmentEvent] = []
        live_rows = 0
        m = plan.m
        if m > 0:
            counts[ServiceClass.PREFIX_HIT] = m
            events.append(SegmentEvent(0, m, ServiceClass.PREFIX_HIT))
            live_rows += m
        for c in range(l_off[ri], l_off[ri + 1]):
            p = m + l_start[c]
            ln = l_len[c]
            if p < carve:
                carved = min(carve - p, ln)
                counts[ServiceClass.CARVEOUT_PREFILL] += carved
                events.append(SegmentEvent(p, carved, ServiceClass.CARVEOUT_PREFILL))
                if ln > carved:
                    counts[ServiceClass.NOVEL_PREFILL] += ln - carved
                    events.append(SegmentEvent(p + carved, ln - carved, ServiceClass.NOVEL_PREFILL))
                live_rows += ln
                continue
            if l_hit[c] == 1:
                counts[ServiceClass.PIC_HIT] += ln
                events.append(SegmentEvent(p, ln, ServiceClass.PIC_HIT, l_fp[c], p - l_psrc[c]))
                if config.mode == Mode.LIVE:
                    live_hits.append((ri, c, len(events) - 1))
                continue
            novel_spans = [(p, ln)]
            hits = s1_hits.get(c)
            if hits:
                w = config.s1_window
                for hs, hf in hits:
                    counts[ServiceClass.S1_HIT] += w
                    events.append(SegmentEvent(hs, w, ServiceClass.S1_HIT, hf))
                novel_spans = _subtract_spans((p, ln), [(hs, w) for hs, _ in hits])
            for s, l in novel_spans:
                counts[ServiceClass.NOVEL_PREFILL] += l
                events.append(SegmentEvent(s, l, ServiceClass.NOVEL_PREFILL))
            live_rows += ln
        assert sum(counts.values()) == n, "service classes must tile the request"
        results.append(ServeResult(counts, events, n, live_rows if config.mode == Mode.LIVE else None, 0))

    if config.mode == Mode.LIVE and live_hits:
        _verify_hits(state, plans, live_hits, h_start, h_len, h_entry, h_psrc, results)
    return results


def _s1_batch(state, tails, ms, off, h_hit, h_start, h_len) -> dict[int, list[tuple[int, int]]]:
    """All S1 probes and sub-window indexing of a batch: one fingerprint launch.
    Returns {chunk index: [(absolute window start, window fingerprint), ...]} for
    the windows that hit, in window order; state.subwindows gains every window."""
    w = state.config.s1_window
    nov = np.nonzero(h_hit == 0)[0]  # probed misses (the inserted chunks), in sequential order
    nwin = h_len[nov] // w
    total = int(nwin.sum())
    if total == 0:
        return {}
    win_chunk = np.repeat(nov, nwin)
    j = np.arange(total) - np.repeat(np.cumsum(nwin) - nwin, nwin)
    req = np.searchsorted(off, win_chunk, side="right") - 1
    tail_base = np.concatenate([[0], np.cumsum([len(t) for t in tails])])
    start_tail = h_start[win_chunk] + j * w
    fps = fingerprint_spans(np.concatenate(tails), tail_base[req] + start_tail, np.full(total, w, np.int64))
    prior = np.fromiter(state.subwindows, dtype=np.uint64, count=len(state.subwindows))
    hit = np.isin(fps, prior)
    # the first novel chunk (in order) carrying each fingerprint; a later chunk's window hits it
    order = np.lexsort((win_chunk, fps))
    fs = fps[order]
    head = np.maximum.accumulate(np.where(np.r_[True, fs[1:] != fs[:-1]], np.arange(total), 0))
    first_chunk = np.empty(total, np.int64)
    first_chunk[order] = win_chunk[order][head]
    hit |= first_chunk < win_chunk
    state.subwindows.update(fps.tolist())
    ms = np.asarray(ms, np.int64)
    out: dict[int, list[tuple[int, int]]] = {}
    for k in np.nonzero(hit)[0]:
        out.setdefault(int(win_chunk[k]), []).append((int(ms[req[k]] + start_tail[k]), int(fps[k])))
    return out


def _verify_hits(state, plans, live_hits, h_start, h_len, h_entry, h_psrc, results):
    """Batched rotation tripwire (engine.py:142-155): materialize every hit with
    one rotate+gather launch, compare with a fresh rotation of fresh rows."""
    config = state.config
    reg = state.registry
    dev = ops._dev()
    ckv = config.kv.ckv_dim
    cs = [c for _, c, _ in live_hits]
    rows = torch.tensor([reg._entry_rows[int(h_entry[c])] for c in cs], dtype=torch.int64, device=dev)
    lens = torch.tensor([int(h_len[c]) for c in cs], dtype=torch.int32, device=dev)
    ps = [plans[ri].m + int(h_start[c]) for ri, c, _ in live_hits]
    deltas = torch.tensor([p - int(h_psrc[c]) for p, c in zip(ps, cs)], dtype=torch.int64, device=dev)
    mat = reg.materialize_device(rows, lens, deltas, config.precision)[0]
    fresh_c, fresh_kr, pos = [], [], []
    for (ri, c, _), p in zip(live_hits, ps):
        toks = plans[ri].flat[p:p + int(h_len[c])]
        fc, fk = reg.fresh_rows(toks)
        fresh_c.append(fc)
        fresh_kr.append(fk)
        pos.append(np.arange(p, p + len(toks), dtype=np.float64))
    fresh_c = torch.from_numpy(np.concatenate(fresh_c)).to(dev)
    fresh_kr = torch.from_numpy(np.concatenate(fresh_kr)).to(dev)
    fresh = rotate_rows_device(fresh_kr, torch.from_numpy(np.concatenate(pos)).to(dev), config.spec)
    bounds = np.concatenate([[0], np.cumsum([int(h_len[c]) for c in cs])])
    seg = torch.repeat_interleave(torch.arange(len(cs), device=dev), lens.to(torch.int64))
    n_rows = int(bounds[-1])
    c_bad = (mat[:n_rows, :ckv] != fresh_c).any(dim=1).to(torch.int64)
    c_bad = torch.zeros(len(cs), dtype=torch.int64, device=dev).index_add_(0, seg, c_bad)
    diff2 = ((mat[:n_rows, ckv:] - fresh) ** 2).sum(dim=1)
    ref2 = (fresh ** 2).sum(dim=1)
    num = torch.zeros(len(cs), dtype=torch.float64, device=dev).index_add_(0, seg, diff2)
    den = torch.zeros(len(cs), dtype=torch.float64, device=dev).index_add_(0, seg, ref2)
    err = (num.sqrt() / den.sqrt()).cpu().numpy()
    c_bad = c_bad.cpu().numpy()
    tol = VERIFY_TOL[config.precision]
    for k, ((ri, c, _), p) in enumerate(zip(live_hits, ps)):
        d = p - int(h_psrc[c])
        if c_bad[k]:
            raise LiveVerificationError(p, int(h_len[c]), d, float("inf"))
        if err[k] > tol:
            raise LiveVerificationError(p, int(h_len[c]), d, float(err[k]))
        results[ri].live_rows += int(h_len[c])
        results[ri].rotation_multiplies += int(h_len[c]) * config.spec.dim


def serve(state: EngineState, request: Request) -> ServeResult:
    """engine.py:158-238 -- one request through the batched B200 path."""
    return serve_batch(state, [request])[0]


@dataclass
class AggregateRow:
    pattern: str
    model_tag: str
    n_req: int
    tprefix: float = 0.0
    pic_unique: float = 0.0
    s1_fraction: float = 0.0
    total: float = 0.0
    warm_tprefix: float = 0.0
    warm_pic_unique: float = 0.0
    warm_s1_fraction: float = 0.0
    warm_total: float = 0.0
    rotation_multiplies: int = 0


def _fractions(results: list[ServeResult]) -> tuple[float, float, float, float]:
    tokens = sum(r.num_tokens for r in results)
    if tokens == 0:
        return 0.0, 0.0, 0.0, 0.0
    tp = sum(r.counts[ServiceClass.PREFIX_HIT] for r in results) / tokens
    pic = sum(r.counts[ServiceClass.PIC_HIT] for r in results) / tokens
    s1 = sum(r.counts[ServiceClass.S1_HIT] for r in results) / tokens
    return tp, pic, s1, tp + pic + s1


def run_trace(state: EngineState, trace: Trace, pattern: str = "trace",
              model_tag: str = "synthetic-oracle", batch: int | None = None) -> tuple[list[ServeResult], AggregateRow]:
    """engine.py:283-306. ``batch`` requests are served per device pass (all by default)."""
    cold_start = state.request_counter == 0
    reqs = list(trace.requests)
    batch = batch or max(len(reqs), 1)
    results: list[ServeResult] = []
    for i in range(0, len(reqs), batch):
        results.extend(serve_batch(state, reqs[i:i + batch]))
    row = AggregateRow(pattern, model_tag, len(results))
    row.tprefix, row.pic_unique, row.s1_fraction, row.total = _fractions(results)
    warm = results[1:] if cold_start and results else results
    row.warm_tprefix, row.warm_pic_unique, row.warm_s1_fraction, row.warm_total = _fractions(warm)
    row.rotation_multiplies = sum(r.rotation_multiplies for r in results)
    return results, row
