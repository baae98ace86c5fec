"""Tensor-level operators over the C ABI (device-resident, batched).

These are the B200 forms of the reference's per-call functions; the drop-in
modules (chunking, fingerprint, rotary, registry, engine) are thin host
adapters over them. All tensors live on the current CUDA device; 64-bit
unsigned values (fingerprints, gear entries) are carried in int64 tensors
holding the same bit patterns, u32 tokens in int32 tensors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N

DEFAULT_GEAR_SEED = 0x49524D494E53554C


def _dev():
    N.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def u64_to_i64(v: int) -> int:
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


def tokens_to_device(tokens) -> torch.Tensor:
    """u32 token ids -> int32 device tensor carrying the same bits."""
    if isinstance(tokens, torch.Tensor):
        t = tokens
        if t.dtype == torch.int64:
            t = (t & 0xFFFFFFFF).to(torch.int64)
            t = torch.where(t >= 2**31, t - 2**32, t).to(torch.int32)
        return t.to(device=_dev(), dtype=torch.int32).contiguous()
    a = np.asarray(tokens, dtype=np.uint64)
    if a.size and int(a.max()) > 0xFFFFFFFF:
        raise ValueError("token ids must be unsigned 32-bit")
    a = a.astype(np.uint32).view(np.int32)
    return torch.from_numpy(np.ascontiguousarray(a)).to(_dev())


# ------------------------------------------------------------------ gear table
_GEAR_DEV: dict[tuple[int, int], torch.Tensor] = {}


def gear_table_device(seed: int = DEFAULT_GEAR_SEED) -> torch.Tensor:
    """65,536-entry splitmix64 table generated on the device (chunking.py:64-76)."""
    dev = _dev()
    key = (seed & (2**64 - 1), dev.index)
    t = _GEAR_DEV.get(key)
    if t is None:
        t = torch.empty(65536, dtype=torch.int64, device=dev)
        N.check(N.lib().irm_gear_table(seed & (2**64 - 1), N.ptr(t), N.stream_ptr()), "irm_gear_table")
        _GEAR_DEV[key] = t
    return t


# ------------------------------------------------------------------ K1: CDC + xxh64
@dataclass
class ChunkTable:
    """Device chunk table: CSR over streams (chunk_off[n_streams+1])."""

    start: torch.Tensor    # int32, stream-relative
    length: torch.Tensor   # int32
    fp: torch.Tensor       # int64 (u64 bits)
    forced: torch.Tensor   # uint8
    chunk_off: torch.Tensor  # int64 [n_streams+1]
    n_chunks: int | None = None

    def to_host(self):
        off = self.chunk_off.cpu().numpy()
        n = int(off[-1])
        return (self.start[:n].cpu().numpy(), self.length[:n].cpu().numpy(),
                self.fp[:n].cpu().numpy().view(np.uint64), self.forced[:n].cpu().numpy(), off)


class CdcWorkspace:
    """Reusable device scratch for irm_cdc_xxh64 (grown on demand until
    ``freeze()``). Output tables are allocated per call, so results never alias
    a later call."""

    def __init__(self):
        self.ws = None
        self.frozen = False

    def freeze(self):
        """No growth from now on (a captured CUDA graph holds the buffer's
        address): a call needing more scratch raises instead of reallocating."""
        self.frozen = True

    def get(self, n_tokens, n_streams, n_pins, min_size):
        L = N.lib()
        wb = int(L.irm_cdc_workspace_bytes(n_tokens, n_streams, n_pins, min_size))
        cap = max(int(L.irm_cdc_chunk_bound(n_tokens, n_streams, n_pins, min_size)), 16)
        dev = _dev()
        if self.ws is None or self.ws.numel() < wb:
            if self.frozen:
                raise ValueError("CdcWorkspace: the call exceeds the frozen (graph-captured) workspace")
            self.ws = torch.empty(max(wb, 256), dtype=torch.uint8, device=dev)
        bufs = (torch.empty(cap, dtype=torch.int32, device=dev),
                torch.empty(cap, dtype=torch.int32, device=dev),
                torch.empty(cap, dtype=torch.int64, device=dev),
                torch.empty(cap, dtype=torch.uint8, device=dev))
        return self.ws, bufs, cap


_DEFAULT_CDC_WS = CdcWorkspace()


def cdc_xxh64(tok: torch.Tensor, stream_off: torch.Tensor, pin_off: torch.Tensor | None,
              pins: torch.Tensor | None, mask_exponent: int = 7, min_size: int = 32,
              max_size: int = 512, marker_pinned: bool = True,
              gear_seed: int = DEFAULT_GEAR_SEED, ws: CdcWorkspace | None = None,
              n_tokens: int | None = None, n_pins: int | None = None,
              gear_from_table: bool = False) -> ChunkTable:
    """Batched CDC + fingerprints over CSR token streams (K1).

    ``tok`` int32 [n_tokens]; ``stream_off`` int64 [n_streams+1]; ``pins``
    int64 sorted per stream (CSR ``pin_off``). Outputs stay on the device.
    The Gear values are computed from ``gear_seed`` in the kernel
    (``irm_cdc_xxh64_seeded``); ``gear_from_table`` reads the device table
    instead (``irm_cdc_xxh64``, same results).
    """
    ws = ws or _DEFAULT_CDC_WS
    n_streams = stream_off.numel() - 1
    n_tokens = tok.numel() if n_tokens is None else n_tokens
    if pins is None or pin_off is None:
        pins = torch.zeros(1, dtype=torch.int64, device=tok.device)
        pin_off = torch.zeros(n_streams + 1, dtype=torch.int64, device=tok.device)
        n_pins = 0
    n_pins = pins.numel() if n_pins is None else n_pins
    wsbuf, (st, ln, fp, fo), cap = ws.get(n_tokens, n_streams, n_pins if marker_pinned else 0,
                                          max(min_size, 1))
    chunk_off = torch.empty(n_streams + 1, dtype=torch.int64, device=tok.device)
    if gear_from_table:
        fn, gear = N.lib().irm_cdc_xxh64, N.ptr(gear_table_device(gear_seed))
    else:
        fn, gear = N.lib().irm_cdc_xxh64_seeded, gear_seed & (2**64 - 1)
    rc = fn(N.ptr(tok), n_tokens, N.ptr(stream_off), n_streams, N.ptr(pin_off), N.ptr(pins), n_pins,
            mask_exponent, min_size, max_size, int(bool(marker_pinned)), gear,
            N.ptr(st), N.ptr(ln), N.ptr(fp), N.ptr(fo), N.ptr(chunk_off), cap, N.ptr(wsbuf),
            wsbuf.numel(), N.stream_ptr())
    N.check(rc, "irm_cdc_xxh64")
    return ChunkTable(st, ln, fp, fo, chunk_off)


# ------------------------------------------------------------------ K2: xxh64 spans
def xxh64_spans(base: torch.Tensor, off: torch.Tensor, length: torch.Tensor, seed: int = 0) -> torch.Tensor:
    """XXH64 of byte spans of a device buffer (offsets/lengths in bytes)."""
    n = off.numel()
    out = torch.empty(max(n, 1), dtype=torch.int64, device=base.device)
    if n:
        N.check(N.lib().irm_xxh64_spans(N.ptr(base), N.ptr(off), N.ptr(length), n, seed & (2**64 - 1),
                                        N.ptr(out), N.stream_ptr()), "irm_xxh64_spans")
    return out[:n]


# ------------------------------------------------------------------ K4: rotation
_DTYPE_CODE = {torch.float64: N.DTYPE_F64, torch.float32: N.DTYPE_F32, torch.bfloat16: N.DTYPE_BF16}


def inv_freq_device(inv_freq) -> torch.Tensor:
    return torch.from_numpy(np.array(inv_freq, dtype=np.float64)).to(_dev())


def rotate_gather(pool: torch.Tensor, out: torch.Tensor, src_row: torch.Tensor, dst_row: torch.Tensor,
                  length: torch.Tensor, delta: torch.Tensor, inv_freq: torch.Tensor,
                  ckv_dim: int = 512, kr_dim: int = 64, layout: int = N.LAYOUT_HALF_SPLIT,
                  out_round: int = N.ROUND_NONE, ws: torch.Tensor | None = None,
                  n_dev: torch.Tensor | None = None, max_sms: int = 0,
                  status: torch.Tensor | None = None) -> None:
    """K4. pool [layers, pool_rows, ckv+kr], out [layers, out_rows, ckv+kr] (same dtype).
    ``n_dev`` (int64 [1], device): process only the first n_dev[0] chunks.
    ``max_sms``: spread over at most this many SMs (0 = all). ``status`` (int64 [1],
    device, optional): sticky OR of 1 (a source run outside the pool) / 2 (a
    destination run outside ``out``); such chunks are skipped. Without ``status``
    the call checks nothing on the host (bench / graph use); see ``check_status``."""
    assert pool.dtype == out.dtype and pool.is_contiguous() and out.is_contiguous()
    assert pool.dim() == 3 and out.dim() == 3 and pool.shape[0] == out.shape[0]
    assert pool.shape[2] == ckv_dim + kr_dim == out.shape[2]
    n = src_row.numel()
    need = int(N.lib().irm_rotate_gather_workspace_bytes(n, kr_dim))
    if ws is None or ws.numel() < need:
        ws = torch.empty(max(need, 256), dtype=torch.uint8, device=pool.device)
    rc = N.lib().irm_rotate_gather(
        N.ptr(pool), pool.shape[1], N.ptr(out), out.shape[1], pool.shape[0], ckv_dim, kr_dim,
        N.ptr(src_row), N.ptr(dst_row), N.ptr(length), N.ptr(delta), n, N.ptr(n_dev), N.ptr(inv_freq), layout,
        _DTYPE_CODE[pool.dtype], out_round, int(max_sms), N.ptr(status), N.ptr(ws), ws.numel(), N.stream_ptr())
    N.check(rc, "irm_rotate_gather")


def check_status(status: torch.Tensor, what: str = "rotate_gather") -> None:
    """Raise if a K4 status word reports skipped out-of-range work (host sync)."""
    v = int(status.item())
    if v:
        parts = [m for b, m in ((1, "a source run outside the latent pool"),
                                (2, "a destination run outside the output"),
                                (4, "a hit past its request's req_stride rows")) if v & b]
        raise ValueError(f"{what}: skipped {' and '.join(parts)} (status {v})")


@dataclass
class SourceGroups:
    """irm_group_by_source output: groups of K4 work sharing a source run."""

    g_src: torch.Tensor     # int64 [cap]
    g_len: torch.Tensor     # int32 [cap]
    g_first: torch.Tensor   # int32 [cap]
    g_count: torch.Tensor   # int32 [cap]
    m_dst: torch.Tensor     # int64 [cap]
    m_delta: torch.Tensor   # int64 [cap]
    n_groups: torch.Tensor  # int64 [1] (device)
    ws: torch.Tensor        # zero-filled group workspace (left zeroed by every call)

    @staticmethod
    def alloc(cap: int, device) -> "SourceGroups":
        i64 = dict(dtype=torch.int64, device=device)
        i32 = dict(dtype=torch.int32, device=device)
        wsb = int(N.lib().irm_group_workspace_bytes(cap))
        return SourceGroups(torch.zeros(cap, **i64), torch.zeros(cap, **i32), torch.zeros(cap, **i32),
                            torch.zeros(cap, **i32), torch.zeros(cap, **i64), torch.zeros(cap, **i64),
                            torch.zeros(1, **i64), torch.zeros(max(wsb, 256), dtype=torch.uint8, device=device))


def group_by_source(src_row: torch.Tensor, dst_row: torch.Tensor, length: torch.Tensor, delta: torch.Tensor,
                    groups: SourceGroups, n_dev: torch.Tensor | None = None) -> SourceGroups:
    """Group K4 work items by source run (irm_group_by_source), into ``groups``'
    static buffers (graph-capturable: nothing is allocated per call)."""
    n = src_row.numel()
    if groups.g_src.numel() < n:
        raise ValueError("group_by_source: group buffers smaller than the work list")
    _expect([(src_row, torch.int64), (dst_row, torch.int64), (length, torch.int32), (delta, torch.int64)],
            "group_by_source")
    rc = N.lib().irm_group_by_source(
        N.ptr(src_row), N.ptr(dst_row), N.ptr(length), N.ptr(delta), n, N.ptr(n_dev), N.ptr(groups.g_src),
        N.ptr(groups.g_len), N.ptr(groups.g_first), N.ptr(groups.g_count), N.ptr(groups.m_dst),
        N.ptr(groups.m_delta), N.ptr(groups.n_groups), N.ptr(groups.ws), groups.ws.numel(), N.stream_ptr())
    N.check(rc, "irm_group_by_source")
    return groups


def rotate_gather_fanout(pool: torch.Tensor, out: torch.Tensor, groups: SourceGroups, inv_freq: torch.Tensor,
                         ckv_dim: int = 512, kr_dim: int = 64, layout: int = N.LAYOUT_HALF_SPLIT,
                         ws: torch.Tensor | None = None, n_members_dev: torch.Tensor | None = None,
                         max_sms: int = 0, status: torch.Tensor | None = None, cta_rounds: int = 1) -> None:
    """K4 fan-out (irm_rotate_gather_fanout): each group's source rows are read
    once and written, rotated by each member's delta, to every member's rows.
    ``cta_rounds`` > 1: CTAs retire after their share so a concurrent
    high-priority stream gets SMs (the overlapped reattach step)."""
    assert pool.dtype == out.dtype and pool.is_contiguous() and out.is_contiguous()
    assert pool.dim() == 3 and out.dim() == 3 and pool.shape[0] == out.shape[0]
    assert pool.shape[2] == ckv_dim + kr_dim == out.shape[2]
    cap = groups.m_dst.numel()
    need = int(N.lib().irm_fanout_workspace_bytes(cap, kr_dim))
    if ws is None or ws.numel() < need:
        ws = torch.empty(max(need, 256), dtype=torch.uint8, device=pool.device)
    rc = N.lib().irm_rotate_gather_fanout(
        N.ptr(pool), pool.shape[1], N.ptr(out), out.shape[1], pool.shape[0], ckv_dim, kr_dim, N.ptr(groups.g_src),
        N.ptr(groups.g_len), N.ptr(groups.g_first), N.ptr(groups.g_count), groups.g_src.numel(),
        N.ptr(groups.n_groups), N.ptr(groups.m_dst), N.ptr(groups.m_delta), cap, N.ptr(n_members_dev),
        N.ptr(inv_freq), layout, _DTYPE_CODE[pool.dtype], int(max_sms), int(cta_rounds), N.ptr(status), N.ptr(ws),
        ws.numel(), N.stream_ptr())
    N.check(rc, "irm_rotate_gather_fanout")


def copy_runs(src_addr: torch.Tensor, src_layer_stride: int, dst_pool: torch.Tensor, dst_row: torch.Tensor,
              length: torch.Tensor, n_dev: torch.Tensor | None = None) -> None:
    """K6 replica fetch: runs of rows from device addresses (peer pools mapped
    over NVLink) into ``dst_pool`` [layers, rows, width]; strides in bytes."""
    assert dst_pool.dim() == 3 and dst_pool.is_contiguous()
    row_bytes = dst_pool.shape[2] * dst_pool.element_size()
    rc = N.lib().irm_copy_runs(N.ptr(src_addr), int(src_layer_stride), N.ptr(dst_pool),
                               dst_pool.stride(0) * dst_pool.element_size(), N.ptr(dst_row), N.ptr(length),
                               src_addr.numel(), N.ptr(n_dev), dst_pool.shape[0], row_bytes, N.stream_ptr())
    N.check(rc, "irm_copy_runs")


def launch_count() -> int:
    """Kernels the library has launched or recorded into a captured graph (process-wide)."""
    return int(N.lib().irm_launch_count())


def rotate_rows(rows: torch.Tensor, positions: torch.Tensor, inv_freq: torch.Tensor,
                layout: int = N.LAYOUT_HALF_SPLIT, out_round: int = N.ROUND_NONE,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """Per-row absolute rotation (rows [n, dim] with arbitrary row stride)."""
    assert rows.dim() == 2 and rows.stride(1) == 1
    if out is None:
        out = torch.empty(rows.shape, dtype=rows.dtype, device=rows.device)
    pos = positions.to(device=rows.device, dtype=torch.float64).contiguous()
    rc = N.lib().irm_rotate_rows(N.ptr(rows), rows.stride(0), N.ptr(out), out.stride(0), rows.shape[0],
                                 rows.shape[1], N.ptr(pos), N.ptr(inv_freq), layout,
                                 _DTYPE_CODE[rows.dtype], out_round, N.stream_ptr())
    N.check(rc, "irm_rotate_rows")
    return out


def rotate_rows_layered(rows: torch.Tensor, positions: torch.Tensor, inv_freq: torch.Tensor,
                        layout: int = N.LAYOUT_HALF_SPLIT, out: torch.Tensor | None = None) -> torch.Tensor:
    """irm_rotate_rows_layered: rows [layers, n, dim] (any row / layer stride, unit
    element stride), every layer's row i rotated by positions[i]; in place when
    ``out`` is ``rows``."""
    assert rows.dim() == 3 and rows.stride(2) == 1
    if out is None:
        out = torch.empty(rows.shape, dtype=rows.dtype, device=rows.device)
    assert out.shape == rows.shape and out.stride(2) == 1
    pos = positions.to(device=rows.device, dtype=torch.float64).contiguous()
    rc = N.lib().irm_rotate_rows_layered(N.ptr(rows), rows.stride(1), rows.stride(0), N.ptr(out), out.stride(1),
                                         out.stride(0), rows.shape[0], rows.shape[1], rows.shape[2], N.ptr(pos),
                                         N.ptr(inv_freq), layout, _DTYPE_CODE[rows.dtype], N.ROUND_NONE,
                                         N.stream_ptr())
    N.check(rc, "irm_rotate_rows_layered")
    return out


def round_f64(x: torch.Tensor, mode: int) -> torch.Tensor:
    x = x.contiguous()
    y = torch.empty_like(x)
    N.check(N.lib().irm_round_f64(N.ptr(x), N.ptr(y), x.numel(), mode, N.stream_ptr()), "irm_round_f64")
    return y


# ------------------------------------------------------------------ K3: chunk store
class ChunkStore:
    """Device content-hash store: fingerprint -> (p_src, len, pool row).

    Host state is only the ctypes view; tables and entries are torch tensors.
    """

    def __init__(self, max_entries: int = 1 << 16, load_factor: float = 0.5, pool_rows: int = 0):
        """pool_rows: rows of the latent pool that new entries' rows are bump-allocated
        in (0 = unbounded); an insert that would pass it is not published and sets
        the sticky pool-full flag that ``counts()`` raises on."""
        dev = _dev()
        n_slots = 1
        while n_slots < max(2, int(max_entries / load_factor)):
            n_slots <<= 1
        self.n_slots, self.max_entries = n_slots, max_entries
        self.slot_key = torch.empty(n_slots, dtype=torch.int64, device=dev)
        self.slot_order = torch.empty(n_slots + 1, dtype=torch.int64, device=dev)
        self.slot_entry = torch.empty(n_slots + 1, dtype=torch.int64, device=dev)
        self.e_fp = torch.empty(max_entries, dtype=torch.int64, device=dev)
        self.e_p_src = torch.empty(max_entries, dtype=torch.int64, device=dev)
        self.e_len = torch.empty(max_entries, dtype=torch.int32, device=dev)
        self.e_row = torch.empty(max_entries, dtype=torch.int64, device=dev)
        self.counters = torch.zeros(4, dtype=torch.int64, device=dev)
        self.view = N.StoreView(
            N.ptr(self.slot_key), N.ptr(self.slot_order), N.ptr(self.slot_entry), n_slots,
            N.ptr(self.e_fp), N.ptr(self.e_p_src), N.ptr(self.e_len), N.ptr(self.e_row),
            max_entries, N.ptr(self.counters), int(pool_rows))
        self._ws = None
        self._ws_frozen = False
        self.reset()

    @property
    def pool_rows(self) -> int:
        return int(self.view.pool_rows)

    def set_pool_rows(self, rows: int) -> None:
        """Bound later inserts to ``rows`` pool rows (0 = unbounded). Read at launch:
        a captured CUDA graph keeps the bound it was captured with."""
        self.view.pool_rows = int(rows)

    def reset(self):
        N.check(N.lib().irm_store_reset(self.view, N.stream_ptr()), "irm_store_reset")

    def reserve(self, n: int) -> None:
        """Size the lookup workspace for batches of up to ``n`` queries once and
        freeze it: a CUDA graph that captured ``lookup_insert`` keeps the buffer's
        address, so it must never be replaced afterwards (a larger call raises).
        An explicit ``reserve`` may still grow it: call it before capturing."""
        self._ws_frozen = False
        self._workspace(n)
        self._ws_frozen = True

    def _workspace(self, n):
        need = int(N.lib().irm_store_workspace_bytes(n))
        if self._ws is None or self._ws.numel() < need:
            if self._ws_frozen:
                raise ValueError(f"ChunkStore: {n} queries exceed the reserved (graph-captured) workspace")
            self._ws = torch.empty(max(need, 256), dtype=torch.uint8, device=self.slot_key.device)
        return self._ws

    def lookup_insert(self, q_fp: torch.Tensor, q_order: torch.Tensor, q_p: torch.Tensor,
                      q_len: torch.Tensor, q_probe: torch.Tensor | None = None):
        n = q_fp.numel()
        dev = q_fp.device
        hit = torch.empty(n, dtype=torch.int32, device=dev)
        entry = torch.empty(n, dtype=torch.int64, device=dev)
        p_src = torch.empty(n, dtype=torch.int64, device=dev)
        row = torch.empty(n, dtype=torch.int64, device=dev)
        ws = self._workspace(n)
        rc = N.lib().irm_store_lookup_insert(
            self.view, N.ptr(q_fp), N.ptr(q_order), N.ptr(q_p), N.ptr(q_len), N.ptr(q_probe), n,
            N.ptr(hit), N.ptr(entry), N.ptr(p_src), N.ptr(row), N.ptr(ws), ws.numel(), N.stream_ptr())
        N.check(rc, "irm_store_lookup_insert")
        return hit, entry, p_src, row

    def lookup(self, q_fp: torch.Tensor) -> torch.Tensor:
        n = q_fp.numel()
        entry = torch.empty(max(n, 1), dtype=torch.int64, device=q_fp.device)
        N.check(N.lib().irm_store_lookup(self.view, N.ptr(q_fp), n, N.ptr(entry), N.stream_ptr()),
                "irm_store_lookup")
        return entry[:n]

    def counts(self) -> tuple[int, int, int]:
        c = self.counters.cpu().tolist()
        if c[2]:
            what = [m for b, m in ((1, "hash table full"), (2, "max_entries reached"),
                                   (4, "latent pool rows exhausted")) if c[2] & b]
            raise RuntimeError(f"chunk store overflow (flags {c[2]}: {', '.join(what)})")
        return c[0], c[1], c[2]


def _expect(pairs, what: str) -> None:
    for t, dt in pairs:
        if t.dtype != dt or not t.is_contiguous() or not t.is_cuda:
            raise ValueError(f"{what}: expected a contiguous CUDA {dt} tensor, got {t.dtype} "
                             f"(contiguous={t.is_contiguous()}, device={t.device})")


def wave_plan(chunk_off: torch.Tensor, n_req: int, start: torch.Tensor, meta_len: torch.Tensor, carve: int,
              order0: int, req: torch.Tensor, p_abs: torch.Tensor, probe: torch.Tensor, order: torch.Tensor) -> None:
    """irm_wave_plan: per chunk slot, owning request, absolute position, probe flag, order key."""
    _expect([(chunk_off, torch.int64), (start, torch.int32), (meta_len, torch.int64), (req, torch.int64),
             (p_abs, torch.int64), (probe, torch.uint8), (order, torch.int64)], "wave_plan")
    if meta_len.numel() < n_req or chunk_off.numel() < n_req + 1 or min(req.numel(), p_abs.numel(), probe.numel(),
                                                                         order.numel()) < start.numel():
        raise ValueError("wave_plan: buffer too small")
    N.check(N.lib().irm_wave_plan(N.ptr(chunk_off), int(n_req), N.ptr(start), N.ptr(meta_len), start.numel(),
                                  int(carve), int(order0), N.ptr(req), N.ptr(p_abs), N.ptr(probe), N.ptr(order),
                                  N.stream_ptr()), "irm_wave_plan")


def wave_rebase(tok: torch.Tensor, off: torch.Tensor, m: torch.Tensor, n_req: int, span_off: torch.Tensor,
                spans: torch.Tensor, tail: torch.Tensor, tail_off: torch.Tensor, pin_off: torch.Tensor,
                pins: torch.Tensor) -> None:
    """irm_wave_rebase: pack the tails tok[off[r] + m[r], off[r+1]) into ``tail``
    (CSR ``tail_off``) and rebase the requests' marker spans (request-relative
    [start, end) pairs, CSR ``span_off``) into tail-relative pins."""
    _expect([(tok, torch.int32), (off, torch.int64), (m, torch.int64), (span_off, torch.int64),
             (spans, torch.int64), (tail, torch.int32), (tail_off, torch.int64), (pin_off, torch.int64),
             (pins, torch.int64)], "wave_rebase")
    if tail.numel() < tok.numel() or tail_off.numel() < n_req + 1 or pin_off.numel() < n_req + 1 \
            or pins.numel() < spans.numel():
        raise ValueError("wave_rebase: output buffers too small")
    N.check(N.lib().irm_wave_rebase(N.ptr(tok), N.ptr(off), N.ptr(m), int(n_req), tok.numel(), N.ptr(span_off),
                                    N.ptr(spans), N.ptr(tail), N.ptr(tail_off), N.ptr(pin_off), N.ptr(pins),
                                    N.stream_ptr()), "irm_wave_rebase")


def wave_compact(hit: torch.Tensor, row: torch.Tensor, req: torch.Tensor, p_abs: torch.Tensor, p_src: torch.Tensor,
                 length: torch.Tensor, req_stride: int, src_out: torch.Tensor, dst_out: torch.Tensor,
                 len_out: torch.Tensor, delta_out: torch.Tensor, n_hit: torch.Tensor, length_out: torch.Tensor,
                 hit_tokens: torch.Tensor | None = None, status: torch.Tensor | None = None) -> None:
    """irm_wave_compact: the hit slots, in slot order, as K4 work; their count on the device.
    A hit whose rows would leave its request's ``req_stride`` rows is dropped and
    sets bit 4 of ``status`` (int64 [1], device, optional)."""
    _expect([(hit, torch.int32), (row, torch.int64), (req, torch.int64), (p_abs, torch.int64), (p_src, torch.int64),
             (length, torch.int32), (src_out, torch.int64), (dst_out, torch.int64), (len_out, torch.int32),
             (delta_out, torch.int64), (n_hit, torch.int64), (length_out, torch.int32)]
            + ([(hit_tokens, torch.int64)] if hit_tokens is not None else []), "wave_compact")
    n = hit.numel()
    if min(t.numel() for t in (row, req, p_abs, p_src, length, src_out, dst_out, len_out, delta_out,
                               length_out)) < n:
        raise ValueError("wave_compact: buffer too small")
    N.check(N.lib().irm_wave_compact(N.ptr(hit), N.ptr(row), N.ptr(req), N.ptr(p_abs), N.ptr(p_src), N.ptr(length),
                                     hit.numel(), int(req_stride), N.ptr(src_out), N.ptr(dst_out), N.ptr(len_out),
                                     N.ptr(delta_out), N.ptr(n_hit), N.ptr(length_out), N.ptr(hit_tokens),
                                     N.ptr(status), N.stream_ptr()), "irm_wave_compact")


# ------------------------------------------------------------------ K5: fused MLA reattach prefill
def chunk_cossin(delta: torch.Tensor, inv_freq: torch.Tensor) -> torch.Tensor:
    """Per-chunk (cos, sin)(delta * inv_freq[j]) from fp64 angles -> float32 [n_chunks, 32, 2]."""
    n = delta.numel()
    cs = torch.empty(max(n, 1), inv_freq.numel(), 2, dtype=torch.float32, device=delta.device)
    if n:
        N.check(N.lib().irm_chunk_cossin(N.ptr(delta.contiguous()), n, N.ptr(inv_freq), N.ptr(cs),
                                         N.stream_ptr()), "irm_chunk_cossin")
    return cs[:n]


def mla_reattach_prefill(q: torch.Tensor, pool: torch.Tensor, n_kv: int, q_pos0: int, scale: float,
                         kv_rows: torch.Tensor | None = None, kv_chunk: torch.Tensor | None = None,
                         chunk_cs: torch.Tensor | None = None, layout: int = N.LAYOUT_HALF_SPLIT,
                         out: torch.Tensor | None = None, lse: torch.Tensor | None = None):
    """K5: absorbed-MLA causal prefill over the 576-wide latent key with the
    reattach rotation of k_r fused into the shared-memory load.

    q [n_q, H, 576] bf16; pool [rows, 576] bf16; returns (out [n_q, H, 512] bf16, lse [n_q, H] fp32).
    """
    assert q.dtype == torch.bfloat16 and pool.dtype == torch.bfloat16 and q.shape[-1] == 576
    q = q.contiguous()
    n_q, heads = q.shape[0], q.shape[1]
    if out is None:
        out = torch.empty(n_q, heads, 512, dtype=torch.bfloat16, device=q.device)
    if lse is None:
        lse = torch.empty(n_q, heads, dtype=torch.float32, device=q.device)
    rc = N.lib().irm_mla_reattach_prefill(
        N.ptr(q), n_q, heads, q_pos0, N.ptr(pool), pool.shape[0], N.ptr(kv_rows), n_kv, N.ptr(kv_chunk), N.ptr(chunk_cs),
        layout, float(scale), N.ptr(out), N.ptr(lse), N.stream_ptr())
    N.check(rc, "irm_mla_reattach_prefill")
    return out, lse
