"""Request data model and the JSONL trace format (reference model.py).

The engine only needs flattened tokens and marker spans; any object with
``.segments`` of ``.kind``/``.tokens`` (e.g. the reference's own
``irminsul.model.Request``) is accepted. Trace ingest (model.py:100-181,
SURVEY §8(f) item 4) is native: ``load_trace_arrays`` turns JSONL text into
flattened u32 token buffers (pinned host memory for one H2D) through
``irm_trace_scan`` / ``irm_trace_fill`` (csrc/ingest.cpp) with no Python
object per token, and ``parse_trace`` builds the reference's ``Trace`` from the
same arrays, with the reference's errors (TraceFormatError line / field).
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass
from typing import IO, Iterable

import numpy as np

MARKER_LEN = 64
TOKEN_MAX = 2**32 - 1
SEGMENT_KINDS = frozenset({"system", "header", "history", "tool", "doc", "marker", "body", "other"})


@dataclass(frozen=True)
class Segment:
    kind: str
    tokens: tuple[int, ...]
    shared_id: str | None = None

    def __post_init__(self):
        if self.kind not in SEGMENT_KINDS:
            raise ValueError(f"unknown segment kind {self.kind!r}")
        if self.kind == "marker" and len(self.tokens) != MARKER_LEN:
            raise ValueError(f"marker segment must hold exactly {MARKER_LEN} tokens")


@dataclass(frozen=True)
class Request:
    session_id: str
    turn_index: int
    segments: tuple[Segment, ...]

    def __post_init__(self):
        if self.turn_index < 0:
            raise ValueError("turn_index must be non-negative")

    @property
    def num_tokens(self) -> int:
        return sum(len(s.tokens) for s in self.segments)


@dataclass(frozen=True)
class Trace:
    requests: tuple[Request, ...] = ()

    def __post_init__(self):  # model.py:68-78
        last_turn: dict[str, int] = {}
        for r in self.requests:
            prev = last_turn.get(r.session_id)
            if prev is not None and r.turn_index <= prev:
                raise ValueError(f"turn_index not strictly increasing in session {r.session_id!r}")
            last_turn[r.session_id] = r.turn_index


class TraceFormatError(ValueError):
    """Malformed trace input; carries the offending line number and field (model.py:27-34)."""

    def __init__(self, line_no: int, fld: str, message: str):
        super().__init__(f"line {line_no}, field {fld!r}: {message}")
        self.line_no = line_no
        self.field = fld


KIND_NAMES = ("system", "header", "history", "tool", "doc", "marker", "body", "other")  # ingest.cpp order


@dataclass
class TraceArrays:
    """A parsed trace as flat arrays (ingest.cpp): tokens u32 [n_tokens] (a
    flattened request is tokens[req_tok_off[i]:req_tok_off[i+1]]), per-segment
    kind codes (KIND_NAMES) and request-relative starts, turns, and strings."""

    tokens: np.ndarray
    req_tok_off: np.ndarray
    req_seg_off: np.ndarray
    turns: np.ndarray
    sessions: list
    seg_kind: np.ndarray
    seg_tok_off: np.ndarray
    shared_ids: list

    @property
    def n_requests(self) -> int:
        return self.turns.size

    def marker_pins(self):
        """CSR of each request's marker spans (start, end) (model.py:89-97)."""
        is_m = self.seg_kind == KIND_NAMES.index("marker")
        req_of_seg = np.repeat(np.arange(self.n_requests), np.diff(self.req_seg_off))
        off = np.zeros(self.n_requests + 1, np.int64)
        np.cumsum(np.bincount(req_of_seg[is_m], minlength=self.n_requests), out=off[1:])
        starts = self.seg_tok_off[is_m]
        return off, np.stack([starts, starts + MARKER_LEN], axis=1) if starts.size else np.zeros((0, 2), np.int64)


def _ingest(text: bytes, universal: bool, pinned: bool = False) -> TraceArrays:
    from . import _native as N

    L = N.lib()
    buf = ctypes.c_char_p(text)  # the bytes object's own buffer: no copy
    sizes = (ctypes.c_int64 * 4)()
    err_line = ctypes.c_int64(0)
    err_field = ctypes.create_string_buffer(256)
    rc = L.irm_trace_scan(buf, len(text), int(universal), sizes, ctypes.byref(err_line), err_field, 256)
    if rc != N.IRM_OK:
        msg = L.irm_last_error().decode(errors="replace")
        raise TraceFormatError(int(err_line.value), err_field.value.decode(errors="surrogatepass"), msg)
    n_req, n_tok, n_seg, n_str = (int(x) for x in sizes)
    if pinned:
        import torch

        tok_t = torch.empty(max(n_tok, 1), dtype=torch.int32, pin_memory=True)
        tokens = tok_t.numpy().view(np.uint32)[:n_tok]
    else:
        tokens = np.empty(n_tok, np.uint32)
    a = lambda n, dt=np.int64: np.empty(max(n, 1), dt)
    req_tok_off, req_seg_off, turns, req_sess = a(n_req + 1), a(n_req + 1), a(n_req), a(2 * n_req)
    seg_kind, seg_tok_off, seg_shared = a(n_seg, np.uint8), a(n_seg), a(2 * n_seg)
    strings = ctypes.create_string_buffer(max(n_str, 1))
    p = lambda x: x.ctypes.data_as(ctypes.c_void_p)
    rc = L.irm_trace_fill(buf, len(text), int(universal), p(tokens) if n_tok else None, p(req_tok_off),
                          p(req_seg_off), p(turns), p(req_sess), p(seg_kind), p(seg_tok_off), p(seg_shared), strings)
    N.check(rc, "irm_trace_fill")
    raw = strings.raw
    dec = lambda o, n: raw[o:o + n].decode("utf-8", errors="surrogatepass")
    sessions = [dec(int(req_sess[2 * i]), int(req_sess[2 * i + 1])) for i in range(n_req)]
    shared = [None if seg_shared[2 * j] < 0 else dec(int(seg_shared[2 * j]), int(seg_shared[2 * j + 1]))
              for j in range(n_seg)]
    out = TraceArrays(tokens, req_tok_off[:n_req + 1], req_seg_off[:n_req + 1], turns[:n_req], sessions,
                      seg_kind[:n_seg], seg_tok_off[:n_seg], shared)
    last: dict[str, int] = {}
    for sid, t in zip(sessions, out.turns.tolist()):  # Trace.__post_init__ (model.py:68-78)
        if sid in last and t <= last[sid]:
            raise ValueError(f"turn_index not strictly increasing in session {sid!r}")
        last[sid] = t
    return out


def load_trace_arrays(path: str | None = None, text: bytes | str | None = None, pinned: bool = True) -> TraceArrays:
    """A JSONL trace file (``path``; universal newlines, as ``open()`` reads it)
    or in-memory ``text`` ('\\n'-separated lines) -> TraceArrays, tokens in pinned
    host memory when ``pinned`` (ready for one H2D into the K0 / K1 buffers)."""
    if (path is None) == (text is None):
        raise ValueError("give exactly one of path / text")
    if path is not None:
        with open(path, "rb") as f:
            return _ingest(f.read(), universal=True, pinned=pinned)
    data = text.encode("utf-8", errors="surrogatepass") if isinstance(text, str) else text
    return _ingest(data, universal=False, pinned=pinned)


def trace_from_arrays(ta: TraceArrays) -> Trace:
    toks = ta.tokens.tolist()
    kinds = ta.seg_kind.tolist()
    starts = ta.seg_tok_off.tolist()
    requests = []
    for i in range(ta.n_requests):
        t0, t1 = int(ta.req_tok_off[i]), int(ta.req_tok_off[i + 1])
        s0, s1 = int(ta.req_seg_off[i]), int(ta.req_seg_off[i + 1])
        segs = []
        for j in range(s0, s1):
            a = t0 + starts[j]
            b = t0 + starts[j + 1] if j + 1 < s1 else t1
            segs.append(Segment(KIND_NAMES[kinds[j]], tuple(toks[a:b]), ta.shared_ids[j]))
        req = Request(ta.sessions[i], int(ta.turns[i]), tuple(segs))
        # the flattened u32 tokens ride along (a view of the ingest buffer), so the
        # engine feeds K0 / K1 without converting Python ints back to an array
        object.__setattr__(req, "_flat_u32", ta.tokens[t0:t1])
        requests.append(req)
    return Trace(tuple(requests))


def parse_trace(source: Iterable[str] | IO[str]) -> Trace:
    """Parse line-delimited request records, preserving input order (model.py:160-166).
    Lines are taken as the source yields them (files: universal newlines)."""
    text = "\n".join(line.rstrip("\n") if line.endswith("\n") else line for line in source)
    return trace_from_arrays(_ingest(text.encode("utf-8", errors="surrogatepass"), universal=False))


def serialize_request(request: Request) -> str:  # model.py:169-178
    obj = {"session_id": request.session_id, "turn": request.turn_index,
           "segments": [{"kind": s.kind, "tokens": list(s.tokens), "shared_id": s.shared_id}
                        for s in request.segments]}
    return json.dumps(obj, separators=(", ", ": "))


def serialize_trace(trace: Trace) -> str:  # model.py:181-183
    return "".join(serialize_request(r) + "\n" for r in trace.requests)


def flatten(request) -> tuple[tuple[int, ...], list[int]]:
    """Concatenated tokens plus each segment's absolute start offset."""
    offsets, tokens = [], []
    for seg in request.segments:
        offsets.append(len(tokens))
        tokens.extend(seg.tokens)
    return tuple(tokens), offsets


def marker_spans(request) -> list[tuple[int, int]]:
    """(start, end) absolute spans of the request's marker segments."""
    spans, pos = [], 0
    for seg in request.segments:
        if seg.kind == "marker":
            spans.append((pos, pos + len(seg.tokens)))
        pos += len(seg.tokens)
    return spans
