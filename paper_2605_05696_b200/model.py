"""Request data model used by the serve path (reference model.py:37-98).

Kept minimal: the engine only needs flattened tokens and marker spans. Any
object with ``.segments`` of ``.kind``/``.tokens`` (e.g. the reference's own
``irminsul.model.Request``) is accepted by the engine. The JSONL trace format
(model.py:100-181) is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

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
