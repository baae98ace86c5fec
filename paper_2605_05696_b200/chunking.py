"""Drop-in for ``irminsul.chunking`` (reference chunking.py) on the B200 path.

Same names, dataclasses, validation and return types as the reference; the
boundary scan and the per-chunk xxh64 run in one batched CUDA pass (K1,
``irm_cdc_xxh64``). ``cdc_chunk_batch`` is the device-resident batched form
used by the engine.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _native as N
from . import ops
from .rng import SplitMix64

DEFAULT_GEAR_SEED = 0x49524D494E53554C
GEAR_TABLE_SIZE = 65536
MARKER_LEN = 64


class Forced(str, Enum):
    NONE = "none"
    MAX_CLAMP = "max_clamp"
    MARKER = "marker"
    STREAM_END = "stream_end"


_FORCED_BY_CODE = (Forced.NONE, Forced.MAX_CLAMP, Forced.MARKER, Forced.STREAM_END)


@dataclass(frozen=True)
class ChunkerParams:
    """chunking.py:37-49 (same defaults and ValueError rules)."""

    mask_exponent: int = 7
    min_size: int = 32
    max_size: int = 512
    gear_seed: int = DEFAULT_GEAR_SEED
    marker_pinned: bool = True

    def __post_init__(self):
        if not (1 <= self.mask_exponent <= 20):
            raise ValueError("mask_exponent must be in [1, 20]")
        if not (1 <= self.min_size < self.max_size):
            raise ValueError("need 1 <= min_size < max_size")


@dataclass(frozen=True)
class Chunk:
    start: int
    len: int
    fingerprint: int
    forced: Forced = Forced.NONE

    @property
    def end(self) -> int:
        return self.start + self.len


def build_gear_table(seed: int) -> list[int]:
    """65,536 splitmix64 outputs for ``seed``, generated on the device."""
    t = torch.empty(GEAR_TABLE_SIZE, dtype=torch.int64, device=ops._dev())
    N.check(N.lib().irm_gear_table(seed & (2**64 - 1), N.ptr(t), N.stream_ptr()), "irm_gear_table")
    return [int(v) for v in t.cpu().numpy().view(np.uint64)]


_TABLE_CACHE: dict[int, list[int]] = {}


def gear_table(seed: int = DEFAULT_GEAR_SEED) -> list[int]:
    table = _TABLE_CACHE.get(seed)
    if table is None:
        table = _TABLE_CACHE[seed] = build_gear_table(seed)
    return table


def canonical_marker(seed: int = DEFAULT_GEAR_SEED) -> tuple[int, ...]:
    """The 64-token marker: a splitmix64 stream re-seeded once (chunking.py:79-86)."""
    gen = SplitMix64(SplitMix64(seed ^ MARKER_LEN).next_u64())
    return tuple(v & 0xFFFFFFFF for v in gen.fill(MARKER_LEN))


def marker_pin_offsets(marker_spans: Iterable[tuple[int, int]]) -> set[int]:
    """Pins after the token before each marker and after its last token."""
    pins: set[int] = set()
    for start, end in marker_spans:
        if start > 0:
            pins.add(start - 1)
        pins.add(end - 1)
    return pins


def _pack_streams(streams: Sequence[Sequence[int]], pins: Sequence[Iterable[int]] | None):
    lens = [len(s) for s in streams]
    stream_off = np.zeros(len(streams) + 1, np.int64)
    np.cumsum(lens, out=stream_off[1:])
    toks = (np.concatenate([np.asarray(s, dtype=np.uint64) for s in streams])
            if streams and stream_off[-1] else np.zeros(0, np.uint64))
    if toks.size and int(toks.max()) > 0xFFFFFFFF:
        raise ValueError("token ids must be unsigned 32-bit")
    pin_lists = [sorted(set(int(p) for p in (pins[i] if pins else ()))) for i in range(len(streams))]
    pin_off = np.zeros(len(streams) + 1, np.int64)
    np.cumsum([len(p) for p in pin_lists], out=pin_off[1:])
    pin_arr = np.array([p for pl in pin_lists for p in pl], dtype=np.int64)
    return toks.astype(np.uint32), stream_off, pin_off, pin_arr


def cdc_chunk_batch(streams: Sequence[Sequence[int]], params: ChunkerParams,
                    marker_positions: Sequence[Iterable[int]] | None = None) -> ops.ChunkTable:
    """Batched K1 over several token streams; results stay on the device."""
    toks, stream_off, pin_off, pin_arr = _pack_streams(streams, marker_positions)
    dev = ops._dev()
    tok_d = torch.from_numpy(toks.view(np.int32)).to(dev) if toks.size else torch.zeros(1, dtype=torch.int32, device=dev)
    use_pins = params.marker_pinned and pin_arr.size > 0
    return ops.cdc_xxh64(
        tok_d, torch.from_numpy(stream_off).to(dev),
        torch.from_numpy(pin_off).to(dev) if use_pins else None,
        torch.from_numpy(pin_arr).to(dev) if use_pins else None,
        params.mask_exponent, params.min_size, params.max_size, params.marker_pinned,
        params.gear_seed, n_tokens=int(toks.size))


def chunks_from_table(table: ops.ChunkTable, stream: int = 0) -> list[Chunk]:
    st, ln, fp, fo, off = table.to_host()
    a, b = int(off[stream]), int(off[stream + 1])
    return [Chunk(int(st[i]), int(ln[i]), int(fp[i]), _FORCED_BY_CODE[fo[i]]) for i in range(a, b)]


def cdc_chunk(tokens: Sequence[int], params: ChunkerParams,
              marker_positions: Iterable[int] = ()) -> list[Chunk]:
    """chunking.py:89-133 -- Gear CDC with marker pins + xxh64, on the device."""
    if len(tokens) == 0:
        return []
    table = cdc_chunk_batch([tokens], params, [marker_positions])
    return chunks_from_table(table, 0)


def fixed_block_chunk(tokens: Sequence[int], block: int) -> list[Chunk]:
    """chunking.py:136-146: aligned fixed-size tiling, fingerprints via K2."""
    if block < 1:
        raise ValueError("block must be >= 1")
    n = len(tokens)
    if n == 0:
        return []
    from .fingerprint import fingerprint_spans

    starts = np.arange(0, n, block, dtype=np.int64)
    lens = np.minimum(starts + block, n) - starts
    fps = fingerprint_spans(tokens, starts, lens)
    return [Chunk(int(s), int(l), int(f), Forced.STREAM_END if l < block else Forced.NONE)
            for s, l, f in zip(starts, lens, fps)]
