"""Drop-in for ``irminsul.fingerprint`` (reference fingerprint.py).

xxHash64 (seed 0) over the little-endian u32 token encoding, computed on the
device by the batched span kernel (K2, ``irm_xxh64_spans``).
"""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import ops

XXH64_EMPTY = 0xEF46DB3751D8E999


def token_bytes(tokens: Sequence[int]) -> bytes:
    """Little-endian u32 encoding of a token sequence (fingerprint.py:16-21)."""
    a = np.asarray(tokens, dtype=np.uint64)
    if a.size and int(a.max()) > 0xFFFFFFFF:
        raise OverflowError("token does not fit in 4 bytes")
    return a.astype("<u4").tobytes()


def _hash_device(buf: np.ndarray, off: np.ndarray, ln: np.ndarray) -> np.ndarray:
    dev = ops._dev()
    b = torch.from_numpy(buf if buf.size else np.zeros(16, np.uint8)).to(dev)
    out = ops.xxh64_spans(b, torch.from_numpy(off).to(dev), torch.from_numpy(ln).to(dev))
    return out.cpu().numpy().view(np.uint64)


def fingerprint_bytes(data: bytes) -> int:
    buf = np.frombuffer(bytes(data), dtype=np.uint8).copy()
    return int(_hash_device(buf, np.zeros(1, np.int64), np.array([len(data)], np.int64))[0])


def fingerprint(tokens: Sequence[int]) -> int:
    """xxHash64 (seed 0) over the little-endian u32 encoding of the tokens."""
    return int(fingerprint_spans(tokens, np.zeros(1, np.int64), np.array([len(tokens)], np.int64))[0])


def fingerprint_spans(tokens: Sequence[int], starts, lens) -> np.ndarray:
    """Batched token-span fingerprints (uint64 array)."""
    buf = np.frombuffer(token_bytes(tokens), dtype=np.uint8).copy()
    return _hash_device(buf, 4 * np.asarray(starts, np.int64), 4 * np.asarray(lens, np.int64))


def sliding_fingerprints(tokens: Sequence[int], window: int = 64) -> list[tuple[int, int]]:
    """One (offset, hash) per window start 0..len-window (fingerprint.py:33-50)."""
    if window < 1:
        raise ValueError("window must be >= 1")
    n = len(tokens)
    if n < window:
        return []
    starts = np.arange(n - window + 1, dtype=np.int64)
    fps = fingerprint_spans(tokens, starts, np.full(starts.size, window, np.int64))
    return [(int(o), int(f)) for o, f in zip(starts, fps)]
