"""TEST INFRASTRUCTURE ONLY -- Python face of the CPU oracle.

Restates the reference algorithm for the cache-reattach hot path so the CUDA
path can be checked without /root/reference (which does not exist on the GPU
box). Integer/byte work (splitmix64, Gear CDC, xxh64) lives in
``irm_oracle.c`` (ctypes); rotary math is numpy f64, as in the reference.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module. The product package never does.

Citations (reference = /root/reference/pkg/src/irminsul):
  gear_table        chunking.py:64-76       canonical_marker   chunking.py:79-86
  cdc_chunk         chunking.py:89-133      marker_pin_offsets chunking.py:149-161
  fingerprint       fingerprint.py:16-30    derive_seed        rng.py:41-51
  make_inv_freq     rotary.py:41-49         rotate_rows        rotary.py:98-108
  round_bf16        rotary.py:63-87         synth_kv           registry.py:37-54
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Iterable, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

FORCED_NAMES = ("none", "max_clamp", "marker", "stream_end")
DEFAULT_GEAR_SEED = 0x49524D494E53554C


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "irm_oracle.c")
        if not os.path.exists(_LIB_PATH) or (
            os.path.exists(src) and os.path.getmtime(src) > os.path.getmtime(_LIB_PATH)
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, i32, u64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
        L.oracle_splitmix64_fill.argtypes = [u64, i64, P]
        L.oracle_derive_seed.argtypes = [u64, P, i32]
        L.oracle_derive_seed.restype = u64
        L.oracle_gear_table.argtypes = [u64, P]
        L.oracle_canonical_marker.argtypes = [u64, P]
        L.oracle_xxh64.argtypes = [P, i64, u64]
        L.oracle_xxh64.restype = u64
        L.oracle_fingerprint.argtypes = [P, i64]
        L.oracle_fingerprint.restype = u64
        L.oracle_cdc_chunk.argtypes = [P, i64, P, i64, i32, i32, i32, P, P, P, P, P, i64]
        L.oracle_cdc_chunk.restype = i64
        L.oracle_gear_states.argtypes = [P, i64, P, i64, P, P]
        L.oracle_cdc_batch.argtypes = [P, P, i32, P, P, i32, i32, i32, P, P, P, P, P, P, P, i32]
        L.oracle_cdc_batch.restype = i64
        L.oracle_rotate_gather_bf16.argtypes = [P, i64, P, i64, i32, P, P, P, P, i64, P, i32, i32]
        L.oracle_max_threads.restype = i32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- constants
def splitmix64_fill(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    lib().oracle_splitmix64_fill(seed & (2**64 - 1), n, _p(out))
    return out


def derive_seed(seed: int, *labels: int) -> int:
    lab = np.array([x & (2**64 - 1) for x in labels], dtype=np.uint64)
    return int(lib().oracle_derive_seed(seed & (2**64 - 1), _p(lab), len(lab)))


_GEAR_CACHE: dict[int, np.ndarray] = {}


def gear_table(seed: int = DEFAULT_GEAR_SEED) -> np.ndarray:
    t = _GEAR_CACHE.get(seed)
    if t is None:
        t = np.empty(65536, dtype=np.uint64)
        lib().oracle_gear_table(seed & (2**64 - 1), _p(t))
        t.setflags(write=False)
        _GEAR_CACHE[seed] = t
    return t


def canonical_marker(seed: int = DEFAULT_GEAR_SEED) -> tuple[int, ...]:
    out = np.empty(64, dtype=np.uint32)
    lib().oracle_canonical_marker(seed & (2**64 - 1), _p(out))
    return tuple(int(x) for x in out)


# ---------------------------------------------------------------- hashing
def xxh64(data: bytes, seed: int = 0) -> int:
    buf = np.frombuffer(data, dtype=np.uint8) if data else np.zeros(1, np.uint8)
    return int(lib().oracle_xxh64(_p(buf), len(data), seed))


def fingerprint(tokens: Sequence[int]) -> int:
    a = np.ascontiguousarray(np.asarray(tokens, dtype=np.uint64).astype(np.uint32))
    if a.size == 0:
        a = np.zeros(1, np.uint32)
        return int(lib().oracle_fingerprint(_p(a), 0))
    return int(lib().oracle_fingerprint(_p(a), a.size))


# ---------------------------------------------------------------- CDC
def marker_pin_offsets(spans: Iterable[tuple[int, int]]) -> set[int]:
    pins: set[int] = set()
    for s, e in spans:
        if s > 0:
            pins.add(s - 1)
        pins.add(e - 1)
    return pins


def cdc_chunk(tokens, k: int = 7, min_size: int = 32, max_size: int = 512,
              pins: Iterable[int] = (), gear_seed: int = DEFAULT_GEAR_SEED,
              marker_pinned: bool = True):
    """Returns (start[int32], len[int32], fp[uint64], forced[uint8]) arrays."""
    tok = np.ascontiguousarray(np.asarray(tokens, dtype=np.uint64).astype(np.uint32))
    n = tok.size
    pin_arr = np.array(sorted(set(int(p) for p in pins)) if marker_pinned else [], dtype=np.int64)
    cap = n // max(min_size, 1) + 2 + pin_arr.size
    st = np.empty(cap, np.int32); ln = np.empty(cap, np.int32)
    fp = np.empty(cap, np.uint64); fo = np.empty(cap, np.uint8)
    g = gear_table(gear_seed)
    tok_p = tok if n else np.zeros(1, np.uint32)
    pin_p = pin_arr if pin_arr.size else np.zeros(1, np.int64)
    nc = lib().oracle_cdc_chunk(_p(tok_p), n, _p(pin_p), pin_arr.size, k, min_size, max_size,
                                _p(g), _p(st), _p(ln), _p(fp), _p(fo), cap)
    assert nc >= 0, "oracle chunk capacity exceeded"
    return st[:nc].copy(), ln[:nc].copy(), fp[:nc].copy(), fo[:nc].copy()


def gear_states(tokens, pins: Iterable[int] = (), gear_seed: int = DEFAULT_GEAR_SEED) -> np.ndarray:
    tok = np.ascontiguousarray(np.asarray(tokens, dtype=np.uint64).astype(np.uint32))
    pin_arr = np.array(sorted(set(pins)), dtype=np.int64)
    out = np.empty(max(tok.size, 1), np.uint64)
    pin_p = pin_arr if pin_arr.size else np.zeros(1, np.int64)
    lib().oracle_gear_states(_p(tok), tok.size, _p(pin_p), pin_arr.size, _p(gear_table(gear_seed)),
                             _p(out))
    return out[: tok.size]


def cdc_batch(tok: np.ndarray, stream_off: np.ndarray, pin_off: np.ndarray, pins: np.ndarray,
              k=7, min_size=32, max_size=512, gear_seed=DEFAULT_GEAR_SEED, n_threads=0):
    """Threaded batched CDC (CPU baseline). Returns per-stream lists of arrays."""
    ns = stream_off.size - 1
    lens = np.diff(stream_off)
    npins = np.diff(pin_off)
    bound = lens // max(min_size, 1) + 2 + npins
    out_off = np.zeros(ns + 1, np.int64)
    np.cumsum(bound, out=out_off[1:])
    cap = int(out_off[-1])
    st = np.empty(cap, np.int32); ln = np.empty(cap, np.int32)
    fp = np.empty(cap, np.uint64); fo = np.empty(cap, np.uint8)
    counts = np.empty(ns, np.int64)
    pins_p = pins if pins.size else np.zeros(1, np.int64)
    lib().oracle_cdc_batch(_p(tok), _p(stream_off), ns, _p(pin_off), _p(pins_p), k, min_size,
                           max_size, _p(gear_table(gear_seed)), _p(out_off), _p(st), _p(ln),
                           _p(fp), _p(fo), _p(counts), n_threads)
    return out_off, counts, st, ln, fp, fo


# ---------------------------------------------------------------- rotary
def make_inv_freq(theta: float, dim: int = 64) -> np.ndarray:
    j = np.arange(dim // 2, dtype=np.float64)
    return np.power(float(theta), -2.0 * j / dim)


def rotate_rows(rows: np.ndarray, positions, inv_freq: np.ndarray,
                interleaved: bool = False) -> np.ndarray:
    """f64 rotation; half-split (reference rotary.py:98-108) or interleaved
    (DSv2-form: pairs (2j, 2j+1), the permutation-conjugate of half-split)."""
    rows = np.asarray(rows, dtype=np.float64)
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, 1)
    ang = pos * inv_freq[np.newaxis, :]
    c, s = np.cos(ang), np.sin(ang)
    half = inv_freq.size
    if not interleaved:
        lo, hi = rows[..., :half], rows[..., half:]
        return np.concatenate([lo * c - hi * s, lo * s + hi * c], axis=-1)
    lo, hi = rows[..., 0::2], rows[..., 1::2]
    out = np.empty_like(rows)
    out[..., 0::2] = lo * c - hi * s
    out[..., 1::2] = lo * s + hi * c
    return out


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Single RNE rounding of f64 onto the bf16 grid (reference rotary.py:63-87)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.array(x, dtype=np.float64)
    fin = np.isfinite(x) & (x != 0.0)
    if not np.any(fin):
        return out
    v = x[fin]
    _, e = np.frexp(v)
    ulp = np.ldexp(1.0, np.maximum(e - 8, -133))
    q = np.rint(v / ulp) * ulp
    mx = float(np.ldexp(2.0 - 2.0**-7, 127))
    out[fin] = np.where(np.abs(q) > mx, np.copysign(np.inf, q), q)
    return out


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ---------------------------------------------------------------- synthetic KV
_CKV_LABEL = 0x434B56
_KR_LABEL = 0x4B52


def synth_kv(token: int, seed: int = 0, ckv_dim: int = 512, kr_dim: int = 64):
    c = np.random.Generator(np.random.PCG64(derive_seed(seed, _CKV_LABEL, token)))
    k = np.random.Generator(np.random.PCG64(derive_seed(seed, _KR_LABEL, token)))
    cv = c.standard_normal(ckv_dim)
    kv = k.standard_normal(kr_dim)
    return cv / np.linalg.norm(cv), kv / np.linalg.norm(kv)


def rotate_gather_bf16(pool_u16: np.ndarray, out_u16: np.ndarray, src_row, dst_row, length,
                       delta, inv_freq, interleaved=False, n_threads=0):
    """CPU baseline of K4 (bf16 pool [L, rows, 576] as uint16 bit patterns)."""
    L, prow, _ = pool_u16.shape
    orow = out_u16.shape[1]
    src_row = np.ascontiguousarray(src_row, np.int64)
    dst_row = np.ascontiguousarray(dst_row, np.int64)
    length = np.ascontiguousarray(length, np.int32)
    delta = np.ascontiguousarray(delta, np.int64)
    inv = np.ascontiguousarray(inv_freq, np.float64)
    lib().oracle_rotate_gather_bf16(_p(pool_u16), prow, _p(out_u16), orow, L, _p(src_row),
                                    _p(dst_row), _p(length), _p(delta), src_row.size, _p(inv),
                                    int(interleaved), n_threads)


def max_threads() -> int:
    return int(lib().oracle_max_threads())


# ----------------------------------------------------------------- K0: exact-prefix match
def prefix_match(inserted, seq):
    """Longest common prefix of ``seq`` with any inserted sequence and the
    earliest-inserted witness reaching it: the brute force the reference pins
    RadixTree with (tests/test_radix.py:15-23, :75-90; radix.py:60-83).
    ``inserted``: list of (handle, tokens) in insert order."""
    q = np.asarray(seq, dtype=np.uint32)
    best, who = 0, None
    for handle, stored in inserted:
        s = np.asarray(stored, dtype=np.uint32)
        n = min(s.size, q.size)
        neq = np.nonzero(s[:n] != q[:n])[0]
        m = int(neq[0]) if neq.size else n
        if m > best:
            best, who = m, handle
    return best, who


def prefix_lengths_sequential(seqs, probe: int = 64):
    """m[i] = the longest common prefix of seqs[i] with any seqs[j], j < i -- the
    phase-1 answer of the serve loop (engine.py:170, 228; radix.py:60-83), exact
    and fast for long sequences: an LCP below ``probe`` is found by comparing
    every earlier sequence's first ``probe`` tokens at once; only sequences
    sharing all ``probe`` first tokens are compared in full."""
    seqs = [np.asarray(s, dtype=np.uint32) for s in seqs]
    heads = np.zeros((len(seqs), probe), np.uint64)
    hlen = np.zeros(len(seqs), np.int64)
    groups: dict[bytes, list[int]] = {}
    out = []
    for i, s in enumerate(seqs):
        h = s[:probe].astype(np.uint64)
        m = 0
        if i:
            n = np.minimum(hlen[:i], h.size)
            eq = heads[:i, :h.size] == h[None, :]
            first_diff = np.where(eq.all(axis=1), h.size, np.argmin(eq, axis=1))
            m = int(np.minimum(first_diff, n).max())
            if h.size == probe:
                for j in groups.get(h.tobytes(), []):  # candidates for an LCP of probe or more
                    t = seqs[j]
                    k = min(t.size, s.size)
                    neq = np.nonzero(t[:k] != s[:k])[0]
                    m = max(m, int(neq[0]) if neq.size else k)
        out.append(m)
        heads[i, :h.size] = h
        hlen[i] = h.size
        if h.size == probe:
            groups.setdefault(h.tobytes(), []).append(i)
    return out
