"""ctypes binding of the C ABI in include/irminsul_b200.h.

The library is built in-tree (paper_2605_05696_b200/_lib/libirminsul_b200.so,
``__graft_entry__.build()``). There is no fallback: if the library or a CUDA
device is missing, every hot-path call raises.
"""

from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libirminsul_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "irminsul_b200.h")

IRM_OK, IRM_EINVAL, IRM_ECUDA, IRM_ECAPACITY = 0, 1, 2, 3
FORCED_NONE, FORCED_MAX_CLAMP, FORCED_MARKER, FORCED_STREAM_END = 0, 1, 2, 3
LAYOUT_HALF_SPLIT, LAYOUT_INTERLEAVED = 0, 1
PEER_HANDLE_BYTES = 64  # IRM_PEER_HANDLE_BYTES
DTYPE_F64, DTYPE_F32, DTYPE_BF16 = 0, 1, 2
ROUND_NONE, ROUND_F32, ROUND_BF16 = 0, 1, 2
EMPTY_KEY = 0xFFFFFFFFFFFFFFFF

P = ctypes.c_void_p
i64, i32, u64, f32 = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_float


class StoreView(ctypes.Structure):
    """irm_store_view (include/irminsul_b200.h)."""

    _fields_ = [
        ("slot_key", P), ("slot_order", P), ("slot_entry", P), ("n_slots", i64),
        ("e_fp", P), ("e_p_src", P), ("e_len", P), ("e_row", P), ("max_entries", i64),
        ("counters", P), ("pool_rows", i64),
    ]


class PrefixView(ctypes.Structure):
    """irm_prefix_view (include/irminsul_b200.h)."""

    _fields_ = [("slots", P), ("n_slots", i64), ("counters", P), ("hash_key", u64)]


_SIGS = {
    "irm_abi_version": ([], i32),
    "irm_last_error": ([], ctypes.c_char_p),
    "irm_device_sm_count": ([], i32),
    "irm_launch_count": ([], i64),
    "irm_gear_table": ([u64, P, P], i32),
    "irm_cdc_chunk_bound": ([i64, i32, i64, i32], i64),
    "irm_cdc_workspace_bytes": ([i64, i32, i64, i32], i64),
    "irm_cdc_xxh64": ([P, i64, P, i32, P, P, i64, i32, i32, i32, i32, P, P, P, P, P, P, i64, P, i64, P], i32),
    "irm_cdc_xxh64_seeded": ([P, i64, P, i32, P, P, i64, i32, i32, i32, i32, u64, P, P, P, P, P, i64, P, i64, P], i32),
    "irm_xxh64_spans": ([P, P, P, i64, u64, P, P], i32),
    "irm_store_reset": ([ctypes.POINTER(StoreView), P], i32),
    "irm_store_workspace_bytes": ([i64], i64),
    "irm_store_lookup_insert": ([ctypes.POINTER(StoreView), P, P, P, P, P, i64, P, P, P, P, P, i64, P], i32),
    "irm_store_lookup": ([ctypes.POINTER(StoreView), P, i64, P, P], i32),
    "irm_wave_rebase": ([P, P, P, i32, i64, P, P, P, P, P, P, P], i32),
    "irm_prefix_wave_prepare": ([ctypes.POINTER(PrefixView), P, i64, P, P, P, i64, P, P, P, i32, P, P], i32),
    "irm_wave_plan": ([P, i32, P, P, i64, i64, i64, P, P, P, P, P], i32),
    "irm_wave_compact": ([P, P, P, P, P, P, i64, i64, P, P, P, P, P, P, P, P, P], i32),
    "irm_rotate_gather_workspace_bytes": ([i64, i32], i64),
    "irm_group_workspace_bytes": ([i64], i64),
    "irm_group_by_source": ([P, P, P, P, i64, P, P, P, P, P, P, P, P, P, i64, P], i32),
    "irm_fanout_workspace_bytes": ([i64, i32], i64),
    "irm_rotate_gather_fanout": ([P, i64, P, i64, i32, i32, i32, P, P, P, P, i64, P, P, P, i64, P, P, i32, i32, i32,
                                  i32, P, P, i64, P], i32),
    "irm_copy_runs": ([P, i64, P, i64, P, P, i64, P, i32, i32, P], i32),
    "irm_peer_export": ([P, P, P], i32),
    "irm_peer_open": ([P, i64, P], i32),
    "irm_exchange_pack": ([P, P, P, P, P, i64, i32, i32, i64, P, P, P, P], i32),
    "irm_exchange_split": ([P, i64, P, P, P, P, P, P], i32),
    "irm_exchange_reply": ([P, i32, i64, P, P, P, P, i64, i64, P, P, i64, P, P, P], i32),
    "irm_exchange_unpack": ([P, P, i64, i64, P, P, P, P, P, P], i32),
    "irm_rotate_gather": ([P, i64, P, i64, i32, i32, i32, P, P, P, P, i64, P, P, i32, i32, i32, i32, P, P, i64, P],
                          i32),
    "irm_rotate_rows": ([P, i64, P, i64, i64, i32, P, P, i32, i32, i32, P], i32),
    "irm_rotate_rows_layered": ([P, i64, i64, P, i64, i64, i32, i64, i32, P, P, i32, i32, i32, P], i32),
    "irm_round_f64": ([P, P, i64, i32, P], i32),
    "irm_chunk_cossin": ([P, i64, P, P, P], i32),
    "irm_trace_scan": ([P, i64, i32, P, P, P, i32], i32),
    "irm_trace_fill": ([P, i64, i32, P, P, P, P, P, P, P, P, P], i32),
    "irm_prefix_reset": ([ctypes.POINTER(PrefixView), P], i32),
    "irm_prefix_workspace_bytes": ([i64, i32], i64),
    "irm_prefix_match_insert": ([ctypes.POINTER(PrefixView), P, P, i32, i64, P, P, P, P, P, P, P, P, P, i64, P], i32),
    "irm_mla_reattach_prefill": ([P, i64, i32, i64, P, i64, P, i32, P, P, i32, f32, P, P, P], i32),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load the in-tree library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def exported_symbols() -> list[str]:
    """Names of the entry points declared in include/irminsul_b200.h."""
    with open(HEADER_PATH) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(irm_\w+)\s*\(", text, re.M)))


def check(rc: int, what: str = "") -> None:
    if rc == IRM_OK:
        return
    msg = lib().irm_last_error().decode(errors="replace")
    if rc in (IRM_EINVAL, IRM_ECAPACITY):
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: CUDA error: {msg}")


_cuda_ok = False


def require_cuda():
    global _cuda_ok
    if _cuda_ok:  # checked once: torch.cuda.is_available() costs milliseconds per call
        return
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("irminsul_b200 requires a CUDA device (B200, sm_100a); no CPU fallback")
    lib()
    _cuda_ok = True


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)
