"""CPU: the C-ABI library loads, exports every declared entry point, and
rejects bad arguments with the reference's error classes before any device
work (ChunkerParams rules chunking.py:45-49 -> IRM_EINVAL -> ValueError)."""

import ctypes

import pytest

from paper_2605_05696_b200 import _native as N


def test_library_exports_every_header_symbol():
    L = N.lib()
    declared = N.exported_symbols()
    assert len(declared) >= 16
    for name in declared:
        assert hasattr(L, name), name
    assert set(N._SIGS) >= set(declared) - {"irm_mla_workspace_bytes", "irm_mla_reattach_prefill"}


def test_abi_version_and_bounds():
    L = N.lib()
    assert L.irm_abi_version() == 1
    assert L.irm_cdc_chunk_bound(32768, 1, 2, 32) == 32768 // 32 + 1 + 2 + 1
    assert L.irm_cdc_chunk_bound(10, 1, 0, 0) == -1
    assert L.irm_cdc_workspace_bytes(1 << 20, 8, 16, 32) > 0
    assert L.irm_store_workspace_bytes(1000) > 0
    assert L.irm_rotate_gather_workspace_bytes(100, 64) >= 100 * 32 * 16


@pytest.mark.parametrize("k,mn,mx", [(0, 32, 512), (21, 32, 512), (7, 0, 512), (7, 512, 512), (7, 600, 512)])
def test_cdc_param_validation(k, mn, mx):
    L = N.lib()
    rc = L.irm_cdc_xxh64(None, 0, None, 0, None, None, 0, k, mn, mx, 1, None, None, None, None,
                         None, None, 0, None, 0, None)
    assert rc == N.IRM_EINVAL
    with pytest.raises(ValueError):
        N.check(rc, "cdc")


def test_cdc_capacity_error():
    L = N.lib()
    buf = ctypes.create_string_buffer(64)
    rc = L.irm_cdc_xxh64(buf, 1000, buf, 1, None, None, 0, 7, 32, 512, 1, buf, buf, buf, buf, buf,
                         buf, 3, buf, 64, None)
    assert rc == N.IRM_ECAPACITY


def test_rotate_validation():
    L = N.lib()
    # odd rotary dim, bad layout, rounding on a non-f64 pool
    g = lambda kr, layout, dtype, rnd, n=1, sms=0: L.irm_rotate_gather(
        None, 0, None, 0, 1, 512, kr, None, None, None, None, n, None, None, layout, dtype, rnd, sms, None, None, 0,
        None)
    assert g(63, 0, 0, 0) == N.IRM_EINVAL
    assert g(64, 7, 0, 0) == N.IRM_EINVAL
    assert g(64, 0, N.DTYPE_BF16, N.ROUND_BF16) == N.IRM_EINVAL
    assert g(64, 0, 0, 0, sms=-1) == N.IRM_EINVAL  # per-call SM limit
    assert L.irm_rotate_rows(None, 0, None, 0, 4, 63, None, None, 0, 0, 0, None) == N.IRM_EINVAL
    # zero work is a no-op success
    assert g(64, 0, 0, 0, n=0) == N.IRM_OK


def test_fanout_validation():
    L = N.lib()
    f = lambda kr, layout, dtype, ng=1, sms=0, rounds=1: L.irm_rotate_gather_fanout(
        None, 0, None, 0, 1, 512, kr, None, None, None, None, ng, None, None, None, 4, None, None, layout, dtype,
        sms, rounds, None, None, 0, None)
    assert f(63, 0, N.DTYPE_BF16) == N.IRM_EINVAL
    assert f(64, 3, N.DTYPE_BF16) == N.IRM_EINVAL
    assert f(64, 0, N.DTYPE_F64) == N.IRM_EINVAL  # bf16 / f32 pools only
    assert f(64, 0, N.DTYPE_BF16, rounds=0) == N.IRM_EINVAL
    assert f(64, 0, N.DTYPE_BF16, ng=0) == N.IRM_OK
    assert L.irm_group_workspace_bytes(1000) >= 2048 * 20
    buf = ctypes.create_string_buffer(64)
    assert L.irm_group_by_source(buf, buf, buf, buf, 100, None, buf, buf, buf, buf, buf, buf, buf, buf, 64,
                                 None) == N.IRM_ECAPACITY


def test_store_view_validation():
    L = N.lib()
    v = N.StoreView()
    v.n_slots = 3  # not a power of two
    assert L.irm_store_reset(ctypes.byref(v), None) == N.IRM_EINVAL
    assert b"power of two" in L.irm_last_error()


def test_wave_ops_reject_wrong_tensors():
    """The wave glue wrappers check dtypes / devices before any library call."""
    import pytest
    import torch

    from paper_2605_05696_b200 import ops

    z64 = torch.zeros(4, dtype=torch.int64)
    z32 = torch.zeros(4, dtype=torch.int32)
    with pytest.raises(ValueError, match="wave_plan"):
        ops.wave_plan(z64, 2, z32, z64, 32, 0, z64, z64, torch.zeros(4, dtype=torch.uint8), z64)  # CPU tensors
    with pytest.raises(ValueError, match="wave_compact"):
        ops.wave_compact(z64, z64, z64, z64, z64, z32, 1, z64, z64, z32, z64, z64[:1], z32)  # hit must be int32


def test_registry_entry_is_frozen():
    """RegistryEntry keeps the reference's frozen-dataclass contract (registry.py:73)
    while its rows are produced lazily."""
    import dataclasses

    import pytest

    from paper_2605_05696_b200.registry import RegistryEntry

    e = RegistryEntry(0xABC, 64, 0, None, (1, 2, 3))
    for field in ("fingerprint", "p_src", "insert_epoch", "c_kv", "kr_base"):
        with pytest.raises(dataclasses.FrozenInstanceError):
            setattr(e, field, 1)
    assert e.chunk_len == 3 and e == RegistryEntry(0xABC, 64, 0, None, (1, 2, 3))
