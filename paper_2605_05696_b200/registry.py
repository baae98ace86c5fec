"""Drop-in for ``irminsul.registry`` (reference registry.py) on the B200 path.

The registry is a device-resident content-hash store (K3, ``ops.ChunkStore``)
over a device latent pool [layers, rows, ckv_dim + kr_dim]:
  * ``insert`` appends the chunk's rows to the pool and stores k_r already
    rotated to p_src + i (the producer rotation, ``irm_rotate_rows``);
  * ``lookup`` probes the device table;
  * ``materialize`` runs the rotate+gather kernel (K4, ``irm_rotate_gather``)
    with delta = p_dest - p_src and the precision tag's store rounding.
Entries keep host mirrors of (c_kv, kr_base) so the reference's object
contract holds: ``materialize(...).c_kv is entry.c_kv`` (registry_test:124).

The synthetic KV oracle (``synth_kv``) stands in for model prefill exactly as
in the reference (registry.py:37-70); it is the input generator, not the path.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _native as N
from . import ops
from .rng import derive_seed
from .rotary import Precision, RotarySpec, _ROUND, inv_freq_device

_CKV_LABEL = 0x434B56
_KR_LABEL = 0x4B52


@dataclass(frozen=True)
class SyntheticKvParams:
    seed: int = 0
    ckv_dim: int = 512
    kr_dim: int = 64

    def __post_init__(self):
        if self.ckv_dim <= 0 or self.kr_dim <= 0:
            raise ValueError("dims must be positive")
        if self.kr_dim % 2 != 0:
            raise ValueError("kr_dim must be even")


def synth_kv(token: int, index_in_chunk: int, params: SyntheticKvParams) -> tuple[np.ndarray, np.ndarray]:
    """Deterministic unit-norm (c_kv row, kr_raw row) for a token id (registry.py:37-54)."""
    ckv_rng = np.random.Generator(np.random.PCG64(derive_seed(params.seed, _CKV_LABEL, token)))
    kr_rng = np.random.Generator(np.random.PCG64(derive_seed(params.seed, _KR_LABEL, token)))
    c_kv = ckv_rng.standard_normal(params.ckv_dim)
    kr_raw = kr_rng.standard_normal(params.kr_dim)
    return c_kv / np.linalg.norm(c_kv), kr_raw / np.linalg.norm(kr_raw)


class _SynthCache:
    def __init__(self, params: SyntheticKvParams):
        self.params = params
        self._rows: dict[int, tuple[np.ndarray, np.ndarray]] = {}

    def rows(self, tokens: Sequence[int]) -> tuple[np.ndarray, np.ndarray]:
        tokens = tokens.tolist() if isinstance(tokens, np.ndarray) else tokens  # Python ints (derive_seed)
        for t in tokens:
            if t not in self._rows:
                self._rows[t] = synth_kv(t, 0, self.params)
        if len(tokens) == 0:
            return np.zeros((0, self.params.ckv_dim)), np.zeros((0, self.params.kr_dim))
        return (np.stack([self._rows[t][0] for t in tokens]),
                np.stack([self._rows[t][1] for t in tokens]))


class RegistryEntry:
    """registry.py:73-84. ``c_kv`` / ``kr_base`` are produced on first use: the
    synthetic prefill rows (PCG64 per token, registry.py:37-54) and their pool
    write + rotation to p_src happen when something reads them (an attribute
    access, materialize, the live tripwire), so observer-mode serving never pays
    for KV it does not look at. The values are the same as an eager insert's."""

    __slots__ = ("fingerprint", "p_src", "insert_epoch", "_reg", "_tokens", "_c_kv", "_kr_base")
    _FROZEN = ("fingerprint", "p_src", "insert_epoch", "c_kv", "kr_base")

    def __init__(self, fingerprint: int, p_src: int, insert_epoch: int, reg, tokens, c_kv=None, kr_base=None):
        sa = object.__setattr__
        sa(self, "fingerprint", fingerprint)
        sa(self, "p_src", p_src)
        sa(self, "insert_epoch", insert_epoch)
        sa(self, "_reg", reg)
        sa(self, "_tokens", tokens)
        sa(self, "_c_kv", c_kv)
        sa(self, "_kr_base", kr_base)

    def __setattr__(self, name, value):
        # frozen like the reference's dataclass (registry.py:73): its public fields never change
        if name in self._FROZEN:
            raise dataclasses.FrozenInstanceError(f"cannot assign to field {name!r}")
        object.__setattr__(self, name, value)

    def __delattr__(self, name):
        if name in self._FROZEN:
            raise dataclasses.FrozenInstanceError(f"cannot delete field {name!r}")
        object.__delattr__(self, name)

    def __eq__(self, other):
        if not isinstance(other, RegistryEntry):
            return NotImplemented
        return (self.fingerprint, self.p_src, self.insert_epoch) == (other.fingerprint, other.p_src,
                                                                     other.insert_epoch) and self._reg is other._reg

    def __hash__(self):
        return hash((self.fingerprint, self.p_src, self.insert_epoch))

    @property
    def c_kv(self) -> np.ndarray:
        if self._c_kv is None:
            self._reg._flush()
        return self._c_kv

    @property
    def kr_base(self) -> np.ndarray:
        if self._kr_base is None:
            self._reg._flush()
        return self._kr_base

    @property
    def chunk_len(self) -> int:
        return len(self._tokens)

    def __repr__(self) -> str:
        return f"RegistryEntry(fingerprint={self.fingerprint:#x}, p_src={self.p_src}, len={self.chunk_len}, " \
               f"insert_epoch={self.insert_epoch})"


@dataclass
class MaterializeResult:
    c_kv: np.ndarray
    k_r: np.ndarray
    delta: int
    multiplies: int


class DevicePool:
    """Latent pool [layers, rows, ckv_dim + kr_dim] on the device, grown by doubling."""

    def __init__(self, ckv_dim: int, kr_dim: int, layers: int = 1, dtype=torch.float64, rows: int = 4096):
        self.ckv_dim, self.kr_dim, self.layers, self.dtype = ckv_dim, kr_dim, layers, dtype
        self.data = torch.zeros(layers, rows, ckv_dim + kr_dim, dtype=dtype, device=ops._dev())

    def ensure(self, rows: int):
        if rows <= self.data.shape[1]:
            return
        cap = self.data.shape[1]
        while cap < rows:
            cap *= 2
        new = torch.zeros(self.layers, cap, self.data.shape[2], dtype=self.dtype, device=self.data.device)
        new[:, : self.data.shape[1]] = self.data
        self.data = new


class KvRegistry:
    """fingerprint -> (c_kv, kr_base, p_src); first writer wins (registry.py:94-170)."""

    def __init__(self, kv_params: SyntheticKvParams, spec: RotarySpec, max_entries: int = 1 << 16):
        self.kv_params = kv_params
        self.spec = spec
        self._synth = _SynthCache(kv_params)
        self._entries: list[RegistryEntry] = []
        self._entry_rows: list[int] = []  # pool row of entry i
        self.store = ops.ChunkStore(max_entries)
        self.pool = DevicePool(kv_params.ckv_dim, kv_params.kr_dim)
        self._rows_used = 0
        self._order = 0
        self._gather_ws = None
        self._pending: list[RegistryEntry] = []  # entries whose rows are not written yet

    # ------------------------------------------------------------ queries
    def __len__(self) -> int:
        return len(self._entries)

    def __contains__(self, fp: int) -> bool:
        return self.lookup(fp) is not None

    def _fp_tensor(self, fps) -> torch.Tensor:
        a = np.asarray([int(f) & (2**64 - 1) for f in fps], dtype=np.uint64).view(np.int64)
        return torch.from_numpy(a).to(ops._dev())

    def lookup(self, fp: int) -> RegistryEntry | None:
        e = int(self.store.lookup(self._fp_tensor([fp])).item())
        return self._entries[e] if e >= 0 else None

    def entries(self) -> list[RegistryEntry]:
        return list(self._entries)  # entry index == insert epoch

    def entry_by_index(self, i: int) -> RegistryEntry:
        return self._entries[i]

    def fresh_rows(self, tokens: Sequence[int]) -> tuple[np.ndarray, np.ndarray]:
        return self._synth.rows(tokens)

    # ------------------------------------------------------------ inserts
    def ensure_capacity(self, n_new: int):
        """Room for n_new more entries: the device store is rebuilt 2x larger from the
        host mirror (same entry ids, rows and p_src; inserting in epoch order gives the
        store's row scan the same rows), so the dict never fills up (registry.py:126)."""
        need = len(self._entries) + n_new
        if need <= self.store.max_entries:
            return
        cap = max(2 * self.store.max_entries, need)
        new = ops.ChunkStore(cap)
        n = len(self._entries)
        if n:
            dev = ops._dev()
            fps = self._fp_tensor([e.fingerprint for e in self._entries])
            order = torch.arange(n, dtype=torch.int64, device=dev)
            p = torch.tensor([e.p_src for e in self._entries], dtype=torch.int64, device=dev)
            ln = torch.tensor([e.chunk_len for e in self._entries], dtype=torch.int32, device=dev)
            hit, entry, _, row = new.lookup_insert(fps, order, p, ln)
            assert bool((hit == 0).all()) and row.cpu().tolist() == self._entry_rows, "store rebuild diverged"
        self.store = new

    def insert(self, fp: int, tokens: Sequence[int], p_src: int) -> RegistryEntry:
        """Store a chunk's KV at p_src (no-op on duplicates, registry.py:126-140)."""
        self.ensure_capacity(1)
        dev = ops._dev()
        hit, entry, _, row = self.store.lookup_insert(
            self._fp_tensor([fp]), torch.tensor([self._order], dtype=torch.int64, device=dev),
            torch.tensor([p_src], dtype=torch.int64, device=dev),
            torch.tensor([len(tokens)], dtype=torch.int32, device=dev))
        self._order += 1
        h, e, r = int(hit.item()), int(entry.item()), int(row.item())
        if h == 1:
            return self._entries[e]
        assert e == len(self._entries), "device store and host mirror diverged"
        return self.commit_rows(fp, tokens, p_src, r)

    def commit_rows(self, fp: int, tokens: Sequence[int], p_src: int, row: int) -> RegistryEntry:
        """Producer side (registry.py:131-136): register the entry whose rows live at
        pool row ``row``; the rows are synthesised and rotated to p_src + i on the
        device at the next ``_flush`` (first read)."""
        toks = tuple(tokens.tolist()) if isinstance(tokens, np.ndarray) else tuple(tokens)
        entry = RegistryEntry(int(fp), int(p_src), len(self._entries), self, toks)
        self._entries.append(entry)
        self._entry_rows.append(row)
        self._pending.append(entry)
        self._rows_used = max(self._rows_used, row + len(tokens))
        return entry

    def _flush(self):
        """Producer (registry.py:131-136), batched: the synthetic rows of every entry
        not yet written go up in ONE host->device copy, k_r is rotated to p_src + i
        for all of them by ONE irm_rotate_rows launch, the rows land in the pool by
        one scatter, and kr_base comes back in one copy."""
        pending, self._pending = self._pending, []
        if not pending:
            return
        ckv, kr = self.kv_params.ckv_dim, self.kv_params.kr_dim
        rows = [self._synth.rows(e._tokens) for e in pending]
        lens = np.array([e.chunk_len for e in pending], np.int64)
        total = int(lens.sum())
        c_all = [r[0] for r in rows]
        if total:
            starts = np.array([self._entry_rows[e.insert_epoch] for e in pending], np.int64)
            self.pool.ensure(int((starts + lens).max()))
            dev = self.pool.data.device
            stage = np.empty((total, ckv + kr), np.float64)
            stage[:, :ckv] = np.concatenate([r[0] for r in rows if len(r[0])])
            stage[:, ckv:] = np.concatenate([r[1] for r in rows if len(r[1])])
            pos = np.concatenate([np.arange(e.p_src, e.p_src + e.chunk_len, dtype=np.float64) for e in pending])
            st = torch.from_numpy(stage).to(dev)
            ops.rotate_rows(st[:, ckv:], torch.from_numpy(pos).to(dev), inv_freq_device(self.spec),
                            self.spec.layout_code, out=st[:, ckv:])
            dst = torch.from_numpy(np.repeat(starts, lens) + (np.arange(total) - np.repeat(np.cumsum(lens) - lens, lens)))
            self.pool.data[0].index_copy_(0, dst.to(dev), st)
            kr_all = st[:, ckv:].cpu().numpy()
        bounds = np.concatenate([[0], np.cumsum(lens)])
        for k, entry in enumerate(pending):
            c_kv = c_all[k].copy()
            kr_base = kr_all[bounds[k]:bounds[k + 1]].copy() if entry.chunk_len else np.zeros((0, kr))
            c_kv.setflags(write=False)
            kr_base.setflags(write=False)
            entry._c_kv, entry._kr_base = c_kv, kr_base

    def pool_bytes(self) -> int:
        """Bytes of the shared latent pool as f64 c_kv rows (one copy per fingerprint)."""
        return sum(e.chunk_len for e in self._entries) * self.kv_params.ckv_dim * 8

    # ------------------------------------------------------------ materialize
    def materialize_device(self, rows: torch.Tensor, lens: torch.Tensor, deltas: torch.Tensor,
                           precision: Precision = Precision.F64, out: torch.Tensor | None = None):
        """Batched K4 over the pool: chunk i -> out rows [sum(lens[:i]), +lens[i])."""
        self._flush()
        n_rows = int(lens.sum().item()) if out is None else out.shape[1]
        if out is None:
            out = torch.empty(1, max(n_rows, 1), self.pool.data.shape[2], dtype=self.pool.data.dtype,
                              device=self.pool.data.device)
        dst = torch.zeros_like(rows)
        if rows.numel() > 1:
            dst[1:] = torch.cumsum(lens[:-1].to(torch.int64), 0)
        need = int(N.lib().irm_rotate_gather_workspace_bytes(rows.numel(), self.kv_params.kr_dim))
        if self._gather_ws is None or self._gather_ws.numel() < need:
            self._gather_ws = torch.empty(max(need, 256), dtype=torch.uint8, device=out.device)
        ops.rotate_gather(self.pool.data, out, rows, dst, lens.to(torch.int32), deltas,
                          inv_freq_device(self.spec), self.kv_params.ckv_dim, self.kv_params.kr_dim,
                          self.spec.layout_code, _ROUND[Precision(precision)], ws=self._gather_ws)
        return out

    def materialize(self, entry: RegistryEntry, p_dest: int,
                    precision: Precision = Precision.F64) -> MaterializeResult:
        """Re-target a stored chunk to p_dest via a uniform delta-rotation (registry.py:146-166)."""
        if p_dest < 0:
            raise ValueError("p_dest must be non-negative")
        delta = p_dest - entry.p_src
        n = entry.chunk_len
        if n == 0:
            return MaterializeResult(entry.c_kv, np.zeros((0, self.spec.dim)), delta, 0)
        dev = ops._dev()
        out = self.materialize_device(
            torch.tensor([self._entry_rows[entry.insert_epoch]], dtype=torch.int64, device=dev),
            torch.tensor([n], dtype=torch.int32, device=dev),
            torch.tensor([delta], dtype=torch.int64, device=dev), precision)
        k_r = out[0, :n, self.kv_params.ckv_dim:].cpu().numpy().copy()
        return MaterializeResult(entry.c_kv, k_r, delta, n * self.spec.dim)

    def naive_reuse(self, entry: RegistryEntry, p_dest: int) -> MaterializeResult:
        """Stored rows with no rotation: the naive-reuse baseline (registry.py:168-170)."""
        return MaterializeResult(entry.c_kv, np.array(entry.kr_base), p_dest - entry.p_src, 0)
