"""Exact-prefix index for phase 1 of the serve path (reference radix.py).

``RadixTree`` is the host form (pointer chasing); ``DeviceRadixTree`` is
K0, the batched device prefix index of SURVEY §8(f) item 1, which the serve
path uses. Edges reference slices of the
inserted sequences (numpy views, no copies) and common-prefix lengths are
computed with vectorised compares, so a 32K-token match is a handful of
numpy calls instead of a per-token Python loop. Semantics follow
radix.py:31-89: longest match, earliest-inserted witness.
"""

from __future__ import annotations

import os

from typing import Hashable, Sequence

import numpy as np


def _lcp(a: np.ndarray, b: np.ndarray) -> int:
    n = min(a.size, b.size)
    if n == 0:
        return 0
    neq = a[:n] != b[:n]
    k = int(np.argmax(neq))
    return n if not neq[k] else k


class _Edge:
    __slots__ = ("label", "children", "witness", "epoch")

    def __init__(self, label: np.ndarray, witness, epoch: int):
        self.label = label
        self.children: dict[int, _Edge] = {}
        self.witness = witness
        self.epoch = epoch


class RadixTree:
    def __init__(self, capacity_hint: int | None = None):
        self._root = _Edge(np.zeros(0, np.uint32), None, -1)
        self._epoch = 0
        self.capacity_hint = capacity_hint

    @staticmethod
    def _arr(seq) -> np.ndarray:
        return np.asarray(seq, dtype=np.uint64).astype(np.uint32) if not isinstance(seq, np.ndarray) else seq.astype(np.uint32, copy=False)

    def insert(self, seq: Sequence[int], handle: Hashable) -> None:
        s = self._arr(seq)
        epoch = self._epoch
        self._epoch += 1
        node = self._root
        if node.epoch < 0:
            node.witness, node.epoch = handle, epoch
        i = 0
        while i < s.size:
            child = node.children.get(int(s[i]))
            if child is None:
                node.children[int(s[i])] = _Edge(s[i:], handle, epoch)
                return
            common = _lcp(child.label, s[i:])
            if common < child.label.size:
                mid = _Edge(child.label[:common], child.witness, child.epoch)
                child.label = child.label[common:]
                mid.children[int(child.label[0])] = child
                node.children[int(s[i])] = mid
                child = mid
            if child.epoch < 0 or epoch < child.epoch:
                child.witness, child.epoch = handle, epoch
            node = child
            i += common

    def match_prefix(self, seq: Sequence[int]) -> tuple[int, Hashable | None]:
        s = self._arr(seq)
        node, matched, witness, i = self._root, 0, None, 0
        while i < s.size:
            child = node.children.get(int(s[i]))
            if child is None:
                break
            common = _lcp(child.label, s[i:])
            if common > 0:
                matched, witness = i + common, child.witness
            if common < child.label.size:
                break
            node = child
            i += common
        return (matched, witness) if matched else (0, None)


class DeviceRadixTree:
    """K0: the exact-prefix index on the B200 (csrc/prefix.cu) behind the
    RadixTree API (radix.py:31-89): ``insert(seq, handle)``,
    ``match_prefix(seq) -> (m, handle)``, plus the batched forms the serve
    path uses (``run_ops``, ``match_insert``), one launch sequence per batch.

    Every prefix of every inserted sequence is a key of a device hash table
    holding the earliest insert epoch that reaches it; a query is a binary
    search over its own prefix keys, verified token by token against the
    witness's stored tokens. The hash is keyed per index (``hash_key``, drawn
    from os.urandom), and a verification failure (a collision) is answered by
    an exact scan on the device: answers are always the reference tree's.
    ``check()`` raises only on a full table. Inserted sequences are kept in a
    device token arena."""

    def __init__(self, capacity_hint: int | None = None, max_prefixes: int = 1 << 22,
                 max_tokens: int = 1 << 24, max_sequences: int = 1 << 16, grow: bool = True,
                 hash_key: int | None = None):
        """Capacities are initial sizes; with ``grow`` (default) the arena, the
        per-sequence arrays and the table are enlarged when a batch would not
        fit (the table by rebuilding it from the arena, epochs unchanged), so a
        long serve run never hits a limit the reference's tree does not have."""
        import torch

        from . import _native as N
        from . import ops

        self._N, self._torch = N, torch
        dev = ops._dev()
        self.hash_key = int.from_bytes(os.urandom(8), "little") if hash_key is None else int(hash_key)
        self.capacity_hint = capacity_hint
        self.grow = grow
        self.counters = torch.zeros(2, dtype=torch.int64, device=dev)
        self._new_table(max_prefixes)
        self.arena = torch.zeros(max_tokens, dtype=torch.int32, device=dev)
        self.wit_off = torch.zeros(max_sequences, dtype=torch.int64, device=dev)
        self.wit_len = torch.zeros(max_sequences, dtype=torch.int64, device=dev)
        self.used = 0        # arena tokens in use
        self._epoch = 0      # inserts so far (radix.py:34-35)
        self._prefix_bound = 0  # upper bound on stored prefixes (inserted tokens since the last count)
        self.handles: list = []
        self._ws = None

    def _new_table(self, max_prefixes: int):
        torch, N = self._torch, self._N
        n_slots = 2
        while n_slots < 2 * max_prefixes:
            n_slots <<= 1
        dev = self.counters.device
        self.n_slots = n_slots
        self.slots = torch.empty(2 * n_slots, dtype=torch.int64, device=dev)  # (key, epoch) pairs
        self.view = N.PrefixView(N.ptr(self.slots), n_slots, N.ptr(self.counters),
                                 self.hash_key & (2**64 - 1))
        N.check(N.lib().irm_prefix_reset(self.view, N.stream_ptr()), "irm_prefix_reset")

    def _reserve(self, n_tok: int, n_ins: int, ins_tok: int):
        """Make room for a batch of n_tok tokens with n_ins inserts (ins_tok of their tokens)."""
        torch = self._torch
        if self.used + n_tok > self.arena.numel():
            if not self.grow:
                raise ValueError("prefix index token arena is full: raise max_tokens")
            new = torch.zeros(max(2 * self.arena.numel(), self.used + n_tok), dtype=torch.int32,
                              device=self.arena.device)
            new[:self.used].copy_(self.arena[:self.used])
            self.arena = new
        if self._epoch + n_ins > self.wit_off.numel():
            if not self.grow:
                raise ValueError("prefix index holds max_sequences inserts: raise max_sequences")
            cap = max(2 * self.wit_off.numel(), self._epoch + n_ins)
            for name in ("wit_off", "wit_len"):
                old = getattr(self, name)
                new = torch.zeros(cap, dtype=torch.int64, device=old.device)
                new[:self._epoch].copy_(old[:self._epoch])
                setattr(self, name, new)
        half = self.n_slots // 2
        if self.grow and self._prefix_bound + ins_tok > half:
            self.check()
            used = int(self.counters[0])  # the real count (one sync, only near the load limit)
            self._prefix_bound = used
            if used + ins_tok > half:
                self._rehash(used + ins_tok)

    def _rehash(self, need: int):
        """Rebuild the table 2x larger from the stored sequences, with their epochs."""
        torch, N = self._torch, self._N
        self.counters.zero_()
        self._new_table(max(2 * need, self.n_slots))
        n = self._epoch
        if n == 0:
            return
        off, ln = self.wit_off[:n], self.wit_len[:n]
        seq_off = torch.zeros(n + 1, dtype=torch.int64, device=off.device)
        seq_off[1:] = torch.cumsum(ln, 0)
        total = int(seq_off[-1])
        idx = torch.repeat_interleave(off - seq_off[:-1], ln) + torch.arange(total, device=off.device)
        tok = self.arena[idx].contiguous()  # every inserted sequence, compacted
        epoch = torch.arange(n, dtype=torch.int64, device=off.device)
        ones = torch.ones(n, dtype=torch.uint8, device=off.device)
        m = torch.empty(n, dtype=torch.int64, device=off.device)
        wit = torch.empty_like(m)
        ws = self._workspace(total, n)
        rc = N.lib().irm_prefix_match_insert(
            self.view, N.ptr(tok), N.ptr(seq_off), n, total, N.ptr(epoch), N.ptr(ones), N.ptr(torch.zeros_like(ones)),
            N.ptr(self.arena), N.ptr(self.wit_off), N.ptr(self.wit_len), N.ptr(m), N.ptr(wit), N.ptr(ws),
            ws.numel(), N.stream_ptr())
        N.check(rc, "irm_prefix_match_insert (rehash)")
        self._prefix_bound = total

    def _workspace(self, n_tok, n_seq):
        need = int(self._N.lib().irm_prefix_workspace_bytes(n_tok, n_seq))
        if self._ws is None or self._ws.numel() < need:
            self._ws = self._torch.empty(max(need, 256), dtype=self._torch.uint8, device=self.arena.device)
        return self._ws

    def run_ops(self, seqs, insert, query, handles=None):
        """A batch of operations in order. ``seqs``: list of token sequences;
        ``insert[i]`` / ``query[i]``: booleans. Returns device tensors
        (m, witness epoch); a query sees every insert before it in the batch
        and before the batch. ``handles[i]`` names inserted sequence i."""
        torch, N = self._torch, self._N
        arrs = [np.asarray(s, dtype=np.uint64).astype(np.uint32) if not isinstance(s, np.ndarray)
                else s.astype(np.uint32, copy=False) for s in seqs]
        n = len(arrs)
        lens = np.array([a.size for a in arrs], np.int64)
        off = np.zeros(n + 1, np.int64)
        np.cumsum(lens, out=off[1:])
        n_tok = int(off[-1])
        ins = np.asarray(insert, bool)
        qry = np.asarray(query, bool)
        n_ins = int(ins.sum())
        ins_tok = int(lens[ins].sum()) if n else 0
        self._reserve(n_tok, n_ins, ins_tok)
        before = np.cumsum(ins) - ins  # inserts earlier in the batch
        # an insert's epoch is its insert index; a query's bound is the number of inserts before it
        epoch = (self._epoch + before).astype(np.int64)
        dev = self.arena.device
        base = self.used
        if n_tok:
            flat = np.concatenate(arrs).view(np.int32)
            self.arena[base:base + n_tok].copy_(torch.from_numpy(flat), non_blocking=False)
        ep_ins = epoch[ins]
        if n_ins:
            self.wit_off[self._epoch:self._epoch + n_ins].copy_(torch.from_numpy(base + off[:-1][ins]))
            self.wit_len[self._epoch:self._epoch + n_ins].copy_(torch.from_numpy(lens[ins]))
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        seq_off, op_epoch = d(off), d(epoch)
        op_ins, op_q = d(ins.astype(np.uint8)), d(qry.astype(np.uint8))
        m = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        wit = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        ws = self._workspace(n_tok, n)
        rc = N.lib().irm_prefix_match_insert(
            self.view, N.ptr(self.arena[base:]) if base < self.arena.numel() else None, N.ptr(seq_off), n,
            n_tok, N.ptr(op_epoch), N.ptr(op_ins), N.ptr(op_q), N.ptr(self.arena), N.ptr(self.wit_off),
            N.ptr(self.wit_len), N.ptr(m), N.ptr(wit), N.ptr(ws), ws.numel(), N.stream_ptr())
        N.check(rc, "irm_prefix_match_insert")
        self.used += n_tok
        self._epoch += n_ins
        self._prefix_bound += ins_tok
        hs = list(handles) if handles is not None else [None] * n
        self.handles += [hs[i] for i in range(n) if ins[i]]
        return m[:n], wit[:n]

    def match_insert(self, seqs, handles):
        """Each sequence is matched against everything inserted before it, then
        inserted (engine.py:170 then :228). Returns host lists (m, witness handle)."""
        n = len(seqs)
        m, wit = self.run_ops(seqs, [True] * n, [True] * n, handles)
        self.check()
        mh, wh = m.cpu().tolist(), wit.cpu().tolist()
        return mh, [self.handles[w] if w >= 0 else None for w in wh]

    def insert(self, seq: Sequence[int], handle: Hashable) -> None:
        self.run_ops([seq], [True], [False], [handle])

    def match_prefix(self, seq: Sequence[int]) -> tuple[int, Hashable | None]:
        m, wit = self.run_ops([seq], [False], [True])
        self.check()
        mm, w = int(m[0]), int(wit[0])
        return (mm, self.handles[w]) if mm else (0, None)

    def check(self):
        flags = int(self.counters[1])
        if flags & 1:
            raise RuntimeError("device prefix index table is full: raise max_prefixes")

    @property
    def collisions_resolved(self) -> bool:
        """True once some query met a hash collision (answered by the exact scan)."""
        return bool(int(self.counters[1]) & 4)

    @property
    def n_prefixes(self) -> int:
        return int(self.counters[0])


class WavePrefixIndex:
    """Phase 1 of the warm-serve step as device work a CUDA graph can capture
    (engine.py:170, 228: every request is matched against everything inserted
    before it -- earlier waves and earlier requests of its own wave -- then
    inserted). The K0 table, token arena and epoch arrays of DeviceRadixTree,
    but with the arena fill level and the next insert epoch as DEVICE counters
    (``irm_prefix_wave_prepare``), so a wave needs no host round trip. Sized
    once; a wave that would overflow is skipped and flagged (``check()``).
    Answers are exact (keyed hash, verified, collisions rescanned)."""

    def __init__(self, max_prefixes: int, arena_tokens: int, max_sequences: int, hash_key: int | None = None):
        import torch

        from . import _native as N
        from . import ops

        self._N, self._torch = N, torch
        dev = ops._dev()
        self.hash_key = int.from_bytes(os.urandom(8), "little") if hash_key is None else int(hash_key)
        n_slots = 2
        while n_slots < 2 * max_prefixes:
            n_slots <<= 1
        self.counters = torch.zeros(2, dtype=torch.int64, device=dev)
        self.n_slots = n_slots
        self.slots = torch.empty(2 * n_slots, dtype=torch.int64, device=dev)  # (key, epoch) pairs
        self.view = N.PrefixView(N.ptr(self.slots), n_slots, N.ptr(self.counters),
                                 self.hash_key & (2**64 - 1))
        N.check(N.lib().irm_prefix_reset(self.view, N.stream_ptr()), "irm_prefix_reset")
        self.arena = torch.zeros(arena_tokens, dtype=torch.int32, device=dev)
        self.wit_off = torch.zeros(max_sequences, dtype=torch.int64, device=dev)
        self.wit_len = torch.zeros(max_sequences, dtype=torch.int64, device=dev)
        self.arena_used = torch.zeros(1, dtype=torch.int64, device=dev)
        self.epoch_next = torch.zeros(1, dtype=torch.int64, device=dev)
        self._ws = None
        self._bufs = {}

    def match_insert_wave(self, tok, seq_off, n_seq: int, m_out, wit_out=None) -> None:
        """tok: int32 [cap] (the wave's requests, CSR ``seq_off`` [n_seq + 1], both on
        the device); m_out int64 [n_seq] <- each request's longest prefix shared with
        an earlier request; then every request is inserted. No host synchronisation."""
        torch, N = self._torch, self._N
        cap = tok.numel()
        key = (cap, n_seq)
        if key not in self._bufs:  # static per shape: a captured graph keeps the addresses
            need = int(N.lib().irm_prefix_workspace_bytes(cap, n_seq))
            self._bufs[key] = (torch.empty(max(need, 256), dtype=torch.uint8, device=tok.device),
                               torch.empty(n_seq, dtype=torch.int64, device=tok.device),
                               torch.ones(n_seq, dtype=torch.uint8, device=tok.device),
                               torch.empty(n_seq, dtype=torch.int64, device=tok.device))
        ws, op_epoch, ones, wit = self._bufs[key]
        wit = wit if wit_out is None else wit_out
        L = N.lib()
        N.check(L.irm_prefix_wave_prepare(self.view, N.ptr(self.arena), self.arena.numel(), N.ptr(self.arena_used),
                                          N.ptr(self.wit_off), N.ptr(self.wit_len), self.wit_off.numel(),
                                          N.ptr(self.epoch_next), N.ptr(tok), N.ptr(seq_off), n_seq, N.ptr(op_epoch),
                                          N.stream_ptr()), "irm_prefix_wave_prepare")
        N.check(L.irm_prefix_match_insert(self.view, N.ptr(tok), N.ptr(seq_off), n_seq, cap, N.ptr(op_epoch),
                                          N.ptr(ones), None, N.ptr(self.arena), N.ptr(self.wit_off),
                                          N.ptr(self.wit_len), N.ptr(m_out), N.ptr(wit), N.ptr(ws), ws.numel(),
                                          N.stream_ptr()), "irm_prefix_match_insert")

    def check(self):
        if int(self.counters[1]) & 1:
            raise RuntimeError("wave prefix index full (table, token arena or epochs): raise its capacities")
