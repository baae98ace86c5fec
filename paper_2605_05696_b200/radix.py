"""Exact-prefix index for phase 1 of the serve path (reference radix.py).

Host-side and pointer-chasing by nature (kept off the GPU; a
batched device prefix index is §8(f) item 1). Edges reference slices of the
inserted sequences (numpy views, no copies) and common-prefix lengths are
computed with vectorised compares, so a 32K-token match is a handful of
numpy calls instead of a per-token Python loop. Semantics follow
radix.py:31-89: longest match, earliest-inserted witness.
"""

from __future__ import annotations

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
