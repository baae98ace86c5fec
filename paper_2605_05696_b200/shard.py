"""K6: the hash-sharded chunk store across the GPUs of one box.

Sessions are data-parallel (session s on rank s mod G). The content store is
sharded by fingerprint prefix: the owner of fp is ``(fp >> 32) * G >> 32``,
which equals ``fp >> (64 - log2 G)`` for a power-of-two G. A lookup wave is one
exchange over ``torch.distributed`` (NCCL over NVLink on B200, gloo in the CPU
tests):

  1. all-to-all of per-owner query counts
  2. all-to-all of the queries (fp, order key, p, len, row hint)
  3. the owner sorts what it received by the global order key (request,
     chunk) and runs the first-writer-wins batch on its shard (K3), so the
     winner is the globally earliest query, exactly as the sequential
     reference (engine.py:197-223)
  4. reverse all-to-all of (hit, p_src, row) to the asking rank

Rows are named globally: ``row = rank << 40 | local_row``. A hit whose rows
live on another rank is fetched once into this rank's replica pool
(``ReplicaCache``), so the rotate+gather (K4) always reads local HBM.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

ROW_SHIFT = 40
ROW_MASK = (1 << ROW_SHIFT) - 1


def owner_of(fp: torch.Tensor, world: int) -> torch.Tensor:
    """Fingerprint-prefix owner rank (fp carried as int64 bits)."""
    hi = (fp >> 32) & 0xFFFFFFFF  # top 32 bits as a non-negative int64
    return ((hi * world) >> 32).to(torch.int64)


def encode_row(rank: int, row: torch.Tensor) -> torch.Tensor:
    return (torch.as_tensor(rank, dtype=torch.int64) << ROW_SHIFT) | row.to(torch.int64)


def decode_row(grow: torch.Tensor):
    return grow >> ROW_SHIFT, grow & ROW_MASK


def _a2a(output: torch.Tensor, inp: torch.Tensor, out_splits, in_splits, group):
    dist.all_to_all_single(output, inp, out_splits, in_splits, group=group)


class ShardedStore:
    """Wraps a local store shard (``ops.ChunkStore`` on GPU; any object with
    the same ``lookup_insert`` contract, e.g. a test dict store on CPU)."""

    def __init__(self, local_store, group=None):
        self.local = local_store
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.last_exchange_bytes = 0

    def lookup_insert(self, q_fp, q_order, q_p, q_len, q_probe=None, q_row_hint=None):
        """Same contract as ops.ChunkStore.lookup_insert, over the sharded store.

        q_order must be globally unique (e.g. (global request << 20) | chunk).
        q_row_hint: global row (encode_row) where this rank keeps the chunk's
        KV if it is the first writer. Returns (hit, p_src, row, owner)."""
        dev = q_fp.device
        n = q_fp.numel()
        probe = torch.ones(n, dtype=torch.bool, device=dev) if q_probe is None else q_probe.to(torch.bool)
        if q_row_hint is None:
            q_row_hint = torch.full((n,), -1, dtype=torch.int64, device=dev)
        sel = torch.nonzero(probe).flatten()
        own = owner_of(q_fp[sel], self.world)
        perm = torch.argsort(own, stable=True)
        sel = sel[perm]
        own = own[perm]
        send = torch.stack([q_fp[sel], q_order[sel], q_p[sel].to(torch.int64), q_len[sel].to(torch.int64),
                            q_row_hint[sel]], dim=1).contiguous()
        counts = torch.bincount(own, minlength=self.world).to(torch.int64)
        recv_counts = torch.empty_like(counts)
        dist.all_to_all_single(recv_counts, counts, group=self.group)
        in_splits = counts.cpu().tolist()
        out_splits = recv_counts.cpu().tolist()
        recv = torch.empty(sum(out_splits), 5, dtype=torch.int64, device=dev)
        _a2a(recv, send, out_splits, in_splits, self.group)

        # owner side: the global first writer is the smallest order key
        o = torch.argsort(recv[:, 1])
        r = recv[o]
        hit, entry, p_src, _row = self.local.lookup_insert(
            r[:, 0].contiguous(), r[:, 1].contiguous(), r[:, 2].contiguous(), r[:, 3].to(torch.int32).contiguous())
        novel = hit == 0
        # the new entry's rows are the winner's (row hint); hits read the entry's row
        e_row = self.local.e_row
        e_row[entry[novel]] = r[novel, 4]
        rows = e_row[entry.clamp_min(0)]
        reply_sorted = torch.stack([hit.to(torch.int64), p_src, rows], dim=1)
        reply = torch.empty_like(reply_sorted)
        reply[o] = reply_sorted
        back = torch.empty(len(sel), 3, dtype=torch.int64, device=dev)
        _a2a(back, reply.contiguous(), in_splits, out_splits, self.group)
        self.last_exchange_bytes = 8 * (5 * (sum(in_splits) + sum(out_splits)) + 3 * (sum(in_splits) + sum(out_splits)))

        out_hit = torch.full((n,), -1, dtype=torch.int32, device=dev)
        out_psrc = torch.zeros(n, dtype=torch.int64, device=dev)
        out_row = torch.full((n,), -1, dtype=torch.int64, device=dev)
        out_owner = torch.full((n,), -1, dtype=torch.int64, device=dev)
        out_hit[sel] = back[:, 0].to(torch.int32)
        out_psrc[sel] = back[:, 1]
        out_row[sel] = back[:, 2]
        out_owner[sel] = own
        return out_hit, out_psrc, out_row, out_owner


class ReplicaCache:
    """Per-rank replica of remote latent rows, keyed by global row.

    ``pool`` is this rank's latent pool [layers, rows, width]; the replica
    region starts at ``replica_base`` and grows. ``localize`` turns global
    rows (encode_row) of hit chunks into local rows, fetching every missing
    remote run once via one all-to-all of row requests and one of row data."""

    def __init__(self, pool: torch.Tensor, replica_base: int, group=None):
        self.pool = pool
        self.base = replica_base
        self.next = replica_base
        self.map: dict[int, int] = {}  # global row of a run start -> local row
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.fetched_rows = 0

    def localize(self, grow: torch.Tensor, length: torch.Tensor) -> torch.Tensor:
        """grow [n] global rows (or -1), length [n] -> local rows (int64)."""
        dev = grow.device
        need: list[list[tuple[int, int]]] = [[] for _ in range(self.world)]
        gt = grow.to(torch.int64)
        remote = (gt >= 0) & ((gt >> ROW_SHIFT) != self.rank)
        if bool(remote.any()):
            uniq, inv = torch.unique(gt[remote], return_inverse=True)
            first = torch.full((uniq.numel(),), -1, dtype=torch.int64, device=dev)
            first.scatter_reduce_(0, inv, length.to(torch.int64)[remote], reduce="amax", include_self=False)
            for gr, l in zip(uniq.cpu().tolist(), first.cpu().tolist()):
                if gr not in self.map:
                    need[gr >> ROW_SHIFT].append((gr & ROW_MASK, l))
        # 1. request counts and (row, len) requests
        counts = torch.tensor([len(x) for x in need], dtype=torch.int64, device=dev)
        recv_counts = torch.empty_like(counts)
        dist.all_to_all_single(recv_counts, counts, group=self.group)
        in_splits, out_splits = counts.cpu().tolist(), recv_counts.cpu().tolist()
        req = torch.tensor([x for lst in need for x in lst], dtype=torch.int64, device=dev).reshape(-1, 2)
        got = torch.empty(sum(out_splits), 2, dtype=torch.int64, device=dev)
        _a2a(got, req, out_splits, in_splits, self.group)
        # 2. serve: gather the requested runs of my pool, row-major [rows, layers, width]
        L, _, W = self.pool.shape
        g_rows = got[:, 0].cpu().tolist()
        g_len = got[:, 1].cpu().tolist()
        send_rows_per_peer = []
        pieces = []
        pos = 0
        for peer in range(self.world):
            cnt = 0
            for i in range(pos, pos + out_splits[peer]):
                pieces.append(self.pool[:, g_rows[i]:g_rows[i] + g_len[i]].transpose(0, 1))
                cnt += g_len[i]
            pos += out_splits[peer]
            send_rows_per_peer.append(cnt)
        send = (torch.cat(pieces) if pieces else torch.empty(0, L, W, dtype=self.pool.dtype, device=dev)).contiguous()
        # 3. row counts back, then the rows
        send_counts = torch.tensor(send_rows_per_peer, dtype=torch.int64, device=dev)
        recv_rows = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_rows, send_counts, group=self.group)
        rr = recv_rows.cpu().tolist()
        data = torch.empty(sum(rr), L, W, dtype=self.pool.dtype, device=dev)
        _a2a(data, send, rr, send_rows_per_peer, self.group)
        # 4. install replicas (requests were issued owner-major, in `need` order)
        total = int(sum(rr))
        if self.next + total > self.pool.shape[1]:
            raise RuntimeError("replica region of the pool is full")
        if total:
            self.pool[:, self.next:self.next + total] = data.transpose(0, 1)
        off = self.next
        for rk in range(self.world):
            for row, l in need[rk]:
                self.map[(rk << ROW_SHIFT) | row] = off
                off += l
        self.next += total
        self.fetched_rows += total
        # 5. map every hit to a local row (vectorised: own rows pass through, remote run
        #    starts are translated with one searchsorted over the replica map)
        gt = grow.to(torch.int64)
        out = torch.where((gt >> ROW_SHIFT) == self.rank, gt & ROW_MASK, torch.zeros_like(gt))
        remote = (gt >= 0) & ((gt >> ROW_SHIFT) != self.rank)
        if bool(remote.any()):
            keys = torch.tensor(sorted(self.map), dtype=torch.int64, device=dev)
            vals = torch.tensor([self.map[k] for k in sorted(self.map)], dtype=torch.int64, device=dev)
            pos = torch.searchsorted(keys, gt[remote]).clamp_max(keys.numel() - 1)
            out[remote] = vals[pos]
        return out
