"""K6: the hash-sharded chunk store across the GPUs of one box.

Sessions are data-parallel (session s on rank s mod G). The content store is
sharded by fingerprint prefix: the owner of fp is ``(fp >> 32) * G >> 32``,
which equals ``fp >> (64 - log2 G)`` for a power-of-two G. A lookup wave is one
exchange over ``torch.distributed`` (NCCL over NVLink on B200, gloo in the CPU
tests), with fixed-capacity buffers so nothing on the path waits for the host:

  1. every probed query goes to slot (owner, position in the owner's bucket)
     of a [G, cap, 4] send buffer (fp, order key, p, len); unused
     slots carry padding order keys that sort after every real key. ``cap``
     is a per-owner bound (fingerprints are uniform, so an owner receives
     ~1/G of a wave: 1.25/G of the wave's capacity + 64 slots); a bucket that
     would overflow sets a sticky flag that ``check()`` raises on
  2. all-to-all of equal splits
  3. the owner sorts what it received by the global order key (request,
     chunk) and runs the first-writer-wins batch on its shard (K3), so the
     winner is the globally earliest query, exactly as the sequential
     reference (engine.py:197-223); a new entry's rows are allocated by the
     owner in its sub-range of the first writer's pool
  4. reverse all-to-all of (hit, p_src, row, fresh) into the same slots;
     fresh = the entry was created by this very exchange (its KV is written
     by the first writer's prefill of this wave, not yet)

Rows are named globally: ``row = rank << 40 | local_row``. A hit whose rows
live on another rank is fetched once into this rank's replica region of its
pool (``ReplicaCache``): the peer pools are mapped into every process (CUDA
IPC over NVLink), a second store keyed by the global row dedupes runs and
assigns replica rows, and ``irm_copy_runs`` pulls the rows peer-to-peer. K4
then always reads local HBM. A hit on an entry created in the same exchange
(``fresh``) is fetched into a per-wave scratch region and never cached: the
writer has not produced those rows yet, so a cached copy would stay stale.
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

ROW_SHIFT = 40
ROW_MASK = (1 << ROW_SHIFT) - 1
PAD_ORDER = 1 << 62  # order keys of padding slots: above every (request << 20 | chunk) key


def owner_of(fp: torch.Tensor, world: int) -> torch.Tensor:
    """Fingerprint-prefix owner rank (fp carried as int64 bits)."""
    hi = (fp >> 32) & 0xFFFFFFFF  # top 32 bits as a non-negative int64
    return ((hi * world) >> 32).to(torch.int64)


def encode_row(rank: int, row: torch.Tensor) -> torch.Tensor:
    return (torch.as_tensor(rank, dtype=torch.int64) << ROW_SHIFT) | row.to(torch.int64)


def decode_row(grow: torch.Tensor):
    return grow >> ROW_SHIFT, grow & ROW_MASK


class ShardedStore:
    """Wraps a local store shard (``ops.ChunkStore`` on GPU; any object with
    the same ``lookup_insert`` contract and an ``e_row`` entry array, e.g. a
    test dict store on CPU)."""

    def __init__(self, local_store, novel_rows: int, group=None, slots: int | None = None,
                 owner_slots: int | None = None):
        """novel_rows: rows [0, novel_rows) of every rank's latent pool hold the
        KV of chunks that rank writes first. Owner o hands out rows of the
        sub-range [o * novel_rows // G, (o + 1) * novel_rows // G) of each
        writer's pool, with one bump counter per writer, so a first writer's
        rows are known in the same exchange that decides it is first.
        slots: the most queries one call may carry; it must be the same on every
        rank (the all-to-all has equal splits). None: the size of each call's
        query array, which then must match across ranks. owner_slots: queries
        per (rank, owner) bucket (default: 1.25 x slots / G + 64, at most slots);
        an overflowing bucket raises in ``check()``."""
        self.local = local_store
        self.group = group
        self.slots = slots
        self.owner_slots = owner_slots
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        e_row = local_store.e_row
        dev = e_row.device
        # global row of every entry of this shard (+1: scatter sink for non-novel queries)
        self.e_grow = torch.full((e_row.numel() + 1,), -1, dtype=torch.int64, device=dev)
        self.region = novel_rows // self.world
        self.base = self.rank * self.region
        self.next = torch.zeros(self.world, dtype=torch.int64, device=dev)  # per-writer bump counters
        self.overflow = torch.zeros((), dtype=torch.bool, device=dev)
        self.bucket_overflow = torch.zeros((), dtype=torch.bool, device=dev)
        self.flags = torch.zeros(1, dtype=torch.int64, device=dev)  # device path: 1 bucket full, 2 rows full
        self.last_exchange_bytes = 0
        self.fresh = None  # per query of the last call: hit on an entry this exchange created

    def lookup_insert(self, q_fp, q_order, q_p, q_len, q_probe=None):
        """Same contract as ops.ChunkStore.lookup_insert, over the sharded store.

        q_order must be globally unique and < 2^62 (e.g. (global request << 20) |
        chunk). Returns (hit, p_src, row, owner); row is the global row
        (encode_row) of the entry's KV: for a novel query, where this rank must
        keep the chunk's KV (a row of its own pool, assigned by the owner).
        No host synchronisation: every buffer has a fixed capacity of ``slots``
        (default q_fp.numel()) queries per owner."""
        dev = q_fp.device
        n, G = q_fp.numel(), self.world
        i64 = dict(dtype=torch.int64, device=dev)
        total = self.slots if self.slots is not None else max(n, 1)
        if n > total:
            raise ValueError(f"{n} queries exceed the exchange's {total} slots")
        cap = self.owner_slots or (total if G == 1 else min(total, (5 * total) // (4 * G) + 64))
        if q_fp.is_cuda:
            return self._lookup_insert_device(q_fp, q_order, q_p, q_len, q_probe, cap)
        # CPU tensors (the gloo tests): the same exchange in torch ops
        probe = torch.ones(n, dtype=torch.bool, device=dev) if q_probe is None else q_probe.to(torch.bool)
        own = torch.where(probe, owner_of(q_fp, G), torch.full_like(q_fp, G))  # bucket G: not probed
        perm = torch.argsort(own, stable=True)
        own_s = own[perm]
        counts = torch.zeros(G + 1, **i64).scatter_add_(0, own, torch.ones(n, **i64))
        start = torch.cumsum(counts, 0) - counts
        pos = torch.arange(n, **i64) - start[own_s]
        self.bucket_overflow |= (counts[:G] > cap).any()  # sticky; check() raises
        valid = (own_s < G) & (pos < cap)
        dest = torch.where(valid, own_s * cap + pos, G * cap)
        send = torch.zeros(G * cap + 1, 4, **i64)  # last row: sink for unprobed queries
        send[:, 1] = PAD_ORDER + self.rank * G * cap + torch.arange(G * cap + 1, **i64)  # unique padding keys
        send.index_copy_(0, dest, torch.stack([q_fp, q_order, q_p.to(torch.int64), q_len.to(torch.int64)],
                                              dim=1)[perm])
        send = send[:G * cap].contiguous()
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=self.group)

        # owner side: the global first writer is the smallest order key (padding sorts last)
        o = torch.argsort(recv[:, 1])
        r = recv[o]
        real = r[:, 1] < PAD_ORDER
        n_before = self._entry_count()  # entries of this shard before the exchange (device)
        hit, entry, p_src, _row = self.local.lookup_insert(
            r[:, 0].contiguous(), r[:, 1].contiguous(), r[:, 2].contiguous(), r[:, 3].to(torch.int32).contiguous(),
            real)
        novel = hit == 0
        # the first writer keeps the new entry's KV: rows of this owner's sub-range of the
        # writer's pool, bump-allocated per writer in slot (= the writer's query) order
        nov_slot = torch.zeros(G * cap, dtype=torch.bool, device=dev).index_copy_(0, o, novel)
        L = torch.where(nov_slot, recv[:, 3], torch.zeros_like(recv[:, 3])).view(G, cap)
        lrow = self.base + self.next[:, None] + torch.cumsum(L, 1) - L
        self.next += L.sum(1)
        self.overflow |= (self.next > self.region).any()
        grow = ((torch.arange(G, **i64)[:, None] << ROW_SHIFT) | lrow).view(-1)[o]
        sink = self.e_grow.numel() - 1
        # each entry has exactly one novel query
        self.e_grow.index_copy_(0, torch.where(novel, entry, torch.full_like(entry, sink)), grow)
        rows = torch.where(entry >= 0, self.e_grow[entry.clamp_min(0)], torch.full_like(entry, -1))
        fresh = ((hit == 1) & (entry >= n_before)).to(torch.int64)
        reply = torch.empty(G * cap, 4, **i64)
        reply.index_copy_(0, o, torch.stack([hit.to(torch.int64), p_src.to(torch.int64), rows, fresh], dim=1))
        back = torch.empty_like(reply)
        dist.all_to_all_single(back, reply, group=self.group)
        self.last_exchange_bytes = 2 * G * cap * (4 + 4) * 8

        res = back[torch.where(valid, dest, torch.zeros_like(dest))]  # sorted position k -> its slot
        out_hit = torch.full((n,), -1, dtype=torch.int32, device=dev)
        out_psrc = torch.zeros(n, **i64)
        out_row = torch.full((n,), -1, **i64)
        out_owner = torch.full((n,), -1, **i64)
        out_hit.index_copy_(0, perm, torch.where(valid, res[:, 0], -1).to(torch.int32))
        out_psrc.index_copy_(0, perm, torch.where(valid, res[:, 1], 0))
        out_row.index_copy_(0, perm, torch.where(valid, res[:, 2], -1))
        out_owner.index_copy_(0, perm, torch.where(valid, own_s, -1))
        out_fresh = torch.zeros(n, dtype=torch.bool, device=dev)
        out_fresh.index_copy_(0, perm, valid & (res[:, 3] == 1))
        self.fresh = out_fresh
        return out_hit, out_psrc, out_row, out_owner

    def _lookup_insert_device(self, q_fp, q_order, q_p, q_len, q_probe, cap):
        """The exchange on the GPU: four native launches (irm_exchange_*) around K3 and
        the two all-to-alls, no host synchronisation (captured whole into the
        pipeline's CUDA graphs)."""
        from . import _native as N

        L, st = N.lib(), N.stream_ptr()
        dev, n, G = q_fp.device, q_fp.numel(), self.world
        m = G * cap
        i64 = dict(dtype=torch.int64, device=dev)
        q_fp, q_order = q_fp.contiguous(), q_order.to(torch.int64).contiguous()
        q_p, q_len = q_p.to(torch.int64).contiguous(), q_len.to(torch.int32).contiguous()
        probe = q_probe.to(torch.uint8).contiguous() if q_probe is not None else None
        send = torch.empty(m, 4, **i64)
        dest = torch.empty(n, **i64)
        N.check(L.irm_exchange_pack(N.ptr(q_fp), N.ptr(q_order), N.ptr(q_p), N.ptr(q_len), N.ptr(probe), n, G,
                                    self.rank, cap, N.ptr(send), N.ptr(dest), N.ptr(self.flags), st),
                "irm_exchange_pack")
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=self.group)
        r_fp, r_order, r_p = torch.empty(m, **i64), torch.empty(m, **i64), torch.empty(m, **i64)
        r_len = torch.empty(m, dtype=torch.int32, device=dev)
        r_real = torch.empty(m, dtype=torch.uint8, device=dev)
        N.check(L.irm_exchange_split(N.ptr(recv), m, N.ptr(r_fp), N.ptr(r_order), N.ptr(r_p), N.ptr(r_len),
                                     N.ptr(r_real), st), "irm_exchange_split")
        n_before = self._entry_count()  # entries of this shard before the exchange (device)
        hit, entry, p_src, _row = self.local.lookup_insert(r_fp, r_order, r_p, r_len, r_real)
        reply = torch.empty(m, 4, **i64)
        N.check(L.irm_exchange_reply(N.ptr(recv), G, cap, N.ptr(hit), N.ptr(entry), N.ptr(p_src), N.ptr(n_before),
                                     self.base, self.region, N.ptr(self.next), N.ptr(self.e_grow),
                                     self.e_grow.numel() - 1, N.ptr(self.flags), N.ptr(reply), st),
                "irm_exchange_reply")
        back = torch.empty_like(reply)
        dist.all_to_all_single(back, reply, group=self.group)
        self.last_exchange_bytes = 2 * m * 4 * 8
        out_hit = torch.empty(n, dtype=torch.int32, device=dev)
        out_psrc, out_row, out_owner = torch.empty(n, **i64), torch.empty(n, **i64), torch.empty(n, **i64)
        fresh = torch.empty(n, dtype=torch.uint8, device=dev)
        N.check(L.irm_exchange_unpack(N.ptr(back), N.ptr(dest), n, cap, N.ptr(out_hit), N.ptr(out_psrc),
                                      N.ptr(out_row), N.ptr(out_owner), N.ptr(fresh), st), "irm_exchange_unpack")
        self.fresh = fresh.view(torch.bool)
        return out_hit, out_psrc, out_row, out_owner

    def _entry_count(self) -> torch.Tensor:
        c = getattr(self.local, "counters", None)
        if c is not None:
            return c[0].clone()
        return torch.tensor(len(getattr(self.local, "map", ())), dtype=torch.int64)

    def check(self):
        """Host check (call outside timed regions): every first writer got its rows and no
        owner bucket of the exchange overflowed."""
        f = int(self.flags[0])
        if bool(self.overflow) or f & 2:
            raise RuntimeError("first-writer row range of the pool is full: raise novel_rows")
        if bool(self.bucket_overflow) or f & 1:
            raise RuntimeError("an owner bucket of the lookup exchange overflowed: raise owner_slots")


class _PeerMapping:
    """A peer allocation mapped into this process, exposed to torch through the
    CUDA array interface (no copy; the mapping lives until the process exits)."""

    def __init__(self, addr: int, shape, itemsize: int):
        self.__cuda_array_interface__ = {"data": (addr, False), "shape": tuple(shape),
                                         "typestr": f"<i{itemsize}", "strides": None, "version": 2}


def map_peer_pools(pool: torch.Tensor, group=None) -> list[torch.Tensor]:
    """Every rank's latent pool, mapped into this process. Index = rank.

    Each rank exports its pool's allocation (``irm_peer_export``: CUDA IPC handle
    + offset) and every other rank maps it on ITS OWN device
    (``irm_peer_open``, peer access over NVLink enabled lazily), so K6's
    ``irm_copy_runs`` on this rank's GPU reads the peer's HBM directly."""
    from . import _native as N

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if world == 1:
        return [pool]
    assert pool.is_cuda and pool.is_contiguous()
    L = N.lib()
    handle = ctypes.create_string_buffer(N.PEER_HANDLE_BYTES)
    offset = ctypes.c_int64(0)
    N.check(L.irm_peer_export(ctypes.c_void_p(pool.data_ptr()), handle, ctypes.byref(offset)), "irm_peer_export")
    objs = [None] * world
    dist.all_gather_object(objs, (handle.raw, offset.value, tuple(pool.shape)), group=group)
    out = []
    with torch.cuda.device(pool.device):
        for r, (h, off, shape) in enumerate(objs):
            if r == rank:
                out.append(pool)
                continue
            assert tuple(shape) == tuple(pool.shape), "peer pools must have the same shape"
            addr = ctypes.c_void_p(0)
            N.check(L.irm_peer_open(ctypes.create_string_buffer(h, len(h)), int(off), ctypes.byref(addr)),
                    "irm_peer_open")
            item = pool.element_size()
            t = torch.as_tensor(_PeerMapping(addr.value, shape, item))
            out.append(t.view(pool.dtype))
    return out


class ReplicaCache:
    """Per-rank replica of remote latent rows, keyed by global row.

    ``pool`` is this rank's latent pool [layers, rows, width]; the replica
    region starts at ``replica_base``. ``peer_pools[r]`` is rank r's pool as
    seen from this process (``map_peer_pools``; same shape on every rank).
    ``map_store`` is a first-writer-wins store (``ops.ChunkStore``) keyed by the
    global row of a run start: a novel key allocates replica rows by the
    store's exclusive scan of run lengths, which is exactly a bump allocator
    that dedupes runs within and across waves."""

    def __init__(self, pool: torch.Tensor, replica_base: int, peer_pools: list[torch.Tensor], rank: int,
                 map_store, scratch_rows: int | None = None):
        """scratch_rows: the last 2 x scratch_rows rows of the pool are a double-buffered
        per-wave scratch for fresh remote hits (rows their writer has not produced yet:
        fetched for this wave, never cached; default: 1/8 of the replica region per
        half). The replica region is [replica_base, pool rows - 2 x scratch_rows)."""
        if scratch_rows is None:
            scratch_rows = max(pool.shape[1] - replica_base, 0) // 8
        self.pool, self.base, self.peers, self.rank, self.map = pool, replica_base, peer_pools, rank, map_store
        self.scratch_rows = scratch_rows
        self.scratch_base = pool.shape[1] - 2 * scratch_rows
        self.limit = self.scratch_base  # replica rows end here
        self._half = 0
        for pp in peer_pools:
            assert pp.shape == pool.shape and pp.dtype == pool.dtype and pp.is_contiguous()
        dev = pool.device
        self.row_bytes = pool.shape[2] * pool.element_size()
        self.layer_bytes = pool.stride(0) * pool.element_size()
        self.peer_base = torch.tensor([pp.data_ptr() for pp in peer_pools], dtype=torch.int64, device=dev)
        self.overflow = torch.zeros((), dtype=torch.bool, device=dev)
        self.fetched_runs = torch.zeros((), dtype=torch.int64, device=dev)
        self.fetched_rows = torch.zeros((), dtype=torch.int64, device=dev)

    def localize(self, grow: torch.Tensor, length: torch.Tensor, fresh: torch.Tensor | None = None,
                 scratch_half: int | None = None) -> torch.Tensor:
        """grow [n] global rows (or -1), length [n] -> local rows (int64).
        Missing remote runs are fetched peer-to-peer first (stream-ordered).
        ``fresh`` [n] (bool, optional): remote hits whose entry was created in this
        wave -- fetched into scratch half ``scratch_half`` (default: alternating per
        call; the two-wave pipeline passes its slot) and NOT cached."""
        dev = grow.device
        n = grow.numel()
        i64 = dict(dtype=torch.int64, device=dev)
        gt = grow.to(torch.int64)
        ln = length.to(torch.int64)
        src_rank = gt >> ROW_SHIFT
        remote = (gt >= 0) & (src_rank != self.rank)
        fresh_remote = remote & fresh if fresh is not None else torch.zeros_like(remote)
        cached = remote & ~fresh_remote
        hit, _e, _p, row = self.map.lookup_insert(gt.contiguous(), torch.arange(n, **i64), torch.zeros(n, **i64),
                                                  ln.to(torch.int32).contiguous(), cached)
        local = self.base + row
        fits = local + ln <= self.limit
        new = cached & (hit == 0)
        self.overflow |= (new & ~fits).any()
        fetch = new & fits
        if fresh is not None:
            half = self._half if scratch_half is None else scratch_half
            if scratch_half is None:
                self._half ^= 1
            # one scratch copy per distinct fresh run of the wave (fixed-size sort, no host sync)
            big = torch.iinfo(torch.int64).max
            sk, sp = torch.sort(torch.where(fresh_remote, gt, torch.full_like(gt, big)))
            first = torch.ones_like(fresh_remote)
            first[1:] = sk[1:] != sk[:-1]
            first &= sk != big
            sl = ln[sp] * first
            off = torch.cumsum(sl, 0) - sl
            head = torch.cummax(torch.where(first, torch.arange(n, **i64), torch.zeros_like(sp)), 0).values
            srow = torch.empty_like(gt)
            srow[sp] = self.scratch_base + half * self.scratch_rows + off[head]
            lead = torch.zeros_like(fresh_remote)
            lead[sp] = first
            sfits = srow + ln <= self.scratch_base + (half + 1) * self.scratch_rows
            self.overflow |= (fresh_remote & ~sfits).any()
            local = torch.where(fresh_remote, srow, local)
            fetch = fetch | (lead & sfits)
        perm = torch.argsort((~fetch).to(torch.int8), stable=True)  # runs to fetch first
        n_fetch = fetch.sum().reshape(1)
        self.fetched_runs += n_fetch[0]
        self.fetched_rows += (ln * fetch).sum()
        src_addr = (self.peer_base[src_rank.clamp(0, len(self.peers) - 1)] +
                    (gt & ROW_MASK) * self.row_bytes)[perm].contiguous()
        self._copy(src_addr, src_rank[perm], (gt & ROW_MASK)[perm], local[perm].contiguous(),
                   ln[perm].to(torch.int32).contiguous(), n_fetch)
        return torch.where(remote, local, torch.where(gt >= 0, gt & ROW_MASK, torch.zeros_like(gt)))

    def _copy(self, src_addr, src_rank, src_row, dst_row, length, n_fetch):
        if self.pool.is_cuda:
            from . import ops

            ops.copy_runs(src_addr, self.layer_bytes, self.pool, dst_row, length, n_dev=n_fetch)
            return
        # CPU tensors (the gloo tests, with shared-memory pools standing in for peer mappings):
        # the same copy, run by torch on the host
        for c in range(int(n_fetch[0])):
            r, s, d, l = int(src_rank[c]), int(src_row[c]), int(dst_row[c]), int(length[c])
            self.pool[:, d:d + l] = self.peers[r][:, s:s + l]

    def check(self):
        """Host check (call outside timed regions): the replica region held every fetch."""
        if bool(self.overflow):
            raise RuntimeError("replica region of the pool is full")
