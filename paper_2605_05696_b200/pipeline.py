"""The warm-serve reattach step as one CUDA graph (B200 production path).

For a wave of requests, one step is

    K0  phase 1 on the device (engine.py:170, 228): every request's longest
        prefix match against all earlier requests, then its insert
        (radix.WavePrefixIndex), and the tails + rebased marker pins packed for
        K1 (irm_wave_rebase) -- when the pipeline has a prefix index; otherwise
        the wave arrives as tails with a host-known m
    K1  CDC + xxh64 over every request tail          (irm_cdc_xxh64)
    K3  first-writer-wins lookup/insert of all chunks (irm_store_lookup_insert)
        -- carve-out chunks (p < 32) neither probed nor inserted (engine.py:184-196)
    K4  rotate+gather of every PIC hit chunk into the per-request KV buffer
        out[l, r * req_stride + p, :] for all layers l (registry.py:146-166)

with no host synchronisation anywhere: every shape is capacity-bounded, the
chunk -> request map comes from the device CSR offsets, and non-hit chunks
are masked to zero rows for K4. That makes the whole step capturable as a
single CUDA graph (no tracing compiler), replayed per wave after the inputs
are copied into the static buffers.

``capture_overlapped`` adds a two-wave software pipeline: one graph per slot
runs K4 of wave i (slot i % 2, on ~120 SMs) while K1 + K3 of wave i + 1 run on
a forked stream over the remaining SMs and fill the other slot. K3 waves stay
in order on that stream, so first-writer-wins across waves is unchanged.

K4 runs in its fan-out form by default (``fanout=True``): the compacted hits
are grouped by source run on the device (``irm_group_by_source``) and every
(entry, layer) slab is read from HBM once for all the requests of the wave that
reattach it (``irm_rotate_gather_fanout``; registry.py:146-166 is a pure
function of (entry, p_dest)). ``fanout=False`` keeps the one-read-per-hit
gather (``irm_rotate_gather``).

Bounds: K4 skips (and reports in ``status``) any source run outside the pool
or destination run outside the output, and the hit compaction refuses a hit
whose request row range would spill past ``req_stride``; ``check()`` raises on
any flag, the store's included (call it outside timed regions).
"""

from __future__ import annotations


import torch

from . import _native as N
from . import ops


def _nvtx(name):
    """NVTX range around a pipeline phase (visible to ncu --nvtx / Nsight on eager runs;
    a captured graph replays without host ranges)."""
    def wrap(fn):
        def inner(*a, **kw):
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*a, **kw)
            finally:
                torch.cuda.nvtx.range_pop()
        inner.__name__, inner.__doc__ = fn.__name__, fn.__doc__
        return inner
    return wrap


class ReattachPipeline:
    def __init__(self, store: ops.ChunkStore, pool: torch.Tensor, inv_freq: torch.Tensor,
                 max_requests: int, max_tokens: int, max_pins: int, req_stride: int,
                 layout: int = N.LAYOUT_INTERLEAVED, mask_exponent: int = 7, min_size: int = 32,
                 max_size: int = 512, carve: int = 32, ckv_dim: int = 512, kr_dim: int = 64,
                 fanout: bool = True, prefix_index=None, max_spans: int = 0):
        """prefix_index (radix.WavePrefixIndex): phase 1 runs on the device inside the
        step -- waves are then loaded as WHOLE requests with their marker spans
        (``load_requests``); K0 matches each request against every earlier one,
        ``irm_wave_rebase`` packs the tails and rebases the pins, then K1 / K3 / K4
        as before. Without it, waves are loaded as tails with a host-known m
        (``load``). max_spans: marker spans per wave (prefix mode)."""
        dev = pool.device
        self.prefix_index = prefix_index
        self.fanout = fanout
        self.k4_sms = 0  # SMs K4 spreads over (0 = all); per launch, captured with it
        self.status = torch.zeros(1, dtype=torch.int64, device=dev)  # sticky K4 / compaction bound flags
        self.store, self.pool, self.inv = store, pool, inv_freq
        self.R, self.req_stride, self.carve = max_requests, req_stride, carve
        self.params = (mask_exponent, min_size, max_size)
        self.layout, self.ckv, self.kr = layout, ckv_dim, kr_dim
        self.max_tokens, self.max_pins = max_tokens, max_pins
        # static inputs, two sets: the overlapped pipeline loads wave i + 2 while wave i + 1 reads the other
        self.inputs = [dict(tok=torch.zeros(max_tokens, dtype=torch.int32, device=dev),
                            stream_off=torch.zeros(max_requests + 1, dtype=torch.int64, device=dev),
                            pin_off=torch.zeros(max_requests + 1, dtype=torch.int64, device=dev),
                            pins=torch.zeros(max(max_pins, 1), dtype=torch.int64, device=dev),
                            m=torch.zeros(max_requests, dtype=torch.int64, device=dev)) for _ in range(2)]
        if prefix_index is not None:  # whole requests + request-relative marker spans, per input set
            assert max_pins >= 2 * max_spans, "two pins per marker span"
            for ins in self.inputs:
                ins.update(full_tok=torch.zeros(max_tokens, dtype=torch.int32, device=dev),
                           full_off=torch.zeros(max_requests + 1, dtype=torch.int64, device=dev),
                           span_off=torch.zeros(max_requests + 1, dtype=torch.int64, device=dev),
                           spans=torch.zeros(max(2 * max_spans, 2), dtype=torch.int64, device=dev))
        self.cur_in = 0  # the input set K1 / K3 read and load() writes
        # static outputs: per-request KV and the chunk service table
        self.out = torch.empty(pool.shape[0], max_requests * req_stride, pool.shape[2], dtype=pool.dtype,
                               device=dev)
        self.cdc_ws = ops.CdcWorkspace()
        bound = int(N.lib().irm_cdc_chunk_bound(max_tokens, max_requests, max_pins, min_size))
        self.gather_ws = torch.empty(int(N.lib().irm_rotate_gather_workspace_bytes(bound, kr_dim)),
                                     dtype=torch.uint8, device=dev)
        self.fan_ws = torch.empty(int(N.lib().irm_fanout_workspace_bytes(max(bound, 16), kr_dim)),
                                  dtype=torch.uint8, device=dev)
        # workspaces sized once for the static capacity and frozen: captured graphs keep their addresses
        self.cdc_ws.get(max_tokens, max_requests, max_pins, max(min_size, 1))
        self.cdc_ws.freeze()
        store.reserve(max(bound, 16))
        if store.pool_rows == 0:  # new entries' rows must fit this pool (sticky flag, check())
            store.set_pool_rows(pool.shape[1])
        self.groups = None  # serial mode's source groups (static: graph-captured)
        self.order0 = 0
        self.fill_slot = None  # overlapped mode: the slot K3 compacts into
        self.slots = None
        self.graph = None
        self.table = self.hit = self.length = self.delta = None

    tok = property(lambda self: self.inputs[self.cur_in]["tok"])
    stream_off = property(lambda self: self.inputs[self.cur_in]["stream_off"])
    pin_off = property(lambda self: self.inputs[self.cur_in]["pin_off"])
    pins = property(lambda self: self.inputs[self.cur_in]["pins"])
    m = property(lambda self: self.inputs[self.cur_in]["m"])

    # ------------------------------------------------------------ device step
    @_nvtx("irm.K0 phase 1 + rebase")
    def k0(self):
        """Phase 1 on the device: m of every request of the wave (K0), then the
        tails and their pins for K1 (irm_wave_rebase). No-op without a prefix index."""
        if self.prefix_index is None:
            return
        ins = self.inputs[self.cur_in]
        self.prefix_index.match_insert_wave(ins["full_tok"], ins["full_off"], self.R, ins["m"])
        ops.wave_rebase(ins["full_tok"], ins["full_off"], ins["m"], self.R, ins["span_off"], ins["spans"],
                        ins["tok"], ins["stream_off"], ins["pin_off"], ins["pins"])

    @_nvtx("irm.K1 cdc+xxh64")
    def k1(self):
        k, mn, mx = self.params
        self.table = ops.cdc_xxh64(self.tok, self.stream_off, self.pin_off, self.pins, k, mn, mx, True,
                                   ws=self.cdc_ws, n_tokens=self.max_tokens, n_pins=self.max_pins)

    def _plan(self):
        """Per-slot request / absolute position / probe flag / order key of the wave
        (irm_wave_plan: the glue of engine.py:181-189, one launch)."""
        t = self.table
        cap = t.start.numel()
        dev = t.start.device
        self.reqc = torch.empty(cap, dtype=torch.int64, device=dev)
        self.p_abs = torch.empty(cap, dtype=torch.int64, device=dev)
        probe = torch.empty(cap, dtype=torch.uint8, device=dev)
        order = torch.empty(cap, dtype=torch.int64, device=dev)
        ops.wave_plan(t.chunk_off, self.R, t.start, self.m, self.carve, self.order0, self.reqc, self.p_abs, probe,
                      order)
        return probe, order

    @_nvtx("irm.K3 store")
    def k3(self):
        t = self.table
        probe, order = self._plan()
        self.hit, self.entry, self.p_src, self.row = self.store.lookup_insert(t.fp, order, self.p_abs,
                                                                              t.length, probe)
        self._compact(self.row)

    def _compact(self, src):
        """PIC hits first, in slot order, with their count left on the device
        (irm_wave_compact, one launch): K4 then walks only real work and the step
        stays free of host synchronisation."""
        t = self.table
        cap = t.start.numel()
        dev = t.start.device
        self.length = torch.empty(cap, dtype=torch.int32, device=dev)
        if self.fill_slot is None:
            self.k4_src = torch.empty(cap, dtype=torch.int64, device=dev)
            self.k4_dst = torch.empty(cap, dtype=torch.int64, device=dev)
            self.k4_len = torch.empty(cap, dtype=torch.int32, device=dev)
            self.k4_delta = torch.empty(cap, dtype=torch.int64, device=dev)
            self.n_hit = torch.empty(1, dtype=torch.int64, device=dev)
            ops.wave_compact(self.hit, src, self.reqc, self.p_abs, self.p_src, t.length, self.req_stride,
                             self.k4_src, self.k4_dst, self.k4_len, self.k4_delta, self.n_hit, self.length,
                             status=self.status)
            if self.fanout:
                if self.groups is None or self.groups.g_src.numel() < cap:
                    self.groups = ops.SourceGroups.alloc(cap, dev)
                ops.group_by_source(self.k4_src, self.k4_dst, self.k4_len, self.k4_delta, self.groups,
                                    n_dev=self.n_hit)
            return
        sl = self.slots[self.fill_slot]  # overlapped mode: static per-slot buffers
        ops.wave_compact(self.hit, src, self.reqc, self.p_abs, self.p_src, t.length, self.req_stride,
                         sl["src"], sl["dst"], sl["len"], sl["delta"], sl["n_hit"], self.length,
                         hit_tokens=self.hit_tokens, status=self.status)
        if self.fanout:
            ops.group_by_source(sl["src"], sl["dst"], sl["len"], sl["delta"], sl["groups"], n_dev=sl["n_hit"])
        sl["hit"].copy_(self.hit)

    @_nvtx("irm.K4 rotate+gather")
    def k4(self, slot: int | None = None, max_sms: int | None = None, cta_rounds: int = 1):
        sms = self.k4_sms if max_sms is None else max_sms
        if slot is None:
            out, src, dst, ln, delta, n_hit, groups = (self.out, self.k4_src, self.k4_dst, self.k4_len,
                                                       self.k4_delta, self.n_hit, self.groups)
        else:
            sl = self.slots[slot]
            out, src, dst, ln, delta, n_hit, groups = (sl["out"], sl["src"], sl["dst"], sl["len"], sl["delta"],
                                                       sl["n_hit"], sl["groups"])
        if self.fanout:
            ops.rotate_gather_fanout(self.pool, out, groups, self.inv, self.ckv, self.kr, self.layout,
                                     ws=self.fan_ws, n_members_dev=n_hit, max_sms=sms, status=self.status,
                                     cta_rounds=cta_rounds)
        else:
            ops.rotate_gather(self.pool, out, src, dst, ln, delta, self.inv, self.ckv, self.kr, self.layout,
                              ws=self.gather_ws, n_dev=n_hit, max_sms=sms, status=self.status)

    def check(self):
        """Host check (outside timed regions): no K4 / compaction bound was hit and
        the store (and the prefix index) did not overflow (raises ValueError /
        RuntimeError)."""
        ops.check_status(self.status, "reattach pipeline")
        self.store.counts()
        if self.prefix_index is not None:
            self.prefix_index.check()

    def step_eager(self):
        self.k0()
        self.k1()
        self.k3()
        self.k4()

    # ------------------------------------------------------------ multi-GPU (K6)
    def enable_sharding(self, sharded_store, replica_cache, rank: int, world: int):
        """Route K3 through the hash-sharded store (shard.ShardedStore) and K4's
        sources through the replica cache. Sharded steps run eagerly (NCCL
        all-to-alls between the kernels) but never wait for the host: every
        buffer is capacity-bounded, so the CPU runs ahead of the GPU."""
        self.sharded, self.replica, self.rank, self.world = sharded_store, replica_cache, rank, world
        # the exchange has equal splits: every rank uses the largest chunk-table capacity
        import torch.distributed as dist

        k, mn, mx = self.params
        cap = torch.tensor([max(int(N.lib().irm_cdc_chunk_bound(self.max_tokens, self.R, self.max_pins, mn)), 16)],
                           dtype=torch.int64, device=self.pool.device)
        if world > 1:
            dist.all_reduce(cap, op=dist.ReduceOp.MAX, group=sharded_store.group)
        sharded_store.slots = int(cap.item())
        # the owner allocates first-writer rows itself (ShardedStore): the shard's own row counter is unused
        self.store.set_pool_rows(0)
        self.store.reserve(world * sharded_store.slots)
        if hasattr(replica_cache.map, "reserve"):
            replica_cache.map.reserve(sharded_store.slots)

    @_nvtx("irm.K3+K6 sharded store")
    def k3_sharded(self, wave: int):
        t = self.table
        cap = t.start.numel()
        dev = t.start.device
        idx = torch.arange(cap, device=dev)
        probe, _ = self._plan()
        probe = probe.to(torch.bool)
        # global order: (global request = (wave * R + r) * G + rank, chunk index within the request);
        # wave: an int, or a device scalar (graph-captured fronts advance it on the device)
        g_req = (wave * self.R + self.reqc) * self.world + self.rank
        order = (g_req << 20) | (idx - t.chunk_off[self.reqc])
        hit, self.p_src, grow, _own = self.sharded.lookup_insert(t.fp, order, self.p_abs, t.length, probe)
        self.hit = hit
        self.grow = grow  # novel chunks: the rows of this rank's pool that keep their KV (prefill writes them)
        is_hit = hit == 1
        # hits on entries this very exchange created (another rank's same-wave first write) are
        # fetched for this wave only: the writer has not produced those rows yet
        src = self.replica.localize(torch.where(is_hit, grow, torch.full_like(grow, -1)),
                                    torch.where(is_hit, t.length, torch.zeros_like(t.length)),
                                    fresh=self.sharded.fresh & is_hit,
                                    scratch_half=self.fill_slot if self.fill_slot is not None else None)
        self._compact(src)

    def step_sharded(self, wave: int):
        self.k0()
        self.k1()
        self.k3_sharded(wave)
        self.k4()

    def run_overlapped_sharded(self, n_waves: int, load_wave, wave0: int = 0, k4_sms: int = 128,
                               after_front=None, after_k4=None):
        """The two-wave pipeline of ``run_overlapped`` for the sharded store, on
        streams instead of graphs: K4 of wave i (main stream, ``k4_sms`` SMs)
        runs while K1 + the sharded lookup + replica fetch of wave i + 1 run on a
        side stream. Waves are numbered ``wave0 + i`` in the global order key."""
        if n_waves <= 0:
            return
        self._alloc_slots()
        main = torch.cuda.current_stream()
        side = self._side if getattr(self, "_side", None) is not None else torch.cuda.Stream(priority=-1)
        self._side = side

        def front(i, s):
            self.fill_slot, self.cur_in = s, s
            self.k0()
            self.k1()
            self.k3_sharded(wave0 + i)
            self.fill_slot, self.cur_in = None, 0

        loader = _Loader(self, load_wave)
        self.k4_sms = k4_sms
        try:
            loader.load(0, main)
            front(0, 0)
            loader.read_done(0, main)
            if after_front:
                after_front(0, 0)
            if n_waves > 1:
                loader.load(1, side)
            for i in range(n_waves):
                s = i & 1
                if i + 1 < n_waves:
                    side.wait_stream(main)
                    with torch.cuda.stream(side):
                        front(i + 1, 1 - s)
                        loader.read_done(i + 1, side)
                self.k4(s, cta_rounds=4 if k4_sms == 0 else 1)
                main.wait_stream(side)
                if i + 2 < n_waves:
                    loader.load(i + 2, side)  # H2D under K4(i + 1); front(i + 2) waits for it
                if after_front and i + 1 < n_waves:
                    after_front(i + 1, 1 - s)
                if after_k4:
                    after_k4(i, s)
        finally:
            self.k4_sms = 0

    # ------------------------------------------------------------ graphs
    def _empty_inputs(self):
        """Zero the CSR offsets of both input sets (every request empty) and return
        a restore function: warm-ups before a capture then touch no store or index."""
        keys = ("full_off", "span_off") if self.prefix_index is not None else ("stream_off", "pin_off")
        saved = [tuple(ins[k].clone() for k in keys) for ins in self.inputs]
        for ins in self.inputs:
            for k in keys:
                ins[k].zero_()

        def restore():
            torch.cuda.synchronize()
            for ins, sv in zip(self.inputs, saved):
                for k, v in zip(keys, sv):
                    ins[k].copy_(v)
            torch.cuda.synchronize()
        return restore

    def capture(self, warmup: int = 2):
        """Capture the step (and K1-, K3- and K4-only graphs for component timing).
        Prefix mode warms up on empty requests (re-serving a wave would match it whole)."""
        restore = self._empty_inputs() if self.prefix_index is not None else None
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.step_eager()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        if restore:
            restore()
        pool = torch.cuda.graph_pool_handle()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, pool=pool):
            self.step_eager()
        self.graph_k1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph_k1, pool=pool):
            self.k1()
        self.graph_k4 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph_k4, pool=pool):
            self.k4()
        self.graph_k3 = torch.cuda.CUDAGraph()  # replays re-probe the same wave: all hits, no inserts
        live = dict(self.__dict__)
        with torch.cuda.graph(self.graph_k3, pool=pool):
            self.k3()
        self.__dict__.update(live)  # k3 rebinds its outputs: the step graph's buffers stay the live ones
        torch.cuda.synchronize()

    def _alloc_slots(self):
        if self.slots is not None:
            return
        if self.table is None:
            self.k1()
        cap = self.table.start.numel()
        dev = self.pool.device
        i64 = dict(dtype=torch.int64, device=dev)
        self.slots = []
        for s in range(2):
            self.slots.append(dict(
                src=torch.zeros(cap, **i64), dst=torch.zeros(cap, **i64), delta=torch.zeros(cap, **i64),
                len=torch.zeros(cap, dtype=torch.int32, device=dev), n_hit=torch.zeros(1, **i64),
                hit=torch.zeros(cap, dtype=torch.int32, device=dev),
                groups=ops.SourceGroups.alloc(cap, dev) if self.fanout else None,
                out=self.out if s == 0 else torch.empty_like(self.out)))
        self.hit_tokens = torch.zeros((), **i64)

    def capture_overlapped(self, k4_sms: int = 128, warmup: int = 2, sharded: bool = False):
        """Capture the two-wave pipeline: ``front[s]`` = K1 + K3 of a wave into
        slot s; ``overlap[s]`` = K4 of slot s on ``k4_sms`` SMs, concurrently with
        front[1 - s] on a forked stream; ``drain[s]`` = K4 of slot s alone.
        Per-slot outputs: ``slots[s]["out"]`` (KV), ``["hit"]`` (service map);
        ``hit_tokens`` accumulates reattached tokens on the device.

        ``sharded``: the front is K1 + the sharded lookup (NCCL all-to-alls
        captured into the graph) + the replica fetch, as in
        ``run_overlapped_sharded``; the wave number of the global order key is a
        device scalar (``wave_t``) each front advances. Every rank captures the
        same sequence of collectives, so replays stay matched across ranks."""
        self._alloc_slots()
        # the next wave's front on a high-priority stream: its kernels take SMs as K4's CTAs retire
        # (K4 runs in cta_rounds=4 rounds of CTAs when it has every SM; profiles/r02_k4_sms.md)
        side = torch.cuda.Stream(priority=-1)
        if sharded:
            self.wave_t = torch.zeros((), dtype=torch.int64, device=self.pool.device)

        def front(s):
            self.fill_slot, self.cur_in = s, s
            self.k0()
            self.k1()
            if sharded:
                self.k3_sharded(self.wave_t)
                self.wave_t += 1
            else:
                self.k3()
            self.fill_slot, self.cur_in = None, 0

        def overlap(s):
            cur = torch.cuda.current_stream()
            side.wait_stream(cur)
            # the rest of the SMs (k4_sms < all), or SMs freed between K4's CTA rounds, run the next front
            self.k4(s, max_sms=k4_sms, cta_rounds=4 if k4_sms == 0 else 1)
            with torch.cuda.stream(side):
                front(1 - s)
            cur.wait_stream(side)

        # warm up and capture over empty streams: no store side effects (nothing is
        # probed or inserted), and every shape is capacity-bounded anyway
        restore = self._empty_inputs()
        s0 = torch.cuda.Stream()
        s0.wait_stream(torch.cuda.current_stream())
        try:
            with torch.cuda.stream(s0):
                for _ in range(warmup):
                    front(0)
                    overlap(0)
                    self.k4(1)
            torch.cuda.current_stream().wait_stream(s0)
            torch.cuda.synchronize()
            mp = torch.cuda.graph_pool_handle()
            self.g_front, self.g_overlap, self.g_drain = [], [], []
            for s in range(2):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, pool=mp):
                    front(s)
                self.g_front.append(g)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, pool=mp):
                    overlap(s)
                self.g_overlap.append(g)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, pool=mp):
                    self.k4(s)
                self.g_drain.append(g)
        finally:
            restore()
        self.hit_tokens.zero_()

    def run_overlapped(self, n_waves: int, load_wave, after_front=None, after_k4=None, wave0: int = 0,
                       readback=None):
        """Process waves 0..n_waves-1 through the two-wave pipeline.
        ``load_wave(i)`` copies wave i's inputs into the static buffers (called on
        the current stream, after the previous graph that read them);
        ``after_front(i, slot)`` is called once wave i's lookup results are in
        ``slots[slot]`` (stream-ordered), e.g. to read the service map back;
        ``after_k4(i, slot)`` once wave i's KV is in ``slots[slot]["out"]``.
        ``readback[i]`` (pinned host tensors, optional): wave i's per-chunk
        service map is copied there on a side stream, off the step's critical
        path; the graph that next overwrites the slot waits for the copy.
        Sharded graphs number the waves ``wave0 + i`` in the global order key."""
        if n_waves <= 0:
            return
        main = torch.cuda.current_stream()
        if getattr(self, "wave_t", None) is not None:
            self.wave_t.fill_(wave0)
        loader = _Loader(self, load_wave)
        if readback is not None and getattr(self, "_d2h", None) is None:
            self._d2h = torch.cuda.Stream()
        rb_done = [None, None]

        def read(j, slot):  # D2H of wave j's service map, after the graph that wrote it
            if readback is not None:
                ev = torch.cuda.Event()
                ev.record(main)
                self._d2h.wait_event(ev)
                with torch.cuda.stream(self._d2h):
                    readback[j].copy_(self.slots[slot]["hit"], non_blocking=True)
                    rb_done[slot] = torch.cuda.Event()
                    rb_done[slot].record(self._d2h)
            if after_front:
                after_front(j, slot)

        loader.load(0, main)
        self.g_front[0].replay()
        loader.read_done(0, main)
        read(0, 0)
        if n_waves > 1:
            loader.load(1, main)
        for i in range(n_waves):
            s = i & 1
            if i + 1 < n_waves:
                if rb_done[1 - s] is not None:
                    main.wait_event(rb_done[1 - s])  # slot 1 - s is rewritten by this graph
                self.g_overlap[s].replay()  # K4(i) || K1 + K3(i + 1) -> slot 1 - s
                loader.read_done(i + 1, main)
                if i + 2 < n_waves:
                    loader.load(i + 2, main)  # H2D under the next graph (other input set)
                read(i + 1, 1 - s)
            else:
                self.g_drain[s].replay()
            if after_k4:
                after_k4(i, s)
        if readback is not None:
            main.wait_stream(self._d2h)

    def load(self, tok, stream_off, pin_off, pins, m):
        """Copy one wave's inputs (device-resident or pinned host) into the static
        buffers of the current input set (``cur_in``), on the current stream.
        Host inputs are validated here (every request's m + tail fits its
        ``req_stride`` rows); device inputs are checked by the compaction on the
        device (``status``), so loading never waits for the GPU."""
        n = tok.numel()
        if n > self.max_tokens or pins.numel() > self.max_pins or m.numel() > self.R:
            raise ValueError("wave exceeds the pipeline's static capacity")
        if not stream_off.is_cuda and not m.is_cuda and m.numel():
            span = (stream_off[1:m.numel() + 1] - stream_off[:m.numel()]) + m
            if int(span.max()) > self.req_stride:
                raise ValueError(f"a request of {int(span.max())} tokens exceeds req_stride {self.req_stride}")
        self.tok[:n].copy_(tok, non_blocking=True)
        r = stream_off.numel()
        self.stream_off[:r].copy_(stream_off, non_blocking=True)
        self.pin_off[:r].copy_(pin_off, non_blocking=True)
        if r < self.R + 1:  # unused request slots are empty streams
            self.stream_off[r:].copy_(self.stream_off[r - 1:r].expand(self.R + 1 - r))
            self.pin_off[r:].copy_(self.pin_off[r - 1:r].expand(self.R + 1 - r))
        self.pins[:pins.numel()].copy_(pins, non_blocking=True)
        self.m[:m.numel()].copy_(m, non_blocking=True)

    def load_requests(self, tok, off, span_off, spans):
        """Prefix mode: copy one wave of WHOLE requests (u32 tokens as int32, CSR
        ``off``) and their request-relative marker spans ([start, end) pairs, CSR
        ``span_off``) into the current input set, on the current stream."""
        assert self.prefix_index is not None, "load_requests needs a prefix index (else: load)"
        ins = self.inputs[self.cur_in]
        n, r = tok.numel(), off.numel()
        if n > ins["full_tok"].numel() or spans.numel() > ins["spans"].numel() or r > self.R + 1:
            raise ValueError("wave exceeds the pipeline's static capacity")
        ins["full_tok"][:n].copy_(tok, non_blocking=True)
        ins["full_off"][:r].copy_(off, non_blocking=True)
        ins["span_off"][:r].copy_(span_off, non_blocking=True)
        if r < self.R + 1:  # unused request slots are empty requests
            ins["full_off"][r:].copy_(ins["full_off"][r - 1:r].expand(self.R + 1 - r))
            ins["span_off"][r:].copy_(ins["span_off"][r - 1:r].expand(self.R + 1 - r))
        ins["spans"][:spans.numel()].copy_(spans, non_blocking=True)

    def replay(self):
        self.graph.replay()


class _Loader:
    """Input loads of the overlapped pipelines on a copy stream. Wave j lands in
    input set j % 2 once the front of wave j - 2 (the set's last reader) is done;
    the stream that runs wave j's front waits for the copy."""

    _stream = None

    def __init__(self, pipe: ReattachPipeline, load_wave):
        self.pipe, self.load_wave = pipe, load_wave
        if _Loader._stream is None:
            _Loader._stream = torch.cuda.Stream()
        self.copy = _Loader._stream
        self.read_ev = [None, None]

    def load(self, j: int, consumer: torch.cuda.Stream):
        s = j & 1
        if self.read_ev[s] is not None:
            self.copy.wait_event(self.read_ev[s])
        else:
            self.copy.wait_stream(consumer)
        with torch.cuda.stream(self.copy):
            self.pipe.cur_in = s
            self.load_wave(j)
            self.pipe.cur_in = 0
        consumer.wait_stream(self.copy)

    def read_done(self, j: int, stream: torch.cuda.Stream):
        ev = torch.cuda.Event()
        ev.record(stream)
        self.read_ev[j & 1] = ev
