"""Decode-step driver: the per-layer select -> cache -> FlashH2D -> attention
sequence of PAPER.md:124 (§3.1 Model Executor) over L layers.

PyTorch is used for device memory, pinned host memory, streams and events only;
every step of the path is a call into libsparseserve.so through `ops`.

Request groups (B200 scheduling): the batch can be split into G
contiguous request groups, each on its own CUDA stream.  Every request's layers
still run strictly in order (layer l+1 of a request only after its layer-l
attention), but while group A waits on the PCIe link for its missed blocks
(FlashH2D), group B's HBM-bound select / attention run on the SMs.  All groups
of a layer share that layer's HBM cache pool; their cache calls are ordered
(group 0 first) and use the same stamp, so a group never evicts a slot that
another group touched in the same step.  A cache call of step t+1 waits for
the layer's attention of every group at step t (no eviction under a reader).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import torch

from . import ops
from ._lib import SS_WS_ATTN, SS_WS_CACHE, SS_WS_SELECT

HEAD_DIM = ops.HEAD_DIM
BLOCK_TOKENS = ops.BLOCK_TOKENS


@dataclasses.dataclass
class EngineConfig:
    batch: int
    layers: int
    num_q_heads: int
    num_kv_heads: int
    max_blk: int               # multiple of 32
    topk: int
    slots_per_layer: int
    num_requests: int          # size of the request-id space (fwd table extent)
    dtype: torch.dtype = torch.bfloat16
    groups: int = 1            # request groups pipelined on separate streams
    h2d_streams: int = 1       # FlashH2D streams shared round-robin by the groups
    select_priority: bool = False  # run select on a high-priority per-group stream
    cache_per_group: bool = False  # per-group cache streams, ordered per layer only
    h2d_server: bool = False   # one persistent FlashH2D launch per step (flash_h2d_serve)
    split_attn: bool = False   # server mode: attend the hits while FlashH2D loads the misses
    pool_per_group: bool = False  # one LRU pool per (layer, request group) of slots/groups slots

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    @property
    def elem_bytes(self) -> int:
        return 2 if self.dtype == torch.bfloat16 else 4

    @property
    def block_bytes(self) -> int:
        return 2 * BLOCK_TOKENS * HEAD_DIM * self.elem_bytes

    @property
    def block_elems(self) -> int:
        return 2 * BLOCK_TOKENS * HEAD_DIM

    @property
    def pairs(self) -> int:
        return self.batch * self.num_kv_heads

    @property
    def fwd_len(self) -> int:
        return self.num_requests * self.layers * self.num_kv_heads * self.max_blk


class RequestGroup:
    """Scratch of one contiguous request range [b0, b1): its selections, cache
    outputs, miss lists, counts, outputs and workspaces, and its stream."""

    def __init__(self, eng: "DecodeEngine", b0: int, b1: int, stream: torch.cuda.Stream):
        c, dev = eng.cfg, eng.device
        self.b0, self.b1 = b0, b1
        nb = b1 - b0
        self.nb = nb
        self.stream = stream
        self.dims = ops.dims(nb, c.num_q_heads, c.num_kv_heads)
        E = nb * c.num_kv_heads * c.topk
        self.E = E
        self.sel = torch.empty(c.layers, nb, c.num_kv_heads, c.topk, dtype=torch.int32, device=dev)
        self.slot = torch.empty_like(self.sel)
        self.hit = torch.empty(c.layers, nb, c.num_kv_heads, c.topk, dtype=torch.uint8, device=dev)
        self.miss_keys = torch.empty(c.layers, E, dtype=torch.int64, device=dev)
        self.miss_slots = torch.empty(c.layers, E, dtype=torch.int32, device=dev)
        self.counts = torch.zeros(c.layers, 4, dtype=torch.int32, device=dev)
        self.out = torch.empty(c.layers, c.num_q_heads, nb, HEAD_DIM, dtype=torch.float32, device=dev)
        self.ws_select = ops.alloc_workspace(SS_WS_SELECT, self.dims, c.max_blk, c.topk, device=dev)
        self.ws_cache = ops.alloc_workspace(SS_WS_CACHE, self.dims, c.max_blk, c.topk,
                                            c.slots_per_layer, device=dev)
        self.ws_attn = ops.alloc_workspace(SS_WS_ATTN, self.dims, c.max_blk, c.topk, device=dev)
        if c.split_attn:
            # split attention (EngineConfig.split_attn): hit-part and miss-part
            # outputs / log-sum-exps, merged into out[l]
            self.out_h = torch.empty(c.num_q_heads, nb, HEAD_DIM, dtype=torch.float32, device=dev)
            self.out_m = torch.empty_like(self.out_h)
            self.lse_h = torch.empty(c.num_q_heads, nb, dtype=torch.float32, device=dev)
            self.lse_m = torch.empty_like(self.lse_h)
        pair_elems = c.max_blk * 2 * HEAD_DIM
        self.meta = [m[b0 * c.num_kv_heads * pair_elems:b1 * c.num_kv_heads * pair_elems]
                     for m in eng.meta]
        self.n_blk = eng.n_blk[b0:b1]
        self.req_ids = eng.req_ids[b0:b1]
        self.tail_len = eng.tail_len[b0:b1]
        self.tail_kv = eng.tail_kv[:, b0:b1]
        self.ev_cache = [torch.cuda.Event() for _ in range(c.layers)]
        self.ev_attn = [torch.cuda.Event() for _ in range(c.layers)]
        self.ev_gather = [torch.cuda.Event() for _ in range(c.layers)]
        self.ev_sel = [torch.cuda.Event() for _ in range(c.layers)]
        # FlashH2D runs on the engine's shared high-priority stream (set below)
        self.h2d_stream = None
        # select on a high-priority stream (EngineConfig.select_priority): the
        # select -> cache -> FlashH2D chain feeds the PCIe link, the bottleneck
        self.sel_stream = None
        self.cache_stream = None      # own cache stream (EngineConfig.cache_per_group)


class DecodeEngine:
    """Device state of one GPU: per-layer metadata, per-layer HBM block-cache
    pools (shared key->slot table), tail blocks, and per-group scratch."""

    def __init__(self, cfg: EngineConfig, device: Optional[torch.device] = None):
        self.cfg = cfg
        dev = torch.device(device or "cuda")
        self.device = dev
        c = cfg
        self.dims = ops.dims(c.batch, c.num_q_heads, c.num_kv_heads)
        meta_elems = ops.meta_numel(c.batch, c.num_kv_heads, c.max_blk)
        self.meta: List[torch.Tensor] = [torch.zeros(meta_elems, dtype=c.dtype, device=dev)
                                         for _ in range(c.layers)]
        self.fwd = torch.full((c.fwd_len,), -1, dtype=torch.int32, device=dev)
        ng0 = max(1, min(c.groups, c.batch))
        # pool_per_group (reading R11b): the slots of a layer are split evenly
        # between the request groups, each group's requests run their own batch
        # LRU over their share, and the groups' cache calls are independent (no
        # cross-group order, 1/groups of the O(S) bookkeeping per call)
        self.per_group_pools = c.pool_per_group and ng0 > 1
        if self.per_group_pools:
            sg = c.slots_per_layer // ng0
            self.gpools = [[ops.CachePool(sg, self.fwd, dev) for _ in range(ng0)] for _ in range(c.layers)]
            self.gpool_kv = [[torch.zeros(sg * c.block_elems, dtype=c.dtype, device=dev) for _ in range(ng0)]
                             for _ in range(c.layers)]
            self.pools = [gp[0] for gp in self.gpools]
            self.pool_kv = [gk[0] for gk in self.gpool_kv]
        else:
            self.pools = [ops.CachePool(c.slots_per_layer, self.fwd, dev) for _ in range(c.layers)]
            self.pool_kv = [torch.zeros(c.slots_per_layer * c.block_elems, dtype=c.dtype, device=dev)
                            for _ in range(c.layers)]
        self.tail_kv = torch.zeros(c.layers, c.batch, c.num_kv_heads, 2, BLOCK_TOKENS, HEAD_DIM,
                                   dtype=c.dtype, device=dev)
        self.tail_len = torch.zeros(c.batch, dtype=torch.int32, device=dev)
        self.n_blk = torch.zeros(c.batch, dtype=torch.int32, device=dev)
        self.req_ids = torch.arange(c.batch, dtype=torch.int32, device=dev)
        self.scale = 1.0 / math.sqrt(HEAD_DIM)
        self.host_kv: Optional[torch.Tensor] = None
        self.host_ptr = 0
        self.host_blocks = 0
        ng = max(1, min(c.groups, c.batch))
        bounds = [round(i * c.batch / ng) for i in range(ng + 1)]
        cur = torch.cuda.current_stream(dev)
        self.groups = [RequestGroup(self, bounds[i], bounds[i + 1],
                                    cur if ng == 1 else torch.cuda.Stream(dev))
                       for i in range(ng)]
        self.h2d_streams = []
        if ng > 1:
            # One high-priority stream carries every group's FlashH2D in issue
            # order (layer l: group 0, 1, ...; then layer l+1): the PCIe link
            # serves one group at a time, which keeps the groups out of phase --
            # while group A's misses stream in, group B runs its HBM-bound
            # attention / next-layer select -- and the gather CTAs are dispatched
            # ahead of queued HBM-kernel CTAs.
            # (h2d_streams > 1: group i uses stream i % h2d_streams, so one group's
            # gather may start while another's is still streaming -- no link gap
            # when a group's cache call finishes late)
            h2d = [torch.cuda.Stream(dev, priority=-1) for _ in range(max(1, c.h2d_streams))]
            for i, g in enumerate(self.groups):
                g.h2d_stream = h2d[i % len(h2d)]
            self.h2d_streams = h2d
        self.cache_stream = torch.cuda.Stream(dev, priority=-1) if ng > 1 else None
        if ng > 1 and (c.cache_per_group or self.per_group_pools):
            # a layer's pool orders its calls group 0, 1, ...; calls of different
            # layers (different pools) need no order, so one shared cache stream
            # would add false cross-layer dependencies
            for g in self.groups:
                g.cache_stream = torch.cuda.Stream(dev, priority=-1)
        if ng > 1 and c.select_priority:
            for g in self.groups:
                g.sel_stream = torch.cuda.Stream(dev, priority=-1)
        # FlashH2D server (EngineConfig.h2d_server, multi-group only): the step's
        # gathers are jobs j = l * groups + gi of ONE persistent launch on the
        # h2d stream; a cache call signals ready[j], the group's attention
        # waits on done[j] (flash_h2d_serve in include/sparseserve.h)
        self.server = ng > 1 and c.h2d_server
        if self.server:
            import os
            import warnings
            if int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8")) < 2 * ng + 2:
                warnings.warn("FlashH2D server with %d request groups: set CUDA_DEVICE_MAX_CONNECTIONS "
                              ">= %d before CUDA starts (a spinning kernel can otherwise sit in front of "
                              "another stream's work until the 3 s timeout)" % (ng, 2 * ng + 2))
            self.njobs = c.layers * ng
            self.h2d_jobs = ops.h2d_jobs([(g.miss_keys[l], g.miss_slots[l], g.counts[l],
                                           self.pool_kv_of(l, gi), g.E)
                                          for l in range(c.layers) for gi, g in enumerate(self.groups)],
                                         device=dev)
            self.h2d_flags = ops.h2d_flags(self.njobs, device=dev)
            # server statistics (link idle time; include/sparseserve.h), zeroed per
            # step; passed to the server only when collect_h2d_stats is set (a few
            # atomics per 8 KiB unit)
            self.h2d_stats = ops.h2d_stats(device=dev)
            ops.preload_kernels()      # no lazy kernel load while the server spins
        self.collect_h2d_stats = False
        self._capturing = False
        g0 = self.groups[0]
        # single-group aliases (tests, smoke)
        self.sel, self.slot, self.hit = g0.sel, g0.slot, g0.hit
        self.miss_keys, self.miss_slots, self.counts, self.out = (g0.miss_keys, g0.miss_slots,
                                                                  g0.counts, g0.out)
        self.E = g0.E

    def pool_of(self, l: int, gi: int) -> "ops.CachePool":
        """The LRU pool request group gi uses at layer l."""
        return self.gpools[l][gi] if self.per_group_pools else self.pools[l]

    def pool_kv_of(self, l: int, gi: int) -> torch.Tensor:
        return self.gpool_kv[l][gi] if self.per_group_pools else self.pool_kv[l]

    # ------------------------------------------------------------------ setup
    def set_host_kv(self, host_kv: torch.Tensor, host_blocks: int, dev_ptr: Optional[int] = None) -> None:
        """host_kv: pinned CPU tensor holding host_blocks blocks [2][32][d] (dtype);
        dev_ptr: its device address if already known (ops.HostPool)."""
        assert host_kv.numel() * host_kv.element_size() >= host_blocks * self.cfg.block_bytes
        self.host_kv = host_kv
        self.host_blocks = host_blocks
        self.host_ptr = dev_ptr if dev_ptr is not None else ops.host_device_pointer(host_kv)

    def key0(self, req: int, layer: int, h: int) -> int:
        c = self.cfg
        return ((req * c.layers + layer) * c.num_kv_heads + h) * c.max_blk

    def build_meta(self, n_blk_host: List[int], dev_host_copy: torch.Tensor,
                   req_ids_host: Optional[List[int]] = None) -> None:
        """S0 over every full block: meta of logical block (b, l, h, j) is built
        from physical host block key % host_blocks.  `dev_host_copy` is a device
        copy of the host blocks (setup only).  Requires host_blocks % max_blk == 0
        (no wrap inside a (b, l, h) run)."""
        c = self.cfg
        assert self.host_blocks % c.max_blk == 0
        req_ids_host = req_ids_host or list(range(c.batch))
        tile_elems = 32 * 2 * HEAD_DIM
        for l in range(c.layers):
            for b in range(c.batch):
                n = int(n_blk_host[b])
                if n == 0:
                    continue
                for h in range(c.num_kv_heads):
                    phys0 = self.key0(req_ids_host[b], l, h) % self.host_blocks
                    keys = dev_host_copy[phys0 * c.block_elems:]
                    pair = b * c.num_kv_heads + h
                    meta = self.meta[l][pair * (c.max_blk // 32) * tile_elems:]
                    ops.block_meta_update(keys, meta, n, key_stride=c.block_elems)

    # ------------------------------------------------------------------- step
    def _group_layer(self, g: RequestGroup, l: int, q: torch.Tensor, stamp: int, gi: int,
                     scores: Optional[torch.Tensor], timers, gather: bool) -> None:
        c = self.cfg

        def timed(name, fn):
            if timers is None or not timers.wants(name):
                fn()
            else:
                s, e = timers.mark(name, gi, l)
                s.record()
                fn()
                e.record()
        multi = len(self.groups) > 1
        if multi and g.sel_stream is not None:
            g.sel_stream.wait_stream(g.stream)       # after this group's previous attention
            with torch.cuda.stream(g.sel_stream):
                timed("select", lambda: ops.ss_block_select(q, g.meta[l], g.n_blk, c.max_blk, c.topk,
                                                            g.dims, g.sel[l], g.ws_select, scores=scores))
                g.ev_sel[l].record(g.sel_stream)
        else:
            timed("select", lambda: ops.ss_block_select(q, g.meta[l], g.n_blk, c.max_blk, c.topk, g.dims,
                                                        g.sel[l], g.ws_select, scores=scores))

        def _cache():
            timed("cache", lambda: ops.kv_cache_lookup_insert(
                self.pool_of(l, gi), g.sel[l], g.req_ids, l, c.layers, c.max_blk, c.topk, g.dims, stamp,
                g.slot[l], g.hit[l], g.miss_keys[l], g.miss_slots[l], g.counts[l], g.ws_cache))

        def _gather():
            self._wait_saved(l, torch.cuda.current_stream(self.device))
            timed("gather", lambda: ops.flash_h2d_gather(self.host_ptr, self.host_blocks,
                                                         g.miss_keys[l], g.miss_slots[l], g.counts[l],
                                                         g.E, self.pool_kv_of(l, gi), c.block_bytes))
        if not multi:
            _cache()
            if gather:
                _gather()
        else:
            # cache calls of all groups go through one high-priority stream in
            # issue order (layer l: group 0, 1, ...): pool order for free, and the
            # small cache kernels are dispatched ahead of queued select CTAs.  The
            # first group of step t also waits for every group's layer-l attention
            # of step t-1 (no eviction under a reader).
            if g.sel_stream is None:
                g.ev_sel[l].record(g.stream)
            cs = g.cache_stream if g.cache_stream is not None else self.cache_stream
            cs.wait_event(g.ev_sel[l])
            if g.cache_stream is not None and gi > 0 and not self.per_group_pools:
                cs.wait_event(self.groups[gi - 1].ev_cache[l])   # same layer pool: in group order
            if gi == 0 and not self._capturing and not self.per_group_pools:
                # (inside a captured graph, successive replays are serialised,
                # which already orders step t+1 after all of step t)
                for other in self.groups[1:]:
                    cs.wait_event(other.ev_attn[l])
            with torch.cuda.stream(cs):
                _cache()
                if gather and self.server:
                    # the job's gather may read a block sealed by an earlier step:
                    # its ready signal waits for that layer's save (if in flight)
                    self._wait_saved(l, cs)
                    # job j's ready signal, then the event the group's stream waits on:
                    # the done-flag wait below is ordered after its own job's signal in
                    # the graph's edges, so it can never sit in a hardware queue in
                    # front of the signal it depends on
                    j = l * len(self.groups) + gi
                    ops.flag_signal(self.h2d_flags[j:j + 1], stream=cs)
                g.ev_cache[l].record(cs)
            if gather and self.server and c.split_attn:
                # the hits (and the tail) are attended while the server loads the
                # misses; then the misses, then the log-sum-exp merge
                g.stream.wait_event(g.ev_cache[l])
                timed("attn", lambda: ops.sparse_decode_attn_part(
                    q, self.pool_kv_of(l, gi), g.slot[l], g.hit[l], 1, c.topk, g.tail_kv[l], g.tail_len, g.dims,
                    self.scale, g.out_h, g.lse_h, g.ws_attn, counts=g.counts[l]))
                ops.flag_wait(self.h2d_flags[self.njobs + j:self.njobs + j + 1], counts=g.counts[l],
                              stream=g.stream)
                timed("attn_miss", lambda: (
                    ops.sparse_decode_attn_part(q, self.pool_kv_of(l, gi), g.slot[l], g.hit[l], 2, c.topk,
                                                g.tail_kv[l], g.tail_len, g.dims, self.scale, g.out_m,
                                                g.lse_m, g.ws_attn, counts=g.counts[l]),
                    ops.sparse_attn_merge(g.out_h, g.lse_h, g.out_m, g.lse_m, g.out[l], counts=g.counts[l])))
                g.ev_attn[l].record(g.stream)
                return
            if gather and self.server:
                g.stream.wait_event(g.ev_cache[l])
                ops.flag_wait(self.h2d_flags[self.njobs + j:self.njobs + j + 1], counts=g.counts[l],
                              stream=g.stream)
            elif gather:
                g.h2d_stream.wait_event(g.ev_cache[l])
                with torch.cuda.stream(g.h2d_stream):
                    _gather()
                    g.ev_gather[l].record(g.h2d_stream)
                g.stream.wait_event(g.ev_gather[l])
            else:
                g.stream.wait_event(g.ev_cache[l])
        timed("attn", lambda: ops.sparse_decode_attn(q, self.pool_kv_of(l, gi), g.slot[l], c.topk,
                                                     g.tail_kv[l], g.tail_len, g.dims, self.scale,
                                                     g.out[l], g.ws_attn, counts=g.counts[l]))
        if len(self.groups) > 1:
            g.ev_attn[l].record(g.stream)

    def layer_step(self, l: int, q: torch.Tensor, stamp: int, scores: Optional[torch.Tensor] = None,
                   gather: bool = True) -> None:
        """One layer of one decode step (S1..S5) for a single-group engine."""
        assert len(self.groups) == 1
        self._group_layer(self.groups[0], l, q, stamp, 0, scores, None, gather)

    def step(self, q_all: torch.Tensor, stamp: int, timers=None, post_attn=None) -> None:
        """q_all: [L][B][Hq][d] on the device.  Enqueues one decode step of every
        layer; outputs land in each group's `out` [L][Hq][nb][d] (float32).
        post_attn(group_index, group, layer), if given, runs on the group's
        stream right after its layer-l attention (e.g. the TP all-gather)."""
        c = self.cfg
        if len(self.groups) == 1:
            for l in range(c.layers):
                self._group_layer(self.groups[0], l, q_all[l], stamp, 0, None, timers, True)
                if post_attn is not None:
                    post_attn(0, self.groups[0], l)
            return
        cur = torch.cuda.current_stream(self.device)
        if self.server:
            self.h2d_flags.zero_()     # before every stream below forks off `cur`
            self.h2d_stats.zero_()
        for g in self.groups:
            g.stream.wait_stream(cur)
        self.cache_stream.wait_stream(cur)
        for g in self.groups:
            if g.cache_stream is not None:
                g.cache_stream.wait_stream(cur)
        # (per-group select streams wait on their group stream, which waits on cur)
        for hs in self.h2d_streams:
            hs.wait_stream(cur)
        if self.server:
            hs = self.h2d_streams[0]
            with torch.cuda.stream(hs):
                tm = timers is not None and timers.wants("gather")
                if tm:
                    ts, te = timers.mark("gather", 0, 0)
                    ts.record()
                ops.flash_h2d_serve(self.host_ptr, self.host_blocks, self.h2d_jobs, self.njobs,
                                    c.block_bytes, self.h2d_flags,
                                    stats=self.h2d_stats if self.collect_h2d_stats else None)
                if tm:
                    te.record()
        # issue layer by layer, group by group: group A's FlashH2D (PCIe) overlaps
        # group B's select / attention (HBM) on the other stream
        for l in range(c.layers):
            for gi, g in enumerate(self.groups):
                with torch.cuda.stream(g.stream):
                    self._group_layer(g, l, q_all[l, g.b0:g.b1], stamp, gi, None, timers, True)
                    if post_attn is not None:
                        post_attn(gi, g, l)
        for g in self.groups:
            cur.wait_stream(g.stream)
        for hs in self.h2d_streams:
            cur.wait_stream(hs)
        # join the cache streams too (their last op, a ready-flag signal, has no
        # other consumer on the host-visible streams)
        cur.wait_stream(self.cache_stream)
        for g in self.groups:
            if g.cache_stream is not None:
                cur.wait_stream(g.cache_stream)

    def outputs(self) -> List[torch.Tensor]:
        return [g.out for g in self.groups]

    def capture_graph(self, q_static: torch.Tensor, post_attn=None, timers=None) -> "torch.cuda.CUDAGraph":
        """Capture one whole decode step (all layers, all request groups and
        streams) into a CUDA graph reading q from `q_static` [L][B][Hq][d].
        Requires device clocks on the pools (`use_device_clock()`), so each
        replay advances the LRU stamps without host-side scalars.  Replaying
        the graph replaces ~10 host launches per layer and group with one."""
        assert getattr(self, "clock", None) is not None, "call use_device_clock() first"
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        self._capturing = True
        try:
            with torch.cuda.graph(g, stream=side):
                self.clock.add_(1)      # one new LRU stamp per replayed step
                self.step(q_static, stamp=0, timers=timers, post_attn=post_attn)
        finally:
            self._capturing = False
        torch.cuda.synchronize(self.device)
        # the step events were recorded inside the capture; fresh ones keep
        # later eager steps from waiting on graph-internal records
        for grp in self.groups:
            for name in ("ev_cache", "ev_attn", "ev_gather", "ev_sel"):
                setattr(grp, name, [torch.cuda.Event() for _ in range(self.cfg.layers)])
        return g

    def use_device_clock(self, start: int) -> None:
        """Switch every pool to one shared device-side stamp counter holding
        `start` (the host `stamp` argument is then ignored).  A captured step
        increments it once per replay; eager steps in this mode must call
        `advance_clock()` before each step."""
        if getattr(self, "clock", None) is None:
            self.clock = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.clock.fill_(start)
        for p in (sum(self.gpools, []) if self.per_group_pools else self.pools):
            p.clock = self.clock

    def advance_clock(self) -> None:
        self.clock.add_(1)

    # ------------------------------------------------------- NEXT-1 save path
    def enable_save_path(self, tail_len_host: List[int], n_blk_host: List[int],
                         d2h_threads: int = 8) -> None:
        """Decode KV append + save: per-layer device staging for
        sealed blocks, a pinned DRAM landing buffer, the FlashD2H CPU-thread pool
        and a save stream.  The host mirrors of tail_len / n_blk decide (without
        a device sync) which requests' tails fill at each step."""
        c, dev = self.cfg, self.device
        self.staging = torch.empty(c.layers, c.batch * c.num_kv_heads * c.block_elems, dtype=c.dtype,
                                   device=dev)
        self.host_stage = torch.empty(c.layers, c.batch * c.num_kv_heads * c.block_elems, dtype=c.dtype,
                                      pin_memory=True)
        self.seal_ws = ops.alloc_workspace(3, self.dims, c.max_blk, c.topk, device=dev)
        self.fill_req = torch.empty(c.batch, dtype=torch.int32, device=dev)
        self.fill_req_host = torch.empty(c.batch, dtype=torch.int32, pin_memory=True)
        self.ev_fill = torch.cuda.Event()       # the last fill_req upload has been read
        self.d2h = ops.D2HEngine(d2h_threads)
        self.d2h_stream = torch.cuda.Stream(dev)
        self.ev_sealed = torch.cuda.Event()
        # ev_saved[l]: layer l's latest FlashD2H save is in DRAM (None: none in flight)
        self.ev_saved: List[Optional[torch.cuda.Event]] = [None] * c.layers
        self.tail_len_host = list(tail_len_host)
        self.n_blk_host = list(n_blk_host)
        self.req_ids_host = self.req_ids.tolist()

    def _wait_saved(self, l: int, stream) -> None:
        """Order `stream` after layer l's in-flight FlashD2H save: only the
        FlashH2D gather of a layer needs the DRAM copy of a freshly sealed
        block (it may select and miss it); select and cache never wait."""
        ev = getattr(self, "ev_saved", None)
        if ev is not None and ev[l] is not None and not self._capturing:
            stream.wait_event(ev[l])

    def append_kv(self, new_kv_all: torch.Tensor) -> None:
        """Append this step's token: new_kv_all [L][B][Hkv][2][d] (device).  Layer 0
        counts the token in tail_len; every layer writes the same tail row."""
        for l in range(self.cfg.layers):
            ops.kv_append(new_kv_all[l], self.tail_kv[l], self.tail_len, advance=(l == 0), d=self.dims)
        self.tail_len_host = [t + 1 for t in self.tail_len_host]

    def seal_full_blocks(self) -> List[int]:
        """After the step's attention: for the requests whose tail is full, build
        the metadata of the new block and stage it (kv_seal_blocks), commit
        (n_blk += 1, tail_len = 0) -- both on the current stream, a few small
        kernels -- then save the staged blocks to DRAM with FlashD2H on the save
        stream, fully in parallel with the next steps' work.  A
        later step's FlashH2D gather of layer l waits for layer l's save only
        (`_wait_saved`).  Returns the sealed request indices."""
        c = self.cfg
        fill = [b for b in range(c.batch) if self.tail_len_host[b] == BLOCK_TOKENS]
        if not fill:
            return []
        n = len(fill)
        full = [b for b in fill if self.n_blk_host[b] >= c.max_blk]
        if full:
            raise ValueError(f"requests {full} have max_blk={c.max_blk} full blocks: no row for a new block")
        cur = torch.cuda.current_stream(self.device)
        # the staging buffers are reused: the previous save of each layer first
        for l in range(c.layers):
            if self.ev_saved[l] is not None:
                cur.wait_event(self.ev_saved[l])
        self.ev_fill.synchronize()              # the pinned upload buffer is free again
        self.fill_req_host[:n].copy_(torch.tensor(fill, dtype=torch.int32))
        self.fill_req[:n].copy_(self.fill_req_host[:n], non_blocking=True)
        self.ev_fill.record(cur)
        for l in range(c.layers):
            ops.kv_seal_blocks(self.fill_req, n, self.tail_kv[l], self.n_blk, c.max_blk, self.meta[l],
                               self.staging[l], self.seal_ws, self.dims)
        ops.kv_commit(self.fill_req, n, self.n_blk, self.tail_len)
        self.ev_sealed.record(cur)
        self.d2h_stream.wait_event(self.ev_sealed)
        with torch.cuda.stream(self.d2h_stream):
            for l in range(c.layers):
                keys = [self.key0(self.req_ids_host[b], l, h) + self.n_blk_host[b]
                        for b in fill for h in range(c.num_kv_heads)]
                ops.flash_d2h_save(self.d2h, self.staging[l], self.host_stage[l], n * c.num_kv_heads,
                                   keys, self.host_kv, self.host_blocks, c.block_bytes)
                ev = torch.cuda.Event()
                ev.record(self.d2h_stream)
                self.ev_saved[l] = ev
        for b in fill:
            self.n_blk_host[b] += 1
            self.tail_len_host[b] = 0
        return fill

    def wait_saves(self) -> None:
        """The current stream waits for every in-flight FlashD2H save."""
        for l in range(self.cfg.layers):
            self._wait_saved(l, torch.cuda.current_stream(self.device))
