"""Decode-step driver: the per-layer select -> cache -> FlashH2D -> attention
sequence of PAPER.md:124 (§3.1 Model Executor) over L layers, on one stream.

PyTorch is used for device memory, pinned host memory and streams only; every
step of the path is a call into libsparseserve.so through `ops`.
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


class DecodeEngine:
    """Device state of one GPU: per-layer metadata, per-layer HBM block-cache
    pools (shared key->slot table), tail blocks, outputs and workspaces."""

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
        self.pools = [ops.CachePool(c.slots_per_layer, self.fwd, dev) for _ in range(c.layers)]
        self.pool_kv = [torch.zeros(c.slots_per_layer * c.block_elems, dtype=c.dtype, device=dev)
                        for _ in range(c.layers)]
        self.tail_kv = torch.zeros(c.layers, c.batch, c.num_kv_heads, 2, BLOCK_TOKENS, HEAD_DIM,
                                   dtype=c.dtype, device=dev)
        self.tail_len = torch.zeros(c.batch, dtype=torch.int32, device=dev)
        self.n_blk = torch.zeros(c.batch, dtype=torch.int32, device=dev)
        self.req_ids = torch.arange(c.batch, dtype=torch.int32, device=dev)
        E = c.pairs * c.topk
        self.E = E
        self.sel = torch.empty(c.layers, c.batch, c.num_kv_heads, c.topk, dtype=torch.int32, device=dev)
        self.slot = torch.empty_like(self.sel)
        self.hit = torch.empty(c.layers, c.batch, c.num_kv_heads, c.topk, dtype=torch.uint8, device=dev)
        self.miss_keys = torch.empty(c.layers, E, dtype=torch.int64, device=dev)
        self.miss_slots = torch.empty(c.layers, E, dtype=torch.int32, device=dev)
        self.counts = torch.zeros(c.layers, 4, dtype=torch.int32, device=dev)
        self.out = torch.empty(c.layers, c.num_q_heads, c.batch, HEAD_DIM, dtype=torch.float32, device=dev)
        self.ws_select = ops.alloc_workspace(SS_WS_SELECT, self.dims, c.max_blk, c.topk, device=dev)
        self.ws_cache = ops.alloc_workspace(SS_WS_CACHE, self.dims, c.max_blk, c.topk,
                                            c.slots_per_layer, device=dev)
        self.ws_attn = ops.alloc_workspace(SS_WS_ATTN, self.dims, c.max_blk, c.topk, device=dev)
        self.scale = 1.0 / math.sqrt(HEAD_DIM)
        self.host_kv: Optional[torch.Tensor] = None
        self.host_ptr = 0
        self.host_blocks = 0

    # ------------------------------------------------------------------ setup
    def set_host_kv(self, host_kv: torch.Tensor, host_blocks: int) -> None:
        """host_kv: pinned CPU tensor holding host_blocks blocks [2][32][d] (dtype)."""
        assert host_kv.is_pinned()
        assert host_kv.numel() * host_kv.element_size() >= host_blocks * self.cfg.block_bytes
        self.host_kv = host_kv
        self.host_blocks = host_blocks
        self.host_ptr = ops.host_device_pointer(host_kv)

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
    def layer_step(self, l: int, q: torch.Tensor, stamp: int, scores: Optional[torch.Tensor] = None,
                   gather: bool = True) -> None:
        """One layer of one decode step (S1..S5)."""
        c = self.cfg
        ops.ss_block_select(q, self.meta[l], self.n_blk, c.max_blk, c.topk, self.dims, self.sel[l],
                            self.ws_select, scores=scores)
        ops.kv_cache_lookup_insert(self.pools[l], self.sel[l], self.req_ids, l, c.layers, c.max_blk,
                                   c.topk, self.dims, stamp, self.slot[l], self.hit[l],
                                   self.miss_keys[l], self.miss_slots[l], self.counts[l],
                                   self.ws_cache)
        if gather:
            ops.flash_h2d_gather(self.host_ptr, self.host_blocks, self.miss_keys[l],
                                 self.miss_slots[l], self.counts[l], self.E, self.pool_kv[l],
                                 c.block_bytes)
        ops.sparse_decode_attn(q, self.pool_kv[l], self.slot[l], c.topk, self.tail_kv[l],
                               self.tail_len, self.dims, self.scale, self.out[l], self.ws_attn,
                               counts=self.counts[l])

    def step(self, q_all: torch.Tensor, stamp: int) -> torch.Tensor:
        """q_all: [L][B][Hq][d]; returns out [L][Hq][B][d] (float32, device)."""
        for l in range(self.cfg.layers):
            self.layer_step(l, q_all[l], stamp)
        return self.out
