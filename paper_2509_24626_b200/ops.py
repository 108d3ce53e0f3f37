"""Thin Python binding of the C ABI (same names as include/sparseserve.h).

Argument marshalling only: torch tensors -> raw pointers + sizes + the current
CUDA stream.  Every step of the hot path runs in the CUDA kernels of
libsparseserve.so; nothing here computes.  Tensors must be contiguous and on
the current CUDA device (host KV: pinned CPU tensor).
"""
from __future__ import annotations

from typing import Optional

import torch

from . import _lib
from ._lib import SSCachePool, SSDims, check

HEAD_DIM = 128
BLOCK_TOKENS = 32


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.SS_BF16
    if t.dtype == torch.float32:
        return _lib.SS_F32
    raise TypeError(f"unsupported dtype {t.dtype} (bf16 or float32)")


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def dims(batch: int, num_q_heads: int, num_kv_heads: int) -> SSDims:
    return SSDims(batch, num_q_heads, num_kv_heads, HEAD_DIM, BLOCK_TOKENS)


def workspace_size(which: int, d: SSDims, max_blk: int, k: int, num_slots: int = 0) -> int:
    return int(_lib.load().ss_workspace_size(which, d, max_blk, k, num_slots))


def alloc_workspace(which: int, d: SSDims, max_blk: int, k: int, num_slots: int = 0,
                    device=None) -> torch.Tensor:
    n = workspace_size(which, d, max_blk, k, num_slots)
    return torch.zeros(max(n, 256), dtype=torch.uint8, device=device or "cuda")


def meta_numel(batch: int, num_kv_heads: int, max_blk: int) -> int:
    """Elements of a (tiled) metadata array for [B][Hkv][max_blk] blocks."""
    assert max_blk % 32 == 0
    return batch * num_kv_heads * max_blk * 2 * HEAD_DIM


# ---------------------------------------------------------------------------
def block_meta_update(keys: torch.Tensor, meta: torch.Tensor, n: int, key_stride: int,
                      dst_idx: Optional[torch.Tensor] = None, stream=None) -> None:
    """S0: meta[dst_idx[i]] = {min, max} over the 32 keys at keys + i*key_stride."""
    if dst_idx is not None:
        assert dst_idx.dtype == torch.int64
    check(_lib.load().block_meta_update(_ptr(keys), key_stride, _ptr(dst_idx), n, _ptr(meta),
                                        _dt(keys), HEAD_DIM, _stream(stream)),
          "block_meta_update")


def ss_block_select(q: torch.Tensor, meta: torch.Tensor, n_blk: torch.Tensor, max_blk: int,
                    k: int, d: SSDims, sel: torch.Tensor, ws: torch.Tensor,
                    scores: Optional[torch.Tensor] = None, stream=None) -> None:
    """S1+S2: sel[b][h][:k] = ascending top-k block ids (-1 padded)."""
    assert n_blk.dtype == torch.int32 and sel.dtype == torch.int32
    if scores is not None:
        assert scores.dtype == torch.float64
    check(_lib.load().ss_block_select(_ptr(q), _ptr(meta), _ptr(n_blk), max_blk, k, d, _dt(q),
                                      _ptr(sel), _ptr(scores), _ptr(ws), ws.numel(),
                                      _stream(stream)), "ss_block_select")


def mean_meta_numel(batch: int, num_kv_heads: int, max_blk: int) -> int:
    """float32 elements of a (tiled) NEXT-3 mean-metadata array."""
    assert max_blk % 32 == 0
    return batch * num_kv_heads * max_blk * HEAD_DIM


def block_meta_update_mean(keys: torch.Tensor, meta: torch.Tensor, n: int, key_stride: int,
                           dst_idx: Optional[torch.Tensor] = None, stream=None) -> None:
    """NEXT-3 S0: meta[dst_idx[i]] = float32 mean of the 32 keys at keys + i*key_stride."""
    assert meta.dtype == torch.float32
    if dst_idx is not None:
        assert dst_idx.dtype == torch.int64
    check(_lib.load().block_meta_update_mean(_ptr(keys), key_stride, _ptr(dst_idx), n, _ptr(meta),
                                             _dt(keys), HEAD_DIM, _stream(stream)),
          "block_meta_update_mean")


def ss_block_select_mean(q: torch.Tensor, meta: torch.Tensor, n_blk: torch.Tensor, max_blk: int,
                         k: int, d: SSDims, sel: torch.Tensor, ws: torch.Tensor,
                         scores: Optional[torch.Tensor] = None, stream=None) -> None:
    """NEXT-3 S1+S2 over mean metadata: top-k of max_g q_g . mu_j."""
    assert n_blk.dtype == torch.int32 and sel.dtype == torch.int32 and meta.dtype == torch.float32
    if scores is not None:
        assert scores.dtype == torch.float64
    check(_lib.load().ss_block_select_mean(_ptr(q), _ptr(meta), _ptr(n_blk), max_blk, k, d, _dt(q),
                                           _ptr(sel), _ptr(scores), _ptr(ws), ws.numel(),
                                           _stream(stream)), "ss_block_select_mean")


class CachePool:
    """Device arrays of one (GPU, layer) HBM block-cache pool (S3 state)."""

    def __init__(self, num_slots: int, fwd: torch.Tensor, device=None, clock: bool = False):
        device = device or fwd.device
        self.fwd = fwd                       # int32 [fwd_len], may be shared across layers
        self.slot_key = torch.full((num_slots,), -1, dtype=torch.int64, device=device)
        self.slot_stamp = torch.full((num_slots,), -1, dtype=torch.int64, device=device)
        self.order = torch.arange(num_slots, dtype=torch.int32, device=device)
        self.order_pos = torch.arange(num_slots, dtype=torch.int32, device=device)
        self.num_slots = num_slots
        # device-side stamp counter (graph-replayable steps); None = host stamps
        self.clock = torch.zeros(1, dtype=torch.int64, device=device) if clock else None

    def c_struct(self) -> SSCachePool:
        return SSCachePool(self.fwd.data_ptr(), self.fwd.numel(), self.slot_key.data_ptr(),
                           self.slot_stamp.data_ptr(), self.order.data_ptr(),
                           self.order_pos.data_ptr(), self.num_slots,
                           self.clock.data_ptr() if self.clock is not None else None)


def kv_cache_lookup_insert(pool: CachePool, sel: torch.Tensor, req_ids: torch.Tensor, layer: int,
                           num_layers: int, max_blk: int, k: int, d: SSDims, stamp: int,
                           slot_out: torch.Tensor, hit_out: torch.Tensor, miss_keys: torch.Tensor,
                           miss_slots: torch.Tensor, counts: torch.Tensor, ws: torch.Tensor,
                           stream=None) -> None:
    """S3: batch-LRU lookup/insert; counts = {hits, misses, evictions, status} (device)."""
    assert sel.dtype == torch.int32 and req_ids.dtype == torch.int32
    assert hit_out.dtype == torch.uint8 and miss_keys.dtype == torch.int64
    assert miss_slots.dtype == torch.int32 and counts.dtype == torch.int32
    check(_lib.load().kv_cache_lookup_insert(pool.c_struct(), _ptr(sel), _ptr(req_ids), layer,
                                             num_layers, max_blk, k, d, int(stamp),
                                             _ptr(slot_out), _ptr(hit_out), _ptr(miss_keys),
                                             _ptr(miss_slots), _ptr(counts), _ptr(ws), ws.numel(),
                                             _stream(stream)), "kv_cache_lookup_insert")


def host_device_pointer(host: torch.Tensor) -> int:
    """Device address of a pinned host tensor."""
    assert host.is_pinned(), "host KV must be pinned (page-locked) memory"
    import ctypes
    out = ctypes.c_void_p()
    check(_lib.load().ss_host_device_pointer(host.data_ptr(), ctypes.byref(out)),
          "ss_host_device_pointer")
    return int(out.value)


class HostPool:
    """Page-locked, device-mapped host memory for the host KV pool, on the NUMA
    node of `device` (ss_host_alloc; freed on close / garbage collection).
    `tensor` is a CPU uint8 view of it, `dev_ptr` its device address."""

    def __init__(self, nbytes: int, device: int = 0, numa_node: Optional[int] = None):
        import ctypes
        lib = _lib.load()
        self.numa_node = int(lib.ss_device_numa_node(device)) if numa_node is None else int(numa_node)
        h, d, bound = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int32(0)
        check(lib.ss_host_alloc(nbytes, self.numa_node, ctypes.byref(h), ctypes.byref(d), ctypes.byref(bound)),
              "ss_host_alloc")
        self.host_ptr, self.dev_ptr, self.nbytes = int(h.value), int(d.value), int(nbytes)
        self.numa_bound = bool(bound.value)
        buf = (ctypes.c_uint8 * nbytes).from_address(self.host_ptr)
        self.tensor = torch.frombuffer(buf, dtype=torch.uint8)

    def close(self) -> None:
        if self.host_ptr:
            self.tensor = None
            _lib.load().ss_host_free(self.host_ptr, self.nbytes)
            self.host_ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def decode_step_host(graph: "torch.cuda.CUDAGraph", q_host: torch.Tensor, q_dev: torch.Tensor,
                     outs_dev, outs_host, stream=None) -> None:
    """One captured decode step from host buffers (ss_decode_step_host): q_host
    (pinned) -> q_dev, graph launch, outs_dev[i] -> outs_host[i] (pinned)."""
    import ctypes
    n = len(outs_dev)
    assert q_host.is_pinned() and all(o.is_pinned() for o in outs_host) and n == len(outs_host)
    assert q_host.numel() * q_host.element_size() == q_dev.numel() * q_dev.element_size()
    dev = (ctypes.c_void_p * max(1, n))(*[_ptr(o) for o in outs_dev])
    host = (ctypes.c_void_p * max(1, n))(*[o.data_ptr() for o in outs_host])
    nbytes = (ctypes.c_size_t * max(1, n))(*[o.numel() * o.element_size() for o in outs_dev])
    for od, oh in zip(outs_dev, outs_host):
        assert od.numel() * od.element_size() == oh.numel() * oh.element_size()
    check(_lib.load().ss_decode_step_host(graph.raw_cuda_graph_exec(), q_host.data_ptr(), _ptr(q_dev),
                                          q_host.numel() * q_host.element_size(), n, dev, host, nbytes,
                                          _stream(stream)), "ss_decode_step_host")


def flash_h2d_gather(host_kv_dev_ptr: int, host_blocks: int, miss_keys: torch.Tensor,
                     miss_slots: torch.Tensor, counts: torch.Tensor, max_misses: int,
                     pool_kv: torch.Tensor, block_bytes: int, stream=None) -> None:
    """S4: pool_kv[miss_slots[i]] <- host_kv[miss_keys[i] % host_blocks], i < counts[1]."""
    check(_lib.load().flash_h2d_gather(host_kv_dev_ptr, host_blocks, _ptr(miss_keys),
                                       _ptr(miss_slots), _ptr(counts), max_misses,
                                       _ptr(pool_kv), block_bytes, _stream(stream)),
          "flash_h2d_gather")


def h2d_jobs(jobs, device=None) -> torch.Tensor:
    """Device array of ss_h2d_job for flash_h2d_serve.  jobs: list of
    (miss_keys int64, miss_slots int32, counts int32[4], pool_kv, max_misses)."""
    arr = (_lib.SSH2DJob * len(jobs))()
    for i, (mk, ms, cnt, pool, mm) in enumerate(jobs):
        assert mk.dtype == torch.int64 and ms.dtype == torch.int32 and cnt.dtype == torch.int32
        arr[i] = _lib.SSH2DJob(_ptr(mk), _ptr(ms), _ptr(cnt), _ptr(pool), int(mm), 0)
    raw = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8)
    return raw.to(device or "cuda")


def h2d_flags(njobs: int, device=None) -> torch.Tensor:
    """Zeroed flag words for flash_h2d_serve (SS_H2D_FLAGS(njobs) = 4*njobs + 1 int32)."""
    return torch.zeros(4 * njobs + 1, dtype=torch.int32, device=device or "cuda")


def h2d_stats(device=None) -> torch.Tensor:
    """Zeroed server statistics words (SS_H2D_STATS uint64, held as int64)."""
    return torch.zeros(_lib.SS_H2D_STATS, dtype=torch.int64, device=device or "cuda")


def flash_h2d_serve(host_kv_dev_ptr: int, host_blocks: int, jobs: torch.Tensor, njobs: int,
                    block_bytes: int, flags: torch.Tensor, timeout_us: int = 0,
                    stats: Optional[torch.Tensor] = None, stream=None) -> None:
    """S4, pipelined: one persistent launch serves njobs gathers (job j once
    flags[j] != 0; sets flags[njobs + j] = 1 when its blocks are in HBM, 2 if
    the server aborted).  timeout_us <= 0: 3 s."""
    assert flags.dtype == torch.int32 and flags.numel() >= 4 * njobs + 1
    if stats is not None:
        assert stats.dtype == torch.int64 and stats.numel() >= _lib.SS_H2D_STATS
    check(_lib.load().flash_h2d_serve(host_kv_dev_ptr, host_blocks, _ptr(jobs), njobs, block_bytes,
                                      _ptr(flags), int(timeout_us), _ptr(stats), _stream(stream)),
          "flash_h2d_serve")


def preload_kernels() -> None:
    """Load every kernel of the library now (see ss_preload_kernels)."""
    check(_lib.load().ss_preload_kernels(), "ss_preload_kernels")


def flag_signal(flag: torch.Tensor, stream=None) -> None:
    """*flag = 1 after prior work on the stream (flag: one int32 element view)."""
    check(_lib.load().ss_flag_signal(flag.data_ptr(), _stream(stream)), "ss_flag_signal")


def flag_wait(flag: torch.Tensor, counts: Optional[torch.Tensor] = None, timeout_us: int = 0,
              stream=None) -> None:
    """Later work on the stream waits until *flag != 0; an aborted job (flag 2)
    or a timed-out wait sets counts[3] = SS_ERR_CUDA (when counts is given)."""
    if counts is not None:
        assert counts.dtype == torch.int32
    check(_lib.load().ss_flag_wait(flag.data_ptr(), _ptr(counts), int(timeout_us), _stream(stream)),
          "ss_flag_wait")


def sparse_decode_attn(q: torch.Tensor, pool_kv: torch.Tensor, slot: torch.Tensor, k: int,
                       tail_kv: torch.Tensor, tail_len: torch.Tensor, d: SSDims, scale: float,
                       out: torch.Tensor, ws: torch.Tensor, counts: Optional[torch.Tensor] = None,
                       stream=None) -> None:
    """S5: out[hq][b][:] = softmax(q K^T * scale) V over the selected blocks + tail."""
    assert out.dtype == torch.float32 and slot.dtype == torch.int32
    check(_lib.load().sparse_decode_attn(_ptr(q), _ptr(pool_kv), _ptr(slot), k, _ptr(tail_kv),
                                         _ptr(tail_len), d, _dt(q), float(scale), _ptr(counts),
                                         _ptr(out), _ptr(ws), ws.numel(), _stream(stream)),
          "sparse_decode_attn")


def sparse_decode_attn_part(q: torch.Tensor, pool_kv: torch.Tensor, slot: torch.Tensor,
                            hit: Optional[torch.Tensor], mode: int, k: int, tail_kv: torch.Tensor,
                            tail_len: torch.Tensor, d: SSDims, scale: float, out: torch.Tensor,
                            lse: torch.Tensor, ws: torch.Tensor, counts: Optional[torch.Tensor] = None,
                            stream=None) -> None:
    """S5 over a subset (mode 0 all, 1 hits + tail, 2 misses) with its log2-domain LSE."""
    assert out.dtype == torch.float32 and lse.dtype == torch.float32 and slot.dtype == torch.int32
    check(_lib.load().sparse_decode_attn_part(_ptr(q), _ptr(pool_kv), _ptr(slot), _ptr(hit), mode, k,
                                              _ptr(tail_kv), _ptr(tail_len), d, _dt(q), float(scale),
                                              _ptr(counts), _ptr(out), _ptr(lse), _ptr(ws), ws.numel(),
                                              _stream(stream)), "sparse_decode_attn_part")


def sparse_attn_merge(out_a: torch.Tensor, lse_a: torch.Tensor, out_b: torch.Tensor,
                      lse_b: torch.Tensor, out: torch.Tensor, counts: Optional[torch.Tensor] = None,
                      stream=None) -> None:
    """out = log-sum-exp combination of two disjoint-subset attention results."""
    rows = lse_a.numel()
    check(_lib.load().sparse_attn_merge(_ptr(out_a), _ptr(lse_a), _ptr(out_b), _ptr(lse_b), rows,
                                        _ptr(counts), _ptr(out), _stream(stream)), "sparse_attn_merge")


# ---------------------------------------------------------------------------
# NEXT-1: decode KV append + save path (FlashD2H)
# ---------------------------------------------------------------------------
def kv_append(new_kv: torch.Tensor, tail_kv: torch.Tensor, tail_len: torch.Tensor, advance: bool,
              d: SSDims, stream=None) -> None:
    """Write this step's K/V rows [B][Hkv][2][d] into row tail_len-1 of the tails
    (tail_len incremented first when `advance`)."""
    assert tail_len.dtype == torch.int32
    check(_lib.load().kv_append(_ptr(new_kv), _ptr(tail_kv), _ptr(tail_len), int(bool(advance)), d,
                                _dt(new_kv), _stream(stream)), "kv_append")


def kv_seal_blocks(fill_req: torch.Tensor, n_fill: int, tail_kv: torch.Tensor, n_blk: torch.Tensor,
                   max_blk: int, meta: torch.Tensor, staging: torch.Tensor, ws: torch.Tensor,
                   d: SSDims, stream=None) -> None:
    """Metadata + contiguous staging copy of the full tails of fill_req[:n_fill]."""
    assert fill_req.dtype == torch.int32 and n_blk.dtype == torch.int32
    check(_lib.load().kv_seal_blocks(_ptr(fill_req), n_fill, _ptr(tail_kv), _ptr(n_blk), max_blk,
                                     _ptr(meta), _ptr(staging), _ptr(ws), ws.numel(), d,
                                     _dt(tail_kv), _stream(stream)), "kv_seal_blocks")


def kv_commit(fill_req: torch.Tensor, n_fill: int, n_blk: torch.Tensor, tail_len: torch.Tensor,
              stream=None) -> None:
    check(_lib.load().kv_commit(_ptr(fill_req), n_fill, _ptr(n_blk), _ptr(tail_len),
                                _stream(stream)), "kv_commit")


class D2HEngine:
    """FlashD2H CPU-thread pool (owned here, freed on close/garbage collection)."""

    def __init__(self, num_threads: int = 8):
        import ctypes
        h = ctypes.c_void_p()
        check(_lib.load().ss_d2h_create(num_threads, ctypes.byref(h)), "ss_d2h_create")
        self.handle = h.value

    def close(self) -> None:
        if self.handle:
            _lib.load().ss_d2h_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def flash_d2h_save(engine: D2HEngine, staging: torch.Tensor, host_buf: torch.Tensor, n_blocks: int,
                   keys_host, host_kv: torch.Tensor, host_blocks: int, block_bytes: int,
                   stream=None) -> None:
    """One D2H copy of n_blocks staged blocks into pinned host_buf, then CPU-thread
    scatter to host_kv[key % host_blocks] (keys: host int64 sequence)."""
    import ctypes
    import numpy as np
    keys = np.ascontiguousarray(np.asarray(keys_host, dtype=np.int64))
    assert keys.shape[0] >= n_blocks
    check(_lib.load().flash_d2h_save(engine.handle, _ptr(staging), host_buf.data_ptr(), n_blocks,
                                     keys.ctypes.data_as(ctypes.c_void_p), host_kv.data_ptr(),
                                     host_blocks, block_bytes, _stream(stream)), "flash_d2h_save")


# ---------------------------------------------------------------------------
# NEXT-2: decoding working set (w-step union of selections) + Algorithm 1
# ---------------------------------------------------------------------------
class WorkingSetState:
    """Per-layer last-selected steps and selection rings + per-request counts."""

    def __init__(self, layers: int, batch: int, num_kv_heads: int, max_blk: int, k: int, w: int = 12,
                 device=None):
        device = device or "cuda"
        self.w = w
        self.last_sel = torch.full((layers, batch, num_kv_heads, max_blk), -(1 << 30),
                                   dtype=torch.int32, device=device)
        self.ring = torch.full((layers, w, batch, num_kv_heads, k), -1, dtype=torch.int32, device=device)
        self.ws_count = torch.zeros(batch, dtype=torch.int32, device=device)


def ws_track(state: WorkingSetState, layer: int, sel: torch.Tensor, k: int, d: SSDims, max_blk: int,
             t: int, stream=None) -> None:
    check(_lib.load().ws_track(_ptr(sel), k, d, max_blk, int(t), state.w, _ptr(state.last_sel[layer]),
                               _ptr(state.ring[layer]), _ptr(state.ws_count), _stream(stream)),
          "ws_track")


def ss_admit(ws_bytes, m_avl: int):
    """Algorithm 1 admission over candidates in order; returns a bool list."""
    import ctypes
    import numpy as np
    ws = np.ascontiguousarray(np.asarray(ws_bytes, dtype=np.int64))
    out = np.zeros(ws.shape[0], dtype=np.uint8)
    n = _lib.load().ss_admit(ws.ctypes.data_as(ctypes.c_void_p), int(ws.shape[0]), int(m_avl),
                             out.ctypes.data_as(ctypes.c_void_p))
    if n < 0:
        raise _lib.SparseServeError("ss_admit: invalid arguments")
    return [bool(x) for x in out]


# ---------------------------------------------------------------------------
# NEXT-4: layer-segmented prefill, storage side
# ---------------------------------------------------------------------------
def prefill_layer_save(k_nhd: torch.Tensor, v_nhd: torch.Tensor, n_tok: int, b: int, req: int,
                       layer: int, num_layers: int, max_blk: int, d: SSDims, staging: torch.Tensor,
                       meta: torch.Tensor, tail_kv: torch.Tensor, n_blk: torch.Tensor,
                       tail_len: torch.Tensor, host_kv: torch.Tensor, host_blocks: int,
                       ws: torch.Tensor, stream=None) -> None:
    """(N,H,D) prefill KV of one layer -> per-head blocks + metadata + DMA save to DRAM + tail."""
    assert host_kv.is_pinned()
    check(_lib.load().prefill_layer_save(_ptr(k_nhd), _ptr(v_nhd), n_tok, b, req, layer, num_layers,
                                         max_blk, d, _dt(k_nhd), _ptr(staging), _ptr(meta),
                                         _ptr(tail_kv), _ptr(n_blk), _ptr(tail_len),
                                         host_kv.data_ptr(), host_blocks, _ptr(ws), ws.numel(),
                                         _stream(stream)), "prefill_layer_save")
