"""Python marshalling for the C oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package.  It never
imports the CUDA path (paper_2509_24626_b200) and the CUDA path never imports
it.  Argument marshalling only: all arithmetic lives in oracle.c.

Arrays are numpy.  Storage arrays are uint16 (bf16 bit patterns) or float32.
Metadata here is in the LOGICAL layout [B][Hkv][max_blk][2][d] (min row, max
row); the CUDA path's tiled HBM layout is a pure permutation of it (see
include/sparseserve.h and tests/layout.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-shared", "-fPIC", "-std=c11"]

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.or_block_meta.argtypes = [P, I64, I64, I32, I32, P]
        L.or_block_score.argtypes = [P, P, P, I32, I32, I32, I32, I32, I32, P]
        L.or_topk.argtypes = [P, P, I32, I32, I32, I32, P]
        L.or_block_mean.argtypes = [P, I64, I64, I32, I32, P]
        L.or_block_score_mean.argtypes = [P, P, P, I32, I32, I32, I32, I32, I32, P]
        L.or_lru.argtypes = [P, I64, P, P, ctypes.c_int32, P, P, I32, I32, I32, I32, I32, I32,
                             I64, P, P, P, P, P]
        L.or_lru.restype = ctypes.c_int
        L.or_gather.argtypes = [P, I64, P, P, ctypes.c_int32, P, I64]
        L.or_attention.argtypes = [P, P, P, I32, P, P, I32, I32, I32, I32, I32, D, P]
        L.or_kv_append.argtypes = [P, P, P, I32, I32, I32, I32, I32]
        L.or_kv_seal.argtypes = [P, I32, P, P, P, I32, P, P, I32, I32, I32]
        L.or_d2h_scatter.argtypes = [P, I64, P, P, I64, I64]
        L.or_prefill_save.argtypes = [P, P, I32, I32, I32, I32, I32, I32, I32, I32, I32, P, P, P, P,
                                      P, I64]
        L.or_ws_estimate.argtypes = [P, I32, I32, I32, I32, I32, I32, I32, P]
        L.or_admit.argtypes = [P, I32, I64, P]
        L.or_admit.restype = ctypes.c_int
        _lib = L
    return _lib


def _dt(a: np.ndarray) -> int:
    if a.dtype == np.uint16:
        return 0
    if a.dtype == np.float32:
        return 1
    raise TypeError(f"storage dtype must be uint16 (bf16 bits) or float32, got {a.dtype}")


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
def block_meta(keys: np.ndarray, key_stride: Optional[int] = None) -> np.ndarray:
    """S0. keys: [n][32][d] (or blocks [n][2][32][d] with key_stride=2*32*d).
    Returns meta [n][2][d] in the same storage dtype."""
    keys = np.ascontiguousarray(keys)
    n = keys.shape[0]
    d = keys.shape[-1]
    if key_stride is None:
        key_stride = int(np.prod(keys.shape[1:]))
    out = np.empty((n, 2, d), dtype=keys.dtype)
    lib().or_block_meta(_p(keys), key_stride, n, _dt(keys), d, _p(out))
    return out


def block_score(q: np.ndarray, meta: np.ndarray, n_blk: np.ndarray) -> np.ndarray:
    """S1. q: [B][Hq][d]; meta: [B][Hkv][max_blk][2][d]; returns float64
    scores [B][Hkv][max_blk] (entries j >= n_blk[b] are NaN)."""
    q = np.ascontiguousarray(q)
    meta = np.ascontiguousarray(meta)
    assert q.dtype == meta.dtype
    B, Hq, d = q.shape
    _, Hkv, max_blk, _, _ = meta.shape
    n_blk = np.ascontiguousarray(n_blk, dtype=np.int32)
    out = np.full((B, Hkv, max_blk), np.nan, dtype=np.float64)
    lib().or_block_score(_p(q), _p(meta), _p(n_blk), B, Hq, Hkv, d, max_blk, _dt(q), _p(out))
    return out


def block_mean(keys: np.ndarray, key_stride: Optional[int] = None) -> np.ndarray:
    """NEXT-3 mean-of-keys metadata. keys: [n][32][d] (or blocks [n][2][32][d]
    with key_stride=2*32*d).  Returns float32 [n][d]."""
    keys = np.ascontiguousarray(keys)
    n = keys.shape[0]
    d = keys.shape[-1]
    if key_stride is None:
        key_stride = int(np.prod(keys.shape[1:]))
    out = np.empty((n, d), dtype=np.float32)
    lib().or_block_mean(_p(keys), key_stride, n, _dt(keys), d, _p(out))
    return out


def block_score_mean(q: np.ndarray, meta: np.ndarray, n_blk: np.ndarray) -> np.ndarray:
    """NEXT-3 score. q: [B][Hq][d] (uint16 bf16 bits or float32); meta: float32
    [B][Hkv][max_blk][d]; returns float64 [B][Hkv][max_blk] (NaN for j >= n_blk)."""
    q = np.ascontiguousarray(q)
    meta = np.ascontiguousarray(meta, dtype=np.float32)
    B, Hq, d = q.shape
    _, Hkv, max_blk, _ = meta.shape
    n_blk = np.ascontiguousarray(n_blk, dtype=np.int32)
    out = np.full((B, Hkv, max_blk), np.nan, dtype=np.float64)
    lib().or_block_score_mean(_p(q), _p(meta), _p(n_blk), B, Hq, Hkv, d, max_blk, _dt(q), _p(out))
    return out


def topk(scores: np.ndarray, n_blk: np.ndarray, k: int) -> np.ndarray:
    """S2. returns sel int32 [B][Hkv][k], ascending, -1 padded."""
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    B, Hkv, max_blk = scores.shape
    n_blk = np.ascontiguousarray(n_blk, dtype=np.int32)
    sel = np.empty((B, Hkv, k), dtype=np.int32)
    lib().or_topk(_p(scores), _p(n_blk), B, Hkv, max_blk, k, _p(sel))
    return sel


class Pool:
    """Oracle-side cache state of one (GPU, layer) pool (S3) plus its KV bytes."""

    def __init__(self, num_slots: int, fwd_len: int, block_bytes: int = 0):
        self.fwd = np.full(fwd_len, -1, dtype=np.int32)
        self.slot_key = np.full(num_slots, -1, dtype=np.int64)
        self.slot_stamp = np.full(num_slots, -1, dtype=np.int64)
        self.kv = np.zeros((num_slots, block_bytes), dtype=np.uint8) if block_bytes else None

    @property
    def num_slots(self) -> int:
        return self.slot_key.shape[0]

    def copy(self) -> "Pool":
        p = Pool.__new__(Pool)
        p.fwd = self.fwd.copy()
        p.slot_key = self.slot_key.copy()
        p.slot_stamp = self.slot_stamp.copy()
        p.kv = None if self.kv is None else self.kv.copy()
        return p


def lru(pool: Pool, sel: np.ndarray, req_ids: np.ndarray, layer: int, num_layers: int,
        max_blk: int, stamp: int):
    """S3. Mutates pool (fwd/slot_key/slot_stamp).  Returns a dict with
    slot, hit, miss_keys, miss_slots, counts."""
    sel = np.ascontiguousarray(sel, dtype=np.int32)
    B, Hkv, k = sel.shape
    req_ids = np.ascontiguousarray(req_ids, dtype=np.int32)
    E = B * Hkv * k
    slot = np.empty((B, Hkv, k), dtype=np.int32)
    hit = np.empty((B, Hkv, k), dtype=np.uint8)
    miss_keys = np.full(max(E, 1), -1, dtype=np.int64)
    miss_slots = np.full(max(E, 1), -1, dtype=np.int32)
    counts = np.zeros(4, dtype=np.int32)
    lib().or_lru(_p(pool.fwd), pool.fwd.shape[0], _p(pool.slot_key), _p(pool.slot_stamp),
                 pool.num_slots, _p(sel), _p(req_ids), layer, num_layers, B, Hkv, max_blk, k,
                 int(stamp), _p(slot), _p(hit), _p(miss_keys), _p(miss_slots), _p(counts))
    m = int(counts[1]) if counts[3] == 0 else 0
    return dict(slot=slot, hit=hit, miss_keys=miss_keys[:m].copy(),
                miss_slots=miss_slots[:m].copy(), counts=counts)


def gather(host_kv: np.ndarray, host_blocks: int, miss_keys: np.ndarray,
           miss_slots: np.ndarray, pool_kv: np.ndarray) -> None:
    """S4. host_kv: uint8 view [host_blocks][block_bytes]; pool_kv: uint8
    [S][block_bytes] (mutated)."""
    host_kv = np.ascontiguousarray(host_kv)
    miss_keys = np.ascontiguousarray(miss_keys, dtype=np.int64)
    miss_slots = np.ascontiguousarray(miss_slots, dtype=np.int32)
    bb = pool_kv.shape[1]
    assert pool_kv.flags["C_CONTIGUOUS"]
    lib().or_gather(_p(host_kv), int(host_blocks), _p(miss_keys), _p(miss_slots),
                    int(miss_keys.shape[0]), _p(pool_kv), bb)


def attention(q: np.ndarray, pool_kv: np.ndarray, slot: np.ndarray, tail: np.ndarray,
              tail_len: np.ndarray, scale: float) -> np.ndarray:
    """S5. q: [B][Hq][d] storage; pool_kv: [S][2][32][d] storage (same dtype);
    slot: [B][Hkv][k]; tail: [B][Hkv][2][32][d]; returns float64 [Hq][B][d]."""
    q = np.ascontiguousarray(q)
    pool_kv = np.ascontiguousarray(pool_kv)
    tail = np.ascontiguousarray(tail)
    assert q.dtype == pool_kv.dtype == tail.dtype
    slot = np.ascontiguousarray(slot, dtype=np.int32)
    tail_len = np.ascontiguousarray(tail_len, dtype=np.int32)
    B, Hq, d = q.shape
    _, Hkv, k = slot.shape
    out = np.empty((Hq, B, d), dtype=np.float64)
    lib().or_attention(_p(q), _p(pool_kv), _p(slot), k, _p(tail), _p(tail_len), B, Hq, Hkv, d,
                       _dt(q), float(scale), _p(out))
    return out


def decode_layer(q, meta, n_blk, k, pool: Pool, req_ids, layer, num_layers, max_blk, stamp,
                 host_kv_u8, host_blocks, tail, tail_len, scale):
    """One layer of the decode step, S1..S5, in the paper's order:
    score -> top-k -> cache lookup/insert -> FlashH2D gather -> attention."""
    scores = block_score(q, meta, n_blk)
    sel = topk(scores, n_blk, k)
    r = lru(pool, sel, req_ids, layer, num_layers, max_blk, stamp)
    out = None
    if r["counts"][3] == 0:
        gather(host_kv_u8, host_blocks, r["miss_keys"], r["miss_slots"], pool.kv)
        d = q.shape[-1]
        pool_view = pool.kv.view(q.dtype).reshape(pool.num_slots, 2, 32, d)
        out = attention(q, pool_view, r["slot"], tail, tail_len, scale)
    return dict(scores=scores, sel=sel, out=out, **r)


# --------------------------------------------------------------------------
# NEXT-1: decode KV append + save path
# --------------------------------------------------------------------------
def kv_append(new_kv: np.ndarray, tail: np.ndarray, tail_len: np.ndarray, advance: bool) -> None:
    """new_kv [B][Hkv][2][d]; tail [B][Hkv][2][32][d] (mutated); tail_len int32 [B] (mutated)."""
    assert new_kv.dtype == tail.dtype and tail.flags["C_CONTIGUOUS"]
    assert tail_len.dtype == np.int32 and tail_len.flags["C_CONTIGUOUS"]
    new_kv = np.ascontiguousarray(new_kv)
    B, Hkv, _, d = new_kv.shape
    lib().or_kv_append(_p(new_kv), _p(tail), _p(tail_len), int(bool(advance)), B, Hkv, d, _dt(new_kv))


def kv_seal(fill_req, tail: np.ndarray, tail_len: np.ndarray, n_blk: np.ndarray, meta: np.ndarray) -> np.ndarray:
    """Seal the full tails of fill_req: metadata into meta [B][Hkv][max_blk][2][d]
    (mutated), counters committed; returns the staging blocks [n][Hkv][2][32][d]."""
    fill = np.ascontiguousarray(np.asarray(fill_req, dtype=np.int32))
    B, Hkv, _, _, d = tail.shape
    max_blk = meta.shape[2]
    staging = np.empty((fill.shape[0], Hkv, 2, 32, d), dtype=tail.dtype)
    assert meta.flags["C_CONTIGUOUS"] and n_blk.dtype == np.int32 and tail_len.dtype == np.int32
    lib().or_kv_seal(_p(fill), int(fill.shape[0]), _p(np.ascontiguousarray(tail)), _p(tail_len),
                     _p(n_blk), max_blk, _p(meta), _p(staging), Hkv, d, _dt(tail))
    return staging


def d2h_scatter(staging_u8: np.ndarray, keys, host_kv_u8: np.ndarray, host_blocks: int) -> None:
    """staging_u8 [n][block_bytes]; host_kv_u8 [host_blocks][block_bytes] (mutated)."""
    keys = np.ascontiguousarray(np.asarray(keys, dtype=np.int64))
    staging_u8 = np.ascontiguousarray(staging_u8)
    bb = staging_u8.shape[1]
    lib().or_d2h_scatter(_p(staging_u8), int(keys.shape[0]), _p(keys), _p(host_kv_u8), host_blocks, bb)


# --------------------------------------------------------------------------
# NEXT-4: layer-segmented prefill, storage side
# --------------------------------------------------------------------------
def prefill_save(k_nhd: np.ndarray, v_nhd: np.ndarray, b: int, req: int, layer: int, num_layers: int,
                 meta: np.ndarray, tail: np.ndarray, n_blk: np.ndarray, tail_len: np.ndarray,
                 host_kv_u8: np.ndarray, host_blocks: int) -> None:
    """k/v [n][Hkv][d]; meta [B][Hkv][max_blk][2][d], tail [B][Hkv][2][32][d], n_blk/tail_len
    int32 [B] and host_kv_u8 [host_blocks][block_bytes] are mutated."""
    k_nhd = np.ascontiguousarray(k_nhd)
    v_nhd = np.ascontiguousarray(v_nhd)
    n, Hkv, d = k_nhd.shape
    max_blk = meta.shape[2]
    for a in (meta, tail, n_blk, tail_len, host_kv_u8):
        assert a.flags["C_CONTIGUOUS"]
    lib().or_prefill_save(_p(k_nhd), _p(v_nhd), n, b, req, layer, num_layers, max_blk, Hkv, d,
                          _dt(k_nhd), _p(meta), _p(tail), _p(n_blk), _p(tail_len), _p(host_kv_u8),
                          int(host_blocks))


def ws_estimate(hist: np.ndarray, max_blk: int, w: int) -> np.ndarray:
    """NEXT-2: hist int32 [T][L][B][Hkv][k] -> ws int64 [T][B] (blocks)."""
    hist = np.ascontiguousarray(hist, dtype=np.int32)
    T, L, B, Hkv, k = hist.shape
    ws = np.zeros((T, B), np.int64)
    lib().or_ws_estimate(_p(hist), T, L, B, Hkv, k, max_blk, w, _p(ws))
    return ws


def admit(m_req, m_avl: int) -> list:
    """Algorithm 1 lines 6-14: per request, True = added, False = reset."""
    m = np.ascontiguousarray(np.asarray(m_req, dtype=np.int64).reshape(-1))
    out = np.zeros(max(len(m), 1), np.uint8)
    lib().or_admit(_p(m), len(m), int(m_avl), _p(out))
    return [bool(x) for x in out[:len(m)]]
