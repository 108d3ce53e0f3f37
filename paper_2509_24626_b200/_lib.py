"""ctypes loader for libsparseserve.so (the C ABI in include/sparseserve.h).

There is no fallback: if the library is missing or fails to load, importing
the ops raises.  Build it with `python -m paper_2509_24626_b200.build` or
`__graft_entry__.build()`.
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# SS_LIB_VARIANT=debug loads libsparseserve_debug.so (built with -DSS_DEBUG_KNOBS:
# the development A/B environment knobs; tools/ and a few subprocess tests only)
LIB_PATH = os.path.join(PKG, "libsparseserve_debug.so" if os.environ.get("SS_LIB_VARIANT") == "debug"
                        else "libsparseserve.so")

SS_OK, SS_ERR_INVALID_ARG, SS_ERR_UNSUPPORTED, SS_ERR_CAPACITY, SS_ERR_CUDA = range(5)
SS_BF16, SS_F32 = 0, 1
SS_H2D_STATS = 8
SS_H2D_DONE_SERVED, SS_H2D_DONE_ABORTED = 1, 2
SS_WS_SELECT, SS_WS_CACHE, SS_WS_ATTN, SS_WS_SEAL, SS_WS_PREFILL = 0, 1, 2, 3, 4

EXPORTS = ("block_meta_update", "ss_block_select", "kv_cache_lookup_insert", "flash_h2d_gather",
           "sparse_decode_attn", "ss_workspace_size", "ss_host_device_pointer",
           "ss_status_string", "ss_version", "kv_append", "kv_seal_blocks", "kv_commit",
           "ss_d2h_create", "ss_d2h_destroy", "flash_d2h_save", "ws_track", "ss_admit", "prefill_layer_save",
           "block_meta_update_mean", "ss_block_select_mean", "flash_h2d_serve", "ss_flag_signal",
           "ss_flag_wait", "ss_preload_kernels",
           "sparse_decode_attn_part", "sparse_attn_merge", "ss_device_numa_node", "ss_host_alloc",
           "ss_host_free", "ss_decode_step_host")


class SSDims(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("block_tokens", ctypes.c_int32)]


class SSCachePool(ctypes.Structure):
    _fields_ = [("fwd", ctypes.c_void_p), ("fwd_len", ctypes.c_int64),
                ("slot_key", ctypes.c_void_p), ("slot_stamp", ctypes.c_void_p),
                ("order", ctypes.c_void_p), ("order_pos", ctypes.c_void_p),
                ("num_slots", ctypes.c_int32),
                ("clock", ctypes.c_void_p)]


class SSH2DJob(ctypes.Structure):
    _fields_ = [("miss_keys", ctypes.c_void_p), ("miss_slots", ctypes.c_void_p),
                ("counts", ctypes.c_void_p), ("pool_kv", ctypes.c_void_p),
                ("max_misses", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class SparseServeError(RuntimeError):
    pass


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(nvcc -gencode arch=compute_100a,code=sm_100a); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, SZ, F = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_float
    L.block_meta_update.argtypes = [P, I64, P, I64, P, I32, I32, P]
    L.ss_block_select.argtypes = [P, P, P, I32, I32, SSDims, I32, P, P, P, SZ, P]
    L.block_meta_update_mean.argtypes = [P, I64, P, I64, P, I32, I32, P]
    L.ss_block_select_mean.argtypes = [P, P, P, I32, I32, SSDims, I32, P, P, P, SZ, P]
    L.kv_cache_lookup_insert.argtypes = [SSCachePool, P, P, I32, I32, I32, I32, SSDims, I64, P, P,
                                         P, P, P, P, SZ, P]
    L.flash_h2d_gather.argtypes = [P, I64, P, P, P, I32, P, I64, P]
    L.flash_h2d_serve.argtypes = [P, I64, P, I32, I64, P, I64, P, P]
    L.ss_flag_signal.argtypes = [P, P]
    L.ss_flag_wait.argtypes = [P, P, I64, P]
    L.ss_preload_kernels.argtypes = []
    L.sparse_decode_attn_part.argtypes = [P, P, P, P, I32, I32, P, P, SSDims, I32, F, P, P, P, P, SZ, P]
    L.sparse_attn_merge.argtypes = [P, P, P, P, I64, P, P, P]
    L.sparse_decode_attn.argtypes = [P, P, P, I32, P, P, SSDims, I32, F, P, P, P, SZ, P]
    L.ss_workspace_size.argtypes = [I32, SSDims, I32, I32, I32]
    L.ss_workspace_size.restype = SZ
    L.ss_host_device_pointer.argtypes = [P, ctypes.POINTER(ctypes.c_void_p)]
    L.ss_device_numa_node.argtypes = [I32]
    L.ss_device_numa_node.restype = I32
    L.ss_host_alloc.argtypes = [SZ, I32, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                                ctypes.POINTER(I32)]
    L.ss_host_alloc.restype = I32
    L.ss_host_free.argtypes = [P, SZ]
    L.ss_host_free.restype = I32
    L.ss_decode_step_host.argtypes = [P, P, P, SZ, I32, P, P, P, P]
    L.ss_decode_step_host.restype = I32
    L.ss_status_string.argtypes = [I32]
    L.ss_status_string.restype = ctypes.c_char_p
    L.ss_version.restype = ctypes.c_char_p
    L.kv_append.argtypes = [P, P, P, I32, SSDims, I32, P]
    L.kv_seal_blocks.argtypes = [P, I32, P, P, I32, P, P, P, SZ, SSDims, I32, P]
    L.kv_commit.argtypes = [P, I32, P, P, P]
    L.ss_d2h_create.argtypes = [I32, ctypes.POINTER(ctypes.c_void_p)]
    L.ss_d2h_destroy.argtypes = [P]
    L.flash_d2h_save.argtypes = [P, P, P, I64, P, P, I64, I64, P]
    L.ws_track.argtypes = [P, I32, SSDims, I32, I64, I32, P, P, P, P]
    L.ws_track.restype = I32
    L.ss_admit.argtypes = [P, I32, I64, P]
    L.prefill_layer_save.argtypes = [P, P, I32, I32, I32, I32, I32, I32, SSDims, I32, P, P, P, P, P,
                                     P, I64, P, SZ, P]
    L.prefill_layer_save.restype = I32
    L.ss_admit.restype = I32
    for name in ("block_meta_update", "ss_block_select", "kv_cache_lookup_insert",
                 "flash_h2d_gather", "sparse_decode_attn", "ss_host_device_pointer", "kv_append",
                 "kv_seal_blocks", "kv_commit", "ss_d2h_create", "ss_d2h_destroy",
                 "flash_d2h_save", "block_meta_update_mean", "ss_block_select_mean", "flash_h2d_serve",
                 "ss_flag_signal", "ss_flag_wait", "ss_preload_kernels",
           "sparse_decode_attn_part", "sparse_attn_merge"):
        getattr(L, name).restype = I32
    _lib = L
    return L


def check(status: int, what: str) -> None:
    if status != SS_OK:
        msg = load().ss_status_string(status).decode()
        raise SparseServeError(f"{what} failed: {msg} ({status})")
