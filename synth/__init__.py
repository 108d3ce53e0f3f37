"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no scoring, selection, cache
or attention logic).  It only draws random numbers with the shapes and value
distributions of the paper's workloads and encodes them in the storage dtypes
(bf16 bit patterns with round-to-nearest-even, or float32).  Both `oracle/`
and `paper_2509_24626_b200/` consume its outputs; neither imports the other.

Recipe:
  * K ~ N(0,1) per element x per-channel scale sigma_c ~ LogNormal(0, 0.5)
    (outlier channels), V ~ N(0,1).
  * q_{t+1} = rho*q_t + sqrt(1-rho^2)*xi, xi ~ N(0, I)   (consecutive-query
    similarity that the paper's LRU relies on, §3.1).
  * optional "needle" tokens: one key per chosen block set to alpha*q_hat.
  * everything rounded to bf16 (RNE) for the bf16 dtype.
Seeds: numpy SeedSequence([config_id, stream_tag, ...]).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

HEAD_DIM = 128
BLOCK_TOKENS = 32  # PAPER.md:39 §1 ("KV block size to 32 tokens")

DT_BF16 = "bf16"
DT_F32 = "f32"


# ----------------------------------------------------------------------------
# dtype encoding (input encoding only)
# ----------------------------------------------------------------------------
def f32_to_bf16_bits(x) -> np.ndarray:
    """Round float32 values to bf16 (round-to-nearest-even); return uint16 bits.

    Finite inputs only (the generators never produce inf/nan)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    b = x.view(np.uint32).astype(np.uint64)
    rounding = ((b >> 16) & 1) + 0x7FFF
    return ((b + rounding) >> 16).astype(np.uint16)


def bf16_bits_to_f32(bits) -> np.ndarray:
    bits = np.ascontiguousarray(np.asarray(bits, dtype=np.uint16))
    return (bits.astype(np.uint32) << 16).view(np.float32)


def encode(x, dtype: str) -> np.ndarray:
    """float array -> storage array (uint16 bf16 bits or float32)."""
    if dtype == DT_BF16:
        return f32_to_bf16_bits(np.asarray(x, dtype=np.float32))
    if dtype == DT_F32:
        return np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    raise ValueError(dtype)


def decode_f64(a, dtype: str) -> np.ndarray:
    """storage array -> exact float64 values."""
    if dtype == DT_BF16:
        return bf16_bits_to_f32(a).astype(np.float64)
    if dtype == DT_F32:
        return np.asarray(a, dtype=np.float32).astype(np.float64)
    raise ValueError(dtype)


def elem_bytes(dtype: str) -> int:
    return 2 if dtype == DT_BF16 else 4


def np_storage_dtype(dtype: str):
    return np.uint16 if dtype == DT_BF16 else np.float32


# ----------------------------------------------------------------------------
# generators
# ----------------------------------------------------------------------------
def rng_for(*tags: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(t) for t in tags]))


def channel_scales(rng: np.random.Generator, d: int = HEAD_DIM, sigma: float = 0.5) -> np.ndarray:
    return rng.lognormal(mean=0.0, sigma=sigma, size=d).astype(np.float32)


def kv_blocks(rng: np.random.Generator, n_blocks: int, d: int = HEAD_DIM,
              scales: Optional[np.ndarray] = None) -> np.ndarray:
    """float32 array [n_blocks][2][32][d]: K (scaled N(0,1)) then V (N(0,1)).

    Layout follows PAPER.md:129/137 §3.2 (H,N,D): the 32 tokens of one head are
    contiguous inside a block; K and V halves of one head-block are adjacent."""
    out = rng.standard_normal((n_blocks, 2, BLOCK_TOKENS, d), dtype=np.float32)
    if scales is not None:
        out[:, 0] *= scales[None, None, :]
    return out


def queries(rng: np.random.Generator, steps: int, shape, rho: float) -> np.ndarray:
    """float32 [steps][*shape] with q_{t+1} = rho q_t + sqrt(1-rho^2) xi."""
    q = np.empty((steps,) + tuple(shape), dtype=np.float32)
    cur = rng.standard_normal(shape, dtype=np.float32)
    s = math.sqrt(max(0.0, 1.0 - rho * rho))
    for t in range(steps):
        if t > 0:
            cur = (rho * cur + s * rng.standard_normal(shape, dtype=np.float32)).astype(np.float32)
        q[t] = cur
    return q


def plant_needles(rng: np.random.Generator, blocks: np.ndarray, qdir: np.ndarray,
                  n_needles: int, alpha: float) -> np.ndarray:
    """Set one key token in `n_needles` random blocks to alpha * qdir/|qdir|.

    blocks: float32 [n][2][32][d] (modified in place); returns the block ids."""
    n = blocks.shape[0]
    ids = rng.choice(n, size=min(n_needles, n), replace=False)
    qhat = qdir / max(float(np.linalg.norm(qdir)), 1e-30)
    tok = rng.integers(0, BLOCK_TOKENS, size=ids.shape[0])
    for i, t in zip(ids, tok):
        blocks[i, 0, t, :] = alpha * qhat
    return np.sort(ids)


@dataclasses.dataclass(frozen=True)
class Workload:
    """Shapes of one decode-step workload."""
    name: str
    batch: int
    layers: int
    num_q_heads: int
    num_kv_heads: int
    context: int           # tokens per request (full blocks * 32 + tail)
    topk: int              # selected blocks per (request, kv head)
    slots_per_layer: int   # HBM cache slots per layer pool
    rho: float
    head_dim: int = HEAD_DIM

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    @property
    def n_blk(self) -> int:
        return self.context // BLOCK_TOKENS

    @property
    def max_blk(self) -> int:
        return ((self.n_blk + 31) // 32) * 32


# configs[0..4] of BASELINE.json, restated
C1 = Workload("C1-8K-MHA-1req-1layer", 1, 1, 32, 32, 8192, 64, 2048, 0.9)
C2 = Workload("C2-LWM7B-128K-b16", 16, 32, 32, 32, 131072, 64, 131072, 0.99)
C3 = Workload("C3-Llama3-8B-GQA-1M-b4", 4, 32, 32, 8, 1048576, 128, 8192, 0.0)


def c4(batch: int) -> Workload:
    return Workload(f"C4-64K-b{batch}", batch, 4, 32, 32, 65536, 64, 262144, 0.95)
