"""Multi-GPU partitioning of the hot path: KV heads are
contiguous per rank; every (request, KV head) pair is independent through
S0..S5, so the only exchange is S6, one all-gather of the per-head outputs per
layer at the tensor-parallel boundary.  The output layout [Hq][B][d] is
head-major, so the rank-major all-gather result is already contiguous.

Host logic only (plumbing); the per-rank work is the single-GPU path.
"""
from __future__ import annotations

from typing import Tuple

import torch


def head_shard(num_q_heads: int, num_kv_heads: int, rank: int, world: int) -> Tuple[int, int, int, int]:
    """(hq0, hq1, hkv0, hkv1): this rank's query-head and KV-head ranges."""
    if num_kv_heads % world:
        raise ValueError(f"{num_kv_heads} KV heads do not split over {world} ranks")
    per = num_kv_heads // world
    g = num_q_heads // num_kv_heads
    hkv0, hkv1 = rank * per, (rank + 1) * per
    return hkv0 * g, hkv1 * g, hkv0, hkv1


def shard_queries(q: torch.Tensor, rank: int, world: int, num_kv_heads: int) -> torch.Tensor:
    """q [..., B, Hq, d] -> this rank's contiguous query heads."""
    hq0, hq1, _, _ = head_shard(q.shape[-2], num_kv_heads, rank, world)
    return q[..., hq0:hq1, :].contiguous()


def gather_outputs(out_local: torch.Tensor, out_full: torch.Tensor, group=None) -> torch.Tensor:
    """S6: all-gather [Hq/N][B][d] shards into [Hq][B][d] (NCCL on GPU, gloo on CPU)."""
    torch.distributed.all_gather_into_tensor(out_full, out_local.contiguous(), group=group)
    return out_full
