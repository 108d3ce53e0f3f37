"""Multi-GPU partitioning of the hot path: KV heads are
contiguous per rank; every (request, KV head) pair is independent through
S0..S5, so the only exchange is S6, one all-gather of the per-head outputs per
layer at the tensor-parallel boundary.  The output layout [Hq][B][d] is
head-major, so the rank-major all-gather result is already contiguous.

The per-rank work is the single-GPU path (request groups, FlashH2D server,
one CUDA graph per step); `OutputGather` adds S6 to it: after each request
group's layer-l attention, on that group's stream, an all-gather of the
group's [Hq/N][nb][d] outputs over a communicator of its own, so the groups'
collectives never order each other and the whole step -- NCCL included -- is
captured as one CUDA graph.  On CPU (tests) the same code runs over gloo.
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


class OutputGather:
    """S6 for one rank's DecodeEngine: per request group, a process group
    (communicator) and a gathered buffer [L][Hq][nb][d] (float32).

    `hook()` is the engine's post_attn callback: it all-gathers layer l's
    output of group gi on the current (the group's) stream, so the group's
    next-layer select is stream-ordered after its TP boundary, as a model's
    next-layer q would be."""

    def __init__(self, eng, world: int, groups=None):
        import torch.distributed as dist
        c = eng.cfg
        self.world = world
        self.pgs = groups if groups is not None else [dist.new_group(list(range(world))) for _ in eng.groups]
        dev = eng.device
        self.full = [torch.empty(c.layers, c.num_q_heads * world, g.nb, g.out.shape[-1], dtype=g.out.dtype,
                                 device=dev) for g in eng.groups]

    def hook(self, timers=None):
        def f(gi, g, l):
            if timers is not None and timers.wants("allgather"):
                s, e = timers.mark("allgather", gi, l)
                s.record()
                gather_outputs(g.out[l], self.full[gi][l], group=self.pgs[gi])
                e.record()
            else:
                gather_outputs(g.out[l], self.full[gi][l], group=self.pgs[gi])
        return f

    def outputs(self):
        return self.full
