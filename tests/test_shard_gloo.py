"""World-size-2 gloo test (CPU) of the multi-GPU host logic: KV-head sharding,
per-rank cache keys/pools, and the S6 all-gather of head-major outputs.  Each
rank runs its shard of the path (oracle on CPU stands in for the kernels); the
gathered output must equal the unsharded computation."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

D = 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rng = synth.rng_for(7000, 1)
    B, Hq, Hkv, n, k = 2, 8, 4, 96, 8
    blocks = synth.encode(synth.kv_blocks(rng, B * Hkv * n, D, synth.channel_scales(rng)), synth.DT_BF16)
    q = synth.encode(rng.standard_normal((B, Hq, D)), synth.DT_BF16)
    tail = synth.encode(synth.kv_blocks(rng, B * Hkv, D).reshape(B, Hkv, 2, 32, D), synth.DT_BF16)
    return B, Hq, Hkv, n, k, blocks.reshape(B, Hkv, n, 2, 32, D), q, tail


def _run_shard(B, Hq, Hkv, n, k, blocks, q, tail, hq0, hq1, hkv0, hkv1):
    hkv = hkv1 - hkv0
    blk = np.ascontiguousarray(blocks[:, hkv0:hkv1]).reshape(-1, 2, 32, D)
    meta = oracle.block_meta(blk, key_stride=2 * 32 * D).reshape(B, hkv, n, 2, D)
    max_blk = n
    fwd_len = B * 1 * hkv * max_blk
    pool = oracle.Pool(B * hkv * k * 2, fwd_len, 16384)
    # rank-local keys: ((req*L + l)*hkv + h_local)*max_blk + j -> host block id of the shard
    host_u8 = blk.view(np.uint8).reshape(B * hkv * n, -1)
    r = oracle.decode_layer(np.ascontiguousarray(q[:, hq0:hq1]), meta, np.full(B, n, np.int32), k, pool,
                            np.arange(B, dtype=np.int32), 0, 1, max_blk, 1, host_u8, B * hkv * n,
                            np.ascontiguousarray(tail[:, hkv0:hkv1]), np.array([3, 0], np.int32),
                            1.0 / math.sqrt(D))
    return r["out"]            # [hq1-hq0][B][d] float64


def _worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_24626_b200.shard import gather_outputs, head_shard
    B, Hq, Hkv, n, k, blocks, q, tail = _problem()
    hq0, hq1, hkv0, hkv1 = head_shard(Hq, Hkv, rank, world)
    out_local = torch.from_numpy(_run_shard(B, Hq, Hkv, n, k, blocks, q, tail, hq0, hq1, hkv0, hkv1))
    out_full = torch.empty((Hq, B, D), dtype=torch.float64)
    gather_outputs(out_local, out_full)
    if rank == 0:
        ret.put(out_full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_head_sharded_allgather_equals_unsharded():
    B, Hq, Hkv, n, k, blocks, q, tail = _problem()
    full = _run_shard(B, Hq, Hkv, n, k, blocks, q, tail, 0, Hq, 0, Hkv)
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, ret)) for r in range(2)]
    for p in procs:
        p.start()
    got = ret.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(got, full)


def test_head_shard_ranges():
    from paper_2509_24626_b200.shard import head_shard
    assert head_shard(32, 8, 1, 4) == (8, 16, 2, 4)
    assert head_shard(32, 32, 7, 8) == (28, 32, 28, 32)
    with pytest.raises(ValueError):
        head_shard(32, 8, 0, 3)


def _og_worker(rank, world, port, ret):
    """OutputGather (the bench's S6 hook) over gloo: per request group its own
    communicator and a [L][Hq][nb][d] gathered buffer."""
    import types
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_24626_b200.shard import OutputGather
    L, hq_local, d = 3, 4, 8
    nbs = [2, 3]
    groups = []
    for gi, nb in enumerate(nbs):
        out = torch.arange(L * hq_local * nb * d, dtype=torch.float32).view(L, hq_local, nb, d)
        groups.append(types.SimpleNamespace(nb=nb, out=out + 1000 * rank + 100 * gi))
    eng = types.SimpleNamespace(cfg=types.SimpleNamespace(layers=L, num_q_heads=hq_local), groups=groups,
                                device=torch.device("cpu"))
    og = OutputGather(eng, world)
    hook = og.hook()
    for l in range(L):
        for gi, g in enumerate(groups):
            hook(gi, g, l)
    if rank == 0:
        ret.put([t.numpy() for t in og.outputs()])
    dist.barrier()
    dist.destroy_process_group()


def test_output_gather_hook_world2():
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_og_worker, args=(r, 2, port, ret)) for r in range(2)]
    for p in procs:
        p.start()
    got = ret.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    L, hq_local, d = 3, 4, 8
    for gi, nb in enumerate([2, 3]):
        base = np.arange(L * hq_local * nb * d, dtype=np.float32).reshape(L, hq_local, nb, d)
        exp = np.concatenate([base + 1000 * r + 100 * gi for r in range(2)], axis=1)   # rank-major heads
        np.testing.assert_array_equal(got[gi], exp)
