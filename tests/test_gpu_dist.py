"""The N > 1 code path on one GPU: a world-size-1 NCCL process group drives the
multi-GPU step exactly as bench.py runs it per rank -- request groups on their
own streams, the FlashH2D server, one CUDA graph per step, and S6 (the NCCL
all-gather of each request group's layer outputs, shard.OutputGather) captured
inside that graph.  The engine holds one rank's KV-head shard of a 2-rank
problem (shard.head_shard); its gathered outputs, selections, counts and slots
are checked step by step against the oracle run on that shard (SURVEY.md §8(e):
(request, KV head) pairs are independent through S0..S5, so a shard's oracle is
the unsharded oracle on its heads).  The world-2 host logic is covered on CPU by
tests/test_shard_gloo.py."""
import json
import math
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
import synth
from layout import D, to_torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl1():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.distributed as dist
    torch.cuda.set_device(0)
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("rank_of_2", [0, 1])
def test_sharded_step_with_nccl_allgather_in_graph(nccl1, rank_of_2):
    from paper_2509_24626_b200.engine import DecodeEngine, EngineConfig
    from paper_2509_24626_b200.shard import OutputGather, head_shard
    dt = synth.DT_BF16
    B, L, Hq_all, Hkv_all, k, steps, graph_after = 5, 3, 16, 8, 24, 8, 3
    hq0, hq1, hkv0, hkv1 = head_shard(Hq_all, Hkv_all, rank_of_2, 2)
    Hq, Hkv = hq1 - hq0, hkv1 - hkv0
    n_blk = [900, 1500, 64, 700, 333]
    tails = [0, 5, 31, 1, 17]
    max_blk = 1504
    ngroups = 3
    S = B * Hkv * k * 2
    cfg = EngineConfig(batch=B, layers=L, num_q_heads=Hq, num_kv_heads=Hkv, max_blk=max_blk, topk=k,
                       slots_per_layer=S, num_requests=B, dtype=torch.bfloat16, groups=ngroups,
                       h2d_server=True, pool_per_group=True)
    eng = DecodeEngine(cfg)
    gather = OutputGather(eng, world=1)
    rng = synth.rng_for(2100, rank_of_2)
    hb = cfg.fwd_len
    host_np = synth.encode(synth.kv_blocks(rng, hb, D, synth.channel_scales(rng)), dt)
    host_t = torch.from_numpy(host_np.view(np.int16)).view(-1).pin_memory().view(torch.bfloat16)
    eng.set_host_kv(host_t, hb)
    eng.n_blk.copy_(torch.tensor(n_blk, dtype=torch.int32))
    eng.tail_len.copy_(torch.tensor(tails, dtype=torch.int32))
    tail_np = synth.encode(synth.kv_blocks(rng, L * B * Hkv, D).reshape(L, B, Hkv, 2, 32, D), dt)
    eng.tail_kv.copy_(to_torch(tail_np))
    eng.build_meta(n_blk, host_t.cuda())
    blocks = host_np.reshape(hb, 2, 32, D)
    metas = []
    for l in range(L):
        m = np.zeros((B, Hkv, max_blk, 2, D), np.uint16)
        for b in range(B):
            for h in range(Hkv):
                k0 = eng.key0(b, l, h)
                m[b, h, :n_blk[b]] = oracle.block_meta(blocks[k0:k0 + n_blk[b]], key_stride=2 * 32 * D)
        metas.append(m)
    Sg = S // ngroups
    gpools = [[oracle.Pool(Sg, cfg.fwd_len, cfg.block_bytes) for _ in range(ngroups)] for _ in range(L)]
    # the full problem's queries; this rank attends its contiguous query heads
    qs_all = synth.encode(synth.queries(rng, steps, (L, B, Hq_all, D), 0.95), dt)
    qs = np.ascontiguousarray(qs_all[:, :, :, hq0:hq1])
    host_u8 = host_np.view(np.uint8).reshape(hb, -1)
    nbk, tl = np.array(n_blk, np.int32), np.array(tails, np.int32)
    graph, q_static = None, None
    for t in range(steps):
        if t == graph_after:
            eng.use_device_clock(start=t)
            q_static = torch.empty_like(to_torch(qs[0]))
            graph = eng.capture_graph(q_static, post_attn=gather.hook())
        if graph is not None:
            q_static.copy_(to_torch(qs[t]))
            graph.replay()
        else:
            eng.step(to_torch(qs[t]), stamp=t + 1, post_attn=gather.hook())
        torch.cuda.synchronize()
        for l in range(L):
            for gi, g in enumerate(eng.groups):
                b0, b1 = g.b0, g.b1
                r = oracle.decode_layer(np.ascontiguousarray(qs[t, l, b0:b1]), np.ascontiguousarray(metas[l][b0:b1]),
                                        nbk[b0:b1], k, gpools[l][gi], np.arange(b0, b1, dtype=np.int32), l, L,
                                        max_blk, t + 1, host_u8, hb, np.ascontiguousarray(tail_np[l, b0:b1]),
                                        tl[b0:b1], 1.0 / math.sqrt(D))
                np.testing.assert_array_equal(g.sel[l].cpu().numpy(), r["sel"])
                np.testing.assert_array_equal(g.counts[l].cpu().numpy(), r["counts"])
                np.testing.assert_array_equal(g.slot[l].cpu().numpy(), r["slot"])
                # S6 result: the all-gathered [Hq * world][nb][d] block of this group
                got = gather.outputs()[gi][l].cpu().numpy()
                assert got.shape == (Hq, b1 - b0, D)
                err = float(np.abs(got - r["out"]).max())
                assert err <= 2e-3, f"step {t} layer {l} group {gi}: {err}"
                np.testing.assert_array_equal(got, g.out[l].cpu().numpy())


def test_bench_torchrun_world1_runs_the_multi_gpu_path():
    """bench.py under torchrun (one rank, NCCL) at a short settle: the N > 1
    launch configuration (groups, server, graph with the NCCL all-gather)
    produces a valid line with no device-side errors."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "1", "--steps", "4", "--warmup", "3", "--settle", "20", "--no-cpu-baseline",
           "--no-gather-alone"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["config"]["cuda_graph"] and line["config"]["h2d_server"]
    assert "NCCL" in line["config"]["parallelism"]
    assert line["errors_in_timed_region"] == 0 and line.get("valid", True)
    assert line["kernels"]["nccl_all_gather"]["launches_per_step"] == 32 * line["config"]["request_groups"]
    assert line["value"] > 0


def test_bench_gpus_beyond_visible_fails_loudly():
    """`bench.py --gpus N` re-launches itself with N ranks; asking for more GPUs
    than are visible must fail with a message, not silently run on one."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    n = torch.cuda.device_count() + 1
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert r.returncode == 2, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])
    assert "visible" in r.stderr
    assert not [x for x in r.stdout.splitlines() if x.startswith("{")]
