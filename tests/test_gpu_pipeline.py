"""End-to-end decode-step parity: the engine (S0..S5 through the C ABI) vs the
oracle pipeline, step by step, on BASELINE.json configs[0] (C1: 1 request,
1 layer, 32 MHA heads, 8K context, k = 64, HBM cache = 25% of blocks) with a
ragged tail, 50 drifting decode steps."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from layout import D, tiled_to_logical, to_numpy, to_torch

pytestmark = pytest.mark.gpu

TOL = {synth.DT_BF16: 2e-3, synth.DT_F32: 1e-5}


def _run_pipeline(dt, B, L, Hq, Hkv, n_blk, k, S, tails, steps, rho, seed):
    from paper_2509_24626_b200.engine import DecodeEngine, EngineConfig
    tdt = torch.bfloat16 if dt == synth.DT_BF16 else torch.float32
    max_blk = ((max(n_blk) + 31) // 32) * 32
    cfg = EngineConfig(batch=B, layers=L, num_q_heads=Hq, num_kv_heads=Hkv, max_blk=max_blk,
                       topk=k, slots_per_layer=S, num_requests=B, dtype=tdt)
    eng = DecodeEngine(cfg)
    rng = synth.rng_for(2000, seed)
    host_blocks = cfg.fwd_len                      # no aliasing in parity runs
    blocks = synth.kv_blocks(rng, host_blocks, D, synth.channel_scales(rng))
    host_np = synth.encode(blocks, dt)
    del blocks
    host_t = torch.from_numpy(host_np.view(np.int16) if dt == synth.DT_BF16 else host_np)
    host_t = host_t.view(-1).pin_memory()
    if dt == synth.DT_BF16:
        host_t = host_t.view(torch.bfloat16)
    eng.set_host_kv(host_t, host_blocks)
    eng.n_blk.copy_(torch.tensor(n_blk, dtype=torch.int32))
    eng.tail_len.copy_(torch.tensor(tails, dtype=torch.int32))
    tail_f = synth.kv_blocks(rng, L * B * Hkv, D).reshape(L, B, Hkv, 2, 32, D)
    tail_np = synth.encode(tail_f, dt)
    eng.tail_kv.copy_(to_torch(tail_np))
    dev_copy = host_t.to("cuda")
    eng.build_meta(n_blk, dev_copy)
    del dev_copy
    torch.cuda.synchronize()

    # oracle side: its own metadata, pools and pipeline
    host_u8 = host_np.view(np.uint8).reshape(host_blocks, -1)
    pools = [oracle.Pool(S, cfg.fwd_len, cfg.block_bytes) for _ in range(L)]
    metas = []
    for l in range(L):
        m = np.zeros((B, Hkv, max_blk, 2, D), dtype=host_np.dtype)
        for b in range(B):
            for h in range(Hkv):
                k0 = eng.key0(b, l, h)
                blk = host_np.reshape(host_blocks, 2, 32, D)[k0:k0 + n_blk[b]]
                if n_blk[b]:
                    m[b, h, :n_blk[b]] = oracle.block_meta(blk, key_stride=2 * 32 * D)
        metas.append(m)
        got_meta = tiled_to_logical(to_numpy(eng.meta[l]), B, Hkv, max_blk)
        for b in range(B):
            np.testing.assert_array_equal(got_meta[b, :, :n_blk[b]].view(np.uint8),
                                          m[b, :, :n_blk[b]].view(np.uint8))

    qs_all = synth.encode(synth.queries(rng, steps, (L, B, Hq, D), rho), dt)
    scale = 1.0 / math.sqrt(D)
    req_ids = np.arange(B, dtype=np.int32)
    stats = dict(hits=0, misses=0, evictions=0, max_err=0.0)
    scores = torch.empty(B, Hkv, max_blk, dtype=torch.float64, device="cuda")
    for t in range(steps):
        for l in range(L):
            q_np = qs_all[t, l]
            eng.layer_step(l, to_torch(q_np), stamp=t + 1, scores=scores)
            torch.cuda.synchronize()
            r = oracle.decode_layer(q_np, metas[l], np.array(n_blk, np.int32), k, pools[l], req_ids,
                                    l, L, max_blk, t + 1, host_u8, host_blocks, tail_np[l],
                                    np.array(tails, np.int32), scale)
            gs = scores.cpu().numpy()
            for b in range(B):
                np.testing.assert_array_equal(gs[b, :, :n_blk[b]].view(np.uint64),
                                              r["scores"][b, :, :n_blk[b]].view(np.uint64))
            np.testing.assert_array_equal(eng.sel[l].cpu().numpy(), r["sel"])
            np.testing.assert_array_equal(eng.counts[l].cpu().numpy(), r["counts"])
            assert r["counts"][3] == 0
            np.testing.assert_array_equal(eng.slot[l].cpu().numpy(), r["slot"])
            np.testing.assert_array_equal(eng.hit[l].cpu().numpy(), r["hit"])
            m = int(r["counts"][1])
            np.testing.assert_array_equal(eng.miss_keys[l].cpu().numpy()[:m], r["miss_keys"])
            np.testing.assert_array_equal(eng.miss_slots[l].cpu().numpy()[:m], r["miss_slots"])
            p = eng.pools[l]
            np.testing.assert_array_equal(p.slot_key.cpu().numpy(), pools[l].slot_key)
            np.testing.assert_array_equal(p.slot_stamp.cpu().numpy(), pools[l].slot_stamp)
            np.testing.assert_array_equal(
                p.order.cpu().numpy(),
                np.lexsort((np.arange(S), pools[l].slot_stamp)).astype(np.int32))
            err = float(np.abs(eng.out[l].cpu().numpy() - r["out"]).max())
            assert err <= TOL[dt], f"step {t} layer {l}: max abs err {err}"
            stats["max_err"] = max(stats["max_err"], err)
            stats["hits"] += int(r["counts"][0])
            stats["misses"] += m
            stats["evictions"] += int(r["counts"][2])
    # the GPU key->slot table is shared by the layer pools (keys are disjoint per layer)
    fwd_exp = sum(pools[l].fwd.astype(np.int64) + 1 for l in range(L)) - 1
    np.testing.assert_array_equal(eng.fwd.cpu().numpy(), fwd_exp.astype(np.int32))
    for l in range(L):
        np.testing.assert_array_equal(to_numpy(eng.pool_kv[l]).view(np.uint8).reshape(S, -1),
                                      pools[l].kv)
    return stats


def test_c1_pipeline_50_steps():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    wl = synth.C1
    st = _run_pipeline(synth.DT_BF16, wl.batch, wl.layers, wl.num_q_heads, wl.num_kv_heads,
                       [wl.n_blk], wl.topk, wl.slots_per_layer, [17], steps=50, rho=wl.rho, seed=1)
    assert st["hits"] > 0 and st["evictions"] > 0
    print("C1 pipeline stats:", st)


def test_gqa_multilayer_ragged_pipeline():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    _run_pipeline(synth.DT_BF16, 3, 2, 16, 4, [2100, 700, 33], 32, 3 * 4 * 32 * 2, [0, 31, 5],
                  steps=12, rho=0.95, seed=2)


def test_f32_pipeline():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    _run_pipeline(synth.DT_F32, 2, 1, 8, 8, [300, 128], 16, 2 * 8 * 16 * 2, [1, 0],
                  steps=8, rho=0.9, seed=3)


@pytest.mark.parametrize("graph_after,server,ngroups,split,ppg", [
    (None, False, 2, False, False), (4, False, 2, False, False), (None, True, 2, False, False),
    (4, True, 2, False, False), (4, True, 3, False, False), (None, True, 2, True, False),
    (4, True, 3, True, False), (None, True, 2, False, True), (4, True, 3, False, True)])
def test_request_groups_pipeline_two_streams(graph_after, server, ngroups, split, ppg):
    """groups=2: the two request groups run on separate streams; per layer the
    oracle makes the same two cache calls (group order, same stamp).  With
    graph_after=4 the steps from 4 on are replays of one captured CUDA graph
    whose LRU stamps come from the pools' device clocks.  server=True: the
    step's gathers are jobs of one persistent flash_h2d_serve launch; split=True:
    each group attends its hits while the misses load, then merges.  ppg=True:
    one LRU pool per (layer, group) of S / groups slots (reading R11b)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2509_24626_b200.engine import DecodeEngine, EngineConfig
    dt = synth.DT_BF16
    B, L, Hq, Hkv, k, steps = 4, 3, 8, 4, 24, 10
    n_blk = [900, 1500, 64, 700]
    tails = [0, 5, 31, 1]
    max_blk = 1504
    S = B * Hkv * k * 2
    cfg = EngineConfig(batch=B, layers=L, num_q_heads=Hq, num_kv_heads=Hkv, max_blk=max_blk, topk=k,
                       slots_per_layer=S, num_requests=B, dtype=torch.bfloat16, groups=ngroups,
                       h2d_server=server, split_attn=split, pool_per_group=ppg)
    eng = DecodeEngine(cfg)
    assert len(eng.groups) == ngroups and eng.server == server
    rng = synth.rng_for(2000, 9)
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
    Sg = S // ngroups if ppg else S
    gpools = [[oracle.Pool(Sg, cfg.fwd_len, cfg.block_bytes) for _ in range(ngroups if ppg else 1)]
              for _ in range(L)]
    qs = synth.encode(synth.queries(rng, steps, (L, B, Hq, D), 0.95), dt)
    host_u8 = host_np.view(np.uint8).reshape(hb, -1)
    nbk = np.array(n_blk, np.int32)
    tl = np.array(tails, np.int32)
    graph = None
    q_static = None
    for t in range(steps):
        if graph_after is not None and t == graph_after:
            eng.use_device_clock(start=t)
            q_static = torch.empty_like(to_torch(qs[0]))
            graph = eng.capture_graph(q_static)
        if graph is not None:
            q_static.copy_(to_torch(qs[t]))
            graph.replay()
        else:
            eng.step(to_torch(qs[t]), stamp=t + 1)
        torch.cuda.synchronize()
        for l in range(L):
            for gi, g in enumerate(eng.groups):
                b0, b1 = g.b0, g.b1
                op = gpools[l][gi if ppg else 0]
                r = oracle.decode_layer(np.ascontiguousarray(qs[t, l, b0:b1]), np.ascontiguousarray(metas[l][b0:b1]),
                                        nbk[b0:b1], k, op, np.arange(b0, b1, dtype=np.int32), l, L,
                                        max_blk, t + 1, host_u8, hb, np.ascontiguousarray(tail_np[l, b0:b1]),
                                        tl[b0:b1], 1.0 / math.sqrt(D))
                np.testing.assert_array_equal(g.sel[l].cpu().numpy(), r["sel"])
                np.testing.assert_array_equal(g.counts[l].cpu().numpy(), r["counts"])
                np.testing.assert_array_equal(g.slot[l].cpu().numpy(), r["slot"])
                err = float(np.abs(g.out[l].cpu().numpy() - r["out"]).max())
                assert err <= TOL[dt], f"step {t} layer {l} group {b0}: {err}"
            for gi in range(ngroups if ppg else 1):
                p_dev, p_or = eng.pool_of(l, gi), gpools[l][gi]
                np.testing.assert_array_equal(p_dev.slot_stamp.cpu().numpy(), p_or.slot_stamp)
                np.testing.assert_array_equal(p_dev.slot_key.cpu().numpy(), p_or.slot_key)
    for l in range(L):
        for gi in range(ngroups if ppg else 1):
            np.testing.assert_array_equal(
                to_numpy(eng.pool_kv_of(l, gi)).view(np.uint8).reshape(Sg, -1), gpools[l][gi].kv)
