"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same
seeded inputs.  Bit-exact for metadata, scores, selections, cache state, miss
lists and gathered bytes; max-abs 2e-3 (bf16) / 1e-5 (f32) for attention
(BASELINE.json north_star tolerances)."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from layout import D, logical_to_tiled, tiled_to_logical, to_numpy, to_torch

pytestmark = pytest.mark.gpu

TOL = {synth.DT_BF16: 2e-3, synth.DT_F32: 1e-5}


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2509_24626_b200 import ops as _ops
    return _ops


def _tdt(dt):
    return torch.bfloat16 if dt == synth.DT_BF16 else torch.float32


# ----------------------------------------------------------------------------
# S0
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("dt", [synth.DT_BF16, synth.DT_F32])
def test_block_meta_update_bit_exact(ops, dt):
    rng = synth.rng_for(1000, 1)
    B, Hkv, max_blk = 2, 3, 64
    n = B * Hkv * max_blk
    blocks = synth.kv_blocks(rng, n, D, synth.channel_scales(rng))
    blocks[3, 0, :, 5] = 0.0
    blocks[3, 0, 7, 5] = -0.0
    blocks[4, 0, :, 9] = -0.0
    store = synth.encode(blocks, dt)
    exp = oracle.block_meta(store, key_stride=2 * 32 * D).reshape(B, Hkv, max_blk, 2, D)
    meta = torch.zeros(B * Hkv * max_blk * 2 * D, dtype=_tdt(dt), device="cuda")
    # scatter in a shuffled order through dst_idx
    perm = rng.permutation(n)
    keys = to_torch(np.ascontiguousarray(store[perm]))
    ops.block_meta_update(keys, meta, n, key_stride=2 * 32 * D,
                          dst_idx=torch.from_numpy(perm.astype(np.int64)).cuda())
    torch.cuda.synchronize()
    got = tiled_to_logical(to_numpy(meta), B, Hkv, max_blk)
    np.testing.assert_array_equal(got.view(np.uint8), exp.view(np.uint8))


# ----------------------------------------------------------------------------
# S1 + S2
# ----------------------------------------------------------------------------
def _select_case(ops, dt, B, Hq, Hkv, n_blk, k, seed, ties=False, needle=False):
    rng = synth.rng_for(1000, 2, seed)
    max_blk = ((max(n_blk) + 31) // 32) * 32 or 32
    nb = B * Hkv * max_blk
    blocks = synth.kv_blocks(rng, nb, D, synth.channel_scales(rng))
    if ties:   # duplicated blocks -> exact score ties (tie rule must hold)
        src = rng.integers(0, nb, size=nb // 3)
        dst = rng.integers(0, nb, size=nb // 3)
        blocks[dst] = blocks[src]
    q = rng.standard_normal((B, Hq, D)).astype(np.float32)
    if needle:
        for b in range(B):
            for h in range(Hkv):
                j = int(rng.integers(0, max(1, n_blk[b])))
                blocks[(b * Hkv + h) * max_blk + j, 0, 3] = 50.0 * q[b, h * (Hq // Hkv)] / np.linalg.norm(q[b, h * (Hq // Hkv)])
    store = synth.encode(blocks, dt)
    qs = synth.encode(q, dt)
    meta_log = oracle.block_meta(store, key_stride=2 * 32 * D).reshape(B, Hkv, max_blk, 2, D)
    nbk = np.array(n_blk, np.int32)
    exp_scores = oracle.block_score(qs, meta_log, nbk)
    exp_sel = oracle.topk(exp_scores, nbk, k)
    # GPU: metadata given in the tiled layout (pure permutation of the same input)
    meta = to_torch(logical_to_tiled(meta_log))
    d = ops.dims(B, Hq, Hkv)
    ws = ops.alloc_workspace(0, d, max_blk, k)
    sel = torch.empty(B, Hkv, k, dtype=torch.int32, device="cuda")
    scores = torch.full((B, Hkv, max_blk), float("nan"), dtype=torch.float64, device="cuda")
    ops.ss_block_select(to_torch(qs), meta, torch.from_numpy(nbk).cuda(), max_blk, k, d, sel, ws,
                        scores=scores)
    # second call: the workspace must have been left clean (tickets reset)
    sel2 = torch.empty_like(sel)
    ops.ss_block_select(to_torch(qs), meta, torch.from_numpy(nbk).cuda(), max_blk, k, d, sel2, ws)
    torch.cuda.synchronize()
    gs = scores.cpu().numpy()
    for b in range(B):
        n = n_blk[b]
        np.testing.assert_array_equal(gs[b, :, :n].view(np.uint64), exp_scores[b, :, :n].view(np.uint64))
    np.testing.assert_array_equal(sel.cpu().numpy(), exp_sel)
    np.testing.assert_array_equal(sel2.cpu().numpy(), exp_sel)
    return exp_sel


@pytest.mark.parametrize("dt", [synth.DT_BF16, synth.DT_F32])
def test_select_c1_shape(ops, dt):
    # C1: 1 request, 32 MHA heads, 8K ctx = 256 blocks, k = 64
    _select_case(ops, dt, 1, 32, 32, [256], 64, seed=1)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_select_gqa_ragged_multichunk(ops, G):
    # n_blk > 2048 exercises the multi-chunk candidate merge; 0 and 17 are ragged tails
    Hkv = 2
    _select_case(ops, synth.DT_BF16, 4, Hkv * G, Hkv, [5000, 2049, 17, 0], 128, seed=10 + G)


@pytest.mark.parametrize("k", [1, 3, 64, 300])
def test_select_ties_and_k_edges(ops, k):
    _select_case(ops, synth.DT_BF16, 2, 4, 4, [300, 96], k, seed=20 + k, ties=True)


@pytest.mark.parametrize("G", [1, 4])
def test_select_large_k_many_chunks_merge_bound(ops, G):
    # 1M-token context (32768 blocks) with k = 300: at the default chunk the pair's
    # candidates (32 x 300 for G = 1, 16 x 300 for G = 4) would exceed the merge's
    # 8192-key shared-memory bound, so the call must widen its chunk, not overflow
    _select_case(ops, synth.DT_BF16, 1, G, 1, [32768], 300, seed=40 + G)


@pytest.mark.parametrize("G,k", [(2, 1), (4, 64), (8, 300), (4, 128)])
def test_select_gqa_ties_tensor_core_path(ops, G, k):
    """GQA bf16 without a scores output runs the tensor-core filter + exact
    rescoring (block_select_tc_kernel): duplicated blocks give exact score ties
    that straddle the k-th place; the selection must equal the oracle's."""
    _select_case(ops, synth.DT_BF16, 2, 2 * G, 2, [3000, 700], k, seed=60 + G + k, ties=True)


def _select_sel_only(ops, q_f, blocks_f, B, Hq, Hkv, n_blk, k):
    """bf16 selection only (the tensor-core path for GQA) vs the oracle."""
    max_blk = ((max(n_blk) + 31) // 32) * 32
    store = synth.encode(blocks_f, synth.DT_BF16)
    qs = synth.encode(q_f, synth.DT_BF16)
    meta_log = oracle.block_meta(store, key_stride=2 * 32 * D).reshape(B, Hkv, max_blk, 2, D)
    nbk = np.array(n_blk, np.int32)
    exp_sel = oracle.topk(oracle.block_score(qs, meta_log, nbk), nbk, k)
    d = ops.dims(B, Hq, Hkv)
    ws = ops.alloc_workspace(0, d, max_blk, k)
    sel = torch.empty(B, Hkv, k, dtype=torch.int32, device="cuda")
    ops.ss_block_select(to_torch(qs), to_torch(logical_to_tiled(meta_log)), torch.from_numpy(nbk).cuda(),
                        max_blk, k, d, sel, ws)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(sel.cpu().numpy(), exp_sel)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_select_gqa_near_ties_below_f32_resolution(ops, G):
    """Blocks whose exact scores differ by far less than the f32 approximation
    can resolve (one key nudged by one bf16 ulp in a copy of another block):
    the exact fp64 rescoring of the candidates must order them as the oracle."""
    rng = synth.rng_for(1000, 7, G)
    B, Hkv, n = 2, 2, 1500
    max_blk = ((n + 31) // 32) * 32
    blocks = synth.kv_blocks(rng, B * Hkv * max_blk, D, synth.channel_scales(rng))
    blocks = synth.bf16_bits_to_f32(synth.f32_to_bf16_bits(blocks)).reshape(blocks.shape)
    src = rng.integers(0, B * Hkv * max_blk, size=400)
    for i, j in enumerate(rng.integers(0, B * Hkv * max_blk, size=400)):
        blocks[j] = blocks[src[i]]
        if i % 2:   # nudge one key element of the copy by one bf16 ulp (exact in bf16)
            t, c = int(rng.integers(0, 32)), int(rng.integers(0, D))
            bits = synth.f32_to_bf16_bits(blocks[j, 0, t, c:c + 1])
            blocks[j, 0, t, c] = synth.bf16_bits_to_f32(bits + np.uint16(1))[0]
    q = rng.standard_normal((B, Hkv * G, D)).astype(np.float32)
    for k in (16, 64):
        _select_sel_only(ops, q, blocks, B, Hkv * G, Hkv, [n, n - 333], k)


@pytest.mark.parametrize("scale_q,scale_k", [(1e10, 1e30), (1e-20, 1e-25), (1.0, 1e-38)])
def test_select_gqa_extreme_magnitudes(ops, scale_q, scale_k):
    """f32 overflow (inf / NaN approximations make every such block a candidate)
    and underflow (covered by the absolute error term) in the tensor-core
    filter: selections still equal the oracle's fp64 ones."""
    rng = synth.rng_for(1000, 8, int(np.log10(scale_k) + 50))
    B, G, Hkv, n = 1, 4, 2, 900
    max_blk = ((n + 31) // 32) * 32
    blocks = synth.kv_blocks(rng, B * Hkv * max_blk, D) * np.float32(scale_k)
    q = (rng.standard_normal((B, Hkv * G, D)) * scale_q).astype(np.float32)
    _select_sel_only(ops, q, blocks, B, Hkv * G, Hkv, [n], 32)


@pytest.mark.parametrize("G", [2, 4])
def test_select_gqa_cluster_shapes(ops, G):
    """The cluster form of the tensor-core select (block_select_tcc_kernel):
    two pairs of 8192 blocks -> 16-CTA clusters of 512-block chunks; request 1
    has 700 blocks, so 14 of its CTAs own no block and still join every cluster
    barrier; request 0 is a copy of ONE block (every L equal: a degenerate
    histogram, every block a candidate, local top-k before the gather)."""
    rng = synth.rng_for(1000, 9, G)
    B, Hkv, max_blk = 2, 1, 8192
    blocks = synth.kv_blocks(rng, B * Hkv * max_blk, D, synth.channel_scales(rng))
    blocks[:max_blk] = blocks[5]
    q = rng.standard_normal((B, Hkv * G, D)).astype(np.float32)
    for k in (1, 128):
        _select_sel_only(ops, q, blocks, B, Hkv * G, Hkv, [max_blk, 700], k)


def test_select_gqa_beyond_cluster_reach_per_chunk_form(ops):
    """max_blk > 16 CTAs x 4096 blocks (2.1M tokens): the tensor-core select
    falls back to its per-chunk form (block_select_tc_kernel: chunk candidates in
    the workspace, last-CTA merge); selections equal the oracle's."""
    rng = synth.rng_for(1000, 10, 0)
    B, G, Hkv, n = 1, 4, 1, 16 * 4096 + 1000
    max_blk = ((n + 31) // 32) * 32
    blocks = synth.kv_blocks(rng, B * Hkv * max_blk, D, synth.channel_scales(rng))
    q = rng.standard_normal((B, Hkv * G, D)).astype(np.float32)
    _select_sel_only(ops, q, blocks, B, Hkv * G, Hkv, [n], 64)


def test_select_needles_selected(ops):
    sel = _select_case(ops, synth.DT_BF16, 2, 8, 8, [700, 64], 4, seed=30, needle=True)
    assert (sel[:, :, 0] >= 0).all()


# ----------------------------------------------------------------------------
# S3
# ----------------------------------------------------------------------------
def _gpu_pool(ops, S, fwd_len):
    fwd = torch.full((fwd_len,), -1, dtype=torch.int32, device="cuda")
    return ops.CachePool(S, fwd)


def _random_sel(rng, B, Hkv, k, n_blk_max, prev=None, keep=0.8):
    sel = np.full((B, Hkv, k), -1, np.int32)
    for b in range(B):
        for h in range(Hkv):
            kk = int(rng.integers(max(1, k // 2), k + 1))
            base = set()
            if prev is not None:
                old = [j for j in prev[b, h] if j >= 0]
                base = set(rng.choice(old, size=int(len(old) * keep), replace=False).tolist()) if old else set()
            while len(base) < kk:
                base.add(int(rng.integers(0, n_blk_max)))
            sel[b, h, :kk] = np.sort(list(base))[:kk]
    return sel


def _cmp_pool(gp, op, S):
    np.testing.assert_array_equal(gp.slot_key.cpu().numpy(), op.slot_key)
    np.testing.assert_array_equal(gp.slot_stamp.cpu().numpy(), op.slot_stamp)
    np.testing.assert_array_equal(gp.fwd.cpu().numpy(), op.fwd)
    exp_order = np.lexsort((np.arange(S), op.slot_stamp)).astype(np.int32)
    np.testing.assert_array_equal(gp.order.cpu().numpy(), exp_order)
    inv = np.empty(S, np.int32)
    inv[exp_order] = np.arange(S, dtype=np.int32)
    np.testing.assert_array_equal(gp.order_pos.cpu().numpy(), inv)


@pytest.mark.parametrize("S", [300, 2048, 5000])
def test_cache_multistep_bit_exact(ops, S):
    rng = synth.rng_for(1000, 3, S)
    B, Hkv, k, L, max_blk = 3, 4, 40, 2, 256
    layer = 1
    fwd_len = B * L * Hkv * max_blk
    gp = _gpu_pool(ops, S, fwd_len)
    op = oracle.Pool(S, fwd_len)
    d = ops.dims(B, Hkv, Hkv)
    ws = ops.alloc_workspace(1, d, max_blk, k, S)
    req_ids = np.array([2, 0, 1], np.int32)
    E = B * Hkv * k
    slot = torch.empty(B, Hkv, k, dtype=torch.int32, device="cuda")
    hit = torch.empty(B, Hkv, k, dtype=torch.uint8, device="cuda")
    mk = torch.empty(E, dtype=torch.int64, device="cuda")
    ms = torch.empty(E, dtype=torch.int32, device="cuda")
    counts = torch.empty(4, dtype=torch.int32, device="cuda")
    prev = None
    saw_capacity = saw_evict = False
    for t in range(60):
        sel = _random_sel(rng, B, Hkv, k, max_blk, prev, keep=0.85)
        prev = sel
        before = op.copy()
        r = oracle.lru(op, sel, req_ids, layer, L, max_blk, stamp=10 + 2 * t)
        ops.kv_cache_lookup_insert(gp, to_torch(sel), to_torch(req_ids), layer, L, max_blk, k, d,
                                   10 + 2 * t, slot, hit, mk, ms, counts, ws)
        torch.cuda.synchronize()
        gc = counts.cpu().numpy()
        np.testing.assert_array_equal(gc, r["counts"])
        if r["counts"][3] == 0:
            np.testing.assert_array_equal(slot.cpu().numpy(), r["slot"])
            np.testing.assert_array_equal(hit.cpu().numpy(), r["hit"])
            m = int(r["counts"][1])
            np.testing.assert_array_equal(mk.cpu().numpy()[:m], r["miss_keys"])
            np.testing.assert_array_equal(ms.cpu().numpy()[:m], r["miss_slots"])
            saw_evict |= r["counts"][2] > 0
        else:
            saw_capacity = True
            np.testing.assert_array_equal(op.slot_stamp, before.slot_stamp)
        _cmp_pool(gp, op, S)
    if S == 300:
        assert saw_capacity
    if S == 2048:
        assert saw_evict


def test_cache_hand_traced_fixture(ops):
    import json, os
    fx = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lru_trace.json")))
    S = fx["num_slots"]
    gp = _gpu_pool(ops, S, fx["max_blk"])
    d = ops.dims(1, 1, 1)
    k = fx["k"]
    ws = ops.alloc_workspace(1, d, fx["max_blk"], k, S)
    slot = torch.empty(1, 1, k, dtype=torch.int32, device="cuda")
    hit = torch.empty(1, 1, k, dtype=torch.uint8, device="cuda")
    mk = torch.empty(k, dtype=torch.int64, device="cuda")
    ms = torch.empty(k, dtype=torch.int32, device="cuda")
    counts = torch.empty(4, dtype=torch.int32, device="cuda")
    for call in fx["calls"]:
        sel = np.array(call["sel"], np.int32).reshape(1, 1, k)
        ops.kv_cache_lookup_insert(gp, to_torch(sel), to_torch(np.array(fx["req_ids"], np.int32)),
                                   fx["layer"], fx["L"], fx["max_blk"], k, d, call["stamp"], slot,
                                   hit, mk, ms, counts, ws)
        torch.cuda.synchronize()
        assert counts.cpu().tolist() == call["counts"]
        assert gp.slot_key.cpu().tolist() == call["slot_key"]
        assert gp.slot_stamp.cpu().tolist() == call["slot_stamp"]
        assert gp.order.cpu().tolist() == call["order"]
        if call["counts"][3] == 0:
            assert slot.cpu().view(-1).tolist() == call["slot"]
            assert hit.cpu().view(-1).tolist() == call["hit"]
            m = call["counts"][1]
            assert mk.cpu().tolist()[:m] == call["miss_keys"]
            assert ms.cpu().tolist()[:m] == call["miss_slots"]


def test_cache_invalid_key(ops):
    S = 8
    gp = _gpu_pool(ops, S, 16)
    d = ops.dims(1, 1, 1)
    ws = ops.alloc_workspace(1, d, 32, 2, S)
    counts = torch.empty(4, dtype=torch.int32, device="cuda")
    ops.kv_cache_lookup_insert(gp, to_torch(np.array([[[3, 20]]], np.int32)),
                               to_torch(np.array([0], np.int32)), 0, 1, 32, 2, d, 1,
                               torch.empty(1, 1, 2, dtype=torch.int32, device="cuda"),
                               torch.empty(1, 1, 2, dtype=torch.uint8, device="cuda"),
                               torch.empty(2, dtype=torch.int64, device="cuda"),
                               torch.empty(2, dtype=torch.int32, device="cuda"), counts, ws)
    torch.cuda.synchronize()
    assert counts.cpu().tolist() == [0, 0, 0, 1]
    assert (gp.slot_stamp.cpu() == -1).all() and (gp.fwd.cpu() == -1).all()


# ----------------------------------------------------------------------------
# S4
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("bb", [16384, 32768, 4096 + 16])
def test_flash_h2d_gather_byte_exact(ops, bb):
    rng = np.random.default_rng(bb)
    HB, S, n = 97, 300, 150
    host_np = rng.integers(0, 256, size=(HB, bb), dtype=np.uint8)
    host = torch.from_numpy(host_np).pin_memory()
    pool_np = rng.integers(0, 256, size=(S, bb), dtype=np.uint8)
    pool = torch.from_numpy(pool_np.copy()).cuda()
    keys = rng.integers(0, 10 * HB, size=n).astype(np.int64)
    slots = rng.choice(S, size=n, replace=False).astype(np.int32)
    m = 120
    counts = torch.tensor([0, m, 0, 0], dtype=torch.int32, device="cuda")
    ops.flash_h2d_gather(ops.host_device_pointer(host), HB, to_torch(keys), to_torch(slots), counts,
                         n, pool, bb)
    torch.cuda.synchronize()
    exp = pool_np.copy()
    oracle.gather(host_np, HB, keys[:m], slots[:m], exp)
    np.testing.assert_array_equal(pool.cpu().numpy(), exp)
    # status != 0 -> no-op
    counts2 = torch.tensor([0, m, 0, 3], dtype=torch.int32, device="cuda")
    pool2 = torch.from_numpy(pool_np.copy()).cuda()
    ops.flash_h2d_gather(ops.host_device_pointer(host), HB, to_torch(keys), to_torch(slots), counts2,
                         n, pool2, bb)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(pool2.cpu().numpy(), pool_np)


# ----------------------------------------------------------------------------
# S5
# ----------------------------------------------------------------------------
def _attn_case(ops, dt, B, Hq, Hkv, k, S, tails, seed, empty_pair=False, q_scale=1.0,
               tail_garbage=False):
    rng = synth.rng_for(1000, 5, seed)
    pool_f = synth.kv_blocks(rng, S, D, synth.channel_scales(rng))
    tail_f = synth.kv_blocks(rng, B * Hkv, D).reshape(B, Hkv, 2, 32, D)
    q = rng.standard_normal((B, Hq, D)).astype(np.float32) * q_scale
    pool, tail, qs = synth.encode(pool_f, dt), synth.encode(tail_f, dt), synth.encode(q, dt)
    if tail_garbage:
        # rows >= tail_len are outside the contract: fill them with NaN / Inf bit
        # patterns, which must not reach the output (0 * NaN = NaN in a P.V product)
        nan = np.uint16(0x7FC0) if dt == synth.DT_BF16 else np.uint32(0x7FC00000)
        inf = np.uint16(0x7F80) if dt == synth.DT_BF16 else np.uint32(0x7F800000)
        tv = tail.view(np.uint16 if dt == synth.DT_BF16 else np.uint32)
        for b in range(B):
            tv[b, :, 0, tails[b]:] = nan
            tv[b, :, 1, tails[b]:] = inf
    slot = np.full((B, Hkv, k), -1, np.int32)
    for b in range(B):
        for h in range(Hkv):
            kk = int(rng.integers(1, k + 1))
            slot[b, h, :kk] = rng.choice(S, size=kk, replace=False)
    if empty_pair:
        slot[0, 0, :] = -1
    tl = np.array(tails, np.int32)
    scale = 1.0 / math.sqrt(D)
    exp = oracle.attention(qs, pool, slot, tail, tl, scale)
    d = ops.dims(B, Hq, Hkv)
    ws = ops.alloc_workspace(2, d, 32, k)
    out = torch.full((Hq, B, D), float("nan"), dtype=torch.float32, device="cuda")
    for rep in range(2):   # second run checks the workspace was left clean
        ops.sparse_decode_attn(to_torch(qs), to_torch(pool), to_torch(slot), k, to_torch(tail),
                               to_torch(tl), d, scale, out, ws)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        err = np.abs(got - exp).max()
        assert np.isfinite(got).all()
        assert err <= TOL[dt], f"max abs err {err}"
    return err


@pytest.mark.parametrize("dt", [synth.DT_BF16, synth.DT_F32])
@pytest.mark.parametrize("G", [1, 4])
def test_attention_tolerance(ops, dt, G):
    Hkv = 8 // G if G <= 8 else 1
    _attn_case(ops, dt, 3, Hkv * G, Hkv, 64, 700, [0, 17, 31], seed=G)


@pytest.mark.parametrize("G", [2, 8])
def test_attention_gqa_more(ops, G):
    _attn_case(ops, synth.DT_BF16, 2, 2 * G, 2, 128, 600, [1, 5], seed=40 + G)


def test_attention_empty_and_tail_only(ops):
    # pair (0,0) has no blocks and tail 0 -> O = 0 ; other pairs mixed
    _attn_case(ops, synth.DT_BF16, 2, 4, 4, 8, 64, [0, 9], seed=50, empty_pair=True)


@pytest.mark.parametrize("dt", [synth.DT_BF16, synth.DT_F32])
def test_attention_tail_rows_beyond_len_ignored(ops, dt):
    _attn_case(ops, dt, 3, 8, 2, 16, 200, [0, 1, 30], seed=70, tail_garbage=True)


@pytest.mark.parametrize("G", [1, 4])
def test_attention_sharp_softmax(ops, G):
    # |q| x 8: logits spread over tens of units, a few tokens carry the weight --
    # the regime where rounding P to bf16 alone (2^-9) would exceed 2e-3
    _attn_case(ops, synth.DT_BF16, 2, 4 * G, 4, 64, 500, [7, 20], seed=80 + G, q_scale=8.0)


def test_attention_many_pairs_stream_k(ops):
    # many pairs, k=64: units split across warp ranges at arbitrary points
    _attn_case(ops, synth.DT_BF16, 16, 32, 32, 64, 4096, [3] * 16, seed=60)


@pytest.mark.parametrize("G,k", [(1, 255), (2, 247), (4, 127), (8, 64)])
def test_attention_one_pair_many_contributors(ops, G, k):
    # one (b, h) pair cut over every warp of the launch (W = U / 8): its last
    # contributor merges up to 32 partials -- G = 1, 2 through the end-of-range
    # bulk-load merge (31 x 2 heads x 528 B: the 32 KiB edge), G = 4, 8 past it
    # (the register merge)
    _attn_case(ops, synth.DT_BF16, 1, G, 1, k, 600, [9], seed=90 + G)


def test_attention_skipped_on_error_status(ops):
    d = ops.dims(1, 1, 1)
    ws = ops.alloc_workspace(2, d, 32, 1)
    out = torch.full((1, 1, D), 7.0, dtype=torch.float32, device="cuda")
    pool = torch.zeros(2 * 32 * D, dtype=torch.bfloat16, device="cuda")
    tail = torch.zeros(2 * 32 * D, dtype=torch.bfloat16, device="cuda")
    ops.sparse_decode_attn(torch.zeros(1, 1, D, dtype=torch.bfloat16, device="cuda"), pool,
                           torch.zeros(1, 1, 1, dtype=torch.int32, device="cuda"), 1, tail,
                           torch.zeros(1, dtype=torch.int32, device="cuda"), d, 0.1, out, ws,
                           counts=torch.tensor([0, 0, 0, 3], dtype=torch.int32, device="cuda"))
    torch.cuda.synchronize()
    assert (out.cpu() == 7.0).all()


def test_cache_device_clock_mode(ops):
    # pool.clock set: the stamp is read on the device (*clock) and the host stamp
    # argument is ignored; several calls may share one stamp (request groups).
    rng = synth.rng_for(1000, 4)
    B, Hkv, k, max_blk, S = 2, 2, 16, 128, 80
    fwd_len = B * Hkv * max_blk
    fwd = torch.full((fwd_len,), -1, dtype=torch.int32, device="cuda")
    gp = ops.CachePool(S, fwd, clock=True)
    op = oracle.Pool(S, fwd_len)
    d = ops.dims(1, Hkv, Hkv)
    ws = ops.alloc_workspace(1, d, max_blk, k, S)
    E = Hkv * k
    slot = torch.empty(1, Hkv, k, dtype=torch.int32, device="cuda")
    hit = torch.empty(1, Hkv, k, dtype=torch.uint8, device="cuda")
    mk = torch.empty(E, dtype=torch.int64, device="cuda")
    ms = torch.empty(E, dtype=torch.int32, device="cuda")
    counts = torch.empty(4, dtype=torch.int32, device="cuda")
    prev = [None, None]
    for t in range(30):
        gp.clock.fill_(t + 1)
        for b in range(B):          # two calls per step (one per request), same stamp
            sel = _random_sel(rng, 1, Hkv, k, max_blk, prev[b], keep=0.7)
            prev[b] = sel
            req = np.array([b], np.int32)
            r = oracle.lru(op, sel, req, 0, 1, max_blk, stamp=t + 1)
            ops.kv_cache_lookup_insert(gp, to_torch(sel), to_torch(req), 0, 1, max_blk, k, d, 999999,
                                       slot, hit, mk, ms, counts, ws)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(counts.cpu().numpy(), r["counts"])
            if r["counts"][3] == 0:
                np.testing.assert_array_equal(slot.cpu().numpy(), r["slot"])
            _cmp_pool(gp, op, S)
        assert int(gp.clock.item()) == t + 1


def test_cache_fused_form_bit_exact(ops):
    """The fused one-launch form of kv_cache_lookup_insert (SS_CACHE_FUSED=1 in
    the debug build, libsparseserve_debug.so) against the oracle: the cache
    parity tests and the request-group pipelines re-run in a subprocess."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    from paper_2509_24626_b200 import build as _build
    if not os.path.exists(_build.LIB_DEBUG):
        pytest.skip("debug library not built (python -m paper_2509_24626_b200.build --debug)")
    env = dict(os.environ, SS_CACHE_FUSED="1", SS_LIB_VARIANT="debug")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_parity.py"),
                        os.path.join(root, "tests", "test_gpu_pipeline.py"),
                        "-k", "(cache or request_groups) and not fused_form"],
                       env=env, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_select_attention_alternative_forms_bit_exact(ops):
    """The forms the default paths fall back to, forced through the debug
    build (libsparseserve_debug.so): the per-chunk tensor-core select with its
    workspace merge (SS_SEL_TCC=0), the MHA select's workspace-merge form
    (SS_SEL_MHA_CLU=0) and the attention's register merge at the range end
    (SS_ATTN_MERGE_BULK=0) -- the select and attention parity tests re-run in a
    subprocess against the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    from paper_2509_24626_b200 import build as _build
    if not os.path.exists(_build.LIB_DEBUG):
        pytest.skip("debug library not built (python -m paper_2509_24626_b200.build --debug)")
    env = dict(os.environ, SS_SEL_TCC="0", SS_SEL_MHA_CLU="0", SS_ATTN_MERGE_BULK="0", SS_LIB_VARIANT="debug")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(root, "tests", "test_gpu_parity.py"),
                        "-k", "(select or attention) and not alternative_forms and not beyond_cluster"],
                       env=env, capture_output=True, text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("dt", [synth.DT_BF16, synth.DT_F32])
@pytest.mark.parametrize("G", [1, 4])
def test_attention_split_hits_misses_merge(ops, dt, G):
    """Split form (sparse_decode_attn_part + sparse_attn_merge): the hit part
    (+ tail) and the miss part each equal the oracle's attention over that
    subset, and their log-sum-exp merge equals the oracle's attention over the
    whole set (PAPER.md:71-72 over disjoint token sets); empty subsets give 0."""
    B, Hkv, k, S = 3, 8 // G, 48, 500
    Hq = Hkv * G
    rng = synth.rng_for(1000, 6, G + (10 if dt == synth.DT_F32 else 0))
    pool = synth.encode(synth.kv_blocks(rng, S, D, synth.channel_scales(rng)), dt)
    tail = synth.encode(synth.kv_blocks(rng, B * Hkv, D).reshape(B, Hkv, 2, 32, D), dt)
    qs = synth.encode(rng.standard_normal((B, Hq, D)).astype(np.float32), dt)
    slot = np.full((B, Hkv, k), -1, np.int32)
    for b in range(B):
        for h in range(Hkv):
            kk = int(rng.integers(1, k + 1))
            slot[b, h, :kk] = rng.choice(S, size=kk, replace=False)
    hit = (rng.random((B, Hkv, k)) < 0.9).astype(np.uint8)
    hit[0, 0, :] = 1          # a pair without misses: empty miss part
    hit[1, 0, :] = 0          # a pair without hits: hit part = tail only
    tl = np.array([0, 17, 31], np.int32)
    scale = 1.0 / math.sqrt(D)
    slot_h = np.where(hit == 1, slot, -1).astype(np.int32)
    slot_m = np.where(hit == 0, slot, -1).astype(np.int32)
    exp_all = oracle.attention(qs, pool, slot, tail, tl, scale)
    exp_h = oracle.attention(qs, pool, slot_h, tail, tl, scale)
    exp_m = oracle.attention(qs, pool, slot_m, tail, np.zeros(B, np.int32), scale)
    d = ops.dims(B, Hq, Hkv)
    ws = ops.alloc_workspace(2, d, 32, k)
    T = lambda x: to_torch(x)
    o_h = torch.full((Hq, B, D), float("nan"), dtype=torch.float32, device="cuda")
    o_m, o = torch.full_like(o_h, float("nan")), torch.full_like(o_h, float("nan"))
    l_h = torch.full((Hq, B), float("nan"), dtype=torch.float32, device="cuda")
    l_m = torch.full_like(l_h, float("nan"))
    ops.sparse_decode_attn_part(T(qs), T(pool), T(slot), T(hit), 1, k, T(tail), T(tl), d, scale, o_h, l_h, ws)
    ops.sparse_decode_attn_part(T(qs), T(pool), T(slot), T(hit), 2, k, T(tail), T(tl), d, scale, o_m, l_m, ws)
    ops.sparse_attn_merge(o_h, l_h, o_m, l_m, o)
    torch.cuda.synchronize()
    for got, exp in ((o_h, exp_h), (o_m, exp_m), (o, exp_all)):
        g = got.cpu().numpy()
        assert np.isfinite(g).all()
        assert np.abs(g - exp).max() <= TOL[dt]
    lm = l_m.cpu().numpy()
    assert np.isneginf(lm[0:G, 0]).all()                         # pair (0, 0): no misses
    assert np.isfinite(l_h.cpu().numpy()).all()                   # every hit part has a tail or hits
    # mode 0 = the one-call attention
    o0, l0 = torch.empty_like(o_h), torch.empty_like(l_h)
    ops.sparse_decode_attn_part(T(qs), T(pool), T(slot), T(hit), 0, k, T(tail), T(tl), d, scale, o0, l0, ws)
    torch.cuda.synchronize()
    assert np.abs(o0.cpu().numpy() - exp_all).max() <= TOL[dt]
