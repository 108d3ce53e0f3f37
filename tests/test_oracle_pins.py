"""Pins for the CPU oracle (oracle/oracle.c) against things other than itself:
library routines, exact rational arithmetic, invariants, special cases that
reduce to textbook definitions, and hand-traced fixtures.  CPU only.

Each test names the PAPER.md passage / DESIGN.md reading it pins.
"""
import collections
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
D = 128


def _bf16(x):
    return synth.f32_to_bf16_bits(np.asarray(x, dtype=np.float32))


def _val(bits):
    return synth.decode_f64(bits, synth.DT_BF16)


# ----------------------------------------------------------------------------
# S0 block metadata (reading R1, R16)
# ----------------------------------------------------------------------------
@pytest.mark.parametrize("dt", [synth.DT_BF16, synth.DT_F32])
def test_meta_matches_numpy_min_max(dt):
    rng = synth.rng_for(900, 1)
    blocks = synth.kv_blocks(rng, 37, D, synth.channel_scales(rng))
    store = synth.encode(blocks, dt)
    meta = oracle.block_meta(store, key_stride=2 * 32 * D)
    vals = synth.decode_f64(store, dt)[:, 0]            # [n][32][d] keys
    got = synth.decode_f64(meta, dt)
    np.testing.assert_array_equal(got[:, 0], vals.min(axis=1))
    np.testing.assert_array_equal(got[:, 1], vals.max(axis=1))


def test_meta_signed_zero_hand_cases():
    # channel 0: tokens hold +0 and -0 only -> min is -0 (0x8000), max is +0 (0x0000)
    # channel 1: all +0 -> both +0; channel 2: all -0 -> both -0
    keys = np.zeros((1, 32, D), dtype=np.uint16)
    keys[0, 5, 0] = 0x8000
    keys[0, :, 2] = 0x8000
    keys[0, 7, 3] = _bf16(-1.5).item()
    keys[0, 9, 3] = _bf16(2.25).item()
    meta = oracle.block_meta(keys)
    assert meta[0, 0, 0] == 0x8000 and meta[0, 1, 0] == 0x0000
    assert meta[0, 0, 1] == 0x0000 and meta[0, 1, 1] == 0x0000
    assert meta[0, 0, 2] == 0x8000 and meta[0, 1, 2] == 0x8000
    assert meta[0, 0, 3] == _bf16(-1.5) and meta[0, 1, 3] == _bf16(2.25)


# ----------------------------------------------------------------------------
# S1 block score (readings R2, R3, R4)
# ----------------------------------------------------------------------------
def _exact_bound(qv, mv, Mv):
    """exact rational Quest bound sum_c max(q_c M_c, q_c m_c)."""
    s = Fraction(0)
    for qc, lo, hi in zip(qv, mv, Mv):
        a, b = Fraction(qc) * Fraction(hi), Fraction(qc) * Fraction(lo)
        s += a if a > b else b
    return s


def _meta_from_blocks(store, n_req, hkv, max_blk):
    meta = oracle.block_meta(store, key_stride=2 * 32 * D)
    return meta.reshape(n_req, hkv, max_blk, 2, D)


def test_score_exact_when_partial_sums_are_representable():
    # small dyadic values: every product and partial sum is exact in fp64,
    # so the oracle must equal the exact rational bound bit-for-bit.
    rng = np.random.default_rng(7)
    q = (rng.integers(-8, 9, size=(1, 1, D)) / 4.0).astype(np.float32)
    keys = (rng.integers(-16, 17, size=(6, 2, 32, D)) / 8.0).astype(np.float32)
    qs, ks = _bf16(q), _bf16(keys)
    meta = _meta_from_blocks(ks, 1, 1, 6)
    sc = oracle.block_score(qs, meta, np.array([6], np.int32))
    qv = _val(qs)[0, 0]
    mv = _val(meta)[0, 0]
    for j in range(6):
        ex = _exact_bound(qv, mv[j, 0], mv[j, 1])
        assert Fraction(sc[0, 0, j]) == ex


def test_score_within_rounding_of_exact_and_sound():
    rng = synth.rng_for(900, 2)
    n = 8
    blocks = synth.kv_blocks(rng, n, D, synth.channel_scales(rng))
    ks = _bf16(blocks)
    qs = _bf16(rng.standard_normal((1, 1, D)))
    meta = _meta_from_blocks(ks, 1, 1, n)
    sc = oracle.block_score(qs, meta, np.array([n], np.int32))
    qv = _val(qs)[0, 0]
    mv = _val(meta)[0, 0]
    kv = _val(ks)[:, 0]                       # [n][32][d]
    u = 2.0 ** -53
    for j in range(n):
        ex = _exact_bound(qv, mv[j, 0], mv[j, 1])
        mag = sum(abs(Fraction(qc)) * max(abs(Fraction(a)), abs(Fraction(b)))
                  for qc, a, b in zip(qv, mv[j, 0], mv[j, 1]))
        assert abs(Fraction(sc[0, 0, j]) - ex) <= Fraction(D * u) * mag
        # bound soundness (P2): exact bound >= exact q.k of every token in the block
        best_dot = max(sum(Fraction(a) * Fraction(b) for a, b in zip(qv, kv[j, t])) for t in range(32))
        assert ex >= best_dot


def test_score_identical_tokens_is_exact_dot_product():
    # special case (P3): all tokens of a block equal -> M = m = k -> bound = q.k
    rng = synth.rng_for(900, 3)
    k1 = rng.standard_normal((5, 1, 1, D)).astype(np.float32)
    blocks = np.broadcast_to(k1, (5, 2, 32, D)).copy()
    ks = _bf16(blocks)
    qs = _bf16(rng.standard_normal((1, 1, D)))
    meta = _meta_from_blocks(ks, 1, 1, 5)
    sc = oracle.block_score(qs, meta, np.array([5], np.int32))
    qv, kv = _val(qs)[0, 0], _val(ks)[:, 0, 0]
    for j in range(5):
        dot = sum(Fraction(a) * Fraction(b) for a, b in zip(qv, kv[j]))
        assert abs(Fraction(sc[0, 0, j]) - dot) <= Fraction(2.0 ** -45) * (1 + abs(dot))
    # and it ranks blocks exactly as numpy's dot products do
    order = np.argsort(-(kv @ qv), kind="stable")
    np.testing.assert_array_equal(np.argsort(-sc[0, 0], kind="stable"), order)


def test_score_gqa_is_max_over_group():
    # reading R4: score of a KV head = max over its G query heads; hq = h*G + g
    rng = synth.rng_for(900, 4)
    B, Hq, Hkv, n = 2, 8, 2, 4
    G = Hq // Hkv
    q = (rng.integers(-4, 5, size=(B, Hq, D)) / 2.0).astype(np.float32)
    keys = (rng.integers(-8, 9, size=(B * Hkv * n, 2, 32, D)) / 4.0).astype(np.float32)
    qs, ks = _bf16(q), _bf16(keys)
    meta = _meta_from_blocks(ks, B, Hkv, n)
    sc = oracle.block_score(qs, meta, np.array([n, n - 1], np.int32))
    qv, mv = _val(qs), _val(meta)
    for b in range(B):
        for h in range(Hkv):
            for j in range(n - b):
                per = [_exact_bound(qv[b, h * G + g], mv[b, h, j, 0], mv[b, h, j, 1]) for g in range(G)]
                assert Fraction(sc[b, h, j]) == max(per)
    assert np.isnan(sc[1, :, n - 1]).all()   # j >= n_blk untouched


# ----------------------------------------------------------------------------
# S2 top-k (readings R5, R6)
# ----------------------------------------------------------------------------
def _lexsort_topk(s, n, k):
    j = np.arange(n)
    order = np.lexsort((j, -s[:n]))
    out = np.sort(order[:min(k, n)])
    return np.concatenate([out, -np.ones(k - out.shape[0], dtype=np.int64)])


@pytest.mark.parametrize("k", [1, 7, 64, 300])
def test_topk_matches_numpy_lexsort(k):
    rng = synth.rng_for(900, 5, k)
    B, Hkv, max_blk = 3, 4, 256
    scores = rng.standard_normal((B, Hkv, max_blk))
    scores[0, 1, 10:20] = scores[0, 1, 5]          # tie suite straddling the boundary
    scores[1, 2, :] = 0.5                          # all ties
    n_blk = np.array([256, 200, 3], np.int32)
    sel = oracle.topk(scores, n_blk, k)
    for b in range(B):
        for h in range(Hkv):
            np.testing.assert_array_equal(sel[b, h], _lexsort_topk(scores[b, h], n_blk[b], k))


def test_topk_invariants():
    rng = synth.rng_for(900, 6)
    s = np.round(rng.standard_normal((1, 1, 500)) * 4) / 4    # many ties
    sel = oracle.topk(s, np.array([500], np.int32), 50)[0, 0]
    chosen = set(sel.tolist())
    assert list(sel) == sorted(sel)
    mn = min(s[0, 0, j] for j in chosen)
    for j in range(500):
        if j not in chosen:
            assert s[0, 0, j] <= mn
            if s[0, 0, j] == mn:
                assert all(c < j for c in chosen if s[0, 0, c] == mn)


def test_needle_block_is_selected():
    # P4: a block holding a key = alpha * q_hat with alpha large enough that its
    # token logit exceeds every other block's bound is provably top-1.
    rng = synth.rng_for(900, 7)
    n = 64
    blocks = synth.kv_blocks(rng, n, D)
    q = rng.standard_normal(D).astype(np.float32)
    jstar = 41
    blocks[jstar, 0, 3] = 100.0 * q / np.linalg.norm(q)
    ks, qs = _bf16(blocks), _bf16(q[None, None])
    meta = _meta_from_blocks(ks, 1, 1, n)
    sc = oracle.block_score(qs, meta, np.array([n], np.int32))
    qv, kv = _val(qs)[0, 0], _val(ks)[:, 0]
    needle_dot = float(kv[jstar, 3] @ qv)
    others = [sc[0, 0, j] for j in range(n) if j != jstar]
    assert needle_dot > max(others)           # the premise of the pin
    for k in (1, 4, 16):
        assert jstar in oracle.topk(sc, np.array([n], np.int32), k)[0, 0]


# ----------------------------------------------------------------------------
# S3 LRU (readings R11, R12)
# ----------------------------------------------------------------------------
def test_lru_hand_traced_fixture():
    fx = json.load(open(os.path.join(GOLDEN, "lru_trace.json")))
    pool = oracle.Pool(fx["num_slots"], fwd_len=fx["max_blk"])
    for call in fx["calls"]:
        sel = np.array(call["sel"], np.int32).reshape(1, 1, -1)
        before = pool.copy()
        r = oracle.lru(pool, sel, np.array(fx["req_ids"], np.int32), fx["layer"], fx["L"],
                       fx["max_blk"], call["stamp"])
        assert r["counts"].tolist() == call["counts"]
        assert pool.slot_key.tolist() == call["slot_key"]
        assert pool.slot_stamp.tolist() == call["slot_stamp"]
        order = np.lexsort((np.arange(pool.num_slots), pool.slot_stamp))
        assert order.tolist() == call["order"]
        if call["counts"][3] == 0:
            assert r["slot"].ravel().tolist() == call["slot"]
            assert r["hit"].ravel().tolist() == call["hit"]
            assert r["miss_keys"].tolist() == call["miss_keys"]
            assert r["miss_slots"].tolist() == call["miss_slots"]
        else:   # P7: capacity error leaves the state byte-identical
            np.testing.assert_array_equal(pool.fwd, before.fwd)
            np.testing.assert_array_equal(pool.slot_key, before.slot_key)
            np.testing.assert_array_equal(pool.slot_stamp, before.slot_stamp)
        # fwd is the inverse of slot_key
        for s, key in enumerate(pool.slot_key):
            if key >= 0:
                assert pool.fwd[key] == s
        assert (pool.fwd >= 0).sum() == (pool.slot_key >= 0).sum()


@pytest.mark.parametrize("S", [1, 2, 3, 5, 8])
def test_lru_one_key_per_call_equals_ordereddict(S):
    # P5: with one key per call, batch-LRU is textbook LRU (collections.OrderedDict)
    rng = np.random.default_rng(100 + S)
    universe = 3 * S + 2
    pool = oracle.Pool(S, fwd_len=64)
    od = collections.OrderedDict()      # key -> slot, LRU first
    used = 0
    for t in range(1, 1500):
        key = int(rng.integers(0, universe))
        r = oracle.lru(pool, np.array([[[key]]], np.int32), np.array([0], np.int32), 0, 1, 64, t)
        if key in od:
            od.move_to_end(key)
            assert r["hit"][0, 0, 0] == 1 and r["slot"][0, 0, 0] == od[key]
        else:
            if len(od) == S:
                _, slot = od.popitem(last=False)
            else:
                slot, used = used, used + 1
            od[key] = slot
            assert r["hit"][0, 0, 0] == 0 and r["slot"][0, 0, 0] == slot
        for k_, s_ in od.items():
            assert pool.slot_key[s_] == k_


def test_lru_invalid_key_is_error_without_mutation():
    pool = oracle.Pool(4, fwd_len=16)
    before = pool.copy()
    r = oracle.lru(pool, np.array([[[3, 20]]], np.int32), np.array([0], np.int32), 0, 1, 32, 1)
    assert r["counts"].tolist() == [0, 0, 0, 1]
    np.testing.assert_array_equal(pool.fwd, before.fwd)
    np.testing.assert_array_equal(pool.slot_stamp, before.slot_stamp)


# ----------------------------------------------------------------------------
# S4 gather
# ----------------------------------------------------------------------------
def test_gather_matches_numpy_fancy_index():
    rng = np.random.default_rng(5)
    host = rng.integers(0, 256, size=(50, 64), dtype=np.uint8)
    pool = rng.integers(0, 256, size=(10, 64), dtype=np.uint8)
    keys = np.array([3, 77, 49, 120], np.int64)        # 77 and 120 alias modulo 50
    slots = np.array([9, 0, 4, 2], np.int32)
    exp = pool.copy()
    exp[slots] = host[keys % 50]
    oracle.gather(host, 50, keys, slots, pool)
    np.testing.assert_array_equal(pool, exp)


# ----------------------------------------------------------------------------
# S5 attention (readings R7, R9, R10)
# ----------------------------------------------------------------------------
def _sdpa(q, k, v, mask=None):
    """torch scaled_dot_product_attention in float64 on CPU (library routine)."""
    q = torch.from_numpy(q)[None, None, None]          # [1,1,1,d]
    k = torch.from_numpy(k)[None, None]                 # [1,1,T,d]
    v = torch.from_numpy(v)[None, None]
    m = None if mask is None else torch.from_numpy(mask)[None, None, None]
    return torch.nn.functional.scaled_dot_product_attention(q, k, v, attn_mask=m)[0, 0, 0].numpy()


@pytest.mark.parametrize("dt", [synth.DT_BF16, synth.DT_F32])
@pytest.mark.parametrize("tail_len", [0, 17])
def test_attention_all_blocks_equals_dense_sdpa(dt, tail_len):
    rng = synth.rng_for(900, 8, tail_len)
    B, Hq, Hkv, n = 2, 4, 2, 6
    G = Hq // Hkv
    blocks = synth.kv_blocks(rng, B * Hkv * n, D)
    tail = synth.kv_blocks(rng, B * Hkv, D).reshape(B, Hkv, 2, 32, D)
    pool = synth.encode(blocks, dt)
    tails = synth.encode(tail, dt)
    qs = synth.encode(rng.standard_normal((B, Hq, D)), dt)
    # pool slot of (b, h, j) = (b*Hkv + h)*n + j; k = n covers every block (shuffled order)
    slot = np.empty((B, Hkv, n), np.int32)
    for b in range(B):
        for h in range(Hkv):
            slot[b, h] = (b * Hkv + h) * n + rng.permutation(n)
    tl = np.array([tail_len, tail_len // 2], np.int32)
    out = oracle.attention(qs, pool, slot, tails, tl, 1.0 / math.sqrt(D))
    pv, tv, qv = synth.decode_f64(pool, dt), synth.decode_f64(tails, dt), synth.decode_f64(qs, dt)
    for b in range(B):
        for hq in range(Hq):
            h = hq // G
            ids = np.arange(n) + (b * Hkv + h) * n
            K = np.concatenate([pv[ids, 0].reshape(-1, D), tv[b, h, 0, :tl[b]]])
            V = np.concatenate([pv[ids, 1].reshape(-1, D), tv[b, h, 1, :tl[b]]])
            np.testing.assert_allclose(out[hq, b], _sdpa(qv[b, hq], K, V), rtol=0, atol=1e-12)


def test_attention_subset_equals_masked_dense():
    # P9: attending only to the selected blocks == dense attention with -inf outside them
    rng = synth.rng_for(900, 9)
    n = 10
    blocks = synth.kv_blocks(rng, n, D)
    pool = synth.encode(blocks, synth.DT_BF16)
    qs = synth.encode(rng.standard_normal((1, 1, D)), synth.DT_BF16)
    chosen = np.array([1, 4, 7, -1, -1], np.int32)
    tails = synth.encode(synth.kv_blocks(rng, 1, D).reshape(1, 1, 2, 32, D), synth.DT_BF16)
    out = oracle.attention(qs, pool, chosen.reshape(1, 1, -1), tails, np.array([5], np.int32),
                           1.0 / math.sqrt(D))
    pv, tv, qv = _val(pool), _val(tails), _val(qs)
    K = np.concatenate([pv[:, 0].reshape(-1, D), tv[0, 0, 0]])
    V = np.concatenate([pv[:, 1].reshape(-1, D), tv[0, 0, 1]])
    mask = np.full(K.shape[0], -np.inf)
    for j in (1, 4, 7):
        mask[j * 32:(j + 1) * 32] = 0.0
    mask[n * 32:n * 32 + 5] = 0.0
    np.testing.assert_allclose(out[0, 0], _sdpa(qv[0, 0], K, V, mask), rtol=0, atol=1e-12)


def test_attention_empty_set_is_zero():
    pool = np.zeros((1, 2, 32, D), np.uint16)
    tails = np.zeros((1, 1, 2, 32, D), np.uint16)
    out = oracle.attention(np.zeros((1, 1, D), np.uint16), pool, np.full((1, 1, 3), -1, np.int32),
                           tails, np.array([0], np.int32), 0.1)
    assert (out == 0).all()


def test_block_geometry_golden():
    fx = json.load(open(os.path.join(GOLDEN, "block_geometry.json")))
    assert fx["block_tokens"] * fx["head_dim"] * 2 * 2 == fx["bytes_per_head_block_kv_2byte"]
    assert synth.BLOCK_TOKENS == fx["block_tokens"] and synth.HEAD_DIM == fx["head_dim"]
    assert fx["token_budget"] // fx["block_tokens"] == synth.C2.topk


# ----------------------------------------------------------------------------
# NEXT-1: append / seal / FlashD2H scatter
# ----------------------------------------------------------------------------
def test_kv_append_and_seal_match_numpy():
    rng = synth.rng_for(900, 20)
    B, Hkv, max_blk = 3, 2, 64
    tail = np.zeros((B, Hkv, 2, 32, D), np.uint16)
    tail_len = np.array([0, 29, 5], np.int32)
    n_blk = np.array([3, 7, 0], np.int32)
    meta = np.zeros((B, Hkv, max_blk, 2, D), np.uint16)
    ref_tail = tail.copy()
    ref_len = tail_len.copy()
    for step in range(3):
        new = synth.encode(rng.standard_normal((B, Hkv, 2, D)), synth.DT_BF16)
        oracle.kv_append(new, tail, tail_len, advance=True)
        for b in range(B):                      # numpy slicing: the definition of "append"
            ref_len[b] += 1
            ref_tail[b, :, :, ref_len[b] - 1] = new[b]
        np.testing.assert_array_equal(tail, ref_tail)
        np.testing.assert_array_equal(tail_len, ref_len)
        # a second layer writes the same row without advancing
        oracle.kv_append(new, tail, tail_len, advance=False)
        np.testing.assert_array_equal(tail, ref_tail)
    assert tail_len[1] == 32
    full = tail[1].copy()
    staging = oracle.kv_seal([1], tail, tail_len, n_blk, meta)
    np.testing.assert_array_equal(staging[0], full)
    vals = _val(full[:, 0])                       # [Hkv][32][d] keys
    np.testing.assert_array_equal(_val(meta[1, :, 7, 0]), vals.min(axis=1))
    np.testing.assert_array_equal(_val(meta[1, :, 7, 1]), vals.max(axis=1))
    assert n_blk.tolist() == [3, 8, 0] and tail_len[1] == 0


def test_d2h_scatter_matches_numpy():
    rng = np.random.default_rng(3)
    st = rng.integers(0, 256, size=(5, 64), dtype=np.uint8)
    host = rng.integers(0, 256, size=(11, 64), dtype=np.uint8)
    keys = np.array([3, 14, 9, 0, 21], np.int64)
    exp = host.copy()
    exp[keys % 11] = st
    oracle.d2h_scatter(st, keys, host, 11)
    np.testing.assert_array_equal(host, exp)


def test_prefill_save_matches_numpy_relayout():
    # NEXT-4: (N,H,D) -> per-head 32-token blocks, metadata,
    # DRAM home of each block, tail -- checked with numpy reshapes / transposes
    rng = synth.rng_for(900, 30)
    n, Hkv, L, layer, max_blk, B, b, req = 32 * 5 + 11, 3, 4, 2, 32, 2, 1, 1
    k = synth.encode(rng.standard_normal((n, Hkv, D)), synth.DT_BF16)
    v = synth.encode(rng.standard_normal((n, Hkv, D)), synth.DT_BF16)
    meta = np.zeros((B, Hkv, max_blk, 2, D), np.uint16)
    tail = np.zeros((B, Hkv, 2, 32, D), np.uint16)
    n_blk = np.zeros(B, np.int32)
    tl = np.zeros(B, np.int32)
    hb = B * L * Hkv * max_blk
    host = np.zeros((hb, 2 * 32 * D * 2), np.uint8)
    oracle.prefill_save(k, v, b, req, layer, L, meta, tail, n_blk, tl, host, hb)
    nb = n // 32
    blocks = np.stack([k[:nb * 32].reshape(nb, 32, Hkv, D), v[:nb * 32].reshape(nb, 32, Hkv, D)], axis=1)
    blocks = blocks.transpose(3, 0, 1, 2, 4)          # [Hkv][nb][2][32][d]
    for h in range(Hkv):
        key0 = ((req * L + layer) * Hkv + h) * max_blk
        got = host[key0:key0 + nb].view(np.uint16).reshape(nb, 2, 32, D)
        np.testing.assert_array_equal(got, blocks[h])
        vals = _val(blocks[h][:, 0])
        np.testing.assert_array_equal(_val(meta[b, h, :nb, 0]), vals.min(axis=1))
        np.testing.assert_array_equal(_val(meta[b, h, :nb, 1]), vals.max(axis=1))
        np.testing.assert_array_equal(tail[b, h, 0, :11], k[nb * 32:, h])
        np.testing.assert_array_equal(tail[b, h, 1, :11], v[nb * 32:, h])
    assert n_blk[b] == nb and tl[b] == 11


# ----------------------------------------------------------------------------
# NEXT-3 mean-of-keys metadata and its score ("simply calculating the mean
# values of the token keys [45]"; reading R18)
# ----------------------------------------------------------------------------
def _f32_of_exact(fr):
    """float32 nearest (RNE) to an exact rational that fits float64 exactly."""
    x = float(fr)
    assert Fraction(x) == fr
    return np.float32(x)


@pytest.mark.parametrize("dt", [synth.DT_BF16, synth.DT_F32])
def test_mean_meta_is_exact_rational_mean(dt):
    # dyadic keys: the exact mean is a float32 value, so mu must equal it exactly
    rng = np.random.default_rng(31)
    keys = (rng.integers(-16, 17, size=(5, 2, 32, D)) / 8.0).astype(np.float32)
    store = synth.encode(keys, dt)
    mu = oracle.block_mean(store, key_stride=2 * 32 * D)
    kv = synth.decode_f64(store, dt)[:, 0]
    for i in range(5):
        for c in range(0, D, 7):
            ex = sum(Fraction(v) for v in kv[i, :, c]) / 32
            assert mu[i, c] == _f32_of_exact(ex)


def test_mean_meta_gaussian_keys_round_once():
    # realistic bf16 keys: the fp64 sum of 32 bf16 values is exact here, so mu is
    # the float32 rounding of the exact mean; numpy's float64 mean agrees to 1 ulp
    rng = synth.rng_for(901, 1)
    blocks = synth.kv_blocks(rng, 9, D, synth.channel_scales(rng))
    store = synth.encode(blocks, synth.DT_BF16)
    mu = oracle.block_mean(store, key_stride=2 * 32 * D)
    kv = synth.decode_f64(store, synth.DT_BF16)[:, 0]
    for i in range(9):
        for c in range(D):
            ex = sum(Fraction(v) for v in kv[i, :, c]) / 32
            if Fraction(float(ex)) == ex:
                assert mu[i, c] == _f32_of_exact(ex)
    np.testing.assert_allclose(mu, kv.mean(axis=1), rtol=2 ** -23, atol=0)


def test_mean_score_exact_and_gqa_max():
    rng = np.random.default_rng(32)
    B, Hq, Hkv, n = 2, 8, 2, 5
    G = Hq // Hkv
    q = (rng.integers(-4, 5, size=(B, Hq, D)) / 2.0).astype(np.float32)
    keys = (rng.integers(-8, 9, size=(B * Hkv * n, 2, 32, D)) / 4.0).astype(np.float32)
    qs, ks = _bf16(q), _bf16(keys)
    mu = oracle.block_mean(ks, key_stride=2 * 32 * D).reshape(B, Hkv, n, D)
    sc = oracle.block_score_mean(qs, mu, np.array([n, n - 2], np.int32))
    qv, kv = _val(qs), _val(ks)[:, 0].reshape(B, Hkv, n, 32, D)
    for b in range(B):
        for h in range(Hkv):
            for j in range(n - 2 * b):
                mean = [sum(Fraction(v) for v in kv[b, h, j, :, c]) / 32 for c in range(D)]
                per = [sum(Fraction(qc) * m for qc, m in zip(qv[b, h * G + g], mean)) for g in range(G)]
                assert Fraction(sc[b, h, j]) == max(per)
    assert np.isnan(sc[1, :, n - 2:]).all()


def test_mean_score_of_identical_tokens_equals_minmax_score():
    # all tokens of a block equal: mean = M = m = the key, so the mean score and
    # the (separately pinned) min/max bound are the same exact dot product
    rng = synth.rng_for(901, 2)
    k1 = rng.standard_normal((6, 1, 1, D)).astype(np.float32)
    ks = _bf16(np.broadcast_to(k1, (6, 2, 32, D)).copy())
    qs = _bf16(rng.standard_normal((1, 4, D)))
    mu = oracle.block_mean(ks, key_stride=2 * 32 * D).reshape(1, 1, 6, D)
    np.testing.assert_array_equal(mu[0, 0], _val(ks)[:, 0, 0])
    s_mean = oracle.block_score_mean(qs, mu, np.array([6], np.int32))
    s_mm = oracle.block_score(qs, _meta_from_blocks(ks, 1, 1, 6), np.array([6], np.int32))
    np.testing.assert_array_equal(s_mean, s_mm)


# ----------------------------------------------------------------------------
# NEXT-2 decoding working set (§3.3) and Algorithm 1
# ----------------------------------------------------------------------------
def test_ws_estimate_closed_forms():
    T, L, B, Hkv, k, mb = 20, 2, 3, 2, 5, 400
    # the same k blocks every step: the union never grows past k per head
    const = np.broadcast_to(np.arange(k, dtype=np.int32), (T, L, B, Hkv, k))
    for w in (1, 4, 12):
        assert (oracle.ws_estimate(const, mb, w) == L * Hkv * k).all()
    # disjoint selections every step: the union is min(t+1, w) * k per head
    disj = (np.arange(T, dtype=np.int32)[:, None, None, None, None] * k
            + np.arange(k, dtype=np.int32)) * np.ones((1, L, B, Hkv, 1), np.int32)
    for w in (1, 3, 12):
        ws = oracle.ws_estimate(disj, mb, w)
        for t in range(T):
            assert (ws[t] == L * Hkv * min(t + 1, w) * k).all()
    # empty selections count nothing; -1 entries are not blocks
    assert (oracle.ws_estimate(np.full((T, L, B, Hkv, k), -1, np.int32), mb, 12) == 0).all()


def test_ws_estimate_brute_force_and_monotone_in_w():
    rng = np.random.default_rng(3)
    T, L, B, Hkv, k, mb = 16, 2, 2, 3, 6, 40
    hist = rng.integers(-1, mb, size=(T, L, B, Hkv, k)).astype(np.int32)
    prev = None
    for w in (1, 2, 5, 12, 16):
        ws = oracle.ws_estimate(hist, mb, w)
        for t in range(T):
            for b in range(B):
                exp = sum(len({int(j) for s in range(max(0, t - w + 1), t + 1)
                               for j in hist[s, l, b, h] if j >= 0})
                          for l in range(L) for h in range(Hkv))
                assert ws[t, b] == exp
        if w == 1:   # w = 1: the working set is this step's distinct selections
            assert (ws == np.array([[sum(len(set(hist[t, l, b, h][hist[t, l, b, h] >= 0].tolist()))
                                         for l in range(L) for h in range(Hkv))
                                     for b in range(B)] for t in range(T)])).all()
        if prev is not None:  # Fig. 8: a longer window never shrinks the union
            assert (ws >= prev).all()
        prev = ws


def test_admit_hand_traced_algorithm1():
    # M_avl = 10: 4 (used 4) add; 7 (11 > 10) reset; 6 (10) add; 1 (11) reset; 0 (10) add
    assert oracle.admit([4, 7, 6, 1, 0], 10) == [True, False, True, False, True]
    # a large request early is reset, later small ones still fit (no early stop)
    assert oracle.admit([20, 3, 3, 3], 9) == [False, True, True, True]
    assert oracle.admit([1, 2], 0) == [False, False]
    assert oracle.admit([0, 0], 0) == [True, True]
    assert oracle.admit([], 5) == []
