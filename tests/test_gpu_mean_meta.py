"""GPU parity for NEXT-3, the mean-of-keys metadata variant (PAPER.md:94 [45],
PAPER.md:124; reading R18): block_meta_update_mean and ss_block_select_mean
through the C ABI vs oracle.block_mean / block_score_mean / topk.  Bit-exact
metadata, float64 scores and selections."""
import numpy as np
import pytest
import torch

import oracle
import synth
from layout import D, mean_logical_to_tiled, mean_tiled_to_logical, to_numpy, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2509_24626_b200 import ops as _ops
    return _ops


@pytest.mark.parametrize("dt", [synth.DT_BF16, synth.DT_F32])
def test_block_meta_update_mean_bit_exact(ops, dt):
    rng = synth.rng_for(1100, 1)
    B, Hkv, max_blk = 2, 3, 64
    n = B * Hkv * max_blk
    blocks = synth.kv_blocks(rng, n, D, synth.channel_scales(rng))
    blocks[5, 0, :, 3] = 1e-30          # tiny and huge magnitudes in one channel sum
    blocks[5, 0, 7, 3] = 3e4
    store = synth.encode(blocks, dt)
    exp = oracle.block_mean(store, key_stride=2 * 32 * D).reshape(B, Hkv, max_blk, D)
    meta = torch.zeros(ops.mean_meta_numel(B, Hkv, max_blk), dtype=torch.float32, device="cuda")
    perm = rng.permutation(n)
    keys = to_torch(np.ascontiguousarray(store[perm]))
    ops.block_meta_update_mean(keys, meta, n, key_stride=2 * 32 * D,
                               dst_idx=torch.from_numpy(perm.astype(np.int64)).cuda())
    torch.cuda.synchronize()
    got = mean_tiled_to_logical(to_numpy(meta), B, Hkv, max_blk)
    np.testing.assert_array_equal(got.view(np.uint32), exp.view(np.uint32))


def _mean_select_case(ops, dt, B, Hq, Hkv, n_blk, k, seed, ties=False):
    rng = synth.rng_for(1100, 2, seed)
    max_blk = ((max(n_blk) + 31) // 32) * 32 or 32
    nb = B * Hkv * max_blk
    blocks = synth.kv_blocks(rng, nb, D, synth.channel_scales(rng))
    if ties:
        src = rng.integers(0, nb, size=nb // 3)
        dst = rng.integers(0, nb, size=nb // 3)
        blocks[dst] = blocks[src]
    store = synth.encode(blocks, dt)
    qs = synth.encode(rng.standard_normal((B, Hq, D)), dt)
    mu = oracle.block_mean(store, key_stride=2 * 32 * D).reshape(B, Hkv, max_blk, D)
    nbk = np.array(n_blk, np.int32)
    exp_scores = oracle.block_score_mean(qs, mu, nbk)
    exp_sel = oracle.topk(exp_scores, nbk, k)
    meta = to_torch(mean_logical_to_tiled(mu))
    d = ops.dims(B, Hq, Hkv)
    ws = ops.alloc_workspace(0, d, max_blk, k)
    sel = torch.empty(B, Hkv, k, dtype=torch.int32, device="cuda")
    scores = torch.full((B, Hkv, max_blk), float("nan"), dtype=torch.float64, device="cuda")
    ops.ss_block_select_mean(to_torch(qs), meta, torch.from_numpy(nbk).cuda(), max_blk, k, d, sel, ws,
                             scores=scores)
    torch.cuda.synchronize()
    gs = scores.cpu().numpy()
    for b in range(B):
        np.testing.assert_array_equal(gs[b, :, :n_blk[b]].view(np.uint64),
                                      exp_scores[b, :, :n_blk[b]].view(np.uint64))
    np.testing.assert_array_equal(sel.cpu().numpy(), exp_sel)


@pytest.mark.parametrize("dt", [synth.DT_BF16, synth.DT_F32])
def test_select_mean_c1_shape(ops, dt):
    _mean_select_case(ops, dt, 1, 32, 32, [256], 64, seed=1)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_select_mean_gqa_ragged_multichunk(ops, G):
    _mean_select_case(ops, synth.DT_BF16, 4, 2 * G, 2, [5000, 2049, 17, 0], 128, seed=10 + G)


@pytest.mark.parametrize("k", [1, 64, 300])
def test_select_mean_ties(ops, k):
    _mean_select_case(ops, synth.DT_BF16, 2, 4, 4, [300, 96], k, seed=20 + k, ties=True)


def test_meta_mean_then_select_end_to_end(ops):
    # the GPU-built mean metadata feeds the GPU select directly (no host layout step)
    rng = synth.rng_for(1100, 3)
    B, Hq, Hkv, max_blk, k = 2, 8, 4, 96, 16
    n = B * Hkv * max_blk
    store = synth.encode(synth.kv_blocks(rng, n, D, synth.channel_scales(rng)), synth.DT_BF16)
    qs = synth.encode(rng.standard_normal((B, Hq, D)), synth.DT_BF16)
    meta = torch.zeros(ops.mean_meta_numel(B, Hkv, max_blk), dtype=torch.float32, device="cuda")
    ops.block_meta_update_mean(to_torch(store), meta, n, key_stride=2 * 32 * D)
    nbk = np.array([96, 50], np.int32)
    d = ops.dims(B, Hq, Hkv)
    ws = ops.alloc_workspace(0, d, max_blk, k)
    sel = torch.empty(B, Hkv, k, dtype=torch.int32, device="cuda")
    ops.ss_block_select_mean(to_torch(qs), meta, torch.from_numpy(nbk).cuda(), max_blk, k, d, sel, ws)
    torch.cuda.synchronize()
    mu = oracle.block_mean(store, key_stride=2 * 32 * D).reshape(B, Hkv, max_blk, D)
    exp = oracle.topk(oracle.block_score_mean(qs, mu, nbk), nbk, k)
    np.testing.assert_array_equal(sel.cpu().numpy(), exp)
