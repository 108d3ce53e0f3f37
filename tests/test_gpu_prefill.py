"""NEXT-4 parity: layer-segmented prefill storage side --
(N,H,D) -> per-head blocks, metadata, DMA save to DRAM, tail -- for every layer
of a request, then a decode step over the saved KV (all misses come from the
blocks saved by the prefill) against the oracle doing the same."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from layout import D, tiled_to_logical, to_numpy, to_torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dt", [synth.DT_BF16, synth.DT_F32])
def test_prefill_layer_save_then_decode(dt):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2509_24626_b200 import ops
    from paper_2509_24626_b200.engine import DecodeEngine, EngineConfig
    tdt = torch.bfloat16 if dt == synth.DT_BF16 else torch.float32
    B, L, Hq, Hkv, k, max_blk = 2, 3, 8, 4, 8, 64
    lens = [32 * 40 + 7, 32 * 9]
    cfg = EngineConfig(batch=B, layers=L, num_q_heads=Hq, num_kv_heads=Hkv, max_blk=max_blk, topk=k,
                       slots_per_layer=B * Hkv * k * 2, num_requests=B, dtype=tdt)
    eng = DecodeEngine(cfg)
    hb = cfg.fwd_len
    npdt = np.uint16 if dt == synth.DT_BF16 else np.float32
    host_np = np.zeros(hb * cfg.block_elems, npdt)
    host_t = torch.from_numpy(host_np.view(np.int16) if dt == synth.DT_BF16 else host_np).pin_memory()
    if dt == synth.DT_BF16:
        host_t = host_t.view(torch.bfloat16)
    eng.set_host_kv(host_t, hb)
    staging = torch.empty(Hkv * max_blk * cfg.block_elems, dtype=tdt, device="cuda")
    ws = ops.alloc_workspace(4, eng.dims, max_blk, k)
    rng = synth.rng_for(9100, 1)
    o_meta = [np.zeros((B, Hkv, max_blk, 2, D), npdt) for _ in range(L)]
    o_tail = np.zeros((L, B, Hkv, 2, 32, D), npdt)
    o_nblk = np.zeros(B, np.int32)
    o_tl = np.zeros(B, np.int32)
    o_host = np.zeros((hb, cfg.block_bytes), np.uint8)
    for b in range(B):
        for l in range(L):
            kk = synth.encode(rng.standard_normal((lens[b], Hkv, D)), dt)
            vv = synth.encode(rng.standard_normal((lens[b], Hkv, D)), dt)
            ops.prefill_layer_save(to_torch(kk), to_torch(vv), lens[b], b, b, l, L, max_blk, eng.dims,
                                   staging, eng.meta[l], eng.tail_kv[l], eng.n_blk, eng.tail_len,
                                   host_t, hb, ws)
            torch.cuda.synchronize()            # staging is reused per layer
            oracle.prefill_save(kk, vv, b, b, l, L, o_meta[l], o_tail[l], o_nblk, o_tl, o_host, hb)
    np.testing.assert_array_equal(eng.n_blk.cpu().numpy(), o_nblk)
    np.testing.assert_array_equal(eng.tail_len.cpu().numpy(), o_tl)
    got_host = (host_t.view(torch.int16).numpy() if dt == synth.DT_BF16 else host_t.numpy()).view(np.uint8)
    np.testing.assert_array_equal(got_host.reshape(hb, -1), o_host)
    for l in range(L):
        got = tiled_to_logical(to_numpy(eng.meta[l]), B, Hkv, max_blk)
        for b in range(B):
            n = o_nblk[b]
            np.testing.assert_array_equal(got[b, :, :n].view(np.uint8), o_meta[l][b, :, :n].view(np.uint8))
            np.testing.assert_array_equal(to_numpy(eng.tail_kv[l, b])[:, :, :o_tl[b]], o_tail[l, b][:, :, :o_tl[b]])
    # one decode step over the saved KV: every selected block misses and is
    # fetched by FlashH2D from what the prefill saved
    pools = [oracle.Pool(cfg.slots_per_layer, cfg.fwd_len, cfg.block_bytes) for _ in range(L)]
    q = synth.encode(rng.standard_normal((L, B, Hq, D)), dt)
    for l in range(L):
        eng.layer_step(l, to_torch(q[l]), stamp=1)
        torch.cuda.synchronize()
        r = oracle.decode_layer(q[l], o_meta[l], o_nblk, k, pools[l], np.arange(B, dtype=np.int32), l, L,
                                max_blk, 1, o_host, hb, o_tail[l], o_tl, 1.0 / math.sqrt(D))
        np.testing.assert_array_equal(eng.sel[l].cpu().numpy(), r["sel"])
        assert r["counts"][0] == 0 and r["counts"][1] > 0
        err = float(np.abs(eng.out[l].cpu().numpy() - r["out"]).max())
        assert err <= (2e-3 if dt == synth.DT_BF16 else 1e-5), err
