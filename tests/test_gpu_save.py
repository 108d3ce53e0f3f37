"""NEXT-1 parity: decode KV append + seal + FlashD2H save path (PAPER.md:151-153,
:125) inside running decode steps, against the oracle replaying the same steps:
tails, counters, metadata of the sealed blocks (bit-exact), the DRAM copies of
the sealed blocks (byte-exact), and the selections / attention of the following
steps (which can select and miss the freshly saved blocks)."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from layout import D, tiled_to_logical, to_numpy, to_torch

pytestmark = pytest.mark.gpu


def test_append_seal_flash_d2h_steps():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2509_24626_b200.engine import DecodeEngine, EngineConfig
    dt = synth.DT_BF16
    B, L, Hq, Hkv, k, steps = 3, 2, 8, 4, 8, 40
    n_blk0 = [40, 70, 5]
    tails0 = [30, 0, 17]
    max_blk = 96
    S = B * Hkv * k * 3
    cfg = EngineConfig(batch=B, layers=L, num_q_heads=Hq, num_kv_heads=Hkv, max_blk=max_blk, topk=k,
                       slots_per_layer=S, num_requests=B, dtype=torch.bfloat16)
    eng = DecodeEngine(cfg)
    rng = synth.rng_for(9000, 1)
    hb = cfg.fwd_len
    host_np = synth.encode(synth.kv_blocks(rng, hb, D, synth.channel_scales(rng)), dt)
    host_t = torch.from_numpy(host_np.view(np.int16).copy()).view(-1).pin_memory().view(torch.bfloat16)
    eng.set_host_kv(host_t, hb)
    eng.n_blk.copy_(torch.tensor(n_blk0, dtype=torch.int32))
    eng.tail_len.copy_(torch.tensor(tails0, dtype=torch.int32))
    tail_np = synth.encode(synth.kv_blocks(rng, L * B * Hkv, D).reshape(L, B, Hkv, 2, 32, D), dt)
    for l in range(L):                      # rows beyond the tail length are zero
        for b in range(B):
            tail_np[l, b, :, :, tails0[b]:] = 0
    eng.tail_kv.copy_(to_torch(tail_np))
    eng.build_meta(n_blk0, host_t.cuda())
    eng.enable_save_path(tails0, n_blk0, d2h_threads=4)

    # oracle state
    o_host = host_np.copy()
    o_tail = tail_np.copy()
    o_tlen = np.array(tails0, np.int32)
    o_nblk = np.array(n_blk0, np.int32)
    metas = []
    for l in range(L):
        m = np.zeros((B, Hkv, max_blk, 2, D), np.uint16)
        for b in range(B):
            for h in range(Hkv):
                k0 = eng.key0(b, l, h)
                m[b, h, :n_blk0[b]] = oracle.block_meta(o_host[k0:k0 + n_blk0[b]], key_stride=2 * 32 * D)
        metas.append(m)
    pools = [oracle.Pool(S, cfg.fwd_len, cfg.block_bytes) for _ in range(L)]
    qs = synth.encode(synth.queries(rng, steps, (L, B, Hq, D), 0.9), dt)
    new_kvs = synth.encode(rng.standard_normal((steps, L, B, Hkv, 2, D)), dt)
    # ---- GPU: all steps back to back, no host synchronisation: each step's
    # FlashD2H save overlaps the following steps (only a later gather of the
    # same layer waits for it); per-step results are cloned on the stream ----
    got = []
    fills = []
    for t in range(steps):
        eng.append_kv(to_torch(new_kvs[t]))
        for l in range(L):
            eng.layer_step(l, to_torch(qs[t, l]), stamp=t + 1)
        got.append([(eng.sel[l].clone(), eng.counts[l].clone(), eng.out[l].clone()) for l in range(L)])
        fills.append(eng.seal_full_blocks())
    eng.wait_saves()
    torch.cuda.synchronize()
    # ---- oracle replay, step by step ----
    sealed_total = 0
    for t in range(steps):
        for l in range(L):
            tl = o_tlen.copy()
            oracle.kv_append(new_kvs[t, l], o_tail[l], tl, advance=True)
        o_tlen = tl
        for l in range(L):
            r = oracle.decode_layer(qs[t, l], metas[l], o_nblk, k, pools[l], np.arange(B, dtype=np.int32),
                                    l, L, max_blk, t + 1, o_host.view(np.uint8).reshape(hb, -1), hb,
                                    o_tail[l], o_tlen, 1.0 / math.sqrt(D))
            g_sel, g_cnt, g_out = got[t][l]
            np.testing.assert_array_equal(g_sel.cpu().numpy(), r["sel"])
            np.testing.assert_array_equal(g_cnt.cpu().numpy(), r["counts"])
            err = float(np.abs(g_out.cpu().numpy() - r["out"]).max())
            assert err <= 2e-3, f"step {t} layer {l}: {err}"
        o_fill = [b for b in range(B) if o_tlen[b] == 32]
        assert fills[t] == o_fill
        if o_fill:
            sealed_total += len(o_fill)
            nb_before = o_nblk.copy()
            for l in range(L):
                tl, nb = o_tlen.copy(), o_nblk.copy()
                staging = oracle.kv_seal(o_fill, o_tail[l], tl, nb, metas[l])
                keys = [eng.key0(b, l, h) + nb_before[b] for b in o_fill for h in range(Hkv)]
                oracle.d2h_scatter(staging.view(np.uint8).reshape(len(keys), -1), keys,
                                   o_host.view(np.uint8).reshape(hb, -1), hb)
            o_tlen, o_nblk = tl, nb
    # ---- final state ----
    np.testing.assert_array_equal(eng.tail_len.cpu().numpy(), o_tlen)
    np.testing.assert_array_equal(eng.n_blk.cpu().numpy(), o_nblk)
    for l in range(L):
        for b in range(B):
            n = o_tlen[b]
            np.testing.assert_array_equal(to_numpy(eng.tail_kv[l, b])[:, :, :n], o_tail[l, b][:, :, :n])
        got_meta = tiled_to_logical(to_numpy(eng.meta[l]), B, Hkv, max_blk)
        for b in range(B):
            np.testing.assert_array_equal(got_meta[b, :, :o_nblk[b]].view(np.uint8),
                                          metas[l][b, :, :o_nblk[b]].view(np.uint8))
    assert sealed_total >= 3
    np.testing.assert_array_equal(host_t.view(torch.int16).numpy().view(np.uint16), o_host.reshape(-1))
