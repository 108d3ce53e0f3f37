"""Per-kernel microbenchmarks at C2 / C3 shapes (CUDA events, many launches,
inputs larger than L2).  Development tool; bench.py is the contract.

  python tools/kbench.py [select|attn|gather|cache|all] [--cfg C2|C3]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2509_24626_b200 import ops  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6550.0

CFG = {"C2": dict(B=16, Hq=32, Hkv=32, n_blk=4096, k=64, S=131072),
       "C3": dict(B=4, Hq=32, Hkv=8, n_blk=32768, k=128, S=8192)}


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def bench_select(c, iters):
    B, Hq, Hkv, n, k = c["B"], c["Hq"], c["Hkv"], c["n_blk"], c["k"]
    nm = 2
    metas = [torch.randn(B * Hkv * n * 2 * 128, device="cuda").to(torch.bfloat16) for _ in range(nm)]
    q = torch.randn(B, Hq, 128, device="cuda").to(torch.bfloat16)
    d = ops.dims(B, Hq, Hkv)
    ws = ops.alloc_workspace(0, d, n, k)
    sel = torch.empty(B, Hkv, k, dtype=torch.int32, device="cuda")
    nb = torch.full((B,), n, dtype=torch.int32, device="cuda")
    i = [0]

    def f():
        ops.ss_block_select(q, metas[i[0] % nm], nb, n, k, d, sel, ws)
        i[0] += 1
    ms = timeit(f, iters)
    byts = B * Hkv * n * 512 + q.numel() * 2
    if os.environ.get("SS_SEL_TRACE"):
        # tensor-core select timeline (debug build): per CTA start / tiles done /
        # threshold / rescoring / chunk top-k / merge start / merge end, n_cand
        import ctypes
        import numpy as np
        from paper_2509_24626_b200 import _lib
        lib = _lib.load()
        torch.cuda.synchronize()
        buf = np.zeros((16384, 12), dtype=np.uint64)
        lib.ss_debug_sel_trace(ctypes.c_void_p(buf.ctypes.data), 16384)
        tr = buf[buf[:, 0] > 0].astype(np.int64)
        t0 = tr[:, 0].min()
        qq = lambda x: [round(float(np.quantile(x, v)), 2) for v in (0.0, 0.5, 0.9, 1.0)] if len(x) else None
        d = lambda i, j, m=None: (tr[m][:, j] - tr[m][:, i]) / 1e3 if m is not None else (tr[:, j] - tr[:, i]) / 1e3
        mg = tr[:, 5] >= tr[:, 0]
        mg &= tr[:, 6] >= tr[:, 5]
        mg &= tr[:, 5] > t0
        if not (tr[:, 2] > 0).any():   # MHA fp64 kernel: start / scored / chunk top-k / merge
            print(json.dumps({"ctas": len(tr), "start_us": qq((tr[:, 0] - t0) / 1e3), "scoring_us": qq(d(0, 1)),
                              "chunk_topk_us": qq(d(1, 4, tr[:, 4] > tr[:, 1])), "scored_end_us": qq((tr[:, 1] - t0) / 1e3),
                              "merges": int(mg.sum()), "merge_us": qq(d(5, 6, mg)) if mg.any() else None,
                              "merge_end_us": qq((tr[mg][:, 6] - t0) / 1e3) if mg.any() else None}))
        else:
          print(json.dumps({"ctas": len(tr), "start_us": qq((tr[:, 0] - t0) / 1e3), "tiles_us": qq(d(0, 1)),
                          "threshold_us": qq(d(1, 2)), "rescore_us": qq(d(2, 3)),
                          "rescore_compaction_us": qq(d(2, 9, tr[:, 9] >= tr[:, 2])), "rescore_data_wait_us": qq(d(9, 8, tr[:, 8] >= tr[:, 9])), "rescore_compute_us": qq(d(8, 3, tr[:, 8] >= tr[:, 2])), "chunk_topk_us": qq(d(3, 4)),
                          "n_cand": qq(tr[:, 7]), "chunk_end_us": qq((tr[:, 4] - t0) / 1e3),
                          "merges": int(mg.sum()), "merge_us": qq(d(5, 6, mg)) if mg.any() else None,
                          "merge_end_us": qq((tr[mg][:, 6] - t0) / 1e3) if mg.any() else None}))
    return {"kernel": "select", "us": ms * 1e3, "GBps": byts / ms / 1e6, "frac": byts / ms / 1e6 / PEAK}


def bench_attn(c, iters):
    B, Hq, Hkv, k, S = c["B"], c["Hq"], c["Hkv"], c["k"], c["S"]
    pool = torch.randn(S * 2 * 32 * 128, device="cuda").to(torch.bfloat16)
    def rand_slots():
        sl = torch.stack([torch.randperm(S, device="cuda")[:k] for _ in range(B * Hkv)]).view(B, Hkv, k)
        return sl.sort(-1).values.to(torch.int32).contiguous()
    slot = rand_slots()
    slot_sets = [slot] + [rand_slots() for _ in range(3)]   # back-to-back timing: no L2 reuse
    q = torch.randn(B, Hq, 128, device="cuda").to(torch.bfloat16)
    tail = torch.zeros(B * Hkv * 2 * 32 * 128, dtype=torch.bfloat16, device="cuda")
    tl = torch.zeros(B, dtype=torch.int32, device="cuda")
    d = ops.dims(B, Hq, Hkv)
    ws = ops.alloc_workspace(2, d, 32, k)
    out = torch.empty(Hq, B, 128, dtype=torch.float32, device="cuda")
    # flush between iterations with a READ of 256 MB (clean L2; a memset would
    # leave 126 MB of dirty lines whose write-back the timed kernel would pay)
    flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
    sink = torch.empty((), dtype=torch.float32, device="cuda")

    def f():
        ops.sparse_decode_attn(q, pool, slot, k, tail, tl, d, 1 / math.sqrt(128), out, ws)
    ms_total = 0.0
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    for _ in range(3):
        f()
    ts = []
    for _ in range(iters):
        torch.sum(flush, dim=0, out=sink)
        # keep the GPU busy ~150 us so the host has enqueued f() before the
        # start event fires (host launch overhead must not count as kernel time)
        torch.cuda._sleep(300000)
        s.record()
        f()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ms = sorted(ts)[len(ts) // 2]
    # back to back (the bench's kernels_solo method): 40 launches over 4 slot sets
    # after a device spin, one event pair -- the average launch duration
    nb2b = 40
    torch.sum(flush, dim=0, out=sink)
    torch.cuda._sleep(3000000)
    s.record()
    for i in range(nb2b):
        ops.sparse_decode_attn(q, pool, slot_sets[i % 4], k, tail, tl, d, 1 / math.sqrt(128), out, ws)
    e.record()
    torch.cuda.synchronize()
    ms_b2b = s.elapsed_time(e) / nb2b
    byts = B * Hkv * k * 16384
    if os.environ.get("SS_ATTN_TRACE"):
        # per-warp globaltimer (ns) at entry / last unit done / exit (debug timeline)
        nw = 148 * 6
        tr = ws.view(torch.uint8)[-nw * 96:].view(torch.int64).view(nw, 12).cpu()
        ok = tr[:, 0] > 0
        widx = torch.arange(nw)[ok]
        tr = tr[ok]
        t0 = int(tr[:, 0].min())
        rel = (tr[:, :3] - t0).double() / 1e3
        q = lambda x: [round(float(x.quantile(v)), 2) for v in (0.0, 0.5, 0.9, 1.0)]
        mg = tr[tr[:, 3] > 0]
        mdur = (mg[:, 4] - mg[:, 3]).double() / 1e3
        mstart = (mg[:, 3] - t0).double() / 1e3
        print(json.dumps({"trace_warps": len(tr), "entry_us_q0/50/90/100": q(rel[:, 0]),
                          "last_unit_us": q(rel[:, 1]), "exit_us": q(rel[:, 2]),
                          "merges": len(mg), "merge_us": q(mdur) if len(mg) else None,
                          "merge_start_us": q(mstart) if len(mg) else None}))
        if len(mg):
            d = lambda i, j: (mg[:, j] - mg[:, i]).double() / 1e3
            print(json.dumps({"merging_warps_us": {"flush_to_ticket": q(d(5, 6)), "ticket_to_merge_start": q(d(6, 3)),
                                                   "merge_m_l_loads": q(d(3, 7)), "merge_o_loads_and_store": q(d(7, 4)),
                                                   "merge_end_to_exit": q(d(4, 2))}}))
            m2 = mg[mg[:, 8] > 0]
            if len(m2):
                d2 = lambda i, j: (m2[:, j] - m2[:, i]).double() / 1e3
                r2 = m2[m2[:, 9] > 0]
                out = {"bulk_merges": len(m2), "round0_load": q(d2(3, 7)), "round0_compute": q(d2(7, 8))}
                if len(r2):
                    d3 = lambda i, j: (r2[:, j] - r2[:, i]).double() / 1e3
                    out.update({"two_round_merges": len(r2), "round1_load": q(d3(8, 9)), "round1_compute": q(d3(9, 10)),
                                "store": q(d3(10, 4))})
                else:
                    out["store"] = q(d2(8, 4))
                print(json.dumps(out))
        # imbalance structure: mean last-unit time by warp slot in the CTA and by SM id
        lu = rel[:, 1]
        slot, sm = widx // 148, widx % 148
        print(json.dumps({"last_unit_by_warp_slot": [round(float(lu[slot == i].mean()), 2) for i in range(6) if (slot == i).any()],
                          "last_unit_by_sm_decile": [round(float(lu[(sm >= 15 * i) & (sm < 15 * i + 15)].mean()), 2) for i in range(10)],
                          "last_unit_even_odd_sm": [round(float(lu[sm % 2 == 0].mean()), 2), round(float(lu[sm % 2 == 1].mean()), 2)]}))
    return {"kernel": "attn", "us": ms * 1e3, "GBps": byts / ms / 1e6, "frac": byts / ms / 1e6 / PEAK,
            "us_b2b": ms_b2b * 1e3, "frac_b2b": byts / ms_b2b / 1e6 / PEAK}


def bench_gather(c, iters, nmiss=2500):
    hb = 1 << 18  # 4 GiB host
    host = torch.empty(hb * 8192, dtype=torch.bfloat16, pin_memory=True)
    ptr = ops.host_device_pointer(host)
    S = c["S"]
    pool = torch.empty(S * 8192, dtype=torch.bfloat16, device="cuda")
    keys = torch.randint(0, hb, (nmiss,), device="cuda", dtype=torch.int64)
    slots = torch.randperm(S, device="cuda")[:nmiss].to(torch.int32)
    counts = torch.tensor([0, nmiss, 0, 0], dtype=torch.int32, device="cuda")

    def f():
        ops.flash_h2d_gather(ptr, hb, keys, slots, counts, nmiss, pool, 16384)
    ms = timeit(f, iters)
    return {"kernel": "gather", "misses": nmiss, "us": ms * 1e3, "GBps": nmiss * 16384 / ms / 1e6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", nargs="?", default="all")
    ap.add_argument("--cfg", default="C2")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--batch", type=int, default=0, help="override the config's batch (e.g. one request group)")
    a = ap.parse_args()
    c = dict(CFG[a.cfg])
    if a.batch:
        c["B"] = a.batch
    res = []
    if a.what in ("select", "all"):
        res.append(bench_select(c, a.iters))
    if a.what in ("attn", "all"):
        res.append(bench_attn(c, a.iters))
    if a.what in ("gather", "all"):
        for m in (64, 2500, 20000):
            res.append(bench_gather(c, a.iters, m))
    for r in res:
        r["cfg"] = a.cfg
        print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}))


if __name__ == "__main__" and not (len(sys.argv) > 1 and sys.argv[1] in ("overlap", "meta", "d2h", "prefill", "h2dsweep",
                                                                          "h2dload")):
    main()


def bench_overlap(c, iters=10, nmiss=1250, host_gib=None):
    """select (half batch) concurrent with a FlashH2D gather on a high-priority stream."""
    B, Hq, Hkv, n, k = c["B"] // 2, c["Hq"], c["Hkv"], c["n_blk"], c["k"]
    meta = torch.randn(B * Hkv * n * 2 * 128, device="cuda").to(torch.bfloat16)
    q = torch.randn(B, Hq, 128, device="cuda").to(torch.bfloat16)
    d = ops.dims(B, Hq, Hkv)
    ws = ops.alloc_workspace(0, d, n, k)
    sel = torch.empty(B, Hkv, k, dtype=torch.int32, device="cuda")
    nb = torch.full((B,), n, dtype=torch.int32, device="cuda")
    hb = (int(os.environ.get("KB_HOST_GIB", "4")) << 30) // 16384
    host = torch.empty(hb * 8192, dtype=torch.bfloat16, pin_memory=True)
    ptr = ops.host_device_pointer(host)
    S = c["S"]
    pool = torch.empty(S * 8192, dtype=torch.bfloat16, device="cuda")
    keys = torch.randint(0, hb, (nmiss,), device="cuda", dtype=torch.int64)
    slots = torch.randperm(S, device="cuda")[:nmiss].to(torch.int32)
    counts = torch.tensor([0, nmiss, 0, 0], dtype=torch.int32, device="cuda")
    hi = torch.cuda.Stream(priority=-1)
    main = torch.cuda.current_stream()

    def sel_f():
        ops.ss_block_select(q, meta, nb, n, k, d, sel, ws)

    def gat_f():
        ops.flash_h2d_gather(ptr, hb, keys, slots, counts, nmiss, pool, 16384)
    res = {}
    res["select_solo_us"] = timeit(sel_f, iters) * 1e3
    res["gather_solo_us"] = timeit(gat_f, iters) * 1e3
    ts, tg = [], []
    for _ in range(iters + 2):
        a0, a1 = torch.cuda.Event(True), torch.cuda.Event(True)
        b0, b1 = torch.cuda.Event(True), torch.cuda.Event(True)
        hi.wait_stream(main)
        with torch.cuda.stream(hi):
            b0.record()
            gat_f()
            b1.record()
        a0.record()
        sel_f()
        a1.record()
        main.wait_stream(hi)
        torch.cuda.synchronize()
        ts.append(a0.elapsed_time(a1))
        tg.append(b0.elapsed_time(b1))
    res["select_with_gather_us"] = sorted(ts[2:])[len(ts[2:]) // 2] * 1e3
    res["gather_with_select_us"] = sorted(tg[2:])[len(tg[2:]) // 2] * 1e3
    res["gather_GBps_solo"] = nmiss * 16384 / res["gather_solo_us"] / 1e3
    return res


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "overlap":
    print(json.dumps({k: round(v, 2) for k, v in bench_overlap(CFG["C2"]).items()}))


def bench_meta(iters=10):
    """S0 block_meta_update over 1M blocks (bulk build, C2 physical pool size)."""
    n = 1 << 20
    keys = torch.randn(n * 2 * 32 * 128 // 16, 16, device="cuda").to(torch.bfloat16).view(-1)
    meta = torch.empty(n * 2 * 128, dtype=torch.bfloat16, device="cuda")
    def f():
        ops.block_meta_update(keys, meta, n, key_stride=2 * 32 * 128)
    ms = timeit(f, iters)
    byts = n * (32 * 128 * 2 + 2 * 128 * 2)        # K half read + meta written
    return {"kernel": "meta_update", "blocks": n, "us": ms * 1e3, "GBps": byts / ms / 1e6,
            "frac": byts / ms / 1e6 / PEAK}


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "meta":
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in bench_meta().items()}))


def bench_d2h(n=2048, threads=8, iters=5):
    """FlashD2H (one D2H memcpy + CPU-thread scatter) vs one cudaMemcpy per 16 KiB
    block (Fig. 4b analog)."""
    bb = 16384
    hb = (4 << 30) // bb
    host = torch.empty(hb * bb, dtype=torch.uint8, pin_memory=True)
    hview = host.view(hb, bb)
    stage_dev = torch.randint(0, 255, (n, bb), dtype=torch.uint8, device="cuda")
    landing = torch.empty(n * bb, dtype=torch.uint8, pin_memory=True)
    keys = torch.randperm(hb)[:n].tolist()
    eng = ops.D2HEngine(threads)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    res = {}
    for _ in range(2):
        ops.flash_d2h_save(eng, stage_dev, landing, n, keys, host, hb, bb)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        ops.flash_d2h_save(eng, stage_dev, landing, n, keys, host, hb, bb)
    e.record()
    torch.cuda.synchronize()
    res["flash_d2h_GBps"] = iters * n * bb / (s.elapsed_time(e) * 1e-3) / 1e9
    ok = all(torch.equal(hview[keys[i]], stage_dev[i].cpu()) for i in range(0, n, max(1, n // 64)))
    s.record()
    for i in range(n):
        hview[keys[i]].copy_(stage_dev[i], non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    res["per_block_memcpy_GBps"] = n * bb / (s.elapsed_time(e) * 1e-3) / 1e9
    res["blocks"] = n
    res["threads"] = threads
    res["byte_exact"] = bool(ok)
    eng.close()
    return res


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "d2h":
    for th in (1, 4, 8, 16):
        print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in bench_d2h(threads=th).items()}))


def bench_prefill(n_tok=131072, Hkv=32, max_blk=4096, iters=3):
    """NEXT-4: one 128K-token prefill layer of one request (LWM-7B heads): GPU
    relayout + metadata + one DMA save per head into pinned DRAM."""
    d = ops.dims(1, Hkv, Hkv)
    k = torch.randn(n_tok, Hkv, 128, device="cuda").to(torch.bfloat16)
    v = torch.randn(n_tok, Hkv, 128, device="cuda").to(torch.bfloat16)
    nb = n_tok // 32
    staging = torch.empty(Hkv * max_blk * 8192, dtype=torch.bfloat16, device="cuda")
    meta = torch.empty(Hkv * max_blk * 256, dtype=torch.bfloat16, device="cuda")
    tail = torch.zeros(Hkv * 8192, dtype=torch.bfloat16, device="cuda")
    n_blk = torch.zeros(1, dtype=torch.int32, device="cuda")
    tl = torch.zeros(1, dtype=torch.int32, device="cuda")
    hb = Hkv * max_blk
    host = torch.empty(hb * 8192, dtype=torch.bfloat16, pin_memory=True)
    ws = ops.alloc_workspace(4, d, max_blk, 64)

    def f():
        ops.prefill_layer_save(k, v, n_tok, 0, 0, 0, 1, max_blk, d, staging, meta, tail, n_blk, tl,
                               host, hb, ws)
    ms = timeit(f, iters, warm=1)
    byts = nb * Hkv * 16384
    return {"kernel": "prefill_layer_save", "tokens": n_tok, "us": ms * 1e3,
            "dram_save_GBps": byts / ms / 1e6}


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "prefill":
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in bench_prefill().items()}))


def bench_h2d_sweep(total_mib=256, iters=3):
    """The paper's Fig. 4a analog: host->HBM loading of
    randomly placed KV blocks, block size swept 4-64 KiB, FlashH2D (one
    zero-copy gather launch) vs one cudaMemcpyAsync per block (the paper's
    memcpy-based loading, issued through torch: host-enqueue bound, as in the
    paper) vs one bulk cudaMemcpyAsync of the same bytes (the copy engine's
    peak).  Device time with CUDA events."""
    host_gib = 4
    host = torch.empty(host_gib << 30, dtype=torch.uint8, pin_memory=True)
    ptr = ops.host_device_pointer(host)
    dev = torch.empty(total_mib << 20, dtype=torch.uint8, device="cuda")
    rows = []
    for kib in (4, 8, 16, 32, 64):
        bb = kib << 10
        n = (total_mib << 20) // bb
        hb = (host_gib << 30) // bb
        keys = torch.randperm(hb, device="cuda")[:n].to(torch.int64)
        slots = torch.randperm(n, device="cuda").to(torch.int32)
        counts = torch.tensor([0, n, 0, 0], dtype=torch.int32, device="cuda")
        ms_fh = timeit(lambda: ops.flash_h2d_gather(ptr, hb, keys, slots, counts, n, dev, bb), iters, 1)
        kh, sh = keys.cpu().tolist(), slots.cpu().tolist()
        hv, dv = host.view(hb, bb), dev.view(n, bb)
        m = min(n, 4096)   # per-block copies: a bounded sample (host-enqueue bound)

        def per_block():
            for i in range(m):
                dv[sh[i]].copy_(hv[kh[i]], non_blocking=True)
        ms_pb = timeit(per_block, 2, 1) * n / m
        ms_bulk = timeit(lambda: dev.copy_(host[:total_mib << 20], non_blocking=True), iters, 1)
        gb = n * bb / 1e9
        rows.append({"block_KiB": kib, "blocks": n, "flash_h2d_GBps": round(gb / (ms_fh * 1e-3), 2),
                     "per_block_memcpy_GBps": round(gb / (ms_pb * 1e-3), 2),
                     "bulk_memcpy_GBps": round(gb / (ms_bulk * 1e-3), 2)})
    return rows


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "h2dsweep":
    for r in bench_h2d_sweep():
        print(json.dumps(r))


def bench_h2d_under_load(nmiss=8192, iters=3):
    """FlashH2D (the per-launch gather, 16 CTAs) alone vs while a device-to-device
    copy keeps HBM busy on another stream (~read + write at full bandwidth): how
    much PCIe goodput the zero-copy loads keep when HBM is saturated, as it is
    inside the decode step."""
    hb = (4 << 30) // 16384
    host = torch.empty(hb * 8192, dtype=torch.bfloat16, pin_memory=True)
    ptr = ops.host_device_pointer(host)
    pool = torch.empty(nmiss * 8192, dtype=torch.bfloat16, device="cuda")
    keys = torch.randint(0, hb, (nmiss,), device="cuda", dtype=torch.int64)
    slots = torch.arange(nmiss, dtype=torch.int32, device="cuda")
    counts = torch.tensor([0, nmiss, 0, 0], dtype=torch.int32, device="cuda")
    a = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    side = torch.cuda.Stream()
    res = {}
    for mode in ("alone", "hbm_copy_concurrent"):
        ts = []
        for _ in range(iters + 1):
            torch.cuda.synchronize()
            if mode != "alone":
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    for _ in range(4):
                        b.copy_(a)
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            torch.cuda._sleep(100000)
            s.record()
            ops.flash_h2d_gather(ptr, hb, keys, slots, counts, nmiss, pool, 16384)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ms = sorted(ts[1:])[len(ts[1:]) // 2]
        res[mode + "_GBps"] = round(nmiss * 16384 / ms / 1e6, 2)
    t0 = torch.cuda.Event(True)
    t1 = torch.cuda.Event(True)
    t0.record()
    for _ in range(4):
        b.copy_(a)
    t1.record()
    torch.cuda.synchronize()
    res["hbm_copy_alone_GBps"] = round(4 * 2 * a.numel() / t0.elapsed_time(t1) / 1e6, 1)
    return res


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "h2dload":
    print(json.dumps(bench_h2d_under_load()))
