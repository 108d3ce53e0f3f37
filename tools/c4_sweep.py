"""BASELINE.json configs[3] (C4): batch-size sweep at 64K context tracking the
decoding working set (union of the last w = 12 selections),
cache hit rate and H2D bytes per step, with a FIXED total HBM cache budget --
the synthetic analog of the paper's Fig. 1 / Fig. 15: as the
batch grows, the working set outgrows the cache and FlashH2D traffic per token
rises.  LWM-7B heads (32 x d=128), 2048 blocks per request, top-64, 4 simulated
layers (32 layers x B=256 would need 256 GiB of metadata), rho = 0.95.

  python tools/c4_sweep.py [--batches 8,16,32,64,128,256] [--steps 12] [--cache-gib 16] [--admission]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_24626_b200 import ops  # noqa: E402
from paper_2509_24626_b200.engine import DecodeEngine, EngineConfig  # noqa: E402


def run(B, args):
    L, H, n_blk, k = 4, 32, 2048, 64
    slots = (args.cache_gib << 30) // L // 16384
    cfg = EngineConfig(batch=B, layers=L, num_q_heads=H, num_kv_heads=H, max_blk=n_blk, topk=k,
                       slots_per_layer=slots, num_requests=B, dtype=torch.bfloat16, groups=1)
    eng = DecodeEngine(cfg)
    phys = 127 * n_blk                                   # 4 GiB physical host pool (aliased)
    hp = ops.HostPool(phys * cfg.block_bytes)
    host_t = hp.tensor.view(torch.bfloat16)
    meta_phys = torch.empty(phys * 2 * 128, dtype=torch.bfloat16, device="cuda")
    bench.gen_host_blocks_on_gpu(eng, host_t, phys, seed=4400, meta_phys=meta_phys)
    eng.set_host_kv(host_t, phys, dev_ptr=hp.dev_ptr)
    tile = 32 * 2 * 128
    mp = meta_phys.view(-1, tile)
    ar = torch.arange(n_blk // 32, device="cuda")
    for l in range(L):
        t0 = torch.tensor([eng.key0(b, l, h) % phys // 32 for b in range(B) for h in range(H)], device="cuda")
        eng.meta[l].view(-1, tile).copy_(mp.index_select(0, (t0[:, None] + ar[None, :]).reshape(-1)))
    del meta_phys, mp
    eng.n_blk.fill_(n_blk)
    eng.tail_len.zero_()
    ws = ops.WorkingSetState(L, B, H, n_blk, k, w=12)
    steps = args.warmup + args.steps
    qs = bench.gen_queries(eng, steps, 0.95, seed=4500)
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    status = 0
    running = [True] * B
    served = 0
    m_avl = args.cache_gib << 30
    for t in range(steps):
        if t == args.warmup:
            torch.cuda.synchronize()
            cnt.zero_()
            served = 0
            s.record()
        if args.admission:
            # Algorithm 1: candidates in FCFS order; M_req = the
            # request's tracked w=12 working set, or (not yet running) the mean of
            # the running ones / one step's demand; reset requests do not run.
            wsc = ws.ws_count.tolist()
            run_ws = [wsc[b] for b in range(B) if running[b] and wsc[b] > 0]
            fresh = (sum(run_ws) / len(run_ws)) if run_ws else H * k * L
            est = [(wsc[b] if running[b] and wsc[b] > 0 else fresh) * 16384 for b in range(B)]
            admit = ops.ss_admit(est, m_avl)
            for b in range(B):
                if admit[b] != running[b]:
                    eng.n_blk[b] = n_blk if admit[b] else 0
                    if not admit[b]:            # S.reset(req): its working-set history is dropped
                        ws.last_sel[:, b].fill_(-(1 << 30))
                        ws.ring[:, :, b].fill_(-1)
                        ws.ws_count[b] = 0
                    running[b] = admit[b]
        served += sum(running)
        for l in range(L):
            eng.layer_step(l, qs[t, l], stamp=t + 1)
            ops.ws_track(ws, l, eng.sel[l], k, eng.dims, n_blk, t)
        cnt += eng.counts.to(torch.int64).sum(0)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    hits, misses, ev, errs = cnt.tolist()
    status = int(eng.counts[:, 3].max().item())
    ws_blocks = int(ws.ws_count.sum().item())
    tok = served / args.steps
    res = {"batch": B, "admission": bool(args.admission), "mean_running": round(tok, 1),
           "layers": L, "cache_gib_total": args.cache_gib, "ms_per_step_4_layers": round(ms, 3),
           "tokens_per_s_4_layers": round(tok / (ms * 1e-3), 1),
           "tokens_per_s_32_layer_equiv": round(tok / (ms * 1e-3) * L / 32, 1),
           "hit_rate": round(hits / max(1, hits + misses), 4),
           "misses_per_step": misses / args.steps,
           "h2d_MB_per_step": round(misses / args.steps * 16384 / 1e6, 1),
           "h2d_KB_per_token": round(misses / args.steps * 16384 / 1e3 / max(tok, 1e-9), 1),
           "demand_blocks_per_step": B * H * k * L,
           "working_set_blocks_w12": ws_blocks,
           "working_set_GiB": round(ws_blocks * 16384 / 2**30, 2),
           "working_set_over_cache": round(ws_blocks * 16384 / (args.cache_gib << 30), 3),
           "capacity_errors": errs, "last_status": status}
    if errs:
        # per-step demand exceeds the cache: every such layer call fails with
        # SS_ERR_CAPACITY and attends nothing, so there is no throughput to report
        for kk in ("ms_per_step_4_layers", "tokens_per_s_4_layers", "tokens_per_s_32_layer_equiv", "hit_rate",
                   "misses_per_step", "h2d_MB_per_step", "h2d_KB_per_token"):
            res[kk] = None
        res["infeasible"] = (f"{B * H * k} selected blocks per layer-step exceed the {slots} slots of a "
                             "layer's cache: SS_ERR_CAPACITY, nothing attended")
    del eng
    hp.close()
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="8,16,32,64,128,256")
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--warmup", type=int, default=14)
    ap.add_argument("--cache-gib", type=int, default=16)
    ap.add_argument("--admission", action="store_true",
                    help="working-set-aware admission (Algorithm 1) over the B candidates")
    args = ap.parse_args()
    for B in [int(x) for x in args.batches.split(",")]:
        print(json.dumps(run(B, args)), flush=True)


if __name__ == "__main__":
    main()
