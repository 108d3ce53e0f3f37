"""NEXT-1 overlap evidence (saving runs "fully in parallel with
model computation"): decode steps of the bench's C2 engine (5 request groups,
FlashH2D server) in which every request's tail fills at step 0, so step 0 seals
16 x 32 heads x 32 layers = 16384 blocks (256 MiB) and saves them with FlashD2H.

  overlap : the save runs on its own stream; a later step's gather of layer l
            waits for layer l's save only (DecodeEngine.seal_full_blocks)
  blocking: the current stream waits for the whole save right after sealing
  none    : the same steps with no block filling (tails start at 0)

Prints one JSON line (one mode per process) with the device time of five eager
steps after 20 settle steps; the HBM cache is the SURVEY's 4x-demand size.

  python tools/save_overlap.py --mode overlap|blocking|none"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import torch  # noqa: E402

import bench  # noqa: E402


def run(mode, args):
    eng, W = bench.setup_engine(args, 0, 1, 0)
    c = eng.cfg
    qs = bench.gen_queries(eng, 40, W["rho"], seed=5000)
    # settle the cache a little (no sealing)
    for t in range(20):
        eng.step(qs[t], t + 1)
    torch.cuda.synchronize()
    tl0 = 31 if mode != "none" else 0
    nb0 = W["n_blk"] - 1                 # 4095 full blocks + a 31-token tail: room for block 4096
    eng.n_blk.fill_(nb0)
    eng.tail_len.fill_(tl0)
    eng.enable_save_path([tl0] * c.batch, [nb0] * c.batch, d2h_threads=8)
    new_kv = torch.randn(c.layers, c.batch, c.num_kv_heads, 2, 128, device="cuda").to(torch.bfloat16)
    ev = [torch.cuda.Event(True) for _ in range(6)]
    torch.cuda.synchronize()
    torch.cuda._sleep(20_000_000)
    ev[0].record()
    sealed = []
    for i, t in enumerate(range(20, 25)):
        eng.append_kv(new_kv)
        eng.step(qs[t], t + 1)
        sealed.append(len(eng.seal_full_blocks()))
        if mode == "blocking":
            eng.wait_saves()
        ev[i + 1].record()
    eng.wait_saves()
    torch.cuda.synchronize()
    steps = [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(5)]
    cnt = sum(g.counts.to(torch.int64).sum(0) for g in eng.groups).tolist()
    return {"mode": mode, "step_ms": steps, "total_ms": round(sum(steps), 3), "sealed_per_step": sealed,
            "blocks_saved": sealed[0] * c.layers * c.num_kv_heads,
            "bytes_saved": sealed[0] * c.layers * c.num_kv_heads * c.block_bytes, "errors": int(cnt[3])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="overlap", choices=["none", "overlap", "blocking"])
    a = ap.parse_args()
    args = argparse.Namespace(config="C2", rho=None, slots=0, groups=5, h2d_streams=1, select_priority=False,
                              cache_per_group=False, h2d_server=1, split_attn=0, pool_per_group=1, host_runs=251)
    print(json.dumps(run(a.mode, args)), flush=True)


if __name__ == "__main__":
    main()
