#!/bin/bash
# Round 2: FlashH2D server spread over more SMs (same bytes in flight, fewer warps
# per SM) -- in-step A/B and the select/gather interference microbench;
# NEXT-1 save overlap step times; ncu capture of attention at the bench shape.
mkdir -p gpurun_out/r02f
{
for v in "16 128 16" "64 32 16" "32 64 16" "128 32 8" "148 32 8"; do
  set -- $v
  echo "== CTAS=$1 THREADS=$2 UNROLL=$3 overlap: $(SS_LIB_VARIANT=debug SS_H2D_CTAS=$1 SS_H2D_THREADS=$2 SS_H2D_UNROLL=$3 python tools/kbench.py overlap)"
done
} > gpurun_out/r02f/overlap_spread.txt 2>&1
{
for v in "16 128 16" "64 32 16" "32 64 16" "128 32 8"; do
  set -- $v
  echo "== CTAS=$1 THREADS=$2 UNROLL=$3"
  SS_LIB_VARIANT=debug SS_H2D_CTAS=$1 SS_H2D_THREADS=$2 SS_H2D_UNROLL=$3 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-gather-alone | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ['value','ms_per_step','step_ms_min_median_max','hit_rate']}), json.dumps(d['flash_h2d']), json.dumps(d['flash_h2d_server']), json.dumps({k: v.get('us_per_launch') for k, v in d['kernels'].items() if isinstance(v, dict)}))"
done
} > gpurun_out/r02f/server_spread.txt 2>&1
for m in none overlap blocking; do timeout 300 python tools/save_overlap.py --mode $m 2>&1 | grep -v Warn | tail -3; done > gpurun_out/r02f/save_overlap.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn_mma -s 3 -c 1 -o gpurun_out/r02f/attn_b3 python tools/kbench.py attn --cfg C2 --batch 3 --iters 3 > gpurun_out/r02f/ncu_attn.log 2>&1
