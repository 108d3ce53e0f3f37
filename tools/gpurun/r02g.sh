#!/bin/bash
# Round 2: FlashH2D server on dedicated SMs (reserved shared memory keeps the
# HBM kernels off the server's SMs): interference microbench + in-step A/B.
mkdir -p gpurun_out/r02g
{
for v in "0 16 128" "227 16 128" "227 8 256" "227 12 128" "227 24 128" "120 16 128"; do
  set -- $v
  echo "== SMEM_KB=$1 CTAS=$2 THREADS=$3 overlap: $(SS_LIB_VARIANT=debug SS_H2D_SMEM_KB=$1 SS_H2D_CTAS=$2 SS_H2D_THREADS=$3 python tools/kbench.py overlap)"
done
} > gpurun_out/r02g/overlap_dedicated.txt 2>&1
{
for v in "0 16 128" "227 16 128" "227 8 256" "227 12 128" "227 24 128" "227 32 128"; do
  set -- $v
  echo "== SMEM_KB=$1 CTAS=$2 THREADS=$3"
  SS_LIB_VARIANT=debug SS_H2D_SMEM_KB=$1 SS_H2D_CTAS=$2 SS_H2D_THREADS=$3 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-gather-alone | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ['value','ms_per_step','step_ms_min_median_max','hit_rate','errors_in_timed_region']}), json.dumps(d['flash_h2d']), json.dumps(d['flash_h2d_server']), json.dumps({k: v.get('us_per_launch') for k, v in d['kernels'].items() if isinstance(v, dict)}), json.dumps({k: (v.get('frac'), v.get('us_per_launch')) for k, v in d['kernels_solo'].items() if isinstance(v, dict) and 'frac' in v or k == 'kv_cache_lookup_insert'}))"
done
} > gpurun_out/r02g/server_dedicated.txt 2>&1
