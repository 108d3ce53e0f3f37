#!/bin/bash
# Round 2 (re-entry): (1) C2 step with the MHA select reading only the min rows
# (debug SS_SEL_L2PF=2: wrong selections, half the select bytes -- the step-time
# bound of a sign-selected half read); (2) attention per-warp timelines at the
# bench's launch shapes (C2 one request group, C3 one request) and full C3.
mkdir -p gpurun_out/r02u
for v in 0 2 0 2; do
  echo "== SS_SEL_L2PF=$v"
  SS_LIB_VARIANT=debug SS_SEL_L2PF=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-gather-alone | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ['value','ms_per_step','step_ms_min_median_max','hit_rate']}), json.dumps(d['flash_h2d']), json.dumps(d.get('flash_h2d_server')), json.dumps({k: v.get('us_per_launch') for k, v in d['kernels'].items() if isinstance(v, dict)}))"
done > gpurun_out/r02u/half_read_experiment.txt 2>&1
{
for c in "--cfg C2 --batch 3" "--cfg C3 --batch 1" "--cfg C3"; do
  echo "== attn $c"; SS_LIB_VARIANT=debug SS_ATTN_TRACE=1 timeout 300 python tools/kbench.py attn $c
done
} > gpurun_out/r02u/attn_trace.txt 2>&1
