#!/bin/bash
# Round 2 experiment: the C2 step with the MHA select reading only half of the
# metadata bytes (debug SS_SEL_L2PF=2: min rows only, WRONG selections -- an
# upper bound on what a half-size metadata read would buy the step).
mkdir -p gpurun_out/r02s
for v in 0 2; do
  echo "== SS_SEL_L2PF=$v"
  SS_LIB_VARIANT=debug SS_SEL_L2PF=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-gather-alone | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ['value','ms_per_step','step_ms_min_median_max','hit_rate','misses_per_step']}), json.dumps(d['flash_h2d']), json.dumps(d['flash_h2d_server']), json.dumps({k: v.get('us_per_launch') for k, v in d['kernels'].items() if isinstance(v, dict)}))"
done > gpurun_out/r02s/half_read_experiment.txt 2>&1
