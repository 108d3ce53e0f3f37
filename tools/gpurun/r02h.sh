#!/bin/bash
# Round 2: pipelined FlashH2D server (next unit's loads issued before the current
# unit's stores / fence / completion atomics): parity, alone rate, in-step A/B.
mkdir -p gpurun_out/r02h
timeout 600 python -m pytest tests/test_gpu_h2d_serve.py tests/test_gpu_pipeline.py -q -k "serve or request_groups" > gpurun_out/r02h/tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02h/tests.log
{
for v in "0 16 128 16" "1 16 128 16" "1 16 128 8" "1 8 256 16" "1 24 128 8" "1 12 128 16"; do
  set -- $v
  echo "== PIPE=$1 CTAS=$2 THREADS=$3 UNROLL=$4"
  SS_LIB_VARIANT=debug SS_H2D_PIPE=$1 SS_H2D_CTAS=$2 SS_H2D_THREADS=$3 SS_H2D_UNROLL=$4 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-gather-alone | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ['value','ms_per_step','step_ms_min_median_max','hit_rate','errors_in_timed_region','errors_in_timing_passes']}), json.dumps(d['flash_h2d']), json.dumps(d['flash_h2d_server']), json.dumps({k: v.get('us_per_launch') for k, v in d['kernels'].items() if isinstance(v, dict)}))"
done
} > gpurun_out/r02h/server_pipe_ab.txt 2>&1
