#!/bin/bash
# Round 2: carve-out A/B (attention launch overhead), gather/select interference,
# split-attention server-timeout reproduction, overlapped FlashD2H save step
# times, ncu full capture of the C3 select.
mkdir -p gpurun_out/r02e
{
for co in -1 100; do
  for a in "--cfg C2 --batch 3" "--cfg C2" "--cfg C3"; do
    echo "carveout=$co $a $(SS_LIB_VARIANT=debug SS_CARVEOUT=$co python tools/kbench.py attn $a)"
  done
  echo "carveout=$co select C3 $(SS_LIB_VARIANT=debug SS_CARVEOUT=$co python tools/kbench.py select --cfg C3)"
done
} > gpurun_out/r02e/carveout_kbench.txt 2>&1
python tools/kbench.py overlap > gpurun_out/r02e/overlap.txt 2>&1
{
echo "== carveout 100 (debug lib)"
SS_LIB_VARIANT=debug SS_CARVEOUT=100 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-gather-alone | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ['value','ms_per_step','step_ms_min_median_max','hit_rate']}), json.dumps(d['flash_h2d']), json.dumps(d['flash_h2d_server']), json.dumps({k: v.get('us_per_launch') for k, v in d['kernels'].items() if isinstance(v, dict)}), json.dumps({k: (v.get('frac'), v.get('us_per_launch')) for k, v in d['kernels_solo'].items() if isinstance(v, dict)}))"
echo "== split attention (release)"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-gather-alone --split-attn 1 | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ['value','ms_per_step','errors_in_timed_region','errors_in_timing_passes','valid']}), json.dumps(d['flash_h2d_server']))"
} > gpurun_out/r02e/bench_ab.txt 2>&1
for m in none overlap blocking; do timeout 300 python tools/save_overlap.py --mode $m; done > gpurun_out/r02e/save_overlap.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_select -s 3 -c 1 -o gpurun_out/r02e/sel_c3 python tools/kbench.py select --cfg C3 --iters 3 > gpurun_out/r02e/ncu_sel.log 2>&1
