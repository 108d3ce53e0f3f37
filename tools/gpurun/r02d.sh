#!/bin/bash
# Round 2: LOP3 operand select in the GQA block select (A/B vs round-1 IMAD form),
# FlashH2D server in-flight A/B in the full step, attention timeline at the bench
# launch shape, overlapped FlashD2H save parity, Fig. 4b analog.
mkdir -p gpurun_out/r02d
{
for cfg in C2 C3; do python tools/kbench.py select --cfg $cfg; done
for ch in 1024 2048 4096; do SS_LIB_VARIANT=debug SS_SEL_CHUNK=$ch python tools/kbench.py select --cfg C3 | sed "s/^/chunk=$ch /"; done
SS_LIB_VARIANT=debug SS_SEL_TT=1 python tools/kbench.py select --cfg C3 | sed "s/^/tt=1 /"
} > gpurun_out/r02d/kbench_select.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "select" > gpurun_out/r02d/select_tests.log 2>&1
timeout 600 python -m pytest tests/test_gpu_save.py -q > gpurun_out/r02d/save_test.log 2>&1
{
for v in "16 128" "24 128" "32 128" "16 256" "24 256" "48 128"; do
  set -- $v
  echo "== CTAS=$1 THREADS=$2"
  SS_LIB_VARIANT=debug SS_H2D_CTAS=$1 SS_H2D_THREADS=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-gather-alone | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({k: d.get(k) for k in ['value','ms_per_step','step_ms_min_median_max','hit_rate']}), json.dumps(d['flash_h2d']), json.dumps(d['flash_h2d_server']), json.dumps({k: v.get('us_per_launch') for k, v in d['kernels'].items() if isinstance(v, dict)}))"
done
} > gpurun_out/r02d/server_ab.txt 2>&1
{
SS_LIB_VARIANT=debug SS_ATTN_TRACE=1 python tools/kbench.py attn --cfg C2 --batch 3
SS_LIB_VARIANT=debug SS_ATTN_TRACE=1 python tools/kbench.py attn --cfg C2
SS_LIB_VARIANT=debug SS_ATTN_TRACE=1 python tools/kbench.py attn --cfg C3
} > gpurun_out/r02d/attn_trace.txt 2>&1
python tools/kbench.py d2h > gpurun_out/r02d/fig4b_d2h.txt 2>&1
