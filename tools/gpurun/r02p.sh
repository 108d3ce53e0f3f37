#!/bin/bash
# Round 2: TC select with the candidates' metadata staged by cp.async (one round
# trip per batch instead of ~8 per candidate); histogram aggregation reverted.
mkdir -p gpurun_out/r02p
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mean_meta.py -q -k "select" > gpurun_out/r02p/tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02p/tests.log
{
python tools/kbench.py select --cfg C3
for ch in 1024 4096; do SS_LIB_VARIANT=debug SS_SEL_CHUNK=$ch python tools/kbench.py select --cfg C3 | sed "s/^/chunk=$ch /"; done
SS_LIB_VARIANT=debug SS_SEL_TC=0 python tools/kbench.py select --cfg C3 | sed 's/^/fp64-only /'
for b in 3 4; do python tools/kbench.py select --cfg C2 --batch $b; done
python tools/kbench.py select --cfg C2
} > gpurun_out/r02p/kbench.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_select_tc -s 3 -c 1 -o gpurun_out/r02p/sel_tc_c3 python tools/kbench.py select --cfg C3 --iters 3 > gpurun_out/r02p/ncu.log 2>&1
