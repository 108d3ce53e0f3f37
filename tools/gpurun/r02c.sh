#!/bin/bash
# Round 2: switch-dispatched GQA select (no per-head select instructions), fixed
# stats test, N>1 path on one GPU, select parity, kbench select C2/C3, bench C2.
mkdir -p gpurun_out/r02c
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c/smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_h2d_serve.py tests/test_gpu_dist.py tests/test_gpu_mean_meta.py -q > gpurun_out/r02c/tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02c/tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "select" >> gpurun_out/r02c/tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02c/tests.log
{
for cfg in C2 C3; do python tools/kbench.py select --cfg $cfg; done
python tools/kbench.py select --cfg C2 --batch 3
for ch in 1024 2048 4096; do SS_LIB_VARIANT=debug SS_SEL_CHUNK=$ch python tools/kbench.py select --cfg C3 | sed "s/^/chunk=$ch /"; done
} > gpurun_out/r02c/kbench_select.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02c/bench_c2.json 2> gpurun_out/r02c/bench_c2.err
echo "rc=$?" >> gpurun_out/r02c/bench_c2.err
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/r02c/fullsize.log 2>&1
