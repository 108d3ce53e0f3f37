#!/bin/bash
# Round 2: tensor-core GQA select (approximate scores + error bound on mma.sync,
# exact fp64 rescoring of the candidates) -- parity (ties, near-ties below f32
# resolution, f32 overflow / underflow, full-size C3), kernels alone, C3 bench.
mkdir -p gpurun_out/r02m
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mean_meta.py tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py -q -k "select or fullsize or gqa_multilayer or request_groups" > gpurun_out/r02m/tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02m/tests.log
{
python tools/kbench.py select --cfg C3
SS_LIB_VARIANT=debug SS_SEL_TC=0 python tools/kbench.py select --cfg C3 | sed 's/^/fp64-only /'
for ch in 1024 2048 4096; do SS_LIB_VARIANT=debug SS_SEL_CHUNK=$ch python tools/kbench.py select --cfg C3 | sed "s/^/tc chunk=$ch /"; done
python tools/kbench.py select --cfg C3 --batch 1
python tools/kbench.py select --cfg C2
python tools/kbench.py attn --cfg C2 --batch 3
python tools/kbench.py attn --cfg C3
} > gpurun_out/r02m/kbench.txt 2>&1
timeout 900 python bench.py --config C3 --no-cpu-baseline > gpurun_out/r02m/bench_c3.json 2> gpurun_out/r02m/bench_c3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_select_tc -s 3 -c 1 -o gpurun_out/r02m/sel_tc_c3 python tools/kbench.py select --cfg C3 --iters 3 > gpurun_out/r02m/ncu.log 2>&1
