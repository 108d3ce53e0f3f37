#!/bin/bash
# Round 2: MHA select chunk chooser (whole waves at the request-group shape) --
# parity, kernels alone at group / full shape, the C2 step.
mkdir -p gpurun_out/r02k
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mean_meta.py tests/test_gpu_fullsize.py -q -k "select or fullsize" > gpurun_out/r02k/tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02k/tests.log
{
for b in 3 4; do python tools/kbench.py select --cfg C2 --batch $b; done
python tools/kbench.py select --cfg C2
python tools/kbench.py select --cfg C3
} > gpurun_out/r02k/kbench_select.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02k/bench_c2.json 2> gpurun_out/r02k/bench_c2.err
