#!/bin/bash
# Round 2: 12-CTA select clusters when 16-CTA ones do not all fit -- parity + kernels alone + C3 bench
mkdir -p gpurun_out/r02ax
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "select" > gpurun_out/r02ax/sel_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02ax/sel_tests.log
{
for rep in 1 2; do for c in "--cfg C3" "--cfg C3 --batch 2" "--cfg C3 --batch 1"; do
  echo "select $c $(timeout 300 python tools/kbench.py select $c)"
done; done
} > gpurun_out/r02ax/kbench.txt 2>&1
timeout 900 python bench.py --config C3 --no-cpu-baseline > gpurun_out/r02ax/bench_c3.json 2> gpurun_out/r02ax/bench_c3.err
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/r02ax/fullsize.log 2>&1
echo "rc=$?" >> gpurun_out/r02ax/fullsize.log
