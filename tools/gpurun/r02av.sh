#!/bin/bash
# Round 2: occupancy-aware cluster size for the GQA select; C3 default of 2 request groups
mkdir -p gpurun_out/r02av
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "select" > gpurun_out/r02av/sel_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02av/sel_tests.log
{
for c in "--cfg C3" "--cfg C3 --batch 2" "--cfg C3 --batch 1"; do
  echo "select $c $(timeout 300 python tools/kbench.py select $c)"
  echo "attn $c $(timeout 300 python tools/kbench.py attn $c)"
done
} > gpurun_out/r02av/kbench.txt 2>&1
timeout 900 python bench.py --config C3 > gpurun_out/r02av/bench_c3.json 2> gpurun_out/r02av/bench_c3.err
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/r02av/fullsize.log 2>&1
echo "rc=$?" >> gpurun_out/r02av/fullsize.log
