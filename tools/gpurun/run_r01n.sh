#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_all2.log 2>&1
for mu in 16 8; do echo "== mma C3 min_units $mu"; SS_ATTN_TRACE=1 SS_ATTN_MIN_UNITS=$mu python tools/kbench.py attn --cfg C3; done > gpurun_out/kbench14.log 2>&1
echo "== mma C2" >> gpurun_out/kbench14.log; SS_ATTN_TRACE=1 python tools/kbench.py attn --cfg C2 >> gpurun_out/kbench14.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config C3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
