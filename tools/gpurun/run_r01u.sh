#!/bin/bash
# full GPU parity suite, C2 (3 request groups) and C3 bench lines, attention C3 traces, select check
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_u.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2_u.json 2> gpurun_out/bench_c2_u.err
timeout 900 python bench.py --config C3 > gpurun_out/bench_c3_u.json 2> gpurun_out/bench_c3_u.err
{
for mu in 16 8 4; do echo "== min_units $mu"; SS_ATTN_TRACE=1 SS_ATTN_MIN_UNITS=$mu python tools/kbench.py attn --cfg C3; done
for cfg in C2 C3; do python tools/kbench.py select --cfg $cfg; done
} > gpurun_out/attn_trace_u.txt 2>&1
