#!/bin/bash
# Session 3 re-entry: parity suite, bench C2/C3 lines, kernels in isolation.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s3a_gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s3a_gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/s3a_bench_c2.json 2> gpurun_out/s3a_bench_c2.err
timeout 900 python bench.py --config C3 > gpurun_out/s3a_bench_c3.json 2> gpurun_out/s3a_bench_c3.err
{ for cfg in C2 C3; do python tools/kbench.py select --cfg $cfg; python tools/kbench.py attn --cfg $cfg; done
  python tools/kbench.py gather; python tools/kbench.py meta; } > gpurun_out/s3a_kbench.txt 2>&1
