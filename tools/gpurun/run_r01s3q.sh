#!/bin/bash
# Session 3 evidence with the new defaults (5 request groups, per-group pools,
# CUDA_DEVICE_MAX_CONNECTIONS=32): full GPU suite, smoke, bench C2 x2 / C3 / reference
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s3q_gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3q_smoke.log 2>&1
for i in 1 2; do timeout 900 python bench.py > gpurun_out/s3q_c2_$i.json 2> gpurun_out/s3q_c2_$i.err; done
timeout 900 python bench.py --config C3 > gpurun_out/s3q_c3.json 2> gpurun_out/s3q_c3.err
timeout 600 python bench.py --impl reference > gpurun_out/s3q_ref.json 2> gpurun_out/s3q_ref.err
timeout 600 python bench.py --no-cpu-baseline --split-attn 1 > gpurun_out/s3q_split.json 2> gpurun_out/s3q_split.err
