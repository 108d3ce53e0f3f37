#!/bin/bash
# Session 3: fused cache call -- parity (fused default + three-kernel form) and A/B in the C2 step
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py tests/test_gpu_h2d_serve.py tests/test_gpu_fullsize.py -x -q > gpurun_out/s3j_tests.log 2>&1
B="python bench.py --no-cpu-baseline"
for i in 1 2; do
  SS_CACHE_FUSED=1 timeout 600 $B > gpurun_out/s3j_fused$i.json 2> gpurun_out/s3j_fused$i.err
  SS_CACHE_FUSED=0 timeout 600 $B > gpurun_out/s3j_three$i.json 2> gpurun_out/s3j_three$i.err
done
SS_CACHE_FUSED=1 SS_CACHE_CTAS=64 timeout 600 $B > gpurun_out/s3j_fused64.json 2> gpurun_out/s3j_fused64.err
