#!/bin/bash
# Session 3: PDL between the cache kernels -- parity + A/B; full-size parity in the bench's launch configuration
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py tests/test_gpu_fullsize.py -x -q > gpurun_out/s3k_tests.log 2>&1
B="python bench.py --no-cpu-baseline"
for i in 1 2; do
  SS_CACHE_PDL=1 timeout 600 $B > gpurun_out/s3k_pdl$i.json 2> gpurun_out/s3k_pdl$i.err
  SS_CACHE_PDL=0 timeout 600 $B > gpurun_out/s3k_nopdl$i.json 2> gpurun_out/s3k_nopdl$i.err
done
