#!/bin/bash
# Session 3: split attention (hits while FlashH2D loads the misses) -- parity + A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py tests/test_gpu_h2d_serve.py tests/test_gpu_fullsize.py -x -q -k "split or request_groups or serve or fullsize or attention" > gpurun_out/s3n_tests.log 2>&1
B="python bench.py --no-cpu-baseline"
for i in 1 2; do
  timeout 600 $B --split-attn 1 > gpurun_out/s3n_split$i.json 2> gpurun_out/s3n_split$i.err
  timeout 600 $B --split-attn 0 > gpurun_out/s3n_nosplit$i.json 2> gpurun_out/s3n_nosplit$i.err
done
timeout 600 $B --split-attn 1 --config C3 > gpurun_out/s3n_split_c3.json 2> gpurun_out/s3n_split_c3.err
