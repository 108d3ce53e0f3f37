#!/bin/bash
# Session 3: out-of-order FlashH2D server + ready-event edge before the done wait
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_h2d_serve.py tests/test_gpu_pipeline.py tests/test_gpu_fullsize.py -x -q > gpurun_out/s3t_tests.log 2>&1
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s3t_c2_$i.json 2> gpurun_out/s3t_c2_$i.err; done
timeout 600 python bench.py --no-cpu-baseline --split-attn 1 > gpurun_out/s3t_split.json 2> gpurun_out/s3t_split.err
timeout 600 python bench.py --no-cpu-baseline --groups 8 > gpurun_out/s3t_g8.json 2> gpurun_out/s3t_g8.err
timeout 900 python bench.py --config C3 --no-cpu-baseline > gpurun_out/s3t_c3.json 2> gpurun_out/s3t_c3.err
