#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mean_meta.py -x -q > gpurun_out/mean_tests.log 2>&1
timeout 900 python bench.py --timeline gpurun_out/timeline_v.json > gpurun_out/bench_c2_v.json 2> gpurun_out/bench_c2_v.err
