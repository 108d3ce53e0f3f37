#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_x.log 2>&1
python tools/kbench.py cache --cfg C2 > gpurun_out/kbench_cache_x.txt 2>&1
python tools/kbench.py cache --cfg C3 >> gpurun_out/kbench_cache_x.txt 2>&1
timeout 900 python bench.py --timeline gpurun_out/timeline_x.json --no-cpu-baseline > gpurun_out/bench_c2_x.json 2> gpurun_out/bench_c2_x.err
