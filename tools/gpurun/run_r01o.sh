#!/bin/bash
timeout 900 python bench.py --groups 4 > gpurun_out/bench_v4_g4.json 2> gpurun_out/bench_v4_g4.err
timeout 900 python bench.py --groups 3 > gpurun_out/bench_v4_g3.json 2> gpurun_out/bench_v4_g3.err
for g in 1 2 4; do timeout 900 python bench.py --config C3 --groups $g > gpurun_out/bench_v4_c3_g$g.json 2> gpurun_out/bench_v4_c3_g$g.err; done
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/gpu_tests_fullsize.log 2>&1
