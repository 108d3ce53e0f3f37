#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py -q -x > gpurun_out/gpu_tests.log 2>&1
python tools/kbench.py attn > gpurun_out/kbench8.log 2>&1
python tools/kbench.py attn --cfg C3 >> gpurun_out/kbench8.log 2>&1
python bench.py --steps 20 --warmup 5 --groups 2 --no-cpu-baseline --timeline gpurun_out/tl_g2.json > gpurun_out/bench_g2.json 2>&1
python bench.py --steps 20 --warmup 5 --groups 3 --no-cpu-baseline > gpurun_out/bench_g3.json 2>&1
