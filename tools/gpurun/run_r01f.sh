#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py -q -x > gpurun_out/gpu_tests.log 2>&1
python tools/kbench.py select --cfg C3 > gpurun_out/kbench7.log 2>&1
python tools/kbench.py select >> gpurun_out/kbench7.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 3 -c 1 -o gpurun_out/prof_attn_c2 python tools/kbench.py attn --iters 1 > gpurun_out/ncu_c2.log 2>&1
