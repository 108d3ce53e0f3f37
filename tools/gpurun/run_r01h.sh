#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_all.log 2>&1
python tools/kbench.py attn --cfg C3 > gpurun_out/kbench9.log 2>&1
SS_ATTN_MIN_UNITS=8 python tools/kbench.py attn --cfg C3 >> gpurun_out/kbench9.log 2>&1
SS_ATTN_MIN_UNITS=4 python tools/kbench.py attn --cfg C3 >> gpurun_out/kbench9.log 2>&1
python tools/kbench.py attn >> gpurun_out/kbench9.log 2>&1
python tools/kbench.py prefill >> gpurun_out/kbench9.log 2>&1
python tools/c4_sweep.py --batches 64,128,256 --admission > gpurun_out/c4_admission.log 2>&1
