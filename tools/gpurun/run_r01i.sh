#!/bin/bash
# tensor-core attention: parity + timing vs the FMA path
timeout 900 python -m pytest tests -m gpu -q -x -k "attn or attention or pipeline or smoke or save or prefill" > gpurun_out/gpu_tests_mma.log 2>&1
echo "== mma" > gpurun_out/kbench10.log
python tools/kbench.py attn --cfg C3 >> gpurun_out/kbench10.log 2>&1
python tools/kbench.py attn >> gpurun_out/kbench10.log 2>&1
echo "== fma" >> gpurun_out/kbench10.log
SS_ATTN_MMA=0 python tools/kbench.py attn --cfg C3 >> gpurun_out/kbench10.log 2>&1
SS_ATTN_MMA=0 python tools/kbench.py attn >> gpurun_out/kbench10.log 2>&1
echo "== mma min_units 8 / 32" >> gpurun_out/kbench10.log
SS_ATTN_MIN_UNITS=8 python tools/kbench.py attn --cfg C3 >> gpurun_out/kbench10.log 2>&1
SS_ATTN_MIN_UNITS=32 python tools/kbench.py attn --cfg C3 >> gpurun_out/kbench10.log 2>&1
