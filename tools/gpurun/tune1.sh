#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
for ch in 2048 1024 512; do
  for cfg in C2 C3; do
    SS_SEL_CHUNK=$ch python tools/kbench.py select --cfg $cfg | sed "s/}/, \"chunk\": $ch}/" >> gpurun_out/kbench2.log 2>&1
  done
done
python tools/kbench.py attn --cfg C2 >> gpurun_out/kbench2.log 2>&1
python tools/kbench.py attn --cfg C3 >> gpurun_out/kbench2.log 2>&1
