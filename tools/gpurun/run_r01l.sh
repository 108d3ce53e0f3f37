#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x -k "attn or attention or pipeline or smoke" > gpurun_out/gpu_tests_mma2.log 2>&1
for cfg in C3 C2; do
  for mu in 16 8 4; do
    echo "== mma $cfg min_units $mu"; SS_ATTN_TRACE=1 SS_ATTN_MIN_UNITS=$mu python tools/kbench.py attn --cfg $cfg
  done
  echo "== fma $cfg"; SS_ATTN_MMA=0 python tools/kbench.py attn --cfg $cfg
done > gpurun_out/kbench12.log 2>&1
