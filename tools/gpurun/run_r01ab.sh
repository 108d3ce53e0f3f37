#!/bin/bash
mkdir -p gpurun_out
{ for tt in 2 1; do for cfg in C3; do echo -n "tt=$tt "; SS_SEL_TT=$tt python tools/kbench.py select --cfg $cfg; done; done
  for ch in 1024 2048; do echo -n "tt=1 ch=$ch "; SS_SEL_TT=1 SS_SEL_CHUNK=$ch python tools/kbench.py select --cfg C3; done
} > gpurun_out/sel_ab.txt 2>&1
SS_SEL_TT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "select" > gpurun_out/sel_parity_ab.log 2>&1
