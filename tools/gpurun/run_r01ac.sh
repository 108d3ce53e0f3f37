#!/bin/bash
mkdir -p gpurun_out
{ for cfg in C3 C2; do python tools/kbench.py select --cfg $cfg; done; } > gpurun_out/sel_ac.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "select" > gpurun_out/sel_parity_ac.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_select -s 3 -c 1 \
  -o gpurun_out/prof_sel_c3_ac python tools/kbench.py select --cfg C3 --iters 2 > /dev/null 2>&1
