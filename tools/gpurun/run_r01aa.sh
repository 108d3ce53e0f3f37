#!/bin/bash
mkdir -p gpurun_out
{ for cfg in C2 C3; do python tools/kbench.py select --cfg $cfg; done; } > gpurun_out/sel_aa.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mean_meta.py -x -q -k "select or meta" > gpurun_out/sel_parity_aa.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_select -s 3 -c 1 \
  -o gpurun_out/prof_sel_c3_aa python tools/kbench.py select --cfg C3 --iters 2 > /dev/null 2>&1
