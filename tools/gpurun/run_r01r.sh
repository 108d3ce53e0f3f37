#!/bin/bash
# ncu --set full of the C3 select (GQA G=4) and C3 attention kernels in isolation
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_select -s 3 -c 1 \
  -o gpurun_out/prof_sel_c3 python tools/kbench.py select --cfg C3 --iters 2 > gpurun_out/ncu_sel_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 3 -c 1 \
  -o gpurun_out/prof_attn_c3 python tools/kbench.py attn --cfg C3 --iters 2 > gpurun_out/ncu_attn_c3.log 2>&1
