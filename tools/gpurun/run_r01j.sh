#!/bin/bash
# C3 attention: timing with host overhead hidden, and ncu full + source of the MMA kernel
echo "== mma" > gpurun_out/kbench11.log
python tools/kbench.py attn --cfg C3 >> gpurun_out/kbench11.log 2>&1
python tools/kbench.py attn >> gpurun_out/kbench11.log 2>&1
echo "== fma" >> gpurun_out/kbench11.log
SS_ATTN_MMA=0 python tools/kbench.py attn --cfg C3 >> gpurun_out/kbench11.log 2>&1
SS_ATTN_MMA=0 python tools/kbench.py attn >> gpurun_out/kbench11.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 3 -c 1 \
   -o gpurun_out/prof_attn_mma_c3 python tools/kbench.py attn --cfg C3 --iters 2 > gpurun_out/ncu_mma_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 3 -c 1 \
   -o gpurun_out/prof_attn_mma_c2 python tools/kbench.py attn --cfg C2 --iters 2 > gpurun_out/ncu_mma_c2.log 2>&1
