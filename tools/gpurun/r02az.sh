#!/bin/bash
# Round 2: ncu full captures of the final select (C3 full batch, two requests) and attention (two C3 requests)
mkdir -p gpurun_out/r02az
timeout 600 ncu --set full --clock-control none -k regex:block_select_tcc -s 3 -c 1 \
   -o gpurun_out/r02az/sel_c3 python tools/kbench.py select --cfg C3 --iters 3 > gpurun_out/r02az/ncu_sel_c3.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:block_select_tcc -s 3 -c 1 \
   -o gpurun_out/r02az/sel_c3b2 python tools/kbench.py select --cfg C3 --batch 2 --iters 3 > gpurun_out/r02az/ncu_sel_c3b2.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:sparse_attn_mma -s 3 -c 1 \
   -o gpurun_out/r02az/attn_c3b2 python tools/kbench.py attn --cfg C3 --batch 2 --iters 3 > gpurun_out/r02az/ncu_attn_c3b2.log 2>&1
for r in sel_c3 sel_c3b2 attn_c3b2; do python tools/ncu_summary.py gpurun_out/r02az/$r.ncu-rep > gpurun_out/r02az/$r.txt 2>&1; done
rm -f gpurun_out/r02az/*.ncu-rep
