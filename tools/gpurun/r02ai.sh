#!/bin/bash
# Round 2: ncu full captures of the reworked kernels (cluster select at C3, attention
# at C3 and at the C2 request-group shape) + the launch list of one C2 step.
mkdir -p gpurun_out/r02ai
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_select_tcc -s 3 -c 1 \
   -o gpurun_out/r02ai/sel_tcc_c3 python tools/kbench.py select --cfg C3 --iters 3 > gpurun_out/r02ai/ncu_sel.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn_mma -s 3 -c 1 \
   -o gpurun_out/r02ai/attn_c3 python tools/kbench.py attn --cfg C3 --iters 3 > gpurun_out/r02ai/ncu_attn_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn_mma -s 3 -c 1 \
   -o gpurun_out/r02ai/attn_c2g python tools/kbench.py attn --cfg C2 --batch 3 --iters 3 > gpurun_out/r02ai/ncu_attn_c2g.log 2>&1
for r in sel_tcc_c3 attn_c3 attn_c2g; do
  python tools/ncu_summary.py gpurun_out/r02ai/$r.ncu-rep > gpurun_out/r02ai/$r.txt 2>&1
  python tools/ncu_source_hot.py gpurun_out/r02ai/$r.ncu-rep >> gpurun_out/r02ai/$r.txt 2>&1
done
KR='regex:block_select|cache_|flash_h2d|sparse_attn'
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 60480 -c 960 --csv \
   --log-file gpurun_out/r02ai/launches_one_step.csv python bench.py --steps 1 --warmup 3 --settle 60 \
   --h2d-server 0 --no-cpu-baseline --no-gather-alone > gpurun_out/r02ai/ncu_list.log 2>&1
python tools/launch_shares.py gpurun_out/r02ai/launches_one_step.csv > gpurun_out/r02ai/launch_shares.txt 2>&1
rm -f gpurun_out/r02ai/*.ncu-rep
