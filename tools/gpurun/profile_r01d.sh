#!/bin/bash
# Round-1 evidence pass (session 2): bench lines C2/C3, per-launch list of one
# graph-replayed timed step (ncu serialises kernels: compare SHARES), ncu --set
# full of the first 6 hot-path launches of that step, and of the attention /
# select kernels alone at C2 and C3.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_d_c2.json 2> gpurun_out/bench_d_c2.err
timeout 900 python bench.py --config C3 > gpurun_out/bench_d_c3.json 2> gpurun_out/bench_d_c3.err
KR='regex:block_select|cache_|flash_h2d|sparse_attn'
# --settle 10 --warmup 3 --steps 1: 13 eager steps x 576 launches (3 groups x 32 layers x 6)
# precede the timed (graph-replayed) step
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 7488 -c 576 --csv \
   --log-file gpurun_out/launches_d.csv python bench.py --steps 1 --warmup 3 --settle 10 --no-cpu-baseline > gpurun_out/ncu_list_d.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k "$KR" -s 7488 -c 6 \
   -o gpurun_out/prof_d_step python bench.py --steps 1 --warmup 3 --settle 10 --no-cpu-baseline > gpurun_out/ncu_full_d.log 2>&1
for cfg in C2 C3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 3 -c 1 \
     -o gpurun_out/prof_d_attn_$cfg python tools/kbench.py attn --cfg $cfg --iters 2 > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_select -s 3 -c 1 \
     -o gpurun_out/prof_d_sel_$cfg python tools/kbench.py select --cfg $cfg --iters 2 > /dev/null 2>&1
done
{ for cfg in C2 C3; do python tools/kbench.py select --cfg $cfg; python tools/kbench.py attn --cfg $cfg; done
  python tools/kbench.py gather; python tools/kbench.py meta; } > gpurun_out/kbench_d.txt 2>&1
