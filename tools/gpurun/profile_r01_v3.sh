#!/bin/bash
# Round-1 evidence pass v3 (tensor-core attention, settle steps): bench lines,
# per-launch list of one graph-replayed timed step (ncu serialises kernels:
# compare SHARES), ncu --set full of the first 6 hot-path launches of that step,
# and of the attention kernel alone (kbench C2 / C3).
set -x
timeout 900 python bench.py > gpurun_out/bench_v3_g2.json 2> gpurun_out/bench_v3_g2.err
timeout 900 python bench.py --groups 3 > gpurun_out/bench_v3_g3.json 2> gpurun_out/bench_v3_g3.err
KR='regex:block_select|cache_|flash_h2d|sparse_attn'
# --settle 10 --warmup 3 --steps 1: 13 eager steps x 384 launches precede the timed (graph) step
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 4992 -c 384 --csv \
   --log-file gpurun_out/launches_v3.csv python bench.py --steps 1 --warmup 3 --settle 10 --no-cpu-baseline > gpurun_out/ncu_list_v3.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k "$KR" -s 4992 -c 6 \
   -o gpurun_out/prof_v3_step python bench.py --steps 1 --warmup 3 --settle 10 --no-cpu-baseline > gpurun_out/ncu_full_v3.log 2>&1
for cfg in C2 C3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 3 -c 1 \
     -o gpurun_out/prof_v3_attn_$cfg python tools/kbench.py attn --cfg $cfg --iters 2 > gpurun_out/ncu_attn_$cfg.log 2>&1
done
