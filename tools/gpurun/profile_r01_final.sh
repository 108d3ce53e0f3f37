#!/bin/bash
# Round-1 evidence pass: per-launch list of one graph-replayed timed step (ncu serialises
# kernels: compare SHARES), ncu --set full of each hot-path kernel, kernel microbenchmarks.
set -x
KR='regex:block_select|cache_|flash_h2d|sparse_attn'
# bench --steps 1 --warmup 3: warm-up 3x384 + e2e 3x384 launches precede the timed step (384)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 2304 -c 384 --csv \
   --log-file gpurun_out/launches_r01.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k "$KR" -s 2304 -c 6 \
   -o gpurun_out/prof_r01_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
for cfg in C2 C3; do
  python tools/kbench.py select --cfg $cfg; python tools/kbench.py attn --cfg $cfg
done > gpurun_out/kbench_final.log 2>&1
python tools/kbench.py gather >> gpurun_out/kbench_final.log 2>&1
python tools/kbench.py meta >> gpurun_out/kbench_final.log 2>&1
