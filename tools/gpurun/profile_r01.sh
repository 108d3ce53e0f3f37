#!/bin/bash
# Round-1 profiling pass: bench line, per-launch list of one timed step, ncu --set full of the top kernels.
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err
KR='regex:block_select|cache_|flash_h2d|sparse_attn'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 2240 -c 320 --csv \
   --log-file gpurun_out/launches_r01.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:block_select|sparse_attn|flash_h2d' -s 288 -c 3 \
   -o gpurun_out/prof_r01 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
