#!/bin/bash
set -x
./tools/tma_host_probe > gpurun_out/tma_host_probe.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err
KR='regex:block_select|cache_|flash_h2d|sparse_attn'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 960 -c 320 --csv \
   --log-file gpurun_out/launches_r01b.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:block_select|sparse_attn' -s 192 -c 2 \
   -o gpurun_out/prof_r01b python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
