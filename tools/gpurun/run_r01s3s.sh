#!/bin/bash
# Session 3 final profiling: Fig. 4a analog (FlashH2D vs per-block / bulk memcpy over block
# sizes), ncu launch list + full capture of the final default step (per-launch FlashH2D form)
mkdir -p gpurun_out
timeout 600 python tools/kbench.py h2dsweep > gpurun_out/s3s_h2dsweep.txt 2>&1
B="python bench.py --no-cpu-baseline --h2d-server 0 --steps 1 --warmup 3 --settle 10 --no-gather-alone"
KR='regex:block_select|cache_|flash_h2d|sparse_attn'
# 5 groups x 32 layers x 6 launches = 960 per step; 11 eager + 2 graph warm-up steps precede the timed one
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 12480 -c 960 --csv \
   --log-file gpurun_out/s3s_launches.csv $B > gpurun_out/s3s_ncu_list.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k "$KR" -s 12480 -c 6 \
   -o /tmp/s3s_step $B > gpurun_out/s3s_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/s3s_step.ncu-rep > gpurun_out/s3s_ncu_step_summary.txt 2>&1
