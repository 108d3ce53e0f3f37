#!/bin/bash
# ncu launch list of one C2 step: the session-start tree (old_tree/, commit 530c8de) vs now
mkdir -p gpurun_out/r02ak
KR='regex:block_select|cache_|flash_h2d|sparse_attn'
(cd old_tree && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 60480 -c 960 --csv \
   --log-file ../gpurun_out/r02ak/launches_old.csv python bench.py --steps 1 --warmup 3 --settle 60 \
   --h2d-server 0 --no-cpu-baseline --no-gather-alone > ../gpurun_out/r02ak/ncu_old.log 2>&1)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 60480 -c 960 --csv \
   --log-file gpurun_out/r02ak/launches_new.csv python bench.py --steps 1 --warmup 3 --settle 60 \
   --h2d-server 0 --no-cpu-baseline --no-gather-alone > gpurun_out/r02ak/ncu_new.log 2>&1
