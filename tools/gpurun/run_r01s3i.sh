#!/bin/bash
# Session 3 evidence pass: full GPU suite, smoke, bench C2/C3 + reference arm,
# ncu launch list of one graph-replayed step (per-launch FlashH2D) and a full
# capture of its first 6 hot-path launches (summarised on the box).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3i_gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3i_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/s3i_c2.json 2> gpurun_out/s3i_c2.err
timeout 900 python bench.py --config C3 > gpurun_out/s3i_c3.json 2> gpurun_out/s3i_c3.err
timeout 600 python bench.py --impl reference > gpurun_out/s3i_ref.json 2> gpurun_out/s3i_ref.err
B="python bench.py --no-cpu-baseline --h2d-server 0 --steps 1 --warmup 3 --settle 10 --no-gather-alone"
KR='regex:block_select|cache_|flash_h2d|sparse_attn'
# settle 10 + warm-up 3 - 2 graph warm-up replays = 11 eager steps x 576 launches, then 2 graph replays x 576
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 7488 -c 576 --csv \
   --log-file gpurun_out/s3i_launches.csv $B > gpurun_out/s3i_ncu_list.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k "$KR" -s 7488 -c 6 \
   -o /tmp/s3i_step $B > gpurun_out/s3i_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/s3i_step.ncu-rep > gpurun_out/s3i_ncu_step_summary.txt 2>&1
du -sh gpurun_out
