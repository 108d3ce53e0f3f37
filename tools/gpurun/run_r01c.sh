#!/bin/bash
python bench.py --steps 10 --warmup 5 --groups 2 --no-cpu-baseline --timeline gpurun_out/tl_g2.json > gpurun_out/bench_g2.json 2>gpurun_out/bench_g2.err
python bench.py --steps 10 --warmup 5 --groups 1 --no-cpu-baseline > gpurun_out/bench_g1.json 2>&1
python bench.py --steps 10 --warmup 5 --groups 3 --no-cpu-baseline --timeline gpurun_out/tl_g3.json > gpurun_out/bench_g3.json 2>&1
SS_H2D_CTAS=24 python bench.py --steps 10 --warmup 5 --groups 2 --no-cpu-baseline > gpurun_out/bench_g2c24.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 3 -c 1 -o gpurun_out/prof_attn_c3 python tools/kbench.py attn --cfg C3 --iters 1 > gpurun_out/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_select -s 3 -c 1 -o gpurun_out/prof_sel_c3 python tools/kbench.py select --cfg C3 --iters 1 >> gpurun_out/ncu_c3.log 2>&1
