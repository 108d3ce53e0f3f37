#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
for ctas in 8 16 24 32; do for u in 16 8; do
  echo -n "ctas=$ctas unroll=$u "; SS_H2D_CTAS=$ctas SS_H2D_UNROLL=$u python tools/kbench.py overlap
done; done > gpurun_out/ab_overlap2.log 2>&1
python tools/kbench.py attn --cfg C3 > gpurun_out/kbench5.log 2>&1
python tools/kbench.py attn >> gpurun_out/kbench5.log 2>&1
for g in 1 2 3; do
  python bench.py --steps 10 --warmup 5 --groups $g --no-cpu-baseline --timeline gpurun_out/tl_g$g.json > gpurun_out/bench_g$g.json 2>&1
done
SS_H2D_CTAS=24 python bench.py --steps 10 --warmup 5 --groups 2 --no-cpu-baseline > gpurun_out/bench_g2c24.json 2>&1
