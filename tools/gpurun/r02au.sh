#!/bin/bash
# Round 2: C3 request-group count (1 / 2 / 4): step time and the kernels' own fractions
mkdir -p gpurun_out/r02au
for g in 4 2 1; do
  timeout 900 python bench.py --config C3 --groups $g --no-cpu-baseline > gpurun_out/r02au/bench_c3_g$g.json 2> gpurun_out/r02au/bench_c3_g$g.err
done
