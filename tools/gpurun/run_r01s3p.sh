#!/bin/bash
# Session 3: per-group pools x request groups
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --pool-per-group 1"
for g in 4 5 6 8; do timeout 600 $B --groups $g > gpurun_out/s3p_g$g.json 2> gpurun_out/s3p_g$g.err; done
timeout 600 $B --groups 4 --split-attn 1 > gpurun_out/s3p_g4_split.json 2> gpurun_out/s3p_g4_split.err
