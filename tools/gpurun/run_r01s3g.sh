#!/bin/bash
# Session 3: request groups x select chunk at the HBM-filling cache (chain-bound regime)
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --settle 250 --steps 10"
for g in 3 4 5 6; do
  for ch in 1024 2048; do
    SS_SEL_CHUNK=$ch timeout 600 $B --groups $g > gpurun_out/s3g_g${g}_ch$ch.json 2> gpurun_out/s3g_g${g}_ch$ch.err
  done
done
SS_H2D_CTAS=24 timeout 600 $B --groups 4 > gpurun_out/s3g_g4_ctas24.json 2> gpurun_out/s3g_g4_ctas24.err
