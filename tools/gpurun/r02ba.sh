#!/bin/bash
mkdir -p gpurun_out/r02ba
{
for rep in 1 2; do for mu in 4 6 8 12; do for c in "--cfg C3 --batch 2" "--cfg C3 --batch 1" "--cfg C2 --batch 3"; do
  echo "min_units=$mu $c $(SS_LIB_VARIANT=debug SS_ATTN_MIN_UNITS=$mu timeout 300 python tools/kbench.py attn $c)"
done; done; done
} > gpurun_out/r02ba/attn_minunits.txt 2>&1
