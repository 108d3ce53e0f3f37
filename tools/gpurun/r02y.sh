#!/bin/bash
# Round 2: bulk vs register merge A/B with per-round timelines.
mkdir -p gpurun_out/r02y
{
for mb in 1 0; do for c in "--cfg C2 --batch 3" "--cfg C3 --batch 1" "--cfg C3"; do
  echo "== merge_bulk=$mb attn $c"; SS_LIB_VARIANT=debug SS_ATTN_MERGE_BULK=$mb SS_ATTN_TRACE=1 timeout 300 python tools/kbench.py attn $c
done; done
for mb in 1 0 1 0; do for c in "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C3"; do
  echo "merge_bulk=$mb $c $(SS_LIB_VARIANT=debug SS_ATTN_MERGE_BULK=$mb timeout 300 python tools/kbench.py attn $c)"
done; done
} > gpurun_out/r02y/attn_trace.txt 2>&1
