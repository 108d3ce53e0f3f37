#!/bin/bash
mkdir -p gpurun_out/r02aa
{
for c in "--cfg C2 --batch 3" "--cfg C3"; do
  echo "== attn $c"; SS_LIB_VARIANT=debug SS_ATTN_TRACE=1 timeout 300 python tools/kbench.py attn $c
done
for c in "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C3" "--cfg C3 --batch 1"; do
  echo "$c $(timeout 300 python tools/kbench.py attn $c)"
done
} > gpurun_out/r02aa/attn_trace.txt 2>&1
