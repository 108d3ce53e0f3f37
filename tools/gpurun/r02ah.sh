#!/bin/bash
mkdir -p gpurun_out/r02ah
{
for c in "--cfg C3" "--cfg C3 --batch 1"; do
  echo "== select $c"; SS_LIB_VARIANT=debug SS_SEL_TRACE=1 timeout 300 python tools/kbench.py select $c
done
} > gpurun_out/r02ah/sel_trace.txt 2>&1
