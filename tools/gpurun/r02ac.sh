#!/bin/bash
# Round 2: tensor-core select timeline (C3 full batch and one request)
mkdir -p gpurun_out/r02ac
{
for c in "--cfg C3" "--cfg C3 --batch 1"; do
  echo "== select $c"; SS_LIB_VARIANT=debug SS_SEL_TRACE=1 timeout 300 python tools/kbench.py select $c
done
} > gpurun_out/r02ac/sel_trace.txt 2>&1
