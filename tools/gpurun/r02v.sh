#!/bin/bash
# Round 2: fixed cost of a one-CTA-per-SM launch (tools/launch_probe.cu) and
# the attention merge path's timeline (flush -> ticket -> merge phases).
mkdir -p gpurun_out/r02v
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/launch_probe tools/launch_probe.cu && timeout 120 /tmp/launch_probe > gpurun_out/r02v/launch_probe.txt 2>&1
{
for c in "--cfg C2 --batch 3" "--cfg C3 --batch 1" "--cfg C3"; do
  echo "== attn $c"; SS_LIB_VARIANT=debug SS_ATTN_TRACE=1 timeout 300 python tools/kbench.py attn $c
done
} > gpurun_out/r02v/attn_trace.txt 2>&1
