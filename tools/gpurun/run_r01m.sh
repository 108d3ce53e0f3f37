#!/bin/bash
for mu in 16 8; do echo "== mma C3 min_units $mu"; SS_ATTN_TRACE=1 SS_ATTN_MIN_UNITS=$mu python tools/kbench.py attn --cfg C3; done > gpurun_out/kbench13.log 2>&1
echo "== mma C2" >> gpurun_out/kbench13.log; SS_ATTN_TRACE=1 python tools/kbench.py attn --cfg C2 >> gpurun_out/kbench13.log 2>&1
