#!/bin/bash
# A/B: select kernel with integer-built float64 operands (SS_SEL_ICV=1, default) vs F2F (0)
mkdir -p gpurun_out
for icv in 0 1; do for cfg in C2 C3; do
  SS_SEL_ICV=$icv python tools/kbench.py select --cfg $cfg | sed "s/^/icv=$icv /"
done; done > gpurun_out/sel_icv.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "select or sel or full or c2 or c3" > gpurun_out/sel_parity.log 2>&1
SS_SEL_ICV=0 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/sel_parity_icv0.log 2>&1
