#!/bin/bash
mkdir -p gpurun_out/r02am
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "beyond_cluster or c1_shape or ragged_multichunk" > gpurun_out/r02am/tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02am/tests.log
{
for c in "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C2"; do
  echo "== select $c"; SS_LIB_VARIANT=debug SS_SEL_TRACE=1 timeout 300 python tools/kbench.py select $c
done
} > gpurun_out/r02am/sel_trace.txt 2>&1
