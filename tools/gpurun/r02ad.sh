#!/bin/bash
# Round 2: select epilogue -- common-prefix radix, one-batch rescoring; parity + timeline
mkdir -p gpurun_out/r02ad
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mean_meta.py -q -k "select" > gpurun_out/r02ad/sel_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02ad/sel_tests.log
{
for c in "--cfg C3" "--cfg C3 --batch 1"; do
  echo "== select $c"; SS_LIB_VARIANT=debug SS_SEL_TRACE=1 timeout 300 python tools/kbench.py select $c
done
for c in "--cfg C2" "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C3" "--cfg C3 --batch 1"; do
  echo "select $c $(timeout 300 python tools/kbench.py select $c)"
done
} > gpurun_out/r02ad/sel_trace.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/r02ad/fullsize.log 2>&1
echo "rc=$?" >> gpurun_out/r02ad/fullsize.log
