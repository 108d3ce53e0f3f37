#!/bin/bash
# Round 2: cluster select rescoring loads by one 2-D TMA per candidate -- parity + timeline
mkdir -p gpurun_out/r02ap
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "select or attention" > gpurun_out/r02ap/tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02ap/tests.log
{
for c in "--cfg C3" "--cfg C3 --batch 1"; do
  echo "== select $c"; SS_LIB_VARIANT=debug SS_SEL_TRACE=1 timeout 300 python tools/kbench.py select $c
done
for rep in 1 2; do for c in "--cfg C3" "--cfg C3 --batch 1" "--cfg C2 --batch 4"; do
  echo "select $c $(timeout 300 python tools/kbench.py select $c)"
done; done
} > gpurun_out/r02ap/sel_trace.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/r02ap/fullsize.log 2>&1
echo "rc=$?" >> gpurun_out/r02ap/fullsize.log
