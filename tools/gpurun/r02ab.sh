#!/bin/bash
mkdir -p gpurun_out/r02ab
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "attention" > gpurun_out/r02ab/attn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02ab/attn_tests.log
{
for c in "--cfg C2 --batch 3" "--cfg C3"; do
  echo "== attn $c"; SS_LIB_VARIANT=debug SS_ATTN_TRACE=1 timeout 300 python tools/kbench.py attn $c
done
for rep in 1 2; do for c in "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C2" "--cfg C3" "--cfg C3 --batch 1"; do
  echo "$c $(timeout 300 python tools/kbench.py attn $c)"
done; done
} > gpurun_out/r02ab/attn_trace.txt 2>&1
