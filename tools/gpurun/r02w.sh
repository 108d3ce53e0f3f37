#!/bin/bash
# Round 2: attention merge with one acq_rel ticket and end-of-range bulk loads of
# the partials -- parity, timelines, min-units sweep.
mkdir -p gpurun_out/r02w
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "attention" > gpurun_out/r02w/attn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02w/attn_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/r02w/fullsize_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02w/fullsize_tests.log
{
for c in "--cfg C2 --batch 3" "--cfg C3 --batch 1" "--cfg C3"; do
  echo "== attn $c"; SS_LIB_VARIANT=debug SS_ATTN_TRACE=1 timeout 300 python tools/kbench.py attn $c
done
for mu in 4 6 8 10 12 16; do for c in "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C2" "--cfg C3 --batch 1" "--cfg C3"; do
  echo "min_units=$mu $c $(SS_LIB_VARIANT=debug SS_ATTN_MIN_UNITS=$mu timeout 300 python tools/kbench.py attn $c)"
done; done
} > gpurun_out/r02w/attn_trace.txt 2>&1
