#!/bin/bash
# Round 2: shuffle-free bulk merge -- parity, timelines, A/B vs register merge, min units.
mkdir -p gpurun_out/r02z
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "attention" > gpurun_out/r02z/attn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02z/attn_tests.log
{
for c in "--cfg C2 --batch 3" "--cfg C3"; do
  echo "== attn $c"; SS_LIB_VARIANT=debug SS_ATTN_TRACE=1 timeout 300 python tools/kbench.py attn $c
done
for rep in 1 2; do for mb in 1 0; do for c in "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C3" "--cfg C3 --batch 1"; do
  echo "merge_bulk=$mb $c $(SS_LIB_VARIANT=debug SS_ATTN_MERGE_BULK=$mb timeout 300 python tools/kbench.py attn $c)"
done; done; done
for mu in 9 10 12; do for c in "--cfg C2 --batch 3" "--cfg C3"; do
  echo "min_units=$mu $c $(SS_LIB_VARIANT=debug SS_ATTN_MIN_UNITS=$mu timeout 300 python tools/kbench.py attn $c)"
done; done
} > gpurun_out/r02z/attn_trace.txt 2>&1
