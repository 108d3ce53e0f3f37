#!/bin/bash
# Round 2: multi-round bulk merge -- parity, timelines, min-units sweep (single
# launch and back to back over 4 slot sets).
mkdir -p gpurun_out/r02x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "attention" > gpurun_out/r02x/attn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02x/attn_tests.log
{
for c in "--cfg C2 --batch 3" "--cfg C3 --batch 1" "--cfg C3"; do
  echo "== attn $c"; SS_LIB_VARIANT=debug SS_ATTN_TRACE=1 timeout 300 python tools/kbench.py attn $c
done
for mu in 4 6 8 10 12 16 24; do for c in "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C2" "--cfg C3 --batch 1" "--cfg C3"; do
  echo "min_units=$mu $c $(SS_LIB_VARIANT=debug SS_ATTN_MIN_UNITS=$mu timeout 300 python tools/kbench.py attn $c)"
done; done
} > gpurun_out/r02x/attn_trace.txt 2>&1
