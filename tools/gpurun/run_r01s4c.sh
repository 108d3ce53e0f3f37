#!/bin/bash
# Session 4: select chunk policy (widen the chunk when the candidate merge would exceed
# its 8192-key bound; chunk cap 2048 -> 4096): select parity incl. the 1M-ctx k=300 case,
# C3 chunk sweep beyond 2048 (one wave of 2 CTAs/SM at 32 pairs needs ~3648), C2 default.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mean_meta.py -q -k "select or mean" > gpurun_out/s4c_tests.log 2>&1
for ch in 2048 2560 3072 3296 3648 4096; do
  echo -n "chunk=$ch "; SS_SEL_CHUNK=$ch timeout 300 python tools/kbench.py select --cfg C3
done > gpurun_out/s4c_sel_chunk_c3.txt 2>&1
for ch in 1024 2048; do
  echo -n "chunk=$ch "; SS_SEL_CHUNK=$ch timeout 300 python tools/kbench.py select --cfg C2
done >> gpurun_out/s4c_sel_chunk_c3.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/s4c_fullsize.log 2>&1
