#!/bin/bash
# attention L2 prefetch distance (C2, C3) + select chunk / persistence at C3, then attention parity
mkdir -p gpurun_out
{
for pf in 0 -1 2 6 12 24; do for cfg in C3 C2; do
  if [ $pf = -1 ]; then unset SS_ATTN_L2PF; lab=auto; else export SS_ATTN_L2PF=$pf; lab=$pf; fi
  echo -n "l2pf=$lab "; python tools/kbench.py attn --cfg $cfg
done; done
unset SS_ATTN_L2PF
for mu in 8 4; do echo -n "min_units=$mu "; SS_ATTN_MIN_UNITS=$mu python tools/kbench.py attn --cfg C3; done
for ch in 512 1024 2048; do echo -n "sel_chunk=$ch "; SS_SEL_CHUNK=$ch python tools/kbench.py select --cfg C3; done
echo -n "sel_persist "; SS_SEL_PERSIST=1 python tools/kbench.py select --cfg C3
} > gpurun_out/attn_pf.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py -x -q > gpurun_out/parity_t.log 2>&1
