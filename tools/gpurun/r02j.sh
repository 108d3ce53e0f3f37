#!/bin/bash
# Round 2: select chunk and attention split at the bench's launch shape (one
# request group: 3 or 4 requests of C2), kernels alone.
mkdir -p gpurun_out/r02j
{
for b in 3 4; do
  for ch in 512 768 1024 1536 2048; do
    echo "batch=$b chunk=$ch $(SS_LIB_VARIANT=debug SS_SEL_CHUNK=$ch python tools/kbench.py select --cfg C2 --batch $b)"
  done
  for mu in 4 8 16; do
    echo "batch=$b attn_min_units=$mu $(SS_LIB_VARIANT=debug SS_ATTN_MIN_UNITS=$mu python tools/kbench.py attn --cfg C2 --batch $b)"
  done
  echo "batch=$b attn_cta_warps=1 $(SS_LIB_VARIANT=debug SS_ATTN_CTA_WARPS=1 python tools/kbench.py attn --cfg C2 --batch $b)"
done
} > gpurun_out/r02j/group_shape_sweep.txt 2>&1
# stages-per-warp A/B for the tensor-core attention (NS x NW = 2x6 | 3x4 | 4x3)
{
for ns in 2 3 4; do
  for a in "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C2" "--cfg C3"; do
    echo "stages=$ns $a $(SS_LIB_VARIANT=debug SS_ATTN_STAGES=$ns python tools/kbench.py attn $a)"
  done
  for mu in 4 16; do
    echo "stages=$ns min_units=$mu C3 $(SS_LIB_VARIANT=debug SS_ATTN_STAGES=$ns SS_ATTN_MIN_UNITS=$mu python tools/kbench.py attn --cfg C3)"
  done
done
} > gpurun_out/r02j/attn_stages.txt 2>&1
for ns in 3 4; do
  SS_LIB_VARIANT=debug SS_ATTN_STAGES=$ns timeout 600 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k attention > gpurun_out/r02j/attn_parity_stages$ns.log 2>&1
  echo "rc=$?" >> gpurun_out/r02j/attn_parity_stages$ns.log
done
