#!/bin/bash
# Round 2: tensor-core select A/B at C3 -- tile stages per warp (1 | 2) x start-tile
# rotation (0 | 13) x chunk (2048 | 4096); parity of the variants.
mkdir -p gpurun_out/r02n
{
for ns in 1 2; do for rot in 0 13; do for ch in 2048 4096; do
  echo "stages=$ns rot=$rot chunk=$ch $(SS_LIB_VARIANT=debug SS_SEL_TC_STAGES=$ns SS_SEL_ROT=$rot SS_SEL_CHUNK=$ch python tools/kbench.py select --cfg C3)"
done; done; done
for rot in 0 13; do echo "fp64 rot=$rot $(SS_LIB_VARIANT=debug SS_SEL_TC=0 SS_SEL_ROT=$rot python tools/kbench.py select --cfg C3)"; done
} > gpurun_out/r02n/sel_tc_ab.txt 2>&1
for v in "2 13" "1 13"; do set -- $v
SS_LIB_VARIANT=debug SS_SEL_TC_STAGES=$1 SS_SEL_ROT=$2 timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_parity.py -k "select" > gpurun_out/r02n/parity_ns$1_rot$2.log 2>&1
echo "rc=$?" >> gpurun_out/r02n/parity_ns$1_rot$2.log
done
