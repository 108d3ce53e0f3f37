#!/bin/bash
mkdir -p gpurun_out
{
for cfg in C2 C3; do echo -n "auto full "; python tools/kbench.py select --cfg $cfg; done
echo -n "auto C2 b5 "; python tools/kbench.py select --cfg C2 --batch 5
echo -n "auto C2 b6 "; python tools/kbench.py select --cfg C2 --batch 6
echo -n "auto C3 b1 "; python tools/kbench.py select --cfg C3 --batch 1
echo -n "auto C3 b2 "; python tools/kbench.py select --cfg C3 --batch 2
for ch in 1024 2048; do
  echo -n "ch=$ch C2 b5 "; SS_SEL_CHUNK=$ch python tools/kbench.py select --cfg C2 --batch 5
  echo -n "ch=$ch C3 full "; SS_SEL_CHUNK=$ch python tools/kbench.py select --cfg C3
  echo -n "ch=$ch C3 b2 "; SS_SEL_CHUNK=$ch python tools/kbench.py select --cfg C3 --batch 2
done
echo -n "ch=512 C3 full "; SS_SEL_CHUNK=512 python tools/kbench.py select --cfg C3
} > gpurun_out/sel_ad.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mean_meta.py -x -q -k "select or meta" > gpurun_out/sel_parity_ad.log 2>&1
