#!/bin/bash
mkdir -p gpurun_out/r02bb
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "attention" > gpurun_out/r02bb/attn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02bb/attn_tests.log
{
for rep in 1 2; do for c in "--cfg C2" "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C3" "--cfg C3 --batch 2" "--cfg C3 --batch 1"; do
  echo "default $c $(timeout 300 python tools/kbench.py attn $c)"
  echo "min_units=8 $c $(SS_LIB_VARIANT=debug SS_ATTN_MIN_UNITS=8 timeout 300 python tools/kbench.py attn $c)"
done; done
} > gpurun_out/r02bb/attn_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py -q -x > gpurun_out/r02bb/other.log 2>&1
echo "rc=$?" >> gpurun_out/r02bb/other.log
