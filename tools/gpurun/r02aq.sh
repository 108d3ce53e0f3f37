#!/bin/bash
# Round 2: conflict-free ordered compactions (cta_compact, cta_topk) -- parity, timelines, kernels alone
mkdir -p gpurun_out/r02aq
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mean_meta.py -q -k "select" > gpurun_out/r02aq/sel_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02aq/sel_tests.log
{
for c in "--cfg C3" "--cfg C3 --batch 1" "--cfg C2 --batch 3"; do
  echo "== select $c"; SS_LIB_VARIANT=debug SS_SEL_TRACE=1 timeout 300 python tools/kbench.py select $c
done
for rep in 1 2; do for c in "--cfg C2" "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C3" "--cfg C3 --batch 1"; do
  echo "select $c $(timeout 300 python tools/kbench.py select $c)"
done; done
} > gpurun_out/r02aq/sel_trace.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py tests/test_gpu_prefill.py tests/test_gpu_save.py -q > gpurun_out/r02aq/other.log 2>&1
echo "rc=$?" >> gpurun_out/r02aq/other.log
