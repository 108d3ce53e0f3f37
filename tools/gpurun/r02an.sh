#!/bin/bash
# Round 2: MHA select as clusters -- parity + timelines + kernels alone
mkdir -p gpurun_out/r02an
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mean_meta.py -q -k "select" > gpurun_out/r02an/sel_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02an/sel_tests.log
{
for c in "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C2"; do
  echo "== select $c"; SS_LIB_VARIANT=debug SS_SEL_TRACE=1 timeout 300 python tools/kbench.py select $c
done
for rep in 1 2; do for clu in 1 0; do for c in "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C2"; do
  echo "mha_clu=$clu $c $(SS_LIB_VARIANT=debug SS_SEL_MHA_CLU=$clu timeout 300 python tools/kbench.py select $c)"
done; done; done
} > gpurun_out/r02an/sel_trace.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py -q -x > gpurun_out/r02an/pipeline.log 2>&1
echo "rc=$?" >> gpurun_out/r02an/pipeline.log
