#!/bin/bash
# Session 3: per-(layer, group) LRU pools -- parity + A/B; split-attention parity after the test fix
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pipeline.py -x -q -k "split or request_groups" > gpurun_out/s3o_tests.log 2>&1
B="python bench.py --no-cpu-baseline"
for i in 1 2; do
  timeout 600 $B --pool-per-group 1 > gpurun_out/s3o_ppg$i.json 2> gpurun_out/s3o_ppg$i.err
  timeout 600 $B --pool-per-group 0 > gpurun_out/s3o_shared$i.json 2> gpurun_out/s3o_shared$i.err
done
timeout 600 $B --pool-per-group 1 --groups 4 > gpurun_out/s3o_ppg_g4.json 2> gpurun_out/s3o_ppg_g4.err
