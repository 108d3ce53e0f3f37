#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k attention > gpurun_out/gpu_tests_attn.log 2>&1
python tools/kbench.py attn > gpurun_out/kbench6.log 2>&1
python tools/kbench.py attn --cfg C3 >> gpurun_out/kbench6.log 2>&1
for c in 16 64 148; do
  SS_H2D_CTAS=$c python bench.py --steps 8 --warmup 4 --groups 1 --no-cpu-baseline > gpurun_out/bench_g1_c$c.json 2>&1
done
