#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gather" > gpurun_out/gather_parity_ae.log 2>&1
python tools/kbench.py gather > gpurun_out/gather_ae.txt 2>&1
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_ae$i.json 2> gpurun_out/bench_c2_ae$i.err; done
