#!/bin/bash
# Session 4: working-set parity against the new oracle (or_ws_estimate / or_admit);
# host-ahead spin A/B (5 vs 20 ms untimed spin before the start event: the first
# timed step was the slowest, 18.4 ms vs a 10.4 ms median, in s4a).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_working_set.py tests/test_abi_cpu.py -q > gpurun_out/s4b_tests.log 2>&1
for i in 1 2; do
  for c in 10000000 40000000; do
    SS_HOST_AHEAD_CYCLES=$c timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s4b_c2_spin${c}_$i.json 2> gpurun_out/s4b_c2_spin${c}_$i.err
  done
done
