#!/bin/bash
# Re-entry check: GPU parity suite, smoke, default bench (C2) and C3 bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config C3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
nvidia-smi -q | grep -i -A3 "link" | head -40 > gpurun_out/pcie.txt
