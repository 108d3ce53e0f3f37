#!/bin/bash
# Session 4 final: full GPU suite, smoke and the default bench line on the final tree.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4d_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s4d_gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/s4d_bench.json 2> gpurun_out/s4d_bench.err
timeout 900 python bench.py --config C3 --no-cpu-baseline > gpurun_out/s4d_bench_c3.json 2> gpurun_out/s4d_bench_c3.err
