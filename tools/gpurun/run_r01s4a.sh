#!/bin/bash
# Session 4 (re-created container): confirm the restored tree end to end on a fresh box —
# smoke(), the full GPU suite, the default bench line (driver's command) and the reference arm.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4a_smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s4a_gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/s4a_bench.json 2> gpurun_out/s4a_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s4a_ref.json 2> gpurun_out/s4a_ref.err
