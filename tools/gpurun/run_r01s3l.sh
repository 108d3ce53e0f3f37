#!/bin/bash
# Session 3 evidence: full GPU suite, smoke, bench C2 (x2) / C3 / reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s3l_gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3l_smoke.log 2>&1
for i in 1 2; do timeout 900 python bench.py > gpurun_out/s3l_c2_$i.json 2> gpurun_out/s3l_c2_$i.err; done
timeout 900 python bench.py --config C3 > gpurun_out/s3l_c3.json 2> gpurun_out/s3l_c3.err
timeout 600 python bench.py --impl reference > gpurun_out/s3l_ref.json 2> gpurun_out/s3l_ref.err
