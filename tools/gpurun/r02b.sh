#!/bin/bash
# Round 2: sticky FlashH2D abort + server stats, NUMA host pool, N>1 path on one GPU
# (world-1 NCCL), new bench (multi-core oracle baseline, server stats), reference arm.
mkdir -p gpurun_out/r02b
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_h2d_serve.py tests/test_gpu_dist.py -x -q > gpurun_out/r02b/tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02b/tests.log
timeout 900 python bench.py > gpurun_out/r02b/bench_c2.json 2> gpurun_out/r02b/bench_c2.err
echo "rc=$?" >> gpurun_out/r02b/bench_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/r02b/bench_ref.json 2> gpurun_out/r02b/bench_ref.err
