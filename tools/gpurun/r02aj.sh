#!/bin/bash
mkdir -p gpurun_out/r02aj
timeout 600 python bench.py --steps 2 --warmup 3 --settle 60 --h2d-server 0 --no-cpu-baseline --no-gather-alone > gpurun_out/r02aj/bench_noserver.json 2> gpurun_out/r02aj/bench_noserver.err
echo "rc=$?" >> gpurun_out/r02aj/bench_noserver.err
CUDA_LAUNCH_BLOCKING=1 timeout 900 python bench.py --steps 1 --warmup 3 --settle 60 --h2d-server 0 --no-cpu-baseline --no-gather-alone > gpurun_out/r02aj/bench_noserver_blocking.json 2> gpurun_out/r02aj/bench_noserver_blocking.err
echo "rc=$?" >> gpurun_out/r02aj/bench_noserver_blocking.err
