#!/bin/bash
# Round 2: the final tree as the driver runs it -- smoke, GPU suite, bench C2 / C3 defaults
mkdir -p gpurun_out/r02bc
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bc/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r02bc/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02bc/bench_c2.json 2> gpurun_out/r02bc/bench_c2.err
timeout 900 python bench.py --config C3 --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02bc/bench_c3.json 2> gpurun_out/r02bc/bench_c3.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02bc/gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02bc/gpu_tests.log
