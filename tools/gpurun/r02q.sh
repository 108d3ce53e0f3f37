#!/bin/bash
# Round 2: TC select L2-prefetch A/B; GPU suite, smoke, C2 / C3 bench on the final select.
mkdir -p gpurun_out/r02q
{
for pf in 0 2 4 8; do echo "pf=$pf $(SS_LIB_VARIANT=debug SS_SEL_TC_PF=$pf python tools/kbench.py select --cfg C3)"; done
for pf in 0 4; do echo "pf=$pf chunk=2048 $(SS_LIB_VARIANT=debug SS_SEL_TC_PF=$pf SS_SEL_CHUNK=2048 python tools/kbench.py select --cfg C3)"; done
} > gpurun_out/r02q/kbench_pf.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02q/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02q/gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02q/gpu_tests.log
timeout 900 python bench.py > gpurun_out/r02q/bench_c2.json 2> gpurun_out/r02q/bench_c2.err
timeout 900 python bench.py --config C3 --no-cpu-baseline > gpurun_out/r02q/bench_c3.json 2> gpurun_out/r02q/bench_c3.err
