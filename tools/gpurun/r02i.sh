#!/bin/bash
# Round-2 evidence pass: GPU suite, smoke, bench lines (C2 default, C3, C2 rho=0.9,
# C2 shared pool R11, C2 with a 112 GiB physical host pool), reference arm, C4 sweep
# to B=256 (+ admission), PCIe under HBM load, ncu launch list of one C2 step.
mkdir -p gpurun_out/r02i
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02i/gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02i/gpu_tests.log
timeout 900 python bench.py > gpurun_out/r02i/bench_c2.json 2> gpurun_out/r02i/bench_c2.err
timeout 900 python bench.py --config C3 > gpurun_out/r02i/bench_c3.json 2> gpurun_out/r02i/bench_c3.err
timeout 900 python bench.py --rho 0.9 --no-cpu-baseline > gpurun_out/r02i/bench_c2_rho09.json 2> gpurun_out/r02i/bench_c2_rho09.err
timeout 900 python bench.py --pool-per-group 0 --no-cpu-baseline > gpurun_out/r02i/bench_c2_shared_pool.json 2> gpurun_out/r02i/bench_c2_shared_pool.err
timeout 1200 python bench.py --host-runs 1789 --no-cpu-baseline > gpurun_out/r02i/bench_c2_hostpool_large.json 2> gpurun_out/r02i/bench_c2_hostpool_large.err
timeout 900 python bench.py --impl reference > gpurun_out/r02i/bench_reference.json 2> gpurun_out/r02i/bench_reference.err
python tools/kbench.py h2dload > gpurun_out/r02i/h2d_under_load.txt 2>&1
timeout 1500 python tools/c4_sweep.py > gpurun_out/r02i/c4_sweep.txt 2>&1
timeout 1500 python tools/c4_sweep.py --admission > gpurun_out/r02i/c4_admission.txt 2>&1
KR='regex:block_select|cache_|flash_h2d|sparse_attn'
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 60480 -c 960 --csv \
   --log-file gpurun_out/r02i/launches_one_step.csv python bench.py --steps 1 --warmup 3 --settle 60 \
   --h2d-server 0 --no-cpu-baseline --no-gather-alone > gpurun_out/r02i/ncu_list.log 2>&1
