#!/bin/bash
# Round-2 final evidence: smoke, GPU suite, bench C2 (x2) / C3 / reference, kernels
# alone, ncu full captures of the step's kernels at the bench launch shape, memcheck
# + racecheck of the tensor-core select.
mkdir -p gpurun_out/r02r
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02r/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02r/gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02r/gpu_tests.log
timeout 900 python bench.py > gpurun_out/r02r/bench_c2.json 2> gpurun_out/r02r/bench_c2.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02r/bench_c2_run2.json 2> gpurun_out/r02r/bench_c2_run2.err
timeout 900 python bench.py --config C3 > gpurun_out/r02r/bench_c3.json 2> gpurun_out/r02r/bench_c3.err
timeout 900 python bench.py --impl reference > gpurun_out/r02r/bench_reference.json 2> gpurun_out/r02r/bench_reference.err
{
for c in "select --cfg C2" "select --cfg C2 --batch 3" "select --cfg C2 --batch 4" "select --cfg C3" "select --cfg C3 --batch 1" \
         "attn --cfg C2" "attn --cfg C2 --batch 3" "attn --cfg C2 --batch 4" "attn --cfg C3" "gather" "meta"; do
  python tools/kbench.py $c
done
} > gpurun_out/r02r/kbench.txt 2>&1
KR='regex:block_select|cache_|flash_h2d|sparse_attn'
timeout 1500 ncu --set full --clock-control none --import-source on -k "$KR" -s 60480 -c 6 \
   -o gpurun_out/r02r/step_kernels python bench.py --steps 1 --warmup 3 --settle 60 --h2d-server 0 \
   --no-cpu-baseline --no-gather-alone > gpurun_out/r02r/ncu_step.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --leak-check no --target-processes all --print-limit 50 \
    python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "gqa_ties or near_ties or extreme or ragged_multichunk" \
    > gpurun_out/r02r/memcheck_tc_select.log 2>&1
echo "exit=$?" >> gpurun_out/r02r/memcheck_tc_select.log
timeout 900 compute-sanitizer --tool racecheck --target-processes all --print-limit 50 \
    python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "gqa_ties or ragged_multichunk" \
    > gpurun_out/r02r/racecheck_tc_select.log 2>&1
echo "exit=$?" >> gpurun_out/r02r/racecheck_tc_select.log
