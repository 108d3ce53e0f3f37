#!/bin/bash
# Round 2 final evidence (after the select compaction fix): smoke, GPU suite, bench C2 (x2, the driver's command
# shape), C3, C2 rho=0.9, reference arm, kernels alone.
mkdir -p gpurun_out/r02ar
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ar/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r02ar/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02ar/bench_c2.json 2> gpurun_out/r02ar/bench_c2.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02ar/bench_c2_run2.json 2> gpurun_out/r02ar/bench_c2_run2.err
timeout 900 python bench.py --config C3 > gpurun_out/r02ar/bench_c3.json 2> gpurun_out/r02ar/bench_c3.err
timeout 900 python bench.py --rho 0.9 --no-cpu-baseline > gpurun_out/r02ar/bench_c2_rho09.json 2> gpurun_out/r02ar/bench_c2_rho09.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02ar/bench_reference.json 2> gpurun_out/r02ar/bench_reference.err
{
for c in "select --cfg C2" "select --cfg C2 --batch 3" "select --cfg C2 --batch 4" "select --cfg C3" "select --cfg C3 --batch 1" \
         "attn --cfg C2" "attn --cfg C2 --batch 3" "attn --cfg C2 --batch 4" "attn --cfg C3" "attn --cfg C3 --batch 1" "gather"; do
  echo "== $c"; timeout 300 python tools/kbench.py $c
done
} > gpurun_out/r02ar/kbench.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02ar/gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02ar/gpu_tests.log
