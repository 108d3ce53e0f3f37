#!/bin/bash
# Round 2: evidence after the attention merge rework and the cluster select --
# smoke, GPU suite, bench C2 / C3, kernels alone (single + back to back).
mkdir -p gpurun_out/r02ag
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ag/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r02ag/smoke.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02ag/bench_c2.json 2> gpurun_out/r02ag/bench_c2.err
timeout 900 python bench.py --config C3 --no-cpu-baseline > gpurun_out/r02ag/bench_c3.json 2> gpurun_out/r02ag/bench_c3.err
{
for c in "select --cfg C2" "select --cfg C2 --batch 3" "select --cfg C2 --batch 4" "select --cfg C3" "select --cfg C3 --batch 1" \
         "attn --cfg C2" "attn --cfg C2 --batch 3" "attn --cfg C2 --batch 4" "attn --cfg C3" "attn --cfg C3 --batch 1"; do
  echo "== $c"; timeout 300 python tools/kbench.py $c
done
} > gpurun_out/r02ag/kbench.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02ag/gpu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02ag/gpu_tests.log
