#!/bin/bash
mkdir -p gpurun_out
{
for cw in 6 1; do for cfg in C2 C3; do echo -n "cta_warps=$cw "; SS_ATTN_CTA_WARPS=$cw python tools/kbench.py attn --cfg $cfg; done; done
} > gpurun_out/attn_ctaw.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k attention > gpurun_out/attn_parity_y.log 2>&1
for cw in 6 1; do
SS_ATTN_CTA_WARPS=$cw timeout 900 python bench.py --no-cpu-baseline --timeline gpurun_out/timeline_y$cw.json > gpurun_out/bench_c2_y$cw.json 2> gpurun_out/bench_c2_y$cw.err
done
