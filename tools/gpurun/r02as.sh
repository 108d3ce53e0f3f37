#!/bin/bash
# Round 2: attention stages per warp (NS x NW = 2x6, 3x4, 4x3) with the bulk-load merge; bench.py link-peak check
mkdir -p gpurun_out/r02as
{
for rep in 1 2; do for ns in 2 3 4; do for c in "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C3" "--cfg C3 --batch 1" "--cfg C2"; do
  echo "stages=$ns $c $(SS_LIB_VARIANT=debug SS_ATTN_STAGES=$ns timeout 300 python tools/kbench.py attn $c)"
done; done; done
} > gpurun_out/r02as/attn_stages.txt 2>&1
timeout 900 python bench.py --config C3 --no-cpu-baseline > gpurun_out/r02as/bench_c3.json 2> gpurun_out/r02as/bench_c3.err
