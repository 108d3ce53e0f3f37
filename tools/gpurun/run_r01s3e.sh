#!/bin/bash
# Session 3: full GPU suite, bench lines with the FlashH2D server, the HBM-filling
# cache and the server-only timing pass; C3; attention alone at C2/C3.
mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/s3e_mem.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3e_gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/s3e_c2.json 2> gpurun_out/s3e_c2.err
timeout 900 python bench.py --config C3 > gpurun_out/s3e_c3.json 2> gpurun_out/s3e_c3.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s3e_ref.json 2> gpurun_out/s3e_ref.err
{ for cfg in C2 C3; do python tools/kbench.py attn --cfg $cfg; python tools/kbench.py select --cfg $cfg; done; } > gpurun_out/s3e_kbench.txt 2>&1
