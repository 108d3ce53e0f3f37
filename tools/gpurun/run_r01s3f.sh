#!/bin/bash
# Session 3: bench lines (C2 with the HBM-filling cache, 300 settle steps; C3).
mkdir -p gpurun_out
timeout 900 python bench.py --hit-trace > gpurun_out/s3f_c2.json 2> gpurun_out/s3f_c2.err
timeout 900 python bench.py --config C3 > gpurun_out/s3f_c3.json 2> gpurun_out/s3f_c3.err
timeout 900 python bench.py --slots 0 --settle 80 > gpurun_out/s3f_c2_slots128k.json 2> gpurun_out/s3f_c2_slots128k.err
