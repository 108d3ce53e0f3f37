#!/bin/bash
# Session 3: run-to-run spread of the default C2 line and scheduling knobs
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline"
for i in 1 2; do timeout 600 $B > gpurun_out/s3h_def$i.json 2> gpurun_out/s3h_def$i.err; done
for i in 1 2; do timeout 600 $B --groups 4 > gpurun_out/s3h_g4_$i.json 2> gpurun_out/s3h_g4_$i.err; done
timeout 600 $B --cache-per-group > gpurun_out/s3h_cpg.json 2> gpurun_out/s3h_cpg.err
timeout 600 $B --select-priority > gpurun_out/s3h_selprio.json 2> gpurun_out/s3h_selprio.err
timeout 600 $B --groups 4 --cache-per-group > gpurun_out/s3h_g4_cpg.json 2> gpurun_out/s3h_g4_cpg.err
