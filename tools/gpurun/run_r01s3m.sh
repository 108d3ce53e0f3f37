#!/bin/bash
# Session 3: in-step scheduling knobs re-measured with per-step medians
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline"
timeout 600 $B > gpurun_out/s3m_def.json 2> gpurun_out/s3m_def.err
for i in 1 2; do SS_SEL_CHUNK=2048 timeout 600 $B > gpurun_out/s3m_ch2048_$i.json 2> gpurun_out/s3m_ch2048_$i.err; done
SS_ATTN_CTA_WARPS=1 timeout 600 $B > gpurun_out/s3m_attn1w.json 2> gpurun_out/s3m_attn1w.err
timeout 600 $B --groups 4 > gpurun_out/s3m_g4.json 2> gpurun_out/s3m_g4.err
timeout 600 $B --groups 2 > gpurun_out/s3m_g2.json 2> gpurun_out/s3m_g2.err
SS_SEL_CHUNK=512 timeout 600 $B > gpurun_out/s3m_ch512.json 2> gpurun_out/s3m_ch512.err
