#!/bin/bash
# Session 3: full GPU suite with the final defaults
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/s3r_gpu_tests.log 2>&1
