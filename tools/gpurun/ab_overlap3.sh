#!/bin/bash
export KB_HOST_GIB=16
for cfg in "8 128 8" "16 128 8" "16 256 8" "16 512 8" "32 256 8" "148 128 8" "8 512 16" "16 256 16"; do
  set -- $cfg
  echo -n "ctas=$1 threads=$2 unroll=$3 "; SS_H2D_CTAS=$1 SS_H2D_THREADS=$2 SS_H2D_UNROLL=$3 python tools/kbench.py overlap
done
