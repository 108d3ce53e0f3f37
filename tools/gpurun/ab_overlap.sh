#!/bin/bash
for ctas in 148 64 32 16 8; do
  for p in 1 0; do
    echo -n "ctas=$ctas persist=$p "; SS_H2D_CTAS=$ctas SS_SEL_PERSIST=$p python tools/kbench.py overlap
  done
done
