#!/bin/bash
# A/B of select / attention variants (env switches) at C2 and C3
for p in 1 0; do for pf in 1 0; do
  SS_SEL_PERSIST=$p SS_SEL_L2PF=$pf python tools/kbench.py select | sed "s/}/, \"persist\": $p, \"l2pf\": $pf}/"
  SS_SEL_PERSIST=$p SS_SEL_L2PF=$pf python tools/kbench.py select --cfg C3 | sed "s/}/, \"persist\": $p, \"l2pf\": $pf}/"
done; done
for pf in 1 0; do
  SS_ATTN_L2PF=$pf python tools/kbench.py attn | sed "s/}/, \"l2pf\": $pf}/"
  SS_ATTN_L2PF=$pf python tools/kbench.py attn --cfg C3 | sed "s/}/, \"l2pf\": $pf}/"
done
