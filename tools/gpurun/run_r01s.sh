#!/bin/bash
# C2 step structure: groups x FlashH2D CTAs, and the step without the gather (HBM chain only)
mkdir -p gpurun_out
run() { # label, env..., args
  local label=$1; shift
  env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $BARGS > /tmp/b.json 2>/tmp/b.err
  python - "$label" <<'PY'
import json, sys
try:
    d = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "FAILED", open('/tmp/b.err').read()[-400:]); sys.exit()
k = d['kernels']
print(f"{sys.argv[1]:28s} tok/s={d['value']:8.1f} ms={d['ms_per_step']:7.3f} hit={d['hit_rate']} e2e={d['e2e']['value']} "
      f"h2d_over_step={d['flash_h2d']['h2d_gbs_over_step']} gather={k['flash_h2d_gather']['achieved']} "
      f"sel_us={k['ss_block_select']['us_per_launch']} attn_us={k['sparse_decode_attn']['us_per_launch']} cache_us={k['kv_cache_lookup_insert']['us_per_launch']}")
PY
}
{
BARGS="--groups 2" run g2 X=1
BARGS="--groups 2" run g2_skipgather SS_H2D_SKIP=1
BARGS="--groups 3" run g3 X=1
BARGS="--groups 4" run g4 X=1
BARGS="--groups 2" run g2_ctas24 SS_H2D_CTAS=24
BARGS="--groups 2" run g2_ctas32 SS_H2D_CTAS=32
BARGS="--groups 3" run g3_ctas24 SS_H2D_CTAS=24
BARGS="--groups 1" run g1 X=1
} > gpurun_out/sweep_s.txt 2>&1
