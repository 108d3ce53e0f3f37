#!/bin/bash
# request groups x FlashH2D streams (C2)
mkdir -p gpurun_out
run() {
  local label=$1; shift
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" > /tmp/b.json 2>/tmp/b.err
  python - "$label" <<'PY'
import json, sys
try:
    d = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "FAILED", open('/tmp/b.err').read()[-400:]); sys.exit()
k = d['kernels']
print(f"{sys.argv[1]:16s} tok/s={d['value']:8.1f} ms={d['ms_per_step']:7.3f} e2e={d['e2e']['value']} "
      f"h2d_over_step={d['flash_h2d']['h2d_gbs_over_step']} gather={k['flash_h2d_gather']['achieved']} "
      f"sel_us={k['ss_block_select']['us_per_launch']} attn_us={k['sparse_decode_attn']['us_per_launch']} cache_us={k['kv_cache_lookup_insert']['us_per_launch']} gather_us={k['flash_h2d_gather']['us_per_launch']}")
PY
}
{
run g3s1 --groups 3 --h2d-streams 1
run g3s2 --groups 3 --h2d-streams 2
run g3s3 --groups 3 --h2d-streams 3
run g4s2 --groups 4 --h2d-streams 2
run g2s2 --groups 2 --h2d-streams 2
run g3s1b --groups 3 --h2d-streams 1
} > gpurun_out/sweep_w.txt 2>&1
