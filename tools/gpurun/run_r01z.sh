#!/bin/bash
# C2 stream scheduling variants (3 request groups)
mkdir -p gpurun_out
run() {
  local label=$1; shift
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" > /tmp/b.json 2>/tmp/b.err
  python - "$label" <<'PY'
import json, sys
try:
    d = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "FAILED", open('/tmp/b.err').read()[-600:]); sys.exit()
k = d['kernels']
print(f"{sys.argv[1]:16s} tok/s={d['value']:8.1f} ms={d['ms_per_step']:7.3f} e2e={d['e2e']['value']} "
      f"h2d_over_step={d['flash_h2d']['h2d_gbs_over_step']} gather={k['flash_h2d_gather']['achieved']} "
      f"sel_us={k['ss_block_select']['us_per_launch']} attn_us={k['sparse_decode_attn']['us_per_launch']} cache_us={k['kv_cache_lookup_insert']['us_per_launch']} gather_us={k['flash_h2d_gather']['us_per_launch']}")
PY
}
{
run base
run selprio --select-priority
run cachepg --cache-per-group
run both --select-priority --cache-per-group
run base2
run both2 --select-priority --cache-per-group
run both_g4 --select-priority --cache-per-group --groups 4
} > gpurun_out/sweep_z.txt 2>&1
