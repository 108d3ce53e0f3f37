#!/bin/bash
# bench.py (groups=2) across FlashH2D grid shapes; one compact line per run
for cfg in "8 8" "16 8" "32 8" "64 8" "16 16" "32 16"; do
  set -- $cfg
  SS_H2D_CTAS=$1 SS_H2D_UNROLL=$2 python bench.py --steps 20 --warmup 5 --groups 2 --no-cpu-baseline > /tmp/b.json 2>&1
  python - "$1" "$2" << 'PY'
import json, sys
d = json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
k = d['kernels']
print(f"ctas={sys.argv[1]} unroll={sys.argv[2]} value={d['value']} ms={d['ms_per_step']} hit={d['hit_rate']} "
      f"gather_ms={k['flash_h2d_gather']['ms_per_step']} sel_ms={k['ss_block_select']['ms_per_step']} "
      f"attn_ms={k['sparse_decode_attn']['ms_per_step']} cache_ms={k['kv_cache_lookup_insert']['ms_per_step']}")
PY
done
