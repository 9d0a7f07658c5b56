#!/bin/bash
# attention work order at 128K: LPT (default) vs kv-group-major (SA_ATTN_ORDER=0)
for M in "--pattern block:64:205" "--mode auto" "--pattern vs:6554:6554" "--mode dense" "--pattern block:8:1"; do
for O in 1 0; do
  SA_ATTN_ORDER=$O timeout 300 python bench.py --ctx 131072 $M --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-128k --no-est --no-ttft 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);r=j['roofline'];print('order=$O $M', 'layer', j['value'], 'attn', r['attn_ms'], 'PF/s', round(r['achieved']/1000,3), 'tiles', r['exec_tiles'])"
done
done
