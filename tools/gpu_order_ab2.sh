#!/bin/bash
# work order for uniform (fixed-pattern / dense) layers: LPT vs kv-group-major at 32K / 64K
for C in "--ctx 32768 --mode dense" "--ctx 32768 --pattern vs:1638:1638" "--ctx 65536 --mode dense" "--ctx 65536 --pattern vs:3277:3277" "--ctx 65536 --pattern tri:6554:0" "--ctx 131072 --pattern tri:13107:0"; do
for O in 1 0; do
  SA_ATTN_ORDER=$O timeout 300 python bench.py $C --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-128k --no-est --no-ttft 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);r=j['roofline'];print('order=$O $C', 'layer', j['value'], 'attn', r['attn_ms'], 'PF/s', round(r['achieved']/1000,3), 'tiles', r['exec_tiles'], j['clocks']['sm_mhz'])"
done
done
