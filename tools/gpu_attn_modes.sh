#!/bin/bash
# attention kernel throughput per family at 32K (fixed modes) + the auto layer
for M in "--mode dense" "--pattern vs:1638:1638" "--pattern tri:3277:0" "--pattern block:8:1" "--pattern block:64:51" "--mode auto"; do
  timeout 300 python bench.py $M --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-128k --no-est --no-ttft 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);r=j['roofline'];print('$M', 'layer', j['value'], 'attn', r['attn_ms'], 'PF/s', round(r['achieved']/1000,3), 'tiles', r['exec_tiles'])"
done
