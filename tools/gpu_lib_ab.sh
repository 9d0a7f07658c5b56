#!/bin/bash
# same-box A/B of two builds of the library: $1 = alternative .so (SA_B200_LIB)
for rep in 1 2; do
for LIB in "" "$1"; do
for M in "--mode dense" "--mode auto" "--pattern vs:1638:1638"; do
  SA_B200_LIB=$LIB timeout 300 python bench.py $M --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-128k --no-est --no-ttft 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);r=j['roofline'];print('lib=${LIB:-default} $M', j['value'], r['attn_ms'], round(r['achieved']/1000,3))"
done
done
done
