#!/bin/bash
set -u
export SA_B200_LIB=paper_2412_06198_b200/_sa_b200_prof.so
for P in "--pattern block:8:1" "--pattern block:64:51"; do
  echo "=== $P"
  timeout 200 python tools/attn_prof.py $P 2>&1 | tail -30
done
for P in "block:8:1" "block:64:51"; do
  timeout 200 python bench.py --pattern $P --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('$P',j['stage_ms']['attention'],j['roofline']['achieved'],j['roofline']['exec_tiles'])"
done
