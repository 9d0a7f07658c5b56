#!/bin/bash
set -u
for rep in 1 2; do
  for P in 4 3 8 2; do
    SA_ATTN_POLY=$P timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('poly=$P auto',j['stage_ms']['attention'],j['ms_per_step'])"
    SA_ATTN_POLY=$P timeout 200 python bench.py --pattern vs:1536:1536 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('poly=$P vs',j['stage_ms']['attention'])"
  done
done
