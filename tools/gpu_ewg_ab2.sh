#!/bin/bash
set -u
B="python bench.py --no-cpu-baseline --no-e2e --no-est --no-ttft --no-128k"
for rep in 1 2; do
for E in 1 0; do
  for P in "" "--pattern block:8:1" "--pattern vs:1536:1536"; do
    SA_ATTN_EWG=$E timeout 300 $B $P 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('ewg=$E $P', j['ms_per_step'], j['stage_ms']['attention'])"
  done
done
done
