#!/bin/bash
# A/B (experiment): attention epilogue cost — SA_ATTN_EPI 1 (full) / 0 (no stores) / 2 (no O read).
set -u
OUT=gpurun_out/${1:-epi}
mkdir -p $OUT
B="python bench.py --no-cpu-baseline --no-e2e --no-128k --no-est --no-ttft"
for rep in 1 2; do
for E in 1 0 2; do
  for P in "" "--pattern block:8:1" "--pattern vs:1536:1536"; do
    SA_ATTN_EPI=$E timeout 200 $B $P 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('epi=$E $P', j['stage_ms']['attention'], j['ms_per_step'])"
  done
done
done
