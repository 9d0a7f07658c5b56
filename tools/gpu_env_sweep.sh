#!/bin/bash
# env-knob sweep of the 32K auto layer: SA_VS_MIN_TILES / SA_OVERLAP_EST
B="python bench.py --no-cpu-baseline --no-e2e --no-est --no-ttft --no-128k"
for rep in 1 2; do
for E in "SA_VS_MIN_TILES=1" "SA_VS_MIN_TILES=2" "SA_VS_MIN_TILES=4" "SA_VS_MIN_TILES=8" "SA_VS_MIN_TILES=16" "SA_OVERLAP_EST=0"; do
  env $E timeout 300 $B 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('$E', j['ms_per_step'], j['stage_ms'])"
done
done
