#!/bin/bash
# Env-variable A/B: bench lines (32K auto x2, 128K auto) for each setting in VARIANTS (";"-separated)
set -u
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for rep in 1 2; do
  for V in "${VS[@]}"; do
    env $V timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('[$V] 32k',j['stage_ms']['attention'],j['stage_ms']['tile_lists'],j['ms_per_step'])"
  done
done
for V in "${VS[@]}"; do
  env $V timeout 300 python bench.py --ctx 131072 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('[$V] 128k',j['stage_ms']['attention'],j['stage_ms']['tile_lists'],j['ms_per_step'])"
done
