#!/bin/bash
# A/B of build variants in scratch/<name> (bench attention stage ms, auto + all-VS).
set -u
ROOT=$(pwd)
for v in ${VARIANTS:-.}; do
  for rep in 1 2; do
    (cd $v && python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('$v auto',j['stage_ms']['attention'],j['roofline']['achieved'])")
  done
  (cd $v && python bench.py --pattern vs:1536:1536 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('$v vs',j['stage_ms']['attention'],j['roofline']['achieved'])")
done
