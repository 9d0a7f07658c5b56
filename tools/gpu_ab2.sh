#!/bin/bash
# A/B of the current tree against scratch/<variant> builds: 32K auto, all-VS, block:8:1 attention ms
set -u
for rep in 1 2; do
  for v in ${VARIANTS:-.}; do
    (cd $v && timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('$v auto',j['stage_ms']['attention'],j['ms_per_step'])")
    (cd $v && timeout 200 python bench.py --pattern block:8:1 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('$v block81',j['stage_ms']['attention'])")
    (cd $v && timeout 200 python bench.py --pattern vs:1536:1536 --steps 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('$v vs',j['stage_ms']['attention'])")
  done
done
