#!/bin/bash
# headline layer time with the finiteness scan / cache fill variants
for ENV in "SA_CHECK_MODE=3" "SA_CHECK_MODE=2" "SA_CHECK_MODE=1" "SA_CHECK_MODE=0" "SA_SCAN_BLOCKS=32" "SA_SCAN_BLOCKS=74" "SA_SCAN_BLOCKS=148" "SA_SCAN_BLOCKS=592"; do
  env $ENV timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-128k --no-est 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('$ENV', j['value'])"
done
