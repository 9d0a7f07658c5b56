#!/bin/bash
# placement of the finiteness scan / cache fill in the headline layer
python -m pytest tests/test_gpu_api.py tests/test_gpu_layers.py tests/test_gpu_bench.py -x -q -m gpu 2>&1 | tail -2
for ENV in "SA_CHECK_MODE=3" "SA_SCAN_AT=2" "SA_SCAN_AT=2 SA_ATTN_PRIO=0" "SA_CHECK_MODE=3" "SA_SCAN_AT=2"; do
  env $ENV timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-128k --no-est --no-ttft 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print('$ENV', j['value'], j['roofline']['attn_ms'])"
done
