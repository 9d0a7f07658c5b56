#!/bin/bash
# two softmax threads per row (SA_ATTN_SPLIT=1) vs one
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py -x -q -m gpu 2>&1 | tail -2
for M in "--mode dense" "--pattern vs:1638:1638" "--mode auto" "--pattern block:8:1" "--pattern tri:3277:0"; do
for SP in 0 1; do
  SA_ATTN_SPLIT=$SP timeout 300 python bench.py $M --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-128k --no-est --no-ttft 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);r=j['roofline'];print('split=$SP $M', 'layer', j['value'], 'attn', r['attn_ms'], 'PF/s', round(r['achieved']/1000,3))"
done
done
