#!/bin/bash
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py -x -q -m gpu 2>&1 | tail -2
for M in "--ctx 131072 --pattern block:64:205" "--pattern block:64:51" "--pattern block:8:1" "--mode auto"; do
  timeout 300 python bench.py $M --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-128k --no-est --no-ttft 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);r=j['roofline'];print('$M', 'layer', j['value'], 'attn', r['attn_ms'], 'PF/s', round(r['achieved']/1000,3), 'tiles', r['exec_tiles'])"
done
