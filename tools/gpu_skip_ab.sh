#!/bin/bash
# attention with / without the dead-warp softmax skip, per family (32K) + Block(64,205) at 128K
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py -x -q -m gpu 2>&1 | tail -2
for SK in 0 1; do
for M in "--pattern block:8:1" "--pattern block:64:51" "--mode auto" "--pattern tri:3277:0" "--ctx 131072 --pattern block:64:205"; do
  SA_ATTN_SKIP=$SK timeout 300 python bench.py $M --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-128k --no-est --no-ttft 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);r=j['roofline'];print('skip=$SK $M', 'layer', j['value'], 'attn', r['attn_ms'], 'PF/s', round(r['achieved']/1000,3), 'tiles', r['exec_tiles'])"
done
done
