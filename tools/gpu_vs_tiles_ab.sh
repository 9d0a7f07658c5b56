#!/bin/bash
# VS estimator: fewest key tiles per CTA (SA_VS_MIN_TILES) — auto layer and all-VS chains
SA_VS_MIN_TILES=16 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "tail or estimator or vs" 2>&1 | tail -2
for T in 1 8 16 32 1 16; do
  L=$(SA_VS_MIN_TILES=$T timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-128k --no-est --no-ttft 2>/dev/null | python -c "import json,sys;j=json.load(sys.stdin);print(j['value'], j['stage_ms'])")
  E=$(SA_VS_MIN_TILES=$T timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import torch, bench
for n in (32768, 131072):
    r = bench.estimator_roofline(n, torch.device('cuda'), reps=3)
    print(n, r['estimator_us'], r['topk_us'], r['chain_us'], end='; ')
" 2>/dev/null)
  echo "min_tiles=$T layer $L | allvs $E"
done
