#!/bin/bash
# all-VS estimator chain (estimator + top-k) with the top-k variants
for ENV in "SA_TOPK_CLUSTER=1" "SA_TOPK_CLUSTER=0"; do
  env $ENV timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import torch, bench
for n in (32768, 131072):
    r = bench.estimator_roofline(n, torch.device('cuda'))
    print('$ENV', n, 'est', r['estimator_us'], 'topk', r['topk_us'], 'chain', r['chain_us'])
"
done
