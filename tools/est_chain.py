import sys; sys.path.insert(0, '.')
import torch, bench
r = bench.estimator_roofline(int(sys.argv[1]) if len(sys.argv) > 1 else 131072, torch.device('cuda'), reps=2)
print(r['topk_us'])
