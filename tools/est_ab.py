#!/usr/bin/env python
"""A/B helper (tool only): the all-VS estimator chain of bench.estimator_roofline at the given n."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or [32768, 131072]:
    r = bench.estimator_roofline(n, torch.device("cuda"), reps=7)
    print(json.dumps({k: r[k] for k in ("n", "estimator_us", "topk_us", "chain_us")}))
