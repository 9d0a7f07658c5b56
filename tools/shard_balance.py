#!/usr/bin/env python
"""Imbalance-limited multi-GPU speedup of the 32K auto layer,
from the executed attention tiles per (head, query tile) of the real device
plan: GQA-group sharding (what bench.py --gpus N runs), per-head LPT, and
(head, query-tile range) LPT units.  Tool only (1 GPU available)."""
import heapq
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_06198_b200 import runtime as R  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q, k, v = bench.synth_inputs(0, n)
dev = torch.device("cuda")
qd, kd, vd = (torch.from_numpy(np.ascontiguousarray(x)).bfloat16().to(dev) for x in (q, k, v))
plan = R.PrefillPlan(1, bench.H, bench.HK, n, bench.D, "auto")
ws = R._workspace(plan.ws_bytes, dev)
out = torch.empty((1, n, bench.H * bench.D), dtype=torch.bfloat16, device=dev)
plan.select(qd, kd, ws)
plan.run(qd, kd, vd, out, ws)
torch.cuda.synchronize()
view = plan.views(ws)
cnt = R._wrap(view.tile_cnt, plan.hh * view.nqt, torch.int32).cpu().numpy().reshape(plan.hh, view.nqt)
per_head = cnt.sum(1).astype(float)
g = bench.H // bench.HK
total = per_head.sum()


def lpt(costs, bins):
    h = [(0.0, i) for i in range(bins)]
    for c in sorted(costs, reverse=True):
        load, i = heapq.heappop(h)
        heapq.heappush(h, (load + c, i))
    return max(x for x, _ in h)


res = {"n": n, "tiles_total": int(total), "tiles_per_head": per_head.astype(int).tolist()}
for N in (2, 4, 8):
    groups = per_head.reshape(bench.HK, g).sum(1)
    group_max = max(groups.reshape(N, -1).sum(1))  # contiguous kv groups per rank
    units = [c for row in cnt for c in np.add.reduceat(row, np.arange(0, view.nqt, 8))]
    res[f"N{N}"] = {"gqa_groups": round(total / group_max, 2), "head_lpt": round(total / lpt(per_head, N), 2),
                    "qtile_range_lpt": round(total / lpt(units, N), 2)}
print(json.dumps(res))
