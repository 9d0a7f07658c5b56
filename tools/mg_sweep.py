#!/usr/bin/env python
"""Randomised sweep of the balanced head-parallel layer (tool): every rank of
a random world (2-8) played in turn on one GPU with the all-gathers emulated
by stacking (as tests/test_gpu_multigpu_sim.py); the assembled output must
equal the single-GPU layer bit for bit and the deal must partition the items.

  python tools/mg_sweep.py [--cases 30] [--seed 0] [--max-n 8192]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_06198_b200 import runtime as R  # noqa: E402
from paper_2412_06198_b200.multigpu import BalancedLayer  # noqa: E402
from paper_2412_06198_b200.patterns import BlockSparse, Triangular, VerticalSlash  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=30)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--max-n", type=int, default=8192)
args = ap.parse_args()
rng = np.random.default_rng(args.seed)
D = 128
fails = 0
t0 = time.time()
for c in range(args.cases):
    HK = int(rng.choice([2, 4, 8]))
    g = int(rng.choice([1, 2, 4]))
    H = HK * g
    world = int(rng.choice([w for w in (2, 4, 8) if HK % w == 0]))
    n = int(rng.integers(1, args.max_n + 1))
    mode = str(rng.choice(["auto", "auto", "fixed", "dense"]))
    fixed = None
    if mode == "fixed":
        fam = int(rng.integers(3))
        fixed = (Triangular(int(rng.integers(1, n + 1)), int(rng.integers(0, 64))) if fam == 0 else
                 VerticalSlash(int(rng.integers(1, n + 1)), int(rng.integers(1, n + 1))) if fam == 1 else
                 BlockSparse(min(int(rng.choice([8, 16, 64])), n), 1))
    rec = {"case": c, "H": H, "HK": HK, "world": world, "n": n, "mode": mode,
           "fixed": None if fixed is None else [type(fixed).__name__, *fixed.__dict__.values()]}
    try:
        gen = torch.Generator(device="cuda")
        gen.manual_seed(int(rng.integers(1 << 30)))
        q, k, v = ((torch.rand((h, n, D), generator=gen, device="cuda") * 2 - 1).bfloat16() for h in (H, HK, HK))
        plan = R.PrefillPlan(1, H, HK, n, D, mode, fixed_pattern=fixed)
        ws = R._workspace(plan.ws_bytes, q.device)
        want = torch.empty((1, n, H * D), dtype=torch.bfloat16, device="cuda")
        if mode == "auto":
            plan.select(q, k, ws)
        plan.run(q, k, v, want, ws)
        ranks = [BalancedLayer(r, world, H, HK, n, D, mode, fixed_pattern=fixed) for r in range(world)]
        packed = torch.stack([rk.estimate(q, k, v) for rk in ranks])
        for rk in ranks:
            rk.load_index(packed)
        blocks = torch.stack([rk.attend(q, k, v) for rk in ranks])
        got = ranks[0].assemble(blocks)
        torch.cuda.synchronize()
        items = torch.cat(ranks[0].owner_items).cpu().numpy()
        rec["partition"] = bool(np.array_equal(np.sort(items), np.arange(H * ranks[0].nqt)))
        rec["equal"] = bool(torch.equal(got, want[0]))
        rec["ok"] = rec["partition"] and rec["equal"]
    except Exception as e:  # noqa: BLE001
        rec.update(ok=False, error=f"{type(e).__name__}: {e}"[:300])
    fails += not rec["ok"]
    print(json.dumps(rec), flush=True)
print(json.dumps({"cases": args.cases, "failures": fails, "seconds": round(time.time() - t0, 1)}))
