#!/usr/bin/env python
"""Where the host-streamed prefill's time goes: pure H2D / D2H copy bandwidth of
the same bytes, then the streamed prefill wall time (tool only)."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_06198_b200 import runtime as R  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, default=131072)
args = ap.parse_args()
n, H, HK, D = args.ctx, 32, 8, 128
g = torch.Generator().manual_seed(0)
q = (torch.rand((1, H, n, D), generator=g) * 2 - 1).bfloat16().pin_memory()
k = (torch.rand((1, HK, n, D), generator=g) * 2 - 1).bfloat16().pin_memory()
v = (torch.rand((1, HK, n, D), generator=g) * 2 - 1).bfloat16().pin_memory()
out_h = torch.empty((1, n, H * D), dtype=torch.bfloat16).pin_memory()
qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
od = torch.empty((1, n, H * D), dtype=torch.bfloat16, device="cuda")
torch.cuda.synchronize()


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3 / reps


h2d = wall(lambda: (qd.copy_(q, non_blocking=True), kd.copy_(k, non_blocking=True), vd.copy_(v, non_blocking=True)))
d2h = wall(lambda: out_h.copy_(od, non_blocking=True))
s2 = torch.cuda.Stream()


def both():
    with torch.cuda.stream(s2):
        out_h.copy_(od, non_blocking=True)
    qd.copy_(q, non_blocking=True)
    kd.copy_(k, non_blocking=True)
    vd.copy_(v, non_blocking=True)


duplex = wall(both)
nb_in = (q.numel() + k.numel() + v.numel()) * 2
nb_out = out_h.numel() * 2
print(f"H2D {nb_in / 1e6:.0f} MB: {h2d:.2f} ms = {nb_in / h2d / 1e6:.1f} GB/s")
print(f"D2H {nb_out / 1e6:.0f} MB: {d2h:.2f} ms = {nb_out / d2h / 1e6:.1f} GB/s")
print(f"H2D || D2H: {duplex:.2f} ms")
cfg = R.ModelConfig(n_heads=H, d_model=H * D, d_head=D, max_context=n)
e2e = wall(lambda: R.prefill(q, k, v, cfg, mode="auto"))
plan = R.PrefillPlan(1, H, HK, n, D, "auto")
ws = R._workspace(plan.ws_bytes, torch.device("cuda"))
dev = wall(lambda: (plan.select(qd, kd, ws), plan.run(qd, kd, vd, od, ws)))
print(f"device-resident layer {dev:.2f} ms; streamed prefill e2e {e2e:.2f} ms; "
      f"ideal ~ max(H2D, D2H) + last group compute + last group D2H")
R._TIMELINE = []
R.prefill(q, k, v, cfg, mode="auto")
print("per group (ms from start): h2d_done, compute_start, compute_end, d2h_done")
for i, row in enumerate(R._TIMELINE[-1]):
    print(i, " ".join(f"{x:7.2f}" for x in row))
