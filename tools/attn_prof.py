#!/usr/bin/env python
"""Phase-cycle profile of attn_fwd_kernel (SA_ATTN_PROF build, `make prof`).

Runs the bench workload (32 q / 8 kv heads, d=128, auto mode) once with the
profiling library and prints the average cycles per 64-key sub-tile that each
warp role spends in each phase.  Tool only; numbers are not bench values.

  SA_B200_LIB=paper_2412_06198_b200/_sa_b200_prof.so python tools/attn_prof.py [--ctx 32768]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_06198_b200 import _lib, runtime as R  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, default=32768)
ap.add_argument("--mode", default="auto")
ap.add_argument("--pattern", default=None, help="fixed pattern for all heads, e.g. block:8:1")
args = ap.parse_args()
n = args.ctx
q, k, v = bench.synth_inputs(0, n)
dev = torch.device("cuda")
qd, kd, vd = (torch.from_numpy(np.ascontiguousarray(x)).bfloat16().to(dev) for x in (q, k, v))
fixed = None
mode = args.mode
if args.pattern:
    from paper_2412_06198_b200.patterns import BlockSparse, Triangular, VerticalSlash

    fam, p1, p2 = args.pattern.split(":")
    fixed = {"tri": Triangular, "vs": VerticalSlash, "block": BlockSparse}[fam](int(p1), int(p2))
    mode = "fixed"
plan = R.PrefillPlan(1, bench.H, bench.HK, n, bench.D, mode, fixed_pattern=fixed)
ws = R._workspace(plan.ws_bytes, dev)
out = torch.empty((1, n, bench.H * bench.D), dtype=torch.bfloat16, device=dev)
lib = _lib.load()
cnt = torch.zeros(48, dtype=torch.int64, device=dev)
for it in range(3):
    if it == 2:
        torch.cuda.synchronize()
        lib.sa_attn_profile_counters(ctypes.c_void_p(cnt.data_ptr()))
    if plan.mode == "auto":
        plan.select(qd, kd, ws)
    plan.run(qd, kd, vd, out, ws)
torch.cuda.synchronize()
lib.sa_attn_profile_counters(ctypes.c_void_p(0))
c = cnt.cpu().numpy().astype(np.float64)
names = {
    0: ("softmax", ["tile-head (mask make/fetch)", "-", "wait S", "tmem ld", "mask+max", "rescale",
                    "exp/sum/pack", "st P + arrive", "epilogue wait O", "epilogue store",
                    "CTA prologue", "CTA lifetime"]),
    16: ("mma", ["-", "wait K (QK)", "issue QK", "-", "wait P", "wait V", "issue PV"]),
    32: ("producer", ["-", "wait empty", "issue TMA"]),
}
for base, (role, ph) in names.items():
    nsub = c[base + 15]
    print(f"{role}: {int(nsub)} sub-tiles (x warps for softmax)")
    for i, nm in enumerate(ph):
        if nm == "-":
            continue
        print(f"   {nm:28s} {c[base + i] / max(nsub, 1):9.1f} cyc/sub-tile")
ctas = c[12] / 4
kern_cyc = c[11] / 4
print(f"CTAs {ctas:.0f}; mean CTA lifetime {kern_cyc / ctas:.0f} cyc, prologue {c[10] / 4 / ctas:.0f} cyc; "
      f"sum of lifetimes / 296 slots = {kern_cyc / 296:.0f} cyc")
