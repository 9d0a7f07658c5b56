#!/usr/bin/env python
"""Randomised decode sweep (tool): prefill (dense) a random prompt, then a few
decode_step calls; each decode output is checked against float64 attention of
the new query over every cached key (the cache holds what the reference
stores: the prompt's and the decoded tokens' k/v in the input dtype).

  python tools/decode_sweep.py [--cases 60] [--seed 0]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_06198_b200 as sa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=60)
ap.add_argument("--seed", type=int, default=0)
args = ap.parse_args()
rng = np.random.default_rng(args.seed)
LAYOUTS = [(1, 1), (4, 4), (8, 2), (8, 1), (6, 3), (32, 8)]
fails = 0
t0 = time.time()
for c in range(args.cases):
    H, HK = LAYOUTS[rng.integers(len(LAYOUTS))]
    B = int(rng.integers(1, 4))
    d = int(rng.choice([128, 64, 8, 5, 100]))
    n0 = int(rng.choice([1, 2, 255, 256, 257])) if rng.random() < 0.3 else int(rng.integers(1, 6000))
    steps = int(rng.integers(1, 4))
    dt = str(rng.choice(["float32", "bf16", "cpu_f32"]))
    rec = {"case": c, "B": B, "H": H, "HK": HK, "d": d, "n0": n0, "steps": steps, "dtype": dt}
    try:
        import torch

        tot = n0 + steps
        q = rng.uniform(-1, 1, (B, H, tot, d)).astype(np.float32)
        k = rng.uniform(-1, 1, (B, HK, tot, d)).astype(np.float32)
        v = rng.uniform(-1, 1, (B, HK, tot, d)).astype(np.float32)
        if dt == "bf16":  # bf16 tensors on the device: the cache keeps bf16
            conv = lambda x: torch.from_numpy(x).cuda().bfloat16()  # noqa: E731
            q, k, v = (torch.from_numpy(x).bfloat16().float().numpy() for x in (q, k, v))
        elif dt == "cpu_f32":  # CPU torch fp32: the host-streamed prefill (d = 128) fills the cache
            conv = lambda x: torch.from_numpy(np.ascontiguousarray(x))  # noqa: E731
        else:
            conv = lambda x: x  # noqa: E731
        cfg = sa.ModelConfig(n_heads=H, d_model=H * d, d_head=d, max_context=tot)
        res = sa.prefill(conv(q[:, :, :n0]), conv(k[:, :, :n0]), conv(v[:, :, :n0]), cfg, mode="dense")
        cache = res.cache
        errs = []
        for s in range(steps):
            t = n0 + s
            out = sa.decode_step(conv(q[:, :, t:t + 1]), conv(k[:, :, t:t + 1]), conv(v[:, :, t:t + 1]), cache, cfg)
            cache = out.cache
            o = out.output
            got = (o.float().cpu().numpy() if hasattr(o, "cpu") else np.asarray(o)).reshape(B, H, d)
            g = H // HK
            kk = np.repeat(k[:, :, : t + 1], g, axis=1).astype(np.float64)
            vv = np.repeat(v[:, :, : t + 1], g, axis=1).astype(np.float64)
            sc = np.einsum("bhd,bhnd->bhn", q[:, :, t].astype(np.float64), kk) / np.sqrt(d)
            w = np.exp(sc - sc.max(-1, keepdims=True))
            w /= w.sum(-1, keepdims=True)
            want = np.einsum("bhn,bhnd->bhd", w, vv)
            errs.append(float(np.abs(got - want).max()))
        rec.update(max_abs=max(errs), cache_len=int(cache.length))
        # fp32 caches: fp32 accumulation; bf16 inputs come back as bf16 (2^-9 relative rounding)
        tol = 4e-3 if dt == "bf16" else 1e-4
        rec["ok"] = bool(max(errs) <= tol and cache.length == n0 + steps)
    except Exception as e:  # noqa: BLE001
        rec.update(ok=False, error=f"{type(e).__name__}: {e}"[:300])
    fails += not rec["ok"]
    print(json.dumps(rec), flush=True)
print(json.dumps({"cases": args.cases, "failures": fails, "seconds": round(time.time() - t0, 1)}))
