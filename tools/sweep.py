#!/usr/bin/env python
"""BASELINE.json configs 3-5 on one GPU:

  C3  128K single layer, per-pattern kernel sweep (fixed Triangular /
      Interval-Slash / Block-Cluster at density 0.1, bench.py:127-138 of the
      reference, plus the auto plan)
  C4  TTFT of a 32-layer Llama-3-8B-shape sparse prefill at 64K: every layer
      has its own synthetic q/k/v (device RNG seeded by (seed, ctx, layer)),
      the layers run back to back on one stream, TTFT = wall of all layers on
      CUDA events (projections excluded, as in the reference runtime.py:1-10)
  C5  context sweep 16K -> 128K: auto ms/layer against dense causal flash
      attention (torch SDPA on the same bf16 tensors, the best installed dense
      kernel on this image) and the TTFT growth gradient (least-squares slope
      of ms vs ctx over the top half of the sweep, reference bench.py:336-378)

Prints one JSON object; `--out` also writes it.  Inputs are uniform [-1, 1]
bf16 generated on the device (not bit-identical to bench.py's host RNG).

  python tools/sweep.py [--ctx 16384,32768,65536,131072] [--ttft-ctx 65536] [--layers 32]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_06198_b200 import runtime as R  # noqa: E402
from paper_2412_06198_b200.patterns import BlockSparse, Triangular, VerticalSlash  # noqa: E402

H, HK, D = 32, 8, 128


def synth(seed: int, ctx: int, layer: int, dev):
    g = torch.Generator(device=dev)
    g.manual_seed(hash((seed, ctx, layer)) & 0x7FFFFFFF)
    mk = lambda heads: (torch.rand((heads, ctx, D), generator=g, device=dev) * 2 - 1).bfloat16()  # noqa: E731
    return mk(H), mk(HK), mk(HK)


def fixed_for(name: str, n: int):
    """fixed_pattern_for at density 0.1 (reference bench.py:127-138, half-even round)."""
    if name == "triangular":
        return Triangular(max(1, round(0.1 * n)), 0)
    if name == "vertical-slash":
        k = max(1, round(0.05 * n))
        return VerticalSlash(k, k)
    b = max(1, min(64, n // 8))
    nb = -(-n // b)
    return BlockSparse(b, max(1, round(0.1 * nb)))


class Layer:
    def __init__(self, n, mode, fixed=None, dev="cuda"):
        self.plan = R.PrefillPlan(1, H, HK, n, D, mode, fixed_pattern=fixed)
        self.ws = R._workspace(self.plan.ws_bytes, dev)
        self.out = torch.empty((1, n, H * D), dtype=torch.bfloat16, device=dev)

    def __call__(self, q, k, v):
        if self.plan.mode == "auto":
            self.plan.select(q, k, self.ws)
        self.plan.run(q, k, v, self.out, self.ws)


def time_ms(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def dense_ms(q, k, v, reps=3):
    qt, kt, vt = q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0)
    f = lambda: torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=True, enable_gqa=True)  # noqa: E731
    return time_ms(f, reps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", default="16384,32768,65536,131072")
    ap.add_argument("--ttft-ctx", type=int, default=65536)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--skip-c3", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda")
    res = {"data": "synthetic uniform [-1,1] bf16, device RNG per (seed, ctx, layer)", "heads": H, "kv_heads": HK,
           "head_dim": D, "gpu": torch.cuda.get_device_name()}

    # C5: context sweep, auto vs dense flash
    sweep = []
    for n in [int(x) for x in args.ctx.split(",")]:
        q, k, v = synth(args.seed, n, 0, dev)
        lay = Layer(n, "auto")
        ms = time_ms(lambda: lay(q, k, v))
        dn = dense_ms(q, k, v)
        fams = [type(hp.pattern).__name__ for hp in lay.plan.plans(lay.ws, with_search=False)[0]]
        sweep.append({"ctx": n, "auto_ms": round(ms, 3), "dense_sdpa_ms": round(dn, 3),
                      "speedup_vs_dense": round(dn / ms, 2),
                      "families": {f: fams.count(f) for f in sorted(set(fams))}})
        del lay, q, k, v
        torch.cuda.empty_cache()
        print(json.dumps(sweep[-1]), file=sys.stderr, flush=True)
    top = sweep[len(sweep) // 2:]
    if len(top) >= 2:
        x = np.array([s["ctx"] for s in top], float)
        for key in ("auto_ms", "dense_sdpa_ms"):
            y = np.array([s[key] for s in top], float)
            res[f"gradient_{key}_per_1k_tokens"] = round(float(np.polyfit(x / 1024, y, 1)[0]), 4)
    res["c5_sweep"] = sweep

    # C3: per-pattern sweep at the largest context
    if not args.skip_c3:
        n = max(s["ctx"] for s in sweep)
        q, k, v = synth(args.seed, n, 0, dev)
        c3 = {}
        for name in ("triangular", "vertical-slash", "block-sparse"):
            p = fixed_for(name, n)
            lay = Layer(n, "fixed", p)
            c3[name] = {"pattern": repr(p), "ms": round(time_ms(lambda: lay(q, k, v), reps=2), 3)}
            del lay
            torch.cuda.empty_cache()
            print(name, c3[name], file=sys.stderr, flush=True)
        res["c3_per_pattern_ms"] = {"ctx": n, **c3}
        del q, k, v
        torch.cuda.empty_cache()

    # C4: TTFT of a multi-layer prefill, layers back to back
    n, L = args.ttft_ctx, args.layers
    layers_in = [synth(args.seed, n, l, dev) for l in range(L)]
    lay = Layer(n, "auto")
    lay(*layers_in[0])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for l in range(L):
        lay(*layers_in[l])
    e1.record()
    torch.cuda.synchronize()
    ttft = e0.elapsed_time(e1)
    qd = layers_in[0][0]
    dense_layer = dense_ms(*layers_in[0])
    res["c4_ttft"] = {"ctx": n, "layers": L, "ttft_ms": round(ttft, 2), "ms_per_layer": round(ttft / L, 3),
                      "dense_sdpa_ttft_ms_est": round(dense_layer * L, 2),
                      "note": "attention path only (no projections/MLP), one stream, 1 GPU"}
    del qd
    print(json.dumps(res))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
