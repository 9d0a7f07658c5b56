#!/usr/bin/env python
"""Randomised parity sweep (tool, not a bench): random shapes, head layouts,
modes and fixed patterns through the public API (paper_2412_06198_b200.prefill)
against the oracle's prefill on identical bf16-rounded inputs.  Checks the
realised plans (family + parameters) and the outputs (max-abs <= 2e-2,
mean-abs <= 2e-3, the north-star tolerance); prints one JSON line per case
and a summary.

  python tools/parity_sweep.py [--cases 40] [--seed 0] [--max-n 6000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import sparse_oracle as O  # noqa: E402
import paper_2412_06198_b200 as sa  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=40)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--max-n", type=int, default=6000)
ap.add_argument("--only", type=int, nargs="*", default=None, help="run only these case numbers")
ap.add_argument("--api-mix", action="store_true",
                help="also randomise the batch (1-3) and the input kind (numpy / CPU torch, pinned or not / "
                     "CUDA torch bf16 or fp32): the host-streamed and device entry paths")
args = ap.parse_args()
rng = np.random.default_rng(args.seed)
LAYOUTS = [(4, 4), (8, 2), (8, 1), (6, 3), (2, 1), (16, 4)]
SPECIAL_N = [1, 2, 63, 64, 65, 127, 128, 129, 255, 257, 1023, 1025]


def rand_fixed(n):
    fam = rng.integers(3)
    if fam == 0:
        return O.Tri(int(rng.integers(1, n + 1)), int(rng.integers(0, min(n, 200) + 1)))
    if fam == 1:
        return O.VS(int(rng.integers(1, n + 1)), int(rng.integers(1, n + 1)))
    b = int(rng.choice([1, 3, 8, 16, 32, 64, 100]))
    b = min(b, n)
    nb = -(-n // b)
    return O.Blk(b, int(rng.integers(1, nb + 1)))


def to_sa(p):
    if p is None:
        return None
    return {O.Tri: sa.Triangular, O.VS: sa.VerticalSlash, O.Blk: sa.BlockSparse}[type(p)](*p.__dict__.values())


def conv(p):
    return None if p is None else (type(p).__name__[0], *[int(x) for x in p.__dict__.values()])


def diagnose(q, k, v, plans, got, d):
    """Per failing head: does the device realise a different index from its own
    fp32 scores (an estimator flip), and does the output then equal the
    oracle's attention over the DEVICE index (i.e. the kernels are right)?"""
    H, HK = q.shape[1], k.shape[1]
    out = []
    for h in range(H):
        qh, kh, vh = q[0, h], k[0, h // (H // HK)], v[0, h // (H // HK)]
        p = plans[h]
        want_idx = O.build_index(qh, kh, p, "estimated", 64) if p is not None else None
        y_want = (O.dense_attention(qh, kh, vh)[1] if p is None else O.sparse_attention(qh, kh, vh, want_idx)[1])
        e = float(np.abs(got[0, :, h * d:(h + 1) * d] - y_want).max())
        if e <= 2e-2:
            continue
        rec = {"head": h, "pattern": conv(p), "max_abs": e}
        if isinstance(p, O.VS):
            dev = sa.build_index(sa.AttnMatrices(qh, kh, vh), to_sa(p), "estimated", 64)
            dc, dd = set(dev.columns), set(dev.diagonals)
            wc, wd = set(want_idx.columns.tolist()), set(want_idx.diagonals.tolist())
            rec.update(col_flips=len(dc ^ wc) // 2, diag_flips=len(dd ^ wd) // 2)
            didx = O.Index(qh.shape[0], np.array(sorted(dc), np.int64), np.array(sorted(dd), np.int64))
            y_dev = O.sparse_attention(qh, kh, vh, didx)[1]
            rec["max_abs_vs_device_index"] = float(np.abs(got[0, :, h * d:(h + 1) * d] - y_dev).max())
            # the flipped candidates' oracle scores: margin of the k-th vs the (k+1)-th
            cs, ds = O.vs_scores(qh, kh, "estimated", 64)
            for name, sc, kk in (("col", cs, p.k_v), ("diag", ds, p.k_s)):
                srt = np.sort(np.asarray(sc, np.float64))[::-1]
                kk = min(kk, len(srt))
                if kk < len(srt):
                    rec[f"{name}_margin"] = float(srt[kk - 1] - srt[kk])
        if isinstance(p, O.Blk):
            dev = sa.build_index(sa.AttnMatrices(qh, kh, vh), to_sa(p), "estimated", 64)
            nb = len(want_idx.block_rows)
            rows = [set() for _ in range(nb)]
            for gq, gk in dev.blocks:
                rows[gq].add(int(gk))
            flips = [g for g in range(nb) if rows[g] != set(want_idx.block_rows[g].tolist())]
            didx = O.Index(qh.shape[0], np.zeros(0, np.int64), np.zeros(0, np.int64), want_idx.block_size,
                           [np.array(sorted(r), np.int64) for r in rows])
            y_dev = O.sparse_attention(qh, kh, vh, didx)[1]
            rec.update(block_row_flips=len(flips),
                       max_abs_vs_device_index=float(np.abs(got[0, :, h * d:(h + 1) * d] - y_dev).max()))
            if flips:  # float64 logit gap between the two choices of the first flipped row
                b = want_idx.block_size
                qb, kb = O.block_mean(qh, b), O.block_mean(kh, b)
                g = flips[0]
                lg = (qb[g].astype(np.float64) @ kb[: g + 1].astype(np.float64).T) * O.head_scale(qh.shape[1])
                a_ = sorted(rows[g] - {g}) or [g]
                b_ = sorted(set(want_idx.block_rows[g].tolist()) - {g}) or [g]
                rec["first_flip"] = {"row": g, "device": a_, "oracle": b_,
                                     "logit_gap": float(abs(lg[a_[0]] - lg[b_[0]]))}
        out.append(rec)
    return out


fails = flips = 0
t0 = time.time()
for c in range(args.cases):
    H, HK = LAYOUTS[rng.integers(len(LAYOUTS))]
    n = int(rng.choice(SPECIAL_N)) if rng.random() < 0.3 else int(rng.integers(1, args.max_n + 1))
    d = int(rng.choice([128, 128, 64]))
    mode = str(rng.choice(["auto", "auto", "fixed", "fixed", "dense"]))
    if H * n > 60000:  # keep the oracle within seconds
        n = max(1, 60000 // H)
    seed = int(rng.integers(1 << 30))
    q, k, v = (O.bf16_round(x) for x in O.synth_qkv_gqa(seed, n, H, HK, d))
    fixed = rand_fixed(n) if mode == "fixed" else None
    B, kind = 1, "numpy"
    if args.api_mix:
        B = int(rng.integers(1, 4))
        kind = str(rng.choice(["numpy", "cpu", "cpu_pinned", "cuda_bf16", "cuda_f32"]))
        if B > 1:
            extra = [[O.bf16_round(x) for x in O.synth_qkv_gqa(seed + 1 + b, n, H, HK, d)] for b in range(B - 1)]
            q, k, v = (np.concatenate([t] + [e[i] for e in extra]) for i, t in enumerate((q, k, v)))
    if args.only is not None and c not in args.only:
        continue
    rec = {"case": c, "H": H, "HK": HK, "n": n, "d": d, "mode": mode, "fixed": conv(fixed), "seed": seed}
    if args.api_mix:
        rec.update(batch=B, inputs=kind)
    try:
        want, wplans = O.prefill(q, k, v, mode, fixed_pattern=fixed)
        cfg = sa.ModelConfig(n_heads=H, d_model=H * d, d_head=d, max_context=max(n, 1))
        kw = {"fixed_pattern": to_sa(fixed)} if fixed is not None else {}
        qi, ki, vi = q, k, v
        if kind != "numpy":
            import torch

            qi, ki, vi = (torch.from_numpy(np.ascontiguousarray(x)) for x in (q, k, v))
            if kind == "cpu_pinned":
                qi, ki, vi = (x.pin_memory() for x in (qi, ki, vi))
            elif kind == "cuda_bf16":
                qi, ki, vi = (x.cuda().bfloat16() for x in (qi, ki, vi))
            elif kind == "cuda_f32":
                qi, ki, vi = (x.cuda() for x in (qi, ki, vi))
        res = sa.prefill(qi, ki, vi, cfg, mode=mode, **kw)
        o = res.outputs
        got = (o.float().cpu().numpy() if hasattr(o, "cpu") else np.asarray(o)).astype(np.float64)
        err = np.abs(got - want)
        gplans = [[conv(hp.pattern) for hp in row] for row in res.plans]
        rec.update(max_abs=float(err.max()), mean_abs=float(err.mean()),
                   plans_equal=gplans == [[conv(p) for p in row] for row in wplans])
        rec["ok"] = bool(rec["max_abs"] <= 2e-2 and rec["mean_abs"] <= 2e-3 and rec["plans_equal"])
        rec["kind"] = "ok" if rec["ok"] else "fail"
        if not rec["ok"] and rec["plans_equal"]:
            rec["diag"] = [dict(x, batch=b) for b in range(B)
                           for x in diagnose(q[b:b + 1], k[b:b + 1], v[b:b + 1], wplans[b], got[b:b + 1], d)]
            # an estimator near-tie (float64 gap below fp32 resolution) realised differently,
            # with the kernels exact on the device's own index
            if rec["diag"] and all(x.get("max_abs_vs_device_index", 1.0) <= 2e-2 and
                                   (x.get("first_flip", {}).get("logit_gap", 1.0) < 1e-5 or
                                    min(x.get("col_margin", 1.0), x.get("diag_margin", 1.0)) < 1e-5)
                                   for x in rec["diag"]):
                rec["kind"] = "near_tie_flip"
    except Exception as e:  # noqa: BLE001 - report and continue
        rec.update(ok=False, kind="fail", error=f"{type(e).__name__}: {e}"[:300])
    fails += rec["kind"] == "fail"
    flips += rec["kind"] == "near_tie_flip"
    print(json.dumps(rec), flush=True)
print(json.dumps({"cases": args.cases if args.only is None else len(args.only), "failures": fails,
                  "near_tie_flips": flips, "seconds": round(time.time() - t0, 1)}))
