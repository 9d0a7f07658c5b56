#!/usr/bin/env python
"""Randomised attention-kernel sweep (tool): arbitrary realised indices — random
column / diagonal sets (with or without the forced diagonal) and random
per-query-block key-block rows of any block size — through
paper_2412_06198_b200.sparse_attention (with and without need_weights)
against the oracle's masked dense attention on the same bf16-rounded inputs.

  python tools/kernel_sweep.py [--cases 100] [--seed 0] [--max-n 4096]
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
ap.add_argument("--cases", type=int, default=100)
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--max-n", type=int, default=4096)
args = ap.parse_args()
rng = np.random.default_rng(args.seed)
fails = 0
t0 = time.time()
for c in range(args.cases):
    n = int(rng.choice([1, 2, 127, 128, 129, 1000])) if rng.random() < 0.25 else int(rng.integers(1, args.max_n + 1))
    d = int(rng.choice([128, 64, 16]))
    q, k, v = (O.bf16_round(x)[0, 0] for x in O.synth_qkv_gqa(int(rng.integers(1 << 30)), n, 1, 1, d))
    m = sa.AttnMatrices(q, k, v)
    kind = str(rng.choice(["vs", "block"]))
    rec = {"case": c, "n": n, "d": d, "kind": kind}
    if kind == "vs":
        dens = float(rng.choice([0.001, 0.01, 0.1, 0.5]))
        cols = np.flatnonzero(rng.random(n) < dens)
        diags = np.flatnonzero(rng.random(n) < dens)
        alw = bool(rng.random() < 0.8)
        if not alw and 0 not in diags and cols.size == 0:
            diags = np.union1d(diags, [0])  # every row needs a key
        if not alw and 0 not in diags:  # rows left empty otherwise: keep row 0 coverable
            cols = np.union1d(cols, [0])
        idx = sa.SparseIndex(n=n, columns=tuple(int(x) for x in cols), diagonals=tuple(int(x) for x in diags),
                             always_diagonal=alw)
        oidx = O.Index(n, cols.astype(np.int64), diags.astype(np.int64), always_diagonal=alw)
        rec.update(cols=int(cols.size), diags=int(diags.size), always_diagonal=alw)
    else:
        b = int(rng.choice([1, 3, 8, 16, 32, 64, 100, 128, 256]))
        b = min(b, n)
        nb = -(-n // b)
        p = float(rng.choice([0.01, 0.1, 0.5]))
        rows, pairs = [], []
        for gq in range(nb):
            ks = set(np.flatnonzero(rng.random(gq + 1) < p).tolist()) | {gq}
            rows.append(np.array(sorted(ks), np.int64))
            pairs += [(gq, gk) for gk in sorted(ks)]
        idx = sa.SparseIndex(n=n, blocks=tuple(pairs), block_size=b, always_diagonal=False)
        oidx = O.Index(n, np.zeros(0, np.int64), np.zeros(0, np.int64), b, rows)
        rec.update(b=b, pairs=len(pairs))
    try:
        want = O.masked_attention(q, k, v, oidx)
        allowed = O.index_mask_rows(oidx, 0, n)
        nw = bool(rng.random() < 0.5)
        r = sa.sparse_attention(m, idx, need_weights=nw)
        y = np.asarray(r[1] if isinstance(r, tuple) else r, np.float64)
        err = np.abs(y - want)
        rec.update(need_weights=nw, max_abs=float(err.max()), mean_abs=float(err.mean()))
        ok = rec["max_abs"] <= 2e-2 and rec["mean_abs"] <= 2e-3
        if nw:
            w = np.asarray(r[0], np.float64)
            rec["masked_weight_max"] = float(np.abs(w[~allowed]).max()) if (~allowed).any() else 0.0
            rec["row_sum_err"] = float(np.abs(w.sum(axis=1) - 1).max())
            ok = ok and rec["masked_weight_max"] == 0.0 and rec["row_sum_err"] <= 1e-5
        rec["ok"] = bool(ok)
    except Exception as e:  # noqa: BLE001
        rec.update(ok=False, error=f"{type(e).__name__}: {e}"[:300])
    fails += not rec["ok"]
    print(json.dumps(rec), flush=True)
print(json.dumps({"cases": args.cases, "failures": fails, "seconds": round(time.time() - t0, 1)}))
