#!/usr/bin/env python
"""Randomised estimator / selector sweep (tool): score_columns,
score_diagonals (exact and estimated, random q_est), build_vertical_slash_index,
block_mean, build_block_index and select_pattern on random single-head inputs
vs the oracle.  Scores: max relative error; index sets: equal, or differing
only where the oracle's float64 scores tie within 1e-5 relative at the top-k
boundary (fp32 device sums vs float64); selection: the same refined pattern,
or the chosen candidates' float64 errors within 1e-6.

  python tools/estimator_sweep.py [--cases 100] [--seed 0] [--max-n 4096]
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


def boundary_tie(scores, got, want, k):
    """Differing members all sit at the k-th score within 1e-5 relative."""
    s = np.asarray(scores, np.float64)
    kth = np.sort(s)[::-1][k - 1]
    diff = np.array(sorted(set(got) ^ set(want)), np.int64)
    return bool(np.all(np.abs(s[diff] - kth) <= 1e-5 * max(np.abs(s).max(), 1e-30)))


def asnp(x):
    return x.float().cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


fails = 0
t0 = time.time()
for c in range(args.cases):
    n = int(rng.choice([1, 2, 63, 64, 65, 128])) if rng.random() < 0.25 else int(rng.integers(1, args.max_n + 1))
    d = int(rng.choice([128, 64, 7]))
    q, k, v = (O.bf16_round(x)[0, 0] for x in O.synth_qkv_gqa(int(rng.integers(1 << 30)), n, 1, 1, d))
    m = sa.AttnMatrices(q, k, v)
    rec = {"case": c, "n": n, "d": d}
    ok = True
    try:
        mode = str(rng.choice(["exact", "estimated"]))
        qe = int(rng.integers(1, 129))
        rows = n if mode == "exact" else min(qe, n)
        if mode == "exact" and n > 4096:
            mode, rows = "estimated", min(qe, n)
        try:
            cs, ds = O.vs_scores(q, k, mode, qe)
        except ValueError as e:  # the reference rejects it: so must the device path, with the same class
            try:
                sa.score_columns(m, mode, qe)
                raised = None
            except sa.SparseAttnError as e2:
                raised = type(e2).__name__
            rec.update(mode=mode, q_est=qe, expected=str(e), raised=raised)
            rec["ok"] = raised == str(e).split(":")[0]
            fails += not rec["ok"]
            print(json.dumps(rec), flush=True)
            continue
        gc = asnp(sa.score_columns(m, mode, qe)).astype(np.float64)
        gd = asnp(sa.score_diagonals(m, mode, qe)).astype(np.float64)
        rec["col_rel"] = float(np.abs(gc - cs).max() / max(np.abs(cs).max(), 1e-30))
        rec["diag_rel"] = float(np.abs(gd - ds).max() / max(np.abs(ds).max(), 1e-30))
        ok &= rec["col_rel"] <= 1e-4 and rec["diag_rel"] <= 1e-4
        kv_, ks_ = int(rng.integers(1, n + 1)), int(rng.integers(1, n + 1))
        gi = sa.build_vertical_slash_index(m, kv_, ks_, mode, qe)
        wi = O.vs_index(q, k, kv_, ks_, mode, qe)
        col_ok = set(gi.columns) == set(wi.columns.tolist()) or boundary_tie(cs, gi.columns, wi.columns.tolist(), kv_)
        diag_ok = set(gi.diagonals) == set(wi.diagonals.tolist()) or \
            boundary_tie(ds, gi.diagonals, wi.diagonals.tolist(), ks_)
        rec.update(mode=mode, q_est=qe, k_v=kv_, k_s=ks_, vs_index_ok=bool(col_ok and diag_ok))
        ok &= col_ok and diag_ok
        b = int(rng.choice([1, 2, 8, 16, 64, 100]))
        b = min(b, n)
        bm = asnp(sa.block_mean(q, b)).astype(np.float64)
        rec["block_mean_rel"] = float(np.abs(bm - O.block_mean(q, b)).max() / max(np.abs(q).max(), 1e-30))
        ok &= rec["block_mean_rel"] <= 1e-6
        nb = -(-n // b)
        kb = int(rng.integers(1, nb + 1))
        gbi = sa.build_block_index(m, b, kb)
        wbi = O.block_index(q, k, b, kb)
        rows_g = [set() for _ in range(nb)]
        for gq, gk in gbi.blocks:
            rows_g[gq].add(int(gk))
        bad = [g for g in range(nb) if rows_g[g] != set(wbi.block_rows[g].tolist())]
        if bad:  # float64 pooled logits of the differing rows: ties within 1e-5 relative
            qb, kbm = O.block_mean(q, b).astype(np.float64), O.block_mean(k, b).astype(np.float64)
            tie = True
            for g in bad:
                lg = qb[g] @ kbm[: g + 1].T
                diff = sorted((rows_g[g] ^ set(wbi.block_rows[g].tolist())) - {g})
                keff = min(kb, g + 1)
                kth = np.sort(lg)[::-1][keff - 1]
                tie &= bool(np.all(np.abs(lg[diff] - kth) <= 1e-5 * max(np.abs(lg).max(), 1e-30)))
                rec.setdefault("block_tie_gaps", []).append(float(np.abs(lg[diff] - kth).max() /
                                                                   max(np.abs(lg).max(), 1e-30)))
            rec["block_rows_tie"] = len(bad)
            ok &= tie
        rec.update(b=b, k_b=kb)
        if n <= 512:
            space = O.default_space(n, d)
            sp = sa.default_search_space(n, d)
            res = sa.select_pattern(m, sp)
            want = O.select(q, k, v, space)
            same = (type(res.chosen).__name__[0], *res.chosen.__dict__.values()) == \
                (type(want[0]).__name__[0], *want[0].__dict__.values())
            rec["select_same"] = bool(same)
            if not same:
                errs = sorted(want[5])
                rec["select_err_gap"] = float(errs[1] - errs[0]) if len(errs) > 1 else 0.0
                ok &= rec["select_err_gap"] <= 1e-6
        rec["ok"] = bool(ok)
    except Exception as e:  # noqa: BLE001
        rec.update(ok=False, error=f"{type(e).__name__}: {e}"[:300])
    fails += not rec["ok"]
    print(json.dumps(rec), flush=True)
print(json.dumps({"cases": args.cases, "failures": fails, "seconds": round(time.time() - t0, 1)}))
