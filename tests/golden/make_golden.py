"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

Every case draws its inputs from a seeded generator (documented per case) so
the tests can regenerate the inputs; the reference's outputs are stored in
``golden.npz`` and plans/patterns in ``golden.json``.  Inputs that feed the
GPU path at d=128 are rounded to bfloat16 first (oracle.bf16_round), so both
sides see identical values.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import sparseattn as ref  # noqa: E402  (the reference, read-only)
from oracle.sparse_oracle import bf16_round, synth_qkv, synth_qkv_gqa  # noqa: E402


def uniform(seed, n, d):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-1, 1, (n, d)), rng.uniform(-1, 1, (n, d)), rng.uniform(-1, 1, (n, d)))


def pat_json(p):
    if p is None:
        return None
    if isinstance(p, ref.Triangular):
        return ["triangular", p.window, p.sinks]
    if isinstance(p, ref.VerticalSlash):
        return ["vertical-slash", p.k_v, p.k_s]
    return ["block-sparse", p.b, p.k_b]


def idx_json(idx):
    return {
        "n": idx.n,
        "columns": list(idx.columns),
        "diagonals": list(idx.diagonals),
        "blocks": [list(b) for b in idx.blocks],
        "block_size": idx.block_size,
    }


def main():
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"cases": {}}

    # 1) tail scoring, exact and estimated (patterns.py:205-228); float64, small d
    sc = []
    for cid, (seed, n, d, mode, qe) in enumerate(
        [(100, 8, 4, "exact", 64), (101, 13, 3, "estimated", 5), (102, 64, 8, "estimated", 16),
         (103, 33, 2, "exact", 1), (104, 1, 2, "exact", 64), (105, 200, 16, "estimated", 64)]
    ):
        q, k, v = uniform(seed, n, d)
        m = ref.AttnMatrices(q, k, v)
        arrays[f"score_{cid}_col"] = ref.score_columns(m, mode, qe)
        arrays[f"score_{cid}_diag"] = ref.score_diagonals(m, mode, qe)
        sc.append([seed, n, d, mode, qe])
    meta["cases"]["scores"] = sc

    # 2) stable top-k on crafted score vectors with ties (patterns.py:231-234)
    tk = []
    rng = np.random.default_rng(7)
    for cid in range(8):
        n = int(rng.integers(1, 300))
        s = rng.integers(0, 5, n).astype(np.float64) * 0.25  # heavy ties
        if cid % 2:
            s = s + rng.random(n) * 1e-3
        k = int(rng.integers(1, n + 1))
        arrays[f"topk_{cid}_scores"] = s
        arrays[f"topk_{cid}_idx"] = np.array(ref.patterns._top_k_stable(s, k), np.int64)
        tk.append(k)
    meta["cases"]["topk"] = tk

    # 3) indices: VS / triangular / block (patterns.py:237-343)
    ix = []
    for cid, (seed, n, d, pat, mode, qe) in enumerate(
        [(200, 16, 4, ("vs", 3, 5), "exact", 64), (201, 40, 8, ("vs", 4, 4), "estimated", 8),
         (202, 13, 4, ("block", 4, 2), None, None), (203, 64, 8, ("block", 8, 1), None, None),
         (204, 100, 6, ("block", 7, 3), None, None), (205, 20, 4, ("tri", 5, 2), None, None),
         (206, 128, 16, ("vs", 10, 12), "estimated", 64), (207, 29, 3, ("block", 29, 1), None, None)]
    ):
        q, k, v = uniform(seed, n, d)
        m = ref.AttnMatrices(q, k, v)
        if pat[0] == "vs":
            idx = ref.build_vertical_slash_index(m, pat[1], pat[2], mode, qe)
        elif pat[0] == "block":
            idx = ref.build_block_index(m, pat[1], pat[2])
        else:
            idx = ref.build_triangular_index(n, pat[1], pat[2])
        ix.append({"seed": seed, "n": n, "d": d, "pat": list(pat), "mode": mode, "q_est": qe,
                   "index": idx_json(idx), "realized": ref.realized_size(idx, n)})
        w, y = ref.sparse_attention(m, idx)
        arrays[f"index_{cid}_w"] = w
        arrays[f"index_{cid}_y"] = y
    meta["cases"]["indices"] = ix

    # 4) block_mean (patterns.py:279-287)
    bm = []
    for cid, (seed, n, d, b) in enumerate([(300, 5, 2, 2), (301, 11, 4, 3), (302, 64, 8, 8), (303, 7, 3, 7)]):
        x = np.random.default_rng(seed).random((n, d))
        arrays[f"bmean_{cid}"] = ref.block_mean(x, b)
        bm.append([seed, n, d, b])
    meta["cases"]["block_mean"] = bm

    # 5) search: default space, refinement, selection (search.py:133-357)
    ss = []
    for n, d, dens in [(64, 128, 0.1), (64, 4, 0.1), (256, 8, 0.05), (4096, 128, 0.1), (40, 16, 0.3)]:
        s = ref.default_search_space(n, d, dens)
        refined = [ref.refine_candidate(c, n, d, s.target_flops, s.epsilon, s.max_refine_iters)
                   for c in s.candidates]
        ss.append({"n": n, "d": d, "density": dens, "candidates": [pat_json(c) for c in s.candidates],
                   "target": s.target_flops,
                   "refined": [[pat_json(r.pattern), r.flops, r.iterations, r.converged] for r in refined]})
    meta["cases"]["space"] = ss
    sel = []
    for cid, (seed, n, d) in enumerate([(400, 32, 4), (401, 64, 8), (402, 48, 16), (403, 64, 128)]):
        q, k, v = uniform(seed, n, d)
        if d == 128:
            q, k, v = (bf16_round(x.astype(np.float32)) for x in (q, k, v))
        m = ref.AttnMatrices(q, k, v)
        r = ref.select_pattern(m, ref.default_search_space(n, d))
        rw = ref.select_pattern_windowed(
            ref.AttnMatrices(*uniform(seed + 50, 4 * n, d)), ref.default_search_space(n, d), n
        )
        sel.append({"seed": seed, "n": n, "d": d, "chosen": pat_json(r.chosen), "error": r.error,
                    "flops": r.realized_flops, "windowed_chosen": pat_json(rw.chosen),
                    "windowed_error": rw.error, "windowed_flops": rw.realized_flops})
    meta["cases"]["select"] = sel

    # 6) prefill at the Llama head shape, bf16-rounded synthetic inputs
    #    (runtime.py:134-206).  Equal-head (reference API) and GQA-expanded.
    pf = []
    for cid, (seed, ctx, H, HK, mode, fixed) in enumerate(
        [(0, 512, 8, 8, "auto", None), (0, 512, 8, 8, "dense", None),
         (1, 1024, 8, 2, "auto", None), (1, 1024, 8, 2, "fixed", "triangular"),
         (1, 1024, 8, 2, "fixed", "vertical-slash"), (1, 1024, 8, 2, "fixed", "block-sparse"),
         (2, 300, 4, 4, "auto", None), (3, 4096, 8, 8, "auto", None)]
    ):
        if H == HK:
            q, k, v = synth_qkv(seed, ctx, H, 128)
        else:
            q, k, v = synth_qkv_gqa(seed, ctx, H, HK, 128)
        q, k, v = (bf16_round(x) for x in (q, k, v))
        g = H // HK
        k, v = np.repeat(k, g, axis=1), np.repeat(v, g, axis=1)
        cfg = ref.ModelConfig(n_heads=H, d_model=H * 128, d_head=128, max_context=ctx)
        kw = {}
        if mode == "fixed":
            kw["fixed_pattern"] = ref.fixed_pattern_for(fixed, ctx, 0.1)
        res = ref.prefill(q, k, v, cfg, mode=mode, **kw)
        out = res.outputs
        arrays[f"prefill_{cid}_rows"] = out[0, :: max(1, ctx // 64)]  # subsample rows
        arrays[f"prefill_{cid}_rowsum"] = out[0].astype(np.float64).sum(axis=1)
        pf.append({"seed": seed, "ctx": ctx, "H": H, "HK": HK, "mode": mode, "fixed": fixed,
                   "plans": [pat_json(p.pattern) for p in res.plans[0]],
                   "errors": [p.search.error if p.search else None for p in res.plans[0]]})
    meta["cases"]["prefill"] = pf

    # 7) BASELINE C1 exactly: synth_qkv(seed=0, 4096, 8 heads, d=128), auto.
    #    bf16-rounded (the GPU-side inputs) -> full plans + sampled outputs; the
    #    unrounded fp32 plans are kept for the record.
    q, k, v = synth_qkv(0, 4096, 8, 128)
    cfg = ref.ModelConfig(n_heads=8, d_model=8 * 128, d_head=128, max_context=4096)
    raw = ref.prefill(q, k, v, cfg, mode="auto")
    qb, kb, vb = (bf16_round(x) for x in (q, k, v))
    res = ref.prefill(qb, kb, vb, cfg, mode="auto")
    arrays["c1_rows"] = res.outputs[0, ::64]
    arrays["c1_rowsum"] = res.outputs[0].astype(np.float64).sum(axis=1)
    meta["cases"]["c1"] = {
        "seed": 0, "ctx": 4096, "H": 8, "mode": "auto",
        "plans": [pat_json(p.pattern) for p in res.plans[0]],
        "errors": [p.search.error for p in res.plans[0]],
        "plans_fp32": [pat_json(p.pattern) for p in raw.plans[0]],
    }

    # 8) Full-size per-head selection (BASELINE C2 32K seeds 0/1, C3 128K seed
    #    0; GQA 32 q / 8 kv, bf16-rounded).  The windowed search reads only the
    #    trailing 64 rows (search.py:276-319), so the reference runs it on the
    #    full-size matrices directly.  For every VS head the reference's own
    #    estimated index (runtime.py:187, patterns.py:237-259) is stored too.
    fw = []
    for seed, ctx in [(0, 32768), (1, 32768), (0, 131072)]:
        q, k, v = synth_qkv_gqa(seed, ctx, 32, 8, 128)
        q, k, v = (bf16_round(x)[0] for x in (q, k, v))
        space = ref.default_search_space(64, 128)
        heads = []
        for h in range(32):
            m = ref.AttnMatrices(q[h], k[h // 4], v[h // 4], causal=True)
            r = ref.select_pattern_windowed(m, space, 64)
            e = {"chosen": pat_json(r.chosen), "error": r.error, "flops": r.realized_flops}
            if isinstance(r.chosen, ref.VerticalSlash) and ctx <= 32768:
                idx = ref.build_index(m, r.chosen, mode="estimated", q_est=64)
                arrays[f"full_{seed}_{ctx}_{h}_cols"] = np.array(idx.columns, np.int32)
                arrays[f"full_{seed}_{ctx}_{h}_diags"] = np.array(idx.diagonals, np.int32)
                e["vs_index"] = True
            heads.append(e)
        fw.append({"seed": seed, "ctx": ctx, "H": 32, "HK": 8, "heads": heads})
        del q, k, v
    meta["cases"]["fullsize_select"] = fw

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
