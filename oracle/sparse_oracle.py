"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the reference's prefill sparse-attention algorithm
(SparseAccelerate, /root/reference/pkg/src/sparseattn).  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference`` legs
of ``bench.py`` may import it, and only as the checker or the timed CPU
baseline.  The shipped path (``paper_2412_06198_b200``) never calls it.

Parity pin: every function is checked against golden vectors produced by the
reference itself (``tests/golden/make_golden.py`` imports the reference in the
build container and records its outputs on seeded inputs) and against the
reference tests' known answers (``tests/test_oracle.py``).

Each function names the reference lines it restates.  Arrays are plain
numpy; per-head inputs are (n, d); multi-head inputs are (B, H, n, d) with
the GQA extension that k/v may carry H // g heads (head h reads kv head
h // g), which the oracle realises by repeating k/v.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# ----------------------------------------------------------------------------
# Patterns (patterns.py:59-94) and realised indices (patterns.py:113-158)


@dataclass(frozen=True)
class Tri:
    window: int
    sinks: int = 0


@dataclass(frozen=True)
class VS:
    k_v: int
    k_s: int


@dataclass(frozen=True)
class Blk:
    b: int
    k_b: int


FAMILIES = ("triangular", "vertical-slash", "block-sparse")  # search.py:322


@dataclass
class Index:
    """Structural index: columns / diagonals, or per-query-block key-block rows."""

    n: int
    columns: np.ndarray  # int64, ascending
    diagonals: np.ndarray  # int64, ascending
    block_size: int = 0
    block_rows: list | None = None  # block_rows[gq] = ascending key-block ids
    always_diagonal: bool = True

    @property
    def is_block(self) -> bool:
        return self.block_rows is not None


def head_scale(d: int) -> float:
    """1/sqrt(d_head) (core.py:84-87)."""
    return 1.0 / math.sqrt(d)


def check_head(q, k, v) -> None:
    """Shape/finiteness contract of AttnMatrices (core.py:61-74)."""
    for x in (q, k, v):
        if x.ndim != 2:
            raise ValueError("DimensionError: per-head inputs must be 2-d")
    if not (q.shape == k.shape == v.shape):
        raise ValueError("DimensionError: q/k/v shapes differ")
    if q.shape[0] < 1 or q.shape[1] < 1:
        raise ValueError("DimensionError: empty head")
    for x in (q, k, v):
        if not np.isfinite(x).all():
            raise ValueError("NonFiniteError")


# ----------------------------------------------------------------------------
# Shared numerics (core.py:113-154)


def row_softmax(x: np.ndarray) -> np.ndarray:
    """Max-subtracted softmax over the last axis; -inf entries become 0
    (core.py:123-135).  Raises on an all -inf row (EmptyRowError)."""
    top = x.max(axis=-1, keepdims=True)
    if np.isneginf(top).any():
        raise ValueError("EmptyRowError")
    e = np.exp(x - top)
    return e / e.sum(axis=-1, keepdims=True)


def dense_attention(q, k, v):
    """Causal dense reference (core.py:138-154): returns (weights, out)."""
    n = q.shape[0]
    s = (q @ k.T) * head_scale(q.shape[1])
    s = np.where(np.tri(n, dtype=bool), s, -np.inf)
    w = row_softmax(s)
    return w, w @ v


# ----------------------------------------------------------------------------
# Estimator: tail-query scores (patterns.py:165-202, 231-234)


def tail_weights(q, k, rows: int):
    """Softmax weights of the last `rows` queries against all keys, causal at the
    global row index (patterns.py:165-179).  Returns (weights, first_row)."""
    n = q.shape[0]
    first = n - rows
    s = (q[first:] @ k.T) * head_scale(q.shape[1])
    keep = np.arange(n)[None, :] <= (first + np.arange(rows))[:, None]
    return row_softmax(np.where(keep, s, -np.inf)), first


def column_mass(w: np.ndarray) -> np.ndarray:
    """score[j] = sum over rows of w[r, j], accumulated in float64 (patterns.py:192-193)."""
    return w.astype(np.float64).sum(axis=0)


def diagonal_mass(w: np.ndarray, first: int, n: int) -> np.ndarray:
    """score[o] = sum of w at (i, i - o), o >= 0 (patterns.py:196-202)."""
    rows = w.shape[0]
    out = np.zeros(n, np.float64)
    ii = first + np.arange(rows)
    for r in range(rows):
        i = ii[r]
        # positions j = 0..i carry offsets o = i - j = i..0
        out[: i + 1] += w[r, i::-1].astype(np.float64)
    return out


def top_k_stable(scores, k: int) -> np.ndarray:
    """Indices of the k largest scores, ties to the lower index, returned in
    ascending index order (patterns.py:231-234)."""
    order = np.argsort(-np.asarray(scores), kind="stable")
    return np.sort(order[:k])


def scoring_rows(n: int, mode: str, q_est: int) -> int:
    """Rows used by the estimator (patterns.py:182-189)."""
    if mode not in ("exact", "estimated"):
        raise ValueError("PatternParamError: scoring mode")
    if mode == "exact":
        return n
    if not 1 <= q_est <= n:
        raise ValueError("PatternParamError: q_est")
    return q_est


def vs_scores(q, k, mode="exact", q_est=64):
    """(column scores, diagonal scores) from one tail pass (patterns.py:205-228, 253-258)."""
    n = q.shape[0]
    w, first = tail_weights(q, k, scoring_rows(n, mode, q_est))
    return column_mass(w), diagonal_mass(w, first, n)


def vs_index(q, k, k_v: int, k_s: int, mode="exact", q_est=64) -> Index:
    """Top-k_v columns and top-k_s diagonals (patterns.py:237-259)."""
    n = q.shape[0]
    if not (1 <= k_v <= n and 1 <= k_s <= n):
        raise ValueError("PatternParamError: k_v/k_s")
    cs, ds = vs_scores(q, k, mode, q_est)
    return Index(n, top_k_stable(cs, k_v), top_k_stable(ds, k_s))


def tri_index(n: int, window: int, sinks: int) -> Index:
    """Band + sinks as a column/diagonal index (patterns.py:262-276)."""
    if not (1 <= window <= n and 0 <= sinks <= n):
        raise ValueError("PatternParamError: window/sinks")
    return Index(n, np.arange(sinks), np.arange(window))


def block_mean(x: np.ndarray, b: int) -> np.ndarray:
    """Row groups of b averaged; the tail group over its true length (patterns.py:279-287)."""
    n = x.shape[0]
    nb = -(-n // b)
    pad = nb * b - n
    xs = np.concatenate([x, np.zeros((pad,) + x.shape[1:], x.dtype)]) if pad else x
    sums = xs.reshape(nb, b, *x.shape[1:]).sum(axis=1)
    cnt = np.full(nb, b, x.dtype)
    cnt[-1] = n - (nb - 1) * b
    return sums / cnt[:, None]


def block_weights(q, k, b: int) -> np.ndarray:
    """Block-causal softmax of pooled logits (patterns.py:305-311)."""
    qb, kb = block_mean(q, b), block_mean(k, b)
    s = (qb @ kb.T) * head_scale(q.shape[1])
    nb = s.shape[0]
    return row_softmax(np.where(np.tri(nb, dtype=bool), s, -np.inf))


def block_index(q, k, b: int, k_b: int) -> Index:
    """Per query block: top-min(k_b, gq+1) causal key blocks plus the diagonal
    block (patterns.py:290-321)."""
    n = q.shape[0]
    if not 1 <= b <= n:
        raise ValueError("PatternParamError: b")
    nb = -(-n // b)
    if not 1 <= k_b <= nb:
        raise ValueError("PatternParamError: k_b")
    w = block_weights(q, k, b)
    rows = []
    for g in range(nb):
        pick = set(top_k_stable(w[g, : g + 1], min(k_b, g + 1)).tolist())
        pick.add(g)
        rows.append(np.array(sorted(pick), np.int64))
    return Index(n, np.zeros(0, np.int64), np.zeros(0, np.int64), b, rows)


def build_index(q, k, pattern, mode="estimated", q_est=64) -> Index:
    """Clamp to n and dispatch by family (patterns.py:324-343)."""
    n = q.shape[0]
    if isinstance(pattern, Tri):
        return tri_index(n, min(pattern.window, n), min(pattern.sinks, n))
    if isinstance(pattern, VS):
        return vs_index(q, k, min(pattern.k_v, n), min(pattern.k_s, n), mode, min(q_est, n))
    if isinstance(pattern, Blk):
        b = min(pattern.b, n)
        return block_index(q, k, b, min(pattern.k_b, -(-n // b)))
    raise ValueError("PatternParamError: unknown pattern")


# ----------------------------------------------------------------------------
# Index semantics, realised size, kernels (patterns.py:113-133, 353-521)


def index_mask_rows(idx: Index, r0: int, r1: int) -> np.ndarray:
    """Boolean mask of rows [r0, r1) x all n columns, from the documented field
    semantics (patterns.py:113-133)."""
    n = idx.n
    ii = np.arange(r0, r1)[:, None]
    jj = np.arange(n)[None, :]
    causal = jj <= ii
    if idx.is_block:
        b = idx.block_size
        nb = -(-n // b)
        m = np.zeros((r1 - r0, n), bool)
        for r, i in enumerate(range(r0, r1)):
            for g in idx.block_rows[i // b]:
                m[r, g * b : min((g + 1) * b, n)] = True
        m &= causal
    else:
        colsel = np.zeros(n, bool)
        colsel[idx.columns] = True
        dsel = np.zeros(n + 1, bool)
        dsel[idx.diagonals] = True
        off = np.clip(ii - jj, -1, n)  # -1 -> acausal; map to the sentinel slot n
        off = np.where(off < 0, n, off)
        m = causal & (colsel[None, :] | dsel[off])
    if idx.always_diagonal:
        m |= ii == jj
    return m


def realized_size(idx: Index) -> int:
    """Distinct causal positions covered (patterns.py:500-521)."""
    n = idx.n
    if idx.is_block:
        b = idx.block_size
        tot = 0
        for gq, row in enumerate(idx.block_rows):
            rq = min(b, n - gq * b)
            for gk in row:
                tot += rq * min(b, n - gk * b) if gk < gq else rq * (rq + 1) // 2
        return tot
    cols = np.sort(idx.columns)
    tot = int((n - cols).sum())
    for o in idx.diagonals:
        tot += (n - int(o)) - int(np.searchsorted(cols, n - int(o)))
    if idx.always_diagonal and 0 not in set(idx.diagonals.tolist()):
        tot += n - cols.size
    return tot


def vs_attention(q, k, v, idx: Index, need_weights=False):
    """Column/diagonal kernel, restating the reference's algorithm: one GEMM over
    the gathered columns, one row-wise dot per diagonal with column duplicates
    removed, the forced diagonal last, then one softmax over the realised
    positions and the matching P.V (patterns.py:353-435)."""
    n, d = q.shape
    sc = head_scale(d)
    cols = np.asarray(idx.columns, np.int64)
    offs = np.asarray(idx.diagonals, np.int64)
    colmask = np.zeros(n, bool)
    colmask[cols] = True
    forced = idx.always_diagonal and not (offs == 0).any()
    width = cols.size + offs.size + int(forced)
    if width == 0:
        raise ValueError("EmptyRowError")
    lg = np.full((n, width), -np.inf, q.dtype)
    rows = np.arange(n)
    if cols.size:
        g = q @ k[cols].T
        lg[:, : cols.size] = np.where(cols[None, :] <= rows[:, None], g, -np.inf)
    for t, o in enumerate(offs):
        o = int(o)
        dots = np.einsum("ij,ij->i", q[o:], k[: n - o])
        lg[o:, cols.size + t] = np.where(colmask[: n - o], -np.inf, dots)
    if forced:
        dots = np.einsum("ij,ij->i", q, k)
        lg[:, -1] = np.where(colmask, -np.inf, dots)
    w = row_softmax(lg * sc)
    out = np.zeros((n, d), q.dtype)
    if cols.size:
        out += w[:, : cols.size] @ v[cols]
    for t, o in enumerate(offs):
        o = int(o)
        out[o:] += w[o:, cols.size + t, None] * v[: n - o]
    if forced:
        out += w[:, -1, None] * v
    dense_w = None
    if need_weights:
        dense_w = np.zeros((n, n), q.dtype)
        if cols.size:
            dense_w[:, cols] = w[:, : cols.size]
        for t, o in enumerate(offs):
            o = int(o)
            keep = ~colmask[: n - o]
            ii = rows[o:][keep]
            dense_w[ii, ii - o] = w[o:, cols.size + t][keep]
        if forced:
            keep = ~colmask
            dense_w[rows[keep], rows[keep]] = w[keep, -1]
    return dense_w, out


def block_attention(q, k, v, idx: Index, need_weights=False):
    """Block kernel: per query block, gather its key blocks, token-causal mask,
    softmax, P.V (patterns.py:438-484)."""
    n, d = q.shape
    b = idx.block_size
    sc = head_scale(d)
    out = np.zeros((n, d), q.dtype)
    dense_w = np.zeros((n, n), q.dtype) if need_weights else None
    for gq, row in enumerate(idx.block_rows):
        if len(row) == 0:
            raise ValueError("EmptyRowError")
        r0, r1 = gq * b, min((gq + 1) * b, n)
        keys = np.concatenate([np.arange(g * b, min((g + 1) * b, n)) for g in row])
        s = (q[r0:r1] @ k[keys].T) * sc
        s = np.where(keys[None, :] <= np.arange(r0, r1)[:, None], s, -np.inf)
        w = row_softmax(s)
        out[r0:r1] = w @ v[keys]
        if dense_w is not None:
            dense_w[r0:r1][:, keys] = w
    return dense_w, out


def sparse_attention(q, k, v, idx: Index, need_weights=False):
    """Dispatch on index structure (patterns.py:487-497)."""
    if idx.is_block:
        return block_attention(q, k, v, idx, need_weights)
    return vs_attention(q, k, v, idx, need_weights)


def masked_attention(q, k, v, idx: Index, chunk=512):
    """Independent brute-force check: dense logits restricted to the index mask,
    row-chunked so large n stays bounded in memory."""
    n, d = q.shape
    sc = head_scale(d)
    out = np.zeros((n, d), np.float64)
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        m = index_mask_rows(idx, r0, r1)
        s = (q[r0:r1].astype(np.float64) @ k[:r1].T.astype(np.float64)) * sc
        w = row_softmax(np.where(m[:, :r1], s, -np.inf))
        out[r0:r1] = w @ v[:r1].astype(np.float64)
    return out


# ----------------------------------------------------------------------------
# Search: FLOPs model, refinement, selection (search.py:103-357)

DENSE_EVAL_CAP = 4096  # search.py:44


def py_round(x: float) -> int:
    """Python's round-half-to-even, as used by _clamped (search.py:153-154)."""
    return int(round(x))


def nominal_positions(p, n: int) -> int:
    """search.py:103-119."""
    cap = n * (n + 1) // 2
    if isinstance(p, Tri):
        return n * (p.window + p.sinks)
    if isinstance(p, VS):
        return min(n * (p.k_v + p.k_s), cap)
    nb = -(-n // p.b)
    return min(p.k_b * p.b * p.b * nb, cap)


def valid_for_n(p, n: int) -> bool:
    """search.py:122-130."""
    if isinstance(p, Tri):
        return 1 <= p.window <= n and 0 <= p.sinks <= n
    if isinstance(p, VS):
        return 1 <= p.k_v <= n and 1 <= p.k_s <= n
    nb = -(-n // p.b)
    return 1 <= p.b <= n and 1 <= p.k_b <= nb


def estimate_flops(p, n: int, d: int, q_est: int = 0):
    """(scoring, logit, output) MACs (search.py:133-150)."""
    if not valid_for_n(p, n):
        raise ValueError("PatternParamError: invalid for n")
    pos = nominal_positions(p, n)
    if isinstance(p, VS):
        scoring = q_est * n * d
    elif isinstance(p, Blk):
        nb = -(-n // p.b)
        scoring = 2 * n * d + nb * nb * d
    else:
        scoring = 0
    return scoring, pos * d, pos * d


def clamp_round(x: float, lo: int, hi: int) -> int:
    return max(lo, min(hi, py_round(x)))


def scale_pattern(p, ratio: float, n: int):
    """search.py:157-171."""
    if isinstance(p, Tri):
        return Tri(clamp_round(p.window * ratio, 1, n), clamp_round(p.sinks * ratio, 0, n))
    if isinstance(p, VS):
        return VS(clamp_round(p.k_v * ratio, 1, n), clamp_round(p.k_s * ratio, 1, n))
    nb = -(-n // p.b)
    return Blk(p.b, clamp_round(p.k_b * ratio, 1, nb))


def refine(p, n: int, d: int, target: int, eps: float, iters: int, q_est: int = 0):
    """Multiplicative refinement toward target (search.py:174-197).
    Returns (pattern, flops, iterations, converged)."""
    cur = p
    est = sum(estimate_flops(cur, n, d, q_est))
    it = 0
    while abs(est - target) > eps * target and it < iters:
        cur = scale_pattern(cur, target / est, n)
        est = sum(estimate_flops(cur, n, d, q_est))
        it += 1
    return cur, est, it, abs(est - target) <= eps * target


def default_space(n: int, d: int, density=0.1, eps=0.05, iters=8, families=FAMILIES):
    """One candidate per family at `density` (search.py:325-357).
    Returns (candidates, target, eps, iters)."""
    b = max(1, min(64, n // 8))
    nb = -(-n // b)
    by = {
        "triangular": Tri(max(1, py_round(density * n)), 0),
        "vertical-slash": VS(max(1, py_round(density * n / 2)), max(1, py_round(density * n / 2))),
        "block-sparse": Blk(b, max(1, min(nb, py_round(density * nb)))),
    }
    return [by[f] for f in families], max(1, int(2 * d * density * n * n)), eps, iters


def frob(a, b) -> float:
    """Frobenius norm of a - b in float64 (core.py:179-186)."""
    return float(np.linalg.norm(a.astype(np.float64) - b.astype(np.float64)))


def select(q, k, v, space, scoring="exact", q_est=64, metric="weights"):
    """Refine, realise, compare to dense, strict-< argmin (search.py:209-258).
    Returns (chosen_pattern, flops, error, iterations, converged, errors)."""
    cands, target, eps, iters = space
    n, d = q.shape
    cost_q = 0 if scoring == "exact" else min(q_est, n)
    refined = [refine(c, n, d, target, eps, iters, cost_q) for c in cands]
    wd, yd = dense_attention(q, k, v)
    best, best_err, errs = None, math.inf, []
    for rc in refined:
        idx = build_index(q, k, rc[0], mode=scoring, q_est=q_est)
        w, y = sparse_attention(q, k, v, idx, need_weights=True)
        e = frob(w, wd) if metric == "weights" else frob(y, yd)
        errs.append(e)
        if e < best_err:
            best, best_err = rc, e
    return best[0], best[1], best_err, best[2], best[3], errs


def rescale_to_full(p, factor: float, n: int):
    """Window-relative sizes scale by n/cal; blocks are kept (search.py:261-273)."""
    if isinstance(p, Tri):
        return Tri(clamp_round(p.window * factor, 1, n), clamp_round(p.sinks * factor, 0, n))
    if isinstance(p, VS):
        return VS(clamp_round(p.k_v * factor, 1, n), clamp_round(p.k_s * factor, 1, n))
    return p


def select_windowed(q, k, v, space, cal: int, scoring="exact", q_est=64):
    """Select on the trailing cal rows, rescale to n (search.py:276-319).
    Returns (pattern_at_n, error, errors)."""
    n, d = q.shape
    if cal == n:
        res = select(q, k, v, space, scoring, q_est)
        return res[0], res[2], res[5]
    res = select(q[-cal:], k[-cal:], v[-cal:], space, scoring, min(q_est, cal))
    return rescale_to_full(res[0], n / cal, n), res[2], res[5]


# ----------------------------------------------------------------------------
# Runtime: prefill (runtime.py:134-206) with the GQA extension


def expand_kv(x: np.ndarray, heads: int) -> np.ndarray:
    """(B, HK, n, d) -> (B, H, n, d): head h reads kv head h // (H // HK)."""
    g = heads // x.shape[1]
    return np.repeat(x, g, axis=1) if g > 1 else x


def prefill(q, k, v, mode="dense", fixed_pattern=None, cal_window=64, q_est=64, heads=None):
    """Per (batch, head): select (auto) -> build_index(estimated) -> kernel;
    outputs packed as (B, L, H * d) (runtime.py:134-206).
    Returns (outputs, patterns[B][H])."""
    B, H, L, d = q.shape
    k = expand_kv(k, H)
    v = expand_kv(v, H)
    cal = min(cal_window, L)
    eq = min(q_est, L)
    space = default_space(cal, d) if mode == "auto" else None
    out = np.empty((B, L, H * d), q.dtype)
    plans = []
    for b in range(B):
        row = []
        for h in (range(H) if heads is None else heads):
            qh, kh, vh = q[b, h], k[b, h], v[b, h]
            check_head(qh, kh, vh)
            if mode == "auto":
                pat = select_windowed(qh, kh, vh, space, cal)[0]
            elif mode == "fixed":
                pat = fixed_pattern
            else:
                pat = None
            if pat is None:
                y = dense_attention(qh, kh, vh)[1]
            else:
                y = sparse_attention(qh, kh, vh, build_index(qh, kh, pat, "estimated", eq))[1]
            out[b, :, h * d : (h + 1) * d] = y
            row.append(pat)
        plans.append(row)
    return out, plans


# ----------------------------------------------------------------------------
# Synthetic inputs (bench.py:111-138) and the bf16 boundary


def synth_qkv(seed: int, ctx: int, n_heads: int, d_head: int, dtype=np.float32):
    """rng([seed, ctx]) draws q, then k, then v, uniform [-1, 1] (bench.py:111-124)."""
    rng = np.random.default_rng([seed, ctx])
    shape = (n_heads, ctx, d_head)
    q = rng.uniform(-1.0, 1.0, shape).astype(dtype)
    k = rng.uniform(-1.0, 1.0, shape).astype(dtype)
    v = rng.uniform(-1.0, 1.0, shape).astype(dtype)
    return q[None], k[None], v[None]


def synth_qkv_gqa(seed: int, ctx: int, n_heads: int, n_kv: int, d_head: int):
    """GQA variant: q (H, n, d), then k (HK, n, d), then v."""
    rng = np.random.default_rng([seed, ctx])
    q = rng.uniform(-1.0, 1.0, (n_heads, ctx, d_head)).astype(np.float32)
    k = rng.uniform(-1.0, 1.0, (n_kv, ctx, d_head)).astype(np.float32)
    v = rng.uniform(-1.0, 1.0, (n_kv, ctx, d_head)).astype(np.float32)
    return q[None], k[None], v[None]


def fixed_pattern_for(method: str, ctx: int, density=0.1):
    """bench.py:127-138."""
    if method == "triangular":
        return Tri(max(1, min(ctx, py_round(density * ctx))), 0)
    if method == "vertical-slash":
        half = max(1, min(ctx, py_round(density * ctx / 2)))
        return VS(half, half)
    if method == "block-sparse":
        b = min(64, ctx)
        nb = -(-ctx // b)
        return Blk(b, max(1, min(nb, py_round(density * nb))))
    raise ValueError(f"no fixed pattern for {method!r}")


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even), returned as
    float32 — the identical inputs both sides see."""
    a = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    lsb = (a >> 16) & 1
    r = ((a + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(np.shape(x))
