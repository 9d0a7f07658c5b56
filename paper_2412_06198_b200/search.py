"""FLOPs-targeted pattern search (reference: search.py).

The cost model and candidate refinement are data-independent integer math and
run on the host, exactly as the reference defines them (including Python's
round-half-to-even).  Selection — dense window weights, candidate
realisation, sparse weights, Frobenius distance, argmin — runs on device:
the one-CTA-per-head selector kernel when the sub-problem fits it (n <= 64,
exact scoring, weight metric: every prefill), else a composition of the
estimator / attention / weights kernels.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _device as D
from . import _lib
from .core import AttnMatrices, MacCounter, frob_norm_diff
from .errors import PatternParamError, SearchError  # noqa: F401
from .patterns import (
    BlockSparse,
    SparsityPattern,
    Triangular,
    VerticalSlash,
    build_index,
    sparse_attention,
)

__all__ = [
    "SearchError",
    "FlopsEstimate",
    "SearchSpace",
    "RefinedCandidate",
    "SearchResult",
    "DEFAULT_FAMILIES",
    "DENSE_EVAL_CAP",
    "nominal_positions",
    "estimate_flops",
    "refine_candidate",
    "refine_search_space",
    "select_pattern",
    "select_pattern_windowed",
    "default_search_space",
]

DENSE_EVAL_CAP = 4096  # search.py:44
SELECTOR_CAL_MAX = 64  # device selector kernel window limit (selector.cu)


@dataclass(frozen=True)
class FlopsEstimate:
    scoring_macs: int
    logit_macs: int
    output_macs: int

    @property
    def total(self) -> int:
        return self.scoring_macs + self.logit_macs + self.output_macs


@dataclass
class SearchSpace:
    """Candidate patterns plus the budget they are refined toward (search.py:64-81)."""

    candidates: list
    target_flops: int
    epsilon: float = 0.05
    max_refine_iters: int = 8

    def __post_init__(self) -> None:
        if not self.candidates:
            raise SearchError("candidate list must be non-empty")
        if not 0.0 < self.epsilon < 1.0:
            raise SearchError(f"epsilon must be in (0, 1), got {self.epsilon}")
        if self.max_refine_iters < 1:
            raise SearchError(f"max_refine_iters must be >= 1, got {self.max_refine_iters}")
        if self.target_flops < 1:
            raise SearchError(f"target_flops must be >= 1, got {self.target_flops}")


@dataclass(frozen=True)
class RefinedCandidate:
    pattern: SparsityPattern
    flops: int
    iterations: int
    converged: bool


@dataclass(frozen=True)
class SearchResult:
    chosen: SparsityPattern
    realized_flops: int
    error: float
    iterations_used: int
    converged: bool


def nominal_positions(p, n: int) -> int:
    """search.py:103-119."""
    cap = n * (n + 1) // 2
    if isinstance(p, Triangular):
        return n * (p.window + p.sinks)
    if isinstance(p, VerticalSlash):
        return min(n * (p.k_v + p.k_s), cap)
    if isinstance(p, BlockSparse):
        return min(p.k_b * p.b * p.b * -(-n // p.b), cap)
    raise PatternParamError(f"unknown pattern {p!r}")


def _validate_for_n(p, n: int) -> None:
    """search.py:122-130."""
    if isinstance(p, Triangular) and not (1 <= p.window <= n and 0 <= p.sinks <= n):
        raise PatternParamError(f"{p} invalid for n={n}")
    if isinstance(p, VerticalSlash) and not (1 <= p.k_v <= n and 1 <= p.k_s <= n):
        raise PatternParamError(f"{p} invalid for n={n}")
    if isinstance(p, BlockSparse):
        nb = -(-n // p.b)
        if not (1 <= p.b <= n and 1 <= p.k_b <= nb):
            raise PatternParamError(f"{p} invalid for n={n}")


def estimate_flops(p, n: int, d_h: int, q_est: int = 0) -> FlopsEstimate:
    """Analytic MAC model (search.py:133-150)."""
    _validate_for_n(p, n)
    pos = nominal_positions(p, n)
    if isinstance(p, VerticalSlash):
        scoring = q_est * n * d_h
    elif isinstance(p, BlockSparse):
        nb = -(-n // p.b)
        scoring = 2 * n * d_h + nb * nb * d_h
    else:
        scoring = 0
    return FlopsEstimate(scoring_macs=scoring, logit_macs=pos * d_h, output_macs=pos * d_h)


def _clamped(value: float, lo: int, hi: int) -> int:
    return max(lo, min(hi, int(round(value))))  # round-half-to-even (search.py:153-154)


def _scale_pattern(p, ratio: float, n: int):
    """search.py:157-171."""
    if isinstance(p, Triangular):
        return Triangular(window=_clamped(p.window * ratio, 1, n), sinks=_clamped(p.sinks * ratio, 0, n))
    if isinstance(p, VerticalSlash):
        return VerticalSlash(k_v=_clamped(p.k_v * ratio, 1, n), k_s=_clamped(p.k_s * ratio, 1, n))
    if isinstance(p, BlockSparse):
        return BlockSparse(b=p.b, k_b=_clamped(p.k_b * ratio, 1, -(-n // p.b)))
    raise PatternParamError(f"unknown pattern {p!r}")


def refine_candidate(p, n: int, d_h: int, target: int, epsilon: float, max_iters: int,
                     q_est: int = 0) -> RefinedCandidate:
    """Multiplicative scaling toward the FLOPs target (search.py:174-197)."""
    cur = p
    est = estimate_flops(cur, n, d_h, q_est).total
    iters = 0
    while abs(est - target) > epsilon * target and iters < max_iters:
        cur = _scale_pattern(cur, target / est, n)
        est = estimate_flops(cur, n, d_h, q_est).total
        iters += 1
    return RefinedCandidate(pattern=cur, flops=est, iterations=iters,
                            converged=abs(est - target) <= epsilon * target)


def refine_search_space(s: SearchSpace, n: int, d_h: int, q_est: int = 0) -> SearchSpace:
    """search.py:200-206."""
    refined = [refine_candidate(c, n, d_h, s.target_flops, s.epsilon, s.max_refine_iters, q_est)
               for c in s.candidates]
    return replace(s, candidates=[rc.pattern for rc in refined])


def _rescale_to_full(p, factor: float, n: int):
    """search.py:261-273."""
    if isinstance(p, Triangular):
        return Triangular(window=_clamped(p.window * factor, 1, n), sinks=_clamped(p.sinks * factor, 0, n))
    if isinstance(p, VerticalSlash):
        return VerticalSlash(k_v=_clamped(p.k_v * factor, 1, n), k_s=_clamped(p.k_s * factor, 1, n))
    return p


DEFAULT_FAMILIES = ("triangular", "vertical-slash", "block-sparse")


def default_search_space(n: int, d_h: int, density: float = 0.1, epsilon: float = 0.05,
                         max_refine_iters: int = 8, families=DEFAULT_FAMILIES) -> SearchSpace:
    """One candidate per requested family at the given density (search.py:325-357)."""
    if not 0.0 < density <= 1.0:
        raise SearchError(f"density must be in (0, 1], got {density}")
    b = max(1, min(64, n // 8))
    nb = -(-n // b)
    by_family = {
        "triangular": Triangular(window=max(1, round(density * n)), sinks=0),
        "vertical-slash": VerticalSlash(k_v=max(1, round(density * n / 2)), k_s=max(1, round(density * n / 2))),
        "block-sparse": BlockSparse(b=b, k_b=max(1, min(nb, round(density * nb)))),
    }
    unknown = [f for f in families if f not in by_family]
    if unknown:
        raise SearchError(f"unknown pattern families {unknown}; choose from {DEFAULT_FAMILIES}")
    target = max(1, int(2 * d_h * density * n * n))
    return SearchSpace(candidates=[by_family[f] for f in families], target_flops=target,
                       epsilon=epsilon, max_refine_iters=max_refine_iters)


# ---------------------------------------------------------------- selection

def family_id(p) -> int:
    if isinstance(p, Triangular):
        return 0
    if isinstance(p, VerticalSlash):
        return 1
    if isinstance(p, BlockSparse):
        return 2
    raise PatternParamError(f"unknown pattern {p!r}")


def pattern_params(p) -> tuple[int, int, int]:
    if isinstance(p, Triangular):
        return 0, p.window, p.sinks
    if isinstance(p, VerticalSlash):
        return 1, p.k_v, p.k_s
    return 2, p.b, p.k_b


def refined_candidates(s: SearchSpace, n: int, d_h: int, cost_q_est: int):
    return [refine_candidate(c, n, d_h, s.target_flops, s.epsilon, s.max_refine_iters, cost_q_est)
            for c in s.candidates]


def _device_select(q, k, heads, kv_heads, n, scale, refined, batch=1):
    """Selector kernel on staged (B*H, n, 128) bf16 q / (B*HK, n, 128) k with
    cal = n: returns (choice[HH] int32 cuda, errors[HH, len(refined)] float64 cuda:
    the written columns of the kernel's [HH, MAX_CAND] table)."""
    hh = batch * heads
    fam = (ctypes_int * _lib.MAX_CAND)()
    p1 = (ctypes_int * _lib.MAX_CAND)()
    p2 = (ctypes_int * _lib.MAX_CAND)()
    for c, rc in enumerate(refined):
        fam[c], p1[c], p2[c] = pattern_params(rc.pattern)
    choice = torch.empty(hh, dtype=torch.int32, device=q.device)
    errs = torch.empty((hh, _lib.MAX_CAND), dtype=torch.float64, device=q.device)
    _lib.call("sa_select_windowed", batch, heads, kv_heads, n, n, scale, q.data_ptr(), k.data_ptr(),
              len(refined), fam, p1, p2, choice.data_ptr(), None, errs.data_ptr(), D.stream())
    return choice, errs[:, :len(refined)]


import ctypes as _ct  # noqa: E402

ctypes_int = _ct.c_int32


def select_pattern(m: AttnMatrices, s: SearchSpace, *, metric: str = "weights", scoring: str = "exact",
                   q_est: int = 64, dense_cap: int = DENSE_EVAL_CAP,
                   counter: MacCounter | None = None) -> SearchResult:
    """Refine candidates, realise each, return the one closest to dense (search.py:209-258)."""
    if metric not in ("weights", "output"):
        raise SearchError(f"metric must be 'weights' or 'output', got {metric!r}")
    if not s.candidates:
        raise SearchError("candidate list must be non-empty")
    if m.n > dense_cap:
        raise SearchError(f"n={m.n} exceeds the dense evaluation cap {dense_cap}; use select_pattern_windowed")
    cost_q_est = 0 if scoring == "exact" else min(q_est, m.n)
    refined = refined_candidates(s, m.n, m.d_head, cost_q_est)
    if any(isinstance(rc.pattern, VerticalSlash) for rc in refined):
        # the reference reaches this check in build_index of its first VS
        # candidate (patterns.py:182-189); raising it before any device work
        # keeps the same exception for the same call
        from .patterns import _check_scoring_args

        _check_scoring_args(m, scoring, min(q_est, m.n))
    fast = (metric == "weights" and scoring == "exact" and m.n <= SELECTOR_CAL_MAX
            and len(refined) <= _lib.MAX_CAND and counter is None)
    if fast:
        q, k, _ = m.staged()
        choice, errs = _device_select(q, k, 1, 1, m.n, m.scale, refined)
        c = int(choice.item())
        err = float(errs[0, c].item())
        best = refined[c]
        return SearchResult(chosen=best.pattern, realized_flops=best.flops, error=err,
                            iterations_used=best.iterations, converged=best.converged)
    # composed device path: dense weights, each candidate's realised weights
    from .core import dense_attention

    dense_w, dense_y = dense_attention(m)
    best, best_err = None, math.inf
    for rc in refined:
        idx = build_index(m, rc.pattern, mode=scoring, q_est=q_est, counter=counter)
        w, y = sparse_attention(m, idx, counter=counter)
        err = frob_norm_diff(w, dense_w) if metric == "weights" else frob_norm_diff(y, dense_y)
        if err < best_err:
            best, best_err = rc, err
    return SearchResult(chosen=best.pattern, realized_flops=best.flops, error=best_err,
                        iterations_used=best.iterations, converged=best.converged)


def select_pattern_windowed(m: AttnMatrices, s: SearchSpace, cal_window: int, *, metric: str = "weights",
                            scoring: str = "exact", q_est: int = 64, dense_cap: int = DENSE_EVAL_CAP,
                            counter: MacCounter | None = None) -> SearchResult:
    """Select on the trailing cal_window rows, rescale to n (search.py:276-319)."""
    if not 1 <= cal_window <= m.n:
        raise SearchError(f"cal_window must be in [1, {m.n}], got {cal_window}")
    if cal_window > dense_cap:
        raise SearchError(f"cal_window {cal_window} exceeds the dense evaluation cap {dense_cap}")
    if cal_window == m.n:
        return select_pattern(m, s, metric=metric, scoring=scoring, q_est=q_est, dense_cap=dense_cap,
                              counter=counter)
    sub = AttnMatrices(m.q[-cal_window:], m.k[-cal_window:], m.v[-cal_window:], causal=m.causal)
    res = select_pattern(sub, s, metric=metric, scoring=scoring, q_est=min(q_est, cal_window),
                         dense_cap=dense_cap, counter=counter)
    full = _rescale_to_full(res.chosen, m.n / cal_window, m.n)
    cost_q_est = 0 if scoring == "exact" else min(q_est, m.n)
    return SearchResult(chosen=full, realized_flops=estimate_flops(full, m.n, m.d_head, cost_q_est).total,
                        error=res.error, iterations_used=res.iterations_used, converged=res.converged)
