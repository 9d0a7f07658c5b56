"""Shared numerics of the drop-in: input validation, dense attention, small
utilities (reference: core.py).

``dense_attention`` runs the tcgen05 attention kernel with the dense causal
index; ``softmax_row`` and ``frob_norm_diff`` are float64 utilities kept with
the reference's exact semantics (they are not on the prefill path)."""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as D
from .errors import (  # noqa: F401  (re-exported names, reference core.py:15-25)
    DimensionError,
    EmptyRowError,
    NonFiniteError,
    SparseAttnError,
)

__all__ = [
    "SparseAttnError",
    "DimensionError",
    "NonFiniteError",
    "EmptyRowError",
    "AttnMatrices",
    "MacCounter",
    "dense_attention",
    "softmax_row",
    "frob_norm_diff",
]


@dataclass(frozen=True)
class AttnMatrices:
    """Per-head q, k, v of shape (n, d_head) plus causal flag (core.py:48-87).

    Accepts numpy arrays or torch tensors (any device); the device copy used by
    the kernels is staged lazily as bf16 [1, n, 128]."""

    q: object
    k: object
    v: object
    causal: bool = True
    _staged: dict = field(default_factory=dict, compare=False, repr=False)

    def __post_init__(self) -> None:
        for name, x in (("q", self.q), ("k", self.k), ("v", self.v)):
            shp = getattr(x, "shape", None)
            if shp is None or len(shp) != 2 or not (D.is_torch(x) or isinstance(x, np.ndarray)):
                raise DimensionError(f"{name} must be a 2-d array, got {shp if shp is not None else type(x)}")
        if not (tuple(self.q.shape) == tuple(self.k.shape) == tuple(self.v.shape)):
            raise DimensionError(
                f"q/k/v shapes differ: {tuple(self.q.shape)}, {tuple(self.k.shape)}, {tuple(self.v.shape)}"
            )
        n, d = self.q.shape
        if n < 1 or d < 1:
            raise DimensionError(f"need n >= 1 and d_head >= 1, got shape {(n, d)}")
        for name, x in (("q", self.q), ("k", self.k), ("v", self.v)):
            if not D.all_finite(x):
                raise NonFiniteError(f"{name} contains NaN or Inf")

    @property
    def n(self) -> int:
        return int(self.q.shape[0])

    @property
    def d_head(self) -> int:
        return int(self.q.shape[1])

    @property
    def scale(self) -> float:
        """Logit scaling factor 1/sqrt(d_head)."""
        return 1.0 / math.sqrt(self.d_head)

    def staged(self):
        """(q, k, v) as bf16 cuda tensors [1, n, 128] (zero-padded head dim)."""
        if "qkv" not in self._staged:
            self._staged["qkv"] = tuple(D.stage_heads(x[None], nm) for x, nm in
                                        ((self.q, "q"), (self.k, "k"), (self.v, "v")))
        return self._staged["qkv"]


@dataclass
class MacCounter:
    """Multiply-accumulate tallies (core.py:90-110)."""

    scoring_macs: int = 0
    logit_macs: int = 0
    output_macs: int = 0

    @property
    def total(self) -> int:
        return self.scoring_macs + self.logit_macs + self.output_macs

    def reset(self) -> None:
        self.scoring_macs = 0
        self.logit_macs = 0
        self.output_macs = 0


def dense_attention(m: AttnMatrices, *, need_weights: bool = True):
    """Causal (or full) softmax(q k^T / sqrt(d)) v on the B200 kernel (core.py:138-154)."""
    from .patterns import SparseIndex, _run_index

    w, y = _run_index(m, SparseIndex(n=m.n), dense=True, need_weights=need_weights)
    return (w if need_weights else None), y


def softmax_row(logits, excluded=frozenset()) -> np.ndarray:
    """Stable float64 softmax over one row with excluded positions exactly 0 (core.py:157-176)."""
    x = np.asarray(logits, dtype=np.float64).ravel()
    keep = np.ones(x.shape[0], dtype=bool)
    if excluded:
        idx = np.fromiter(excluded, dtype=np.intp)
        if idx.min() < 0 or idx.max() >= x.shape[0]:
            raise DimensionError("excluded position out of range")
        keep[idx] = False
    if not keep.any():
        raise EmptyRowError("empty attention row")
    out = np.zeros(x.shape[0], dtype=np.float64)
    vals = x[keep]
    e = np.exp(vals - vals.max())
    out[keep] = e / e.sum()
    return out


def frob_norm_diff(a, b) -> float:
    """Frobenius norm of (a - b), accumulated in float64 (core.py:179-186)."""
    if tuple(np.shape(a)) != tuple(np.shape(b)):
        raise DimensionError(f"shape mismatch: {np.shape(a)} vs {np.shape(b)}")
    if D.is_torch(a) or D.is_torch(b):
        ta = torch.as_tensor(a).double()
        tb = torch.as_tensor(b).double().to(ta.device)
        return float(torch.linalg.norm((ta - tb).reshape(-1)).item())
    diff = np.asarray(a, np.float64) - np.asarray(b, np.float64)
    return float(np.linalg.norm(diff))
