"""Pattern families, realised indices, estimators and sparse attention on the
B200 kernels (reference: patterns.py).

Per-head entry points stage the head onto the GPU, call the C ABI and return
results in the caller's array type (numpy in -> numpy out, torch in -> torch
out).  Index objects keep the reference's structural tuples; the device
encodings live in ``device_index``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Union

import numpy as np
import torch

from . import _device as D
from . import _lib
from . import device_index as DI
from .core import AttnMatrices, MacCounter
from .errors import DimensionError, EmptyRowError, PatternParamError, SparseAttnError  # noqa: F401

__all__ = [
    "PatternParamError",
    "Triangular",
    "VerticalSlash",
    "BlockSparse",
    "SparsityPattern",
    "SparseIndex",
    "pattern_label",
    "score_columns",
    "score_diagonals",
    "build_vertical_slash_index",
    "build_triangular_index",
    "build_block_index",
    "build_index",
    "block_mean",
    "vertical_slash_attention",
    "block_sparse_attention",
    "sparse_attention",
    "realized_size",
]

INT32_MAX = 2**31 - 1


@dataclass(frozen=True)
class Triangular:
    """Causal band of width `window` plus `sinks` leading global columns (patterns.py:59-70)."""

    window: int
    sinks: int = 0

    def __post_init__(self) -> None:
        if self.window < 1:
            raise PatternParamError(f"window must be >= 1, got {self.window}")
        if self.sinks < 0:
            raise PatternParamError(f"sinks must be >= 0, got {self.sinks}")


@dataclass(frozen=True)
class VerticalSlash:
    """Top k_v columns plus top k_s diagonals (patterns.py:73-82)."""

    k_v: int
    k_s: int

    def __post_init__(self) -> None:
        if self.k_v < 1 or self.k_s < 1:
            raise PatternParamError(f"k_v and k_s must be >= 1, got {self.k_v}, {self.k_s}")


@dataclass(frozen=True)
class BlockSparse:
    """Top k_b key blocks of side b per query block (patterns.py:85-94)."""

    b: int
    k_b: int

    def __post_init__(self) -> None:
        if self.b < 1 or self.k_b < 1:
            raise PatternParamError(f"b and k_b must be >= 1, got {self.b}, {self.k_b}")


SparsityPattern = Union[Triangular, VerticalSlash, BlockSparse]


def pattern_label(p) -> str:
    """Compact, comma-free description for report cells (patterns.py:97-110)."""
    if p is None:
        return "-"
    if isinstance(p, Triangular):
        return f"triangular(window={p.window} sinks={p.sinks})"
    if isinstance(p, VerticalSlash):
        return f"vertical-slash(kv={p.k_v} ks={p.k_s})"
    if isinstance(p, BlockSparse):
        return f"block-sparse(b={p.b} kb={p.k_b})"
    raise PatternParamError(f"unknown pattern {p!r}")


def _num_blocks(n: int, b: int) -> int:
    return -(-n // b)


@dataclass(frozen=True)
class SparseIndex:
    """Realised causal positions, stored structurally (patterns.py:113-158)."""

    n: int
    columns: tuple = ()
    diagonals: tuple = ()
    blocks: tuple = ()
    block_size: int = 0
    always_diagonal: bool = True

    def __post_init__(self) -> None:
        if self.n < 1:
            raise PatternParamError(f"index length must be >= 1, got {self.n}")
        if self.blocks and (self.columns or self.diagonals):
            raise PatternParamError("index mixes block and column/diagonal structure")
        for name, entries in (("columns", self.columns), ("diagonals", self.diagonals),
                              ("blocks", self.blocks)):
            if len(set(entries)) != len(entries):
                raise PatternParamError(f"duplicate entries in {name}")
        for c in self.columns:
            if not 0 <= c < self.n:
                raise PatternParamError(f"column {c} out of range for n={self.n}")
        for o in self.diagonals:
            if not 0 <= o < self.n:
                raise PatternParamError(f"diagonal offset {o} out of range for n={self.n}")
        if self.blocks:
            if self.block_size < 1:
                raise PatternParamError("block index requires block_size >= 1")
            nb = _num_blocks(self.n, self.block_size)
            for gq, gk in self.blocks:
                if not 0 <= gq < nb or not 0 <= gk < nb:
                    raise PatternParamError(f"block pair {(gq, gk)} out of range")
                if gk > gq:
                    raise PatternParamError(f"block pair {(gq, gk)} violates causality")


# ---------------------------------------------------------------- device index

def _index_builder(idx: SparseIndex, n: int, hh: int = 1, dense: bool = False):
    """One head's SparseIndex -> HostIndexBuilder (device encodings)."""
    b = DI.HostIndexBuilder(n, hh)
    if dense:
        b.set_dense(0)
        return b
    if idx.blocks:
        nb = _num_blocks(n, idx.block_size)
        rows: list[list[int]] = [[] for _ in range(nb)]
        for gq, gk in idx.blocks:
            rows[gq].append(gk)
        b.set_block(0, idx.block_size, [np.array(sorted(r), np.int32) for r in rows])
        return b
    cols = sorted(idx.columns)
    diags = sorted(idx.diagonals)
    if idx.always_diagonal and diags and diags == list(range(len(diags))) and cols == list(range(len(cols))):
        # build_triangular_index form: band + sinks (patterns.py:262-276)
        b.set_triangular(0, len(diags), len(cols))
        return b
    b.set_vertical_slash(0, cols, diags)
    if not idx.always_diagonal:
        b.family[0] = DI.FAM_VS_NOEYE
    return b


def _check_nonempty(idx: SparseIndex) -> None:
    if idx.blocks:
        present = {gq for gq, _ in idx.blocks}
        nb = _num_blocks(idx.n, idx.block_size)
        missing = [g for g in range(nb) if g not in present]
        if missing:
            raise EmptyRowError(f"query block {missing[0]} has no selected key blocks")
        return
    if not idx.always_diagonal and 0 not in idx.columns and 0 not in idx.diagonals:
        raise EmptyRowError("empty attention row")


def _run_index(m: AttnMatrices, idx: SparseIndex, *, dense: bool = False, need_weights: bool = False):
    """Attention of one head under `idx` on the tcgen05 kernel -> (weights|None, y).
    dense with m.causal False: every key of every row (core.py:150)."""
    n = m.n
    q, k, v = m.staged()
    noncausal = dense and not m.causal
    builder = _index_builder(idx, n, dense=dense)
    if noncausal:
        builder.set_dense(0, causal=False)
    dix = builder.upload(q.device)
    off, cnt, tiles = DI.noncausal_dense_tiles(n, 1, q.device) if noncausal else DI.build_tiles(dix)
    out = torch.empty((n, DI.HEAD_DIM), dtype=torch.bfloat16, device=q.device)
    lse = torch.empty((1, n), dtype=torch.float32, device=q.device) if need_weights else None
    view = dix.view()
    st = D.stream()
    _lib.call("sa_attn_sparse", 1, 1, 1, n, m.scale, q.data_ptr(), k.data_ptr(), v.data_ptr(),
              out.data_ptr(), view, off.data_ptr(), cnt.data_ptr(), tiles.data_ptr(),
              lse.data_ptr() if lse is not None else None, st)
    y = D.to_host_or_keep(out[:, : m.d_head], m.q)
    w = None
    if need_weights:
        wt = torch.empty((n, n), dtype=torch.float32, device=q.device)
        _lib.call("sa_attn_weights", 1, 1, n, 0, m.scale, q.data_ptr(), k.data_ptr(),
                  lse.data_ptr(), view, wt.data_ptr(), st)
        w = D.to_host_or_keep(wt, m.q)
    return w, y


# ---------------------------------------------------------------- estimators

def _check_scoring_args(m: AttnMatrices, mode: str, q_est: int) -> int:
    """patterns.py:182-189."""
    if mode not in ("exact", "estimated"):
        raise PatternParamError(f"scoring mode must be 'exact' or 'estimated', got {mode!r}")
    if mode == "estimated":
        if not 1 <= q_est <= m.n:
            raise PatternParamError(f"q_est must be in [1, {m.n}], got {q_est}")
        return q_est
    return m.n


def _tail_scores(m: AttnMatrices, rows: int, counter: MacCounter | None):
    """Column and diagonal mass of the last `rows` queries on the tcgen05
    estimator (patterns.py:165-202) -> two fp32 cuda vectors of length n."""
    n = m.n
    q, k, _ = m.staged()
    col = torch.empty(n, dtype=torch.float32, device=q.device)
    diag = torch.empty(n, dtype=torch.float32, device=q.device)
    lib = _lib.load()
    ws_bytes = int(lib.sa_score_tail_workspace(1, 1, n, n))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    st = D.stream()
    r_first = n - rows
    g = 0
    r_hi = n
    while r_hi > r_first:
        r_lo = max(r_first, r_hi - 128)
        _lib.call("sa_score_tail", 1, 1, 1, n, m.scale, q.data_ptr(), k.data_ptr(), r_lo, r_hi,
                  col.data_ptr(), diag.data_ptr(), int(g > 0), None, 0, ws.data_ptr(), ws_bytes, st)
        r_hi = r_lo
        g += 1
    if counter is not None:
        counter.scoring_macs += rows * n * m.d_head
    return col, diag


def _scores_out(t: torch.Tensor, m: AttnMatrices):
    if D.is_torch(m.q):
        return t.double()
    return t.double().cpu().numpy()


def score_columns(m: AttnMatrices, mode: str = "exact", q_est: int = 64, counter: MacCounter | None = None):
    """Per-column attention mass (patterns.py:205-215)."""
    rows = _check_scoring_args(m, mode, q_est)
    return _scores_out(_tail_scores(m, rows, counter)[0], m)


def score_diagonals(m: AttnMatrices, mode: str = "exact", q_est: int = 64, counter: MacCounter | None = None):
    """Per-offset attention mass (patterns.py:218-228)."""
    rows = _check_scoring_args(m, mode, q_est)
    return _scores_out(_tail_scores(m, rows, counter)[1], m)


def _topk_device(scores: torch.Tensor, k: int) -> list[int]:
    """Stable top-k on device (patterns.py:231-234): ascending ids."""
    n = scores.shape[-1]
    out = torch.empty(k, dtype=torch.int32, device=scores.device)
    _lib.call("sa_topk_stable_f32", scores.data_ptr(), 1, n, n, k, out.data_ptr(), k, D.stream())
    return out.cpu().tolist()


def build_vertical_slash_index(m: AttnMatrices, k_v: int, k_s: int, mode: str = "exact",
                               q_est: int = 64, counter: MacCounter | None = None) -> SparseIndex:
    """Top-k_v columns and top-k_s diagonals by attention mass (patterns.py:237-259)."""
    n = m.n
    if not 1 <= k_v <= n:
        raise PatternParamError(f"k_v must be in [1, {n}], got {k_v}")
    if not 1 <= k_s <= n:
        raise PatternParamError(f"k_s must be in [1, {n}], got {k_s}")
    rows = _check_scoring_args(m, mode, q_est)
    col, diag = _tail_scores(m, rows, counter)
    return SparseIndex(n=n, columns=tuple(_topk_device(col, k_v)),
                       diagonals=tuple(_topk_device(diag, k_s)), always_diagonal=True)


def build_triangular_index(n: int, window: int, sinks: int) -> SparseIndex:
    """Causal band of width `window` plus `sinks` leading columns (patterns.py:262-276)."""
    if not 1 <= window <= n:
        raise PatternParamError(f"window must be in [1, {n}], got {window}")
    if not 0 <= sinks <= n:
        raise PatternParamError(f"sinks must be in [0, {n}], got {sinks}")
    return SparseIndex(n=n, columns=tuple(range(sinks)), diagonals=tuple(range(window)),
                       always_diagonal=True)


def block_mean(x, b: int):
    """Mean-pool rows in groups of b; the last partial block averages its true
    length (patterns.py:279-287).  fp32 on device."""
    if b < 1:
        raise PatternParamError(f"block side must be >= 1, got {b}")
    dev = D.require_cuda()
    t = torch.as_tensor(x) if not D.is_torch(x) else x
    if t.dim() != 2:
        raise DimensionError(f"block_mean expects a 2-d array, got {tuple(t.shape)}")
    n, d = t.shape
    src = t.to(device=dev, dtype=torch.float32).contiguous()
    nb = _num_blocks(n, b)
    out = torch.empty((nb, d), dtype=torch.float32, device=dev)
    _lib.call("sa_block_mean_f32", src.data_ptr(), n, d, b, out.data_ptr(), D.stream())
    return D.to_host_or_keep(out, x)


def _block_rows(m: AttnMatrices, b: int, k_b: int) -> list[list[int]]:
    """Device block estimator -> per query block ascending key-block ids."""
    n = m.n
    q, k, _ = m.staged()
    nb = _num_blocks(n, b)
    qp = torch.empty((1, nb, 384), dtype=torch.bfloat16, device=q.device)
    kp = torch.empty((1, nb, 256), dtype=torch.bfloat16, device=q.device)
    st = D.stream()
    _lib.call("sa_block_pool", 1, n, b, 0, q.data_ptr(), qp.data_ptr(), None, st)
    _lib.call("sa_block_pool", 1, n, b, 1, k.data_ptr(), kp.data_ptr(), None, st)
    idx = torch.empty((nb, k_b + 1), dtype=torch.int32, device=q.device)
    row_off = torch.empty(nb + 1, dtype=torch.int32, device=q.device)
    lib = _lib.load()
    ws_bytes = int(lib.sa_block_select_workspace(n, b, k_b))
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=q.device)
    _lib.call("sa_block_select", 1, 1, 1, n, b, k_b, m.scale, qp.data_ptr(), kp.data_ptr(),
              idx.data_ptr(), row_off.data_ptr(), ws.data_ptr(), ws_bytes, st)
    rows = idx.cpu().numpy()
    return [[int(g) for g in r if g != INT32_MAX] for r in rows]


def build_block_index(m: AttnMatrices, b: int, k_b: int, counter: MacCounter | None = None) -> SparseIndex:
    """Top-k_b causal key blocks per query block by pooled attention (patterns.py:290-321)."""
    n, d = m.n, m.d_head
    if not 1 <= b <= n:
        raise PatternParamError(f"b must be in [1, {n}], got {b}")
    nb = _num_blocks(n, b)
    if not 1 <= k_b <= nb:
        raise PatternParamError(f"k_b must be in [1, {nb}], got {k_b}")
    rows = _block_rows(m, b, k_b)
    if counter is not None:
        counter.scoring_macs += 2 * n * d + nb * nb * d
    blocks = tuple((gq, gk) for gq, r in enumerate(rows) for gk in r)
    return SparseIndex(n=n, blocks=blocks, block_size=b, always_diagonal=True)


def build_index(m: AttnMatrices, pattern, mode: str = "estimated", q_est: int = 64,
                counter: MacCounter | None = None) -> SparseIndex:
    """Realise any pattern family against an input (patterns.py:324-343)."""
    if isinstance(pattern, Triangular):
        return build_triangular_index(m.n, min(pattern.window, m.n), min(pattern.sinks, m.n))
    if isinstance(pattern, VerticalSlash):
        return build_vertical_slash_index(m, min(pattern.k_v, m.n), min(pattern.k_s, m.n), mode,
                                          min(q_est, m.n), counter)
    if isinstance(pattern, BlockSparse):
        b = min(pattern.b, m.n)
        return build_block_index(m, b, min(pattern.k_b, _num_blocks(m.n, b)), counter)
    raise PatternParamError(f"unknown pattern {pattern!r}")


# ---------------------------------------------------------------- kernels

def _check_kernel_inputs(m: AttnMatrices, idx: SparseIndex) -> None:
    if not m.causal:
        raise PatternParamError("sparse kernels require causal attention")
    if idx.n != m.n:
        raise DimensionError(f"index realized for n={idx.n}, input has n={m.n}")


def _count(counter, idx, m):
    if counter is not None:
        pos = realized_size(idx, m.n)
        counter.logit_macs += pos * m.d_head
        counter.output_macs += pos * m.d_head


def vertical_slash_attention(m: AttnMatrices, idx: SparseIndex, *, need_weights: bool = True,
                             counter: MacCounter | None = None):
    """Sparse attention over a column/diagonal index (patterns.py:353-435)."""
    _check_kernel_inputs(m, idx)
    if idx.blocks:
        raise PatternParamError("block index passed to the vertical-slash kernel")
    if not idx.columns and not idx.diagonals and not idx.always_diagonal:
        raise EmptyRowError("empty attention row")
    _check_nonempty(idx)
    w, y = _run_index(m, idx, need_weights=need_weights)
    _count(counter, idx, m)
    return w, y


def block_sparse_attention(m: AttnMatrices, idx: SparseIndex, *, need_weights: bool = True,
                           counter: MacCounter | None = None):
    """Sparse attention over a block index (patterns.py:438-484)."""
    _check_kernel_inputs(m, idx)
    if idx.columns or idx.diagonals:
        raise PatternParamError("column/diagonal index passed to the block-sparse kernel")
    if not idx.blocks:
        raise EmptyRowError("empty attention row")
    _check_nonempty(idx)
    w, y = _run_index(m, idx, need_weights=need_weights)
    _count(counter, idx, m)
    return w, y


def sparse_attention(m: AttnMatrices, idx: SparseIndex, *, need_weights: bool = True,
                     counter: MacCounter | None = None):
    """Dispatch to the kernel matching the index structure (patterns.py:487-497)."""
    if idx.blocks:
        return block_sparse_attention(m, idx, need_weights=need_weights, counter=counter)
    return vertical_slash_attention(m, idx, need_weights=need_weights, counter=counter)


def realized_size(idx: SparseIndex, n: int) -> int:
    """Exact count of distinct causal positions covered (patterns.py:500-521)."""
    if idx.n != n:
        raise DimensionError(f"index realized for n={idx.n}, asked about n={n}")
    if idx.blocks:
        total = 0
        b = idx.block_size
        for gq, gk in idx.blocks:
            rows = min(b, n - gq * b)
            total += rows * min(b, n - gk * b) if gk < gq else rows * (rows + 1) // 2
        return total
    cols = np.sort(np.fromiter(idx.columns, dtype=np.int64, count=len(idx.columns)))
    total = int((n - cols).sum()) if cols.size else 0
    for o in idx.diagonals:
        total += (n - o) - int(np.searchsorted(cols, n - o, side="left"))
    if idx.always_diagonal and 0 not in idx.diagonals:
        total += n - cols.size
    return total
