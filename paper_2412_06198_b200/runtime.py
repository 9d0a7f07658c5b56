"""Multi-head prefill runtime on the B200 kernels (reference: runtime.py).

``prefill`` runs one whole layer on device in two C-ABI calls: the selector
(auto mode, timed as ``select_s``) and ``sa_prefill`` (estimators, top-k,
index encodings, tile lists and the tcgen05 attention), with no host
synchronisation until the outputs are returned.  Inputs may be numpy arrays
(the reference's types; outputs come back as numpy) or torch tensors (outputs
stay on device).  As a strict extension of runtime.py:119-131, k and v may
carry fewer heads than q (GQA: query head h reads kv head h // (H // HK)).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib
from .errors import CacheOverflowError, DimensionError, NonFiniteError, SearchError, SparseAttnError
from .patterns import BlockSparse, PatternParamError, Triangular, VerticalSlash
from .search import (
    DENSE_EVAL_CAP,
    SELECTOR_CAL_MAX,
    SearchResult,
    SearchSpace,
    _rescale_to_full,
    default_search_space,
    estimate_flops,
    pattern_params,
    refined_candidates,
)

__all__ = [
    "CacheOverflowError",
    "ModelConfig",
    "KvCache",
    "HeadPlan",
    "PrefillResult",
    "DecodeResult",
    "prefill",
    "decode_step",
]

MODE_DENSE, MODE_FIXED, MODE_AUTO = 0, 1, 2


@dataclass(frozen=True)
class ModelConfig:
    """Head layout: d_model must equal n_heads * d_head (runtime.py:39-54)."""

    n_heads: int
    d_model: int
    d_head: int
    max_context: int

    def __post_init__(self) -> None:
        if min(self.n_heads, self.d_model, self.d_head, self.max_context) < 1:
            raise DimensionError("all ModelConfig fields must be >= 1")
        if self.d_model != self.n_heads * self.d_head:
            raise DimensionError(f"d_model={self.d_model} != n_heads*d_head={self.n_heads * self.d_head}")


class KvCache:
    """Append-only per-head key/value rows, resident on the GPU (runtime.py:57-90).

    ``kv_heads`` (default n_heads) sizes the cache for GQA inputs.  ``keys()`` /
    ``values()`` return numpy when the appended rows were numpy, else tensors."""

    def __init__(self, batch: int, n_heads: int, d_head: int, capacity: int, dtype=np.float32,
                 kv_heads: int | None = None, _rows=None):
        dev = D.require_cuda()
        tdt = dtype if isinstance(dtype, torch.dtype) else torch.from_numpy(np.zeros(0, dtype)).dtype
        h = n_heads if kv_heads is None else kv_heads
        if _rows is not None:  # full-capacity device rows held in place (see adopt)
            self._k, self._v = _rows
            if tuple(self._k.shape) != (batch, h, capacity, d_head) or self._k.dtype != tdt:
                raise DimensionError("adopted cache rows do not match the cache shape")
            self._np = not isinstance(dtype, torch.dtype)
            self.length = capacity
            return
        # rows past `length` are never read (keys()/values() slice), so no zero fill
        self._k = torch.empty((batch, h, capacity, d_head), dtype=tdt, device=dev)
        self._v = torch.empty((batch, h, capacity, d_head), dtype=tdt, device=dev)
        self._np = not isinstance(dtype, torch.dtype)
        self.length = 0

    @property
    def capacity(self) -> int:
        return self._k.shape[2]

    def append(self, k_rows, v_rows) -> None:
        """Append (batch, heads, t, d_head) rows to both caches."""
        if tuple(k_rows.shape) != tuple(v_rows.shape):
            raise DimensionError(f"key/value shapes differ: {tuple(k_rows.shape)} vs {tuple(v_rows.shape)}")
        if tuple(k_rows.shape[:2]) != tuple(self._k.shape[:2]) or k_rows.shape[3] != self._k.shape[3]:
            raise DimensionError(f"rows shaped {tuple(k_rows.shape)} do not fit cache {tuple(self._k.shape)}")
        t = k_rows.shape[2]
        if self.length + t > self.capacity:
            raise CacheOverflowError(f"cache of capacity {self.capacity} cannot hold {self.length + t} rows")
        kk = torch.as_tensor(k_rows) if not D.is_torch(k_rows) else k_rows
        vv = torch.as_tensor(v_rows) if not D.is_torch(v_rows) else v_rows
        self._k[:, :, self.length:self.length + t] = kk.to(self._k.device, self._k.dtype)
        self._v[:, :, self.length:self.length + t] = vv.to(self._v.device, self._v.dtype)
        self._np = not D.is_torch(k_rows)
        self.length += t

    def _out(self, t):
        return t.cpu().numpy() if self._np else t

    def keys(self):
        return self._out(self._k[:, :, : self.length])

    def values(self):
        return self._out(self._v[:, :, : self.length])


@dataclass(frozen=True)
class HeadPlan:
    """Per-head execution choice: a sparse pattern or dense (None) (runtime.py:93-99)."""

    head: int
    pattern: object
    search: SearchResult | None = None


@dataclass
class PrefillResult:
    outputs: object  # (batch, length, d_model)
    cache: KvCache
    plans: list
    elapsed_s: float  # selection + index building + kernels (+ cache fill)
    select_s: float
    kernel_s: float


@dataclass
class DecodeResult:
    output: object  # (batch, 1, d_model)
    cache: KvCache
    elapsed_s: float


def _check_qkv(q, k, v, cfg: ModelConfig):
    """runtime.py:119-131, extended to k/v with H // g heads."""
    for name, x in (("q", q), ("k", k), ("v", v)):
        if len(x.shape) != 4:
            raise DimensionError(f"{name} must be (batch, n_heads, length, d_head), got {tuple(x.shape)}")
    if tuple(k.shape) != tuple(v.shape):
        raise DimensionError(f"q/k/v shapes differ: {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
    batch, heads, length, d_head = (int(s) for s in q.shape)
    kb, kh, kl, kd = (int(s) for s in k.shape)
    if (kb, kl, kd) != (batch, length, d_head) or kh < 1 or heads % kh != 0:
        raise DimensionError(f"q/k/v shapes differ: {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
    if heads != cfg.n_heads or d_head != cfg.d_head:
        raise DimensionError(
            f"inputs have (heads, d_head)=({heads}, {d_head}), config expects ({cfg.n_heads}, {cfg.d_head})"
        )
    return batch, length, kh


def _pat(fam: int, p1: int, p2: int):
    return (Triangular(p1, p2), VerticalSlash(p1, p2), BlockSparse(p1, p2))[fam]


_WS_CACHE: dict = {}


def _workspace(nbytes: int, device) -> torch.Tensor:
    key = device
    buf = _WS_CACHE.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        _WS_CACHE[key] = buf
    return buf


class PrefillPlan:
    """Host half of one prefill call: validated shapes, the C descriptor and
    the candidate bookkeeping needed to report plans (reused by bench.py)."""

    def __init__(self, batch, heads, kv_heads, length, d_head, mode, *, search=None, fixed_pattern=None,
                 cal_window=64, q_est=64):
        if mode not in ("dense", "auto", "fixed"):
            raise SparseAttnError(f"unknown prefill mode {mode!r}")
        if mode == "fixed" and fixed_pattern is None:
            raise SparseAttnError("mode 'fixed' requires fixed_pattern")
        self.batch, self.heads, self.kv_heads, self.length, self.d_head = batch, heads, kv_heads, length, d_head
        self.mode = mode
        self.scale = 1.0 / math.sqrt(d_head)
        self.cal = min(cal_window, length)
        self.q_est = min(q_est, length)
        if mode == "auto" and self.cal < 1:  # select_pattern_windowed (search.py:290-291)
            raise SearchError(f"cal_window must be in [1, {length}], got {self.cal}")
        d = _lib.sa_prefill_desc()
        d.batch, d.heads, d.kv_heads, d.n = batch, heads, kv_heads, length
        d.scale = self.scale
        d.q_est = self.q_est
        d.cal = self.cal
        self.refined = None
        self.full = None
        self.fixed_pattern = fixed_pattern
        if mode == "dense":
            d.mode = MODE_DENSE
        elif mode == "fixed":
            d.mode = MODE_FIXED
            f, p1, p2 = pattern_params(fixed_pattern)
            d.fixed.family, d.fixed.p1, d.fixed.p2 = f, p1, p2
        else:
            d.mode = MODE_AUTO
            space = search if search is not None else default_search_space(self.cal, d_head)
            if len(space.candidates) > _lib.MAX_CAND:
                raise SearchError(f"the device selector holds at most {_lib.MAX_CAND} candidates, "
                                  f"got {len(space.candidates)}")
            # select_pattern(scoring="exact") refines with cost_q_est = 0 (search.py:235)
            self.refined = refined_candidates(space, self.cal, d_head, 0)
            if self.cal == length:
                self.full = [rc.pattern for rc in self.refined]
            else:
                self.full = [_rescale_to_full(rc.pattern, length / self.cal, length) for rc in self.refined]
            d.ncand = len(self.refined)
            for c, (rc, fp) in enumerate(zip(self.refined, self.full)):
                d.cand[c].family, d.cand[c].p1, d.cand[c].p2 = pattern_params(rc.pattern)
                d.full[c].family, d.full[c].p1, d.full[c].p2 = pattern_params(fp)
            d.preselected = 1
        # build_index(mode="estimated", q_est) of a vertical-slash head rejects
        # q_est < 1 (runtime.py:187, patterns.py:182-189); raised before any work
        vs_possible = (mode == "fixed" and isinstance(fixed_pattern, VerticalSlash)) or \
            (mode == "auto" and any(isinstance(p, VerticalSlash) for p in self.full))
        if vs_possible and self.q_est < 1:
            raise PatternParamError(f"q_est must be in [1, {length}], got {self.q_est}")
        self.desc = d
        self.ws_bytes = int(_lib.load().sa_prefill_workspace_size(d))
        if self.ws_bytes == 0:  # the plan was rejected: re-run it for its status code
            _lib.check(_lib.load().sa_prefill_views(d, None, None))

    @property
    def hh(self) -> int:
        return self.batch * self.heads

    def views(self, ws: torch.Tensor) -> _lib.sa_prefill_view:
        v = _lib.sa_prefill_view()
        _lib.call("sa_prefill_views", self.desc, ws.data_ptr(), v)
        return v

    def select(self, q: torch.Tensor, k: torch.Tensor, ws: torch.Tensor) -> None:
        """Per-head selection into the workspace's choice slot (auto mode)."""
        if self.cal <= SELECTOR_CAL_MAX:
            # the device selector; its last CTA per head applies the choice, so
            # sa_prefill (preselected = 2) starts straight at the estimators
            self.desc.preselected = 2
            _lib.call("sa_prefill_select", self.desc, q.data_ptr(), k.data_ptr(), ws.data_ptr(), ws.numel(),
                      D.stream())
            return
        self.desc.preselected = 1
        v = self.views(ws)
        # wide calibration windows: composed device selection per head, the
        # weights in fp32 like the reference's (search.py:242-250); every
        # candidate's error lands in the error rows like the selector kernel's
        from .core import AttnMatrices, dense_attention, frob_norm_diff
        from .patterns import build_index, sparse_attention

        g = self.heads // self.kv_heads
        choices = []
        errs = torch.full((self.hh, _lib.MAX_CAND), math.inf, dtype=torch.float64)
        for hh in range(self.hh):
            b, h = divmod(hh, self.heads)
            kvh = b * self.kv_heads + h // g
            qs = q[hh, -self.cal:, : self.d_head].float()
            ks = k[kvh, -self.cal:, : self.d_head].float()
            sub = AttnMatrices(qs, ks, ks)  # weights only: v is not read
            dw, _ = dense_attention(sub)
            best, best_err = 0, math.inf
            for c, rc in enumerate(self.refined):
                w, _ = sparse_attention(sub, build_index(sub, rc.pattern, mode="exact"))
                e = frob_norm_diff(w, dw)
                errs[hh, c] = e
                if e < best_err:  # strict <: the earlier candidate wins ties (search.py:249)
                    best, best_err = c, e
            choices.append(best)
        _copy_into(v.choice, torch.tensor(choices, dtype=torch.int32, device=q.device))
        _copy_into(v.errors, errs.to(q.device).reshape(-1))

    def run(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor, ws: torch.Tensor) -> None:
        _lib.call("sa_prefill", self.desc, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                  ws.data_ptr(), ws.numel(), D.stream())

    def graph(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor,
              ws: torch.Tensor) -> torch.cuda.CUDAGraph:
        """Capture selection + the whole layer into a CUDA graph bound to these
        buffers; `replay()` recomputes `out` for whatever q/k/v then hold (same
        shapes).  Saves the per-kernel launch gaps of the eager path."""
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            if self.mode == "auto":  # warm the lazy per-kernel attributes outside capture
                self.select(q, k, ws)
            self.run(q, k, v, out, ws)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=side):
                if self.mode == "auto":
                    self.select(q, k, ws)
                self.run(q, k, v, out, ws)
        torch.cuda.current_stream().wait_stream(side)
        return g

    def plans(self, ws: torch.Tensor, with_search: bool = True, flag: torch.Tensor | None = None):
        """Per (batch, head) HeadPlan list from the device choice (one small D2H).
        With `flag` (the device finiteness flag of desc.check_flag) the same
        readback carries it and NonFiniteError is raised when it is set."""
        v = self.views(ws)
        hh = self.hh
        parts = [] if flag is None else [flag.double()]
        nc = len(self.refined) if self.mode == "auto" else 0
        if self.mode == "auto":  # only the written error columns (the rest of the table is scratch)
            errs_dev = _wrap(v.errors, hh * _lib.MAX_CAND, torch.float64).view(hh, _lib.MAX_CAND)[:, :nc]
            parts += [_wrap(v.choice, hh, torch.int32).double(), errs_dev.reshape(-1)]
        small = torch.cat(parts).cpu().numpy() if parts else None
        if flag is not None:
            if int(small[0]):
                raise NonFiniteError("q, k or v contains NaN or Inf")
            small = small[1:]
        if self.mode != "auto":
            return self.plans_from(None, None, self.batch, self.heads, with_search)
        choice = small[:hh].astype(np.int64)
        errs = small[hh:].reshape(hh, nc)
        return self.plans_from(choice, errs, self.batch, self.heads, with_search)

    def plans_from(self, choice, errs, batch: int, heads: int, with_search: bool = True):
        """HeadPlan rows from host copies of the per-head choice and window errors."""
        if self.mode == "dense":
            return [[HeadPlan(head=h, pattern=None) for h in range(heads)] for _ in range(batch)]
        if self.mode == "fixed":
            return [[HeadPlan(head=h, pattern=self.fixed_pattern) for h in range(heads)] for _ in range(batch)]
        out = []
        for b in range(batch):
            row = []
            for h in range(heads):
                c = int(choice[b * heads + h])
                rc, fp = self.refined[c], self.full[c]
                res = None
                if with_search:
                    res = SearchResult(chosen=fp, realized_flops=estimate_flops(fp, self.length, self.d_head, 0).total,
                                       error=float(errs[b * heads + h, c]), iterations_used=rc.iterations,
                                       converged=rc.converged)
                row.append(HeadPlan(head=h, pattern=fp, search=res))
            out.append(row)
        return out


import ctypes as _ct  # noqa: E402

_ct_i32 = _ct.c_int32


def _wrap(ptr: int, count: int, dtype) -> torch.Tensor:
    """Device tensor view of `count` elements at raw pointer `ptr` (workspace slice)."""
    esize = torch.empty(0, dtype=dtype).element_size()
    base = _WS_OWNER_FIND(ptr)
    off = ptr - base.data_ptr()
    return base[off: off + count * esize].view(dtype)


def _WS_OWNER_FIND(ptr: int) -> torch.Tensor:
    for buf in _WS_CACHE.values():
        if buf.data_ptr() <= ptr < buf.data_ptr() + buf.numel():
            return buf
    raise RuntimeError("pointer outside the prefill workspace")


def _read_i32(ptr, count):
    return _wrap(ptr, count, torch.int32).cpu().numpy()


def _read_f64(ptr, count):
    return _wrap(ptr, count, torch.float64).cpu().numpy()


def _copy_into(ptr, src: torch.Tensor):
    _wrap(ptr, src.numel(), src.dtype).copy_(src.reshape(-1))


def stage_layer(q, k, v):
    """(B, H, L, d) numpy/torch -> (B*H, L, 128), (B*HK, L, 128), ... bf16 cuda."""
    B, H, L, d = (int(s) for s in q.shape)
    HK = int(k.shape[1])
    qd = D.stage_heads(_flat(q, B * H, L, d), "q")
    kd = D.stage_heads(_flat(k, B * HK, L, d), "k")
    vd = D.stage_heads(_flat(v, B * HK, L, d), "v")
    return qd, kd, vd


def _flat(x, g, L, d):
    if D.is_torch(x):
        return x.reshape(g, L, d)
    return np.ascontiguousarray(x).reshape(g, L, d)


def _check_plan_args(mode, fixed_pattern, search, cal_window, q_est, length, d_head):
    """The reference's argument errors that surface inside its per-head loop,
    raised up front: select_pattern_windowed's window check (search.py:290-291)
    and build_index's q_est check for a vertical-slash head (runtime.py:187,
    patterns.py:182-189)."""
    cal = min(cal_window, length)
    if mode == "auto" and cal < 1:
        raise SearchError(f"cal_window must be in [1, {length}], got {cal}")
    qe = min(q_est, length)
    if qe >= 1:
        return
    if mode == "fixed":
        vs = isinstance(fixed_pattern, VerticalSlash)
    elif mode == "auto":
        space = search if search is not None else default_search_space(cal, d_head)
        vs = any(isinstance(c, VerticalSlash) for c in space.candidates)
    else:
        vs = False
    if vs:
        raise PatternParamError(f"q_est must be in [1, {length}], got {qe}")


def prefill(q, k, v, cfg: ModelConfig, search: SearchSpace | None = None, mode: str = "dense", *,
            fixed_pattern=None, cal_window: int = 64, q_est: int = 64, dense_cap: int = DENSE_EVAL_CAP) -> PrefillResult:
    """Process all prompt tokens at once; the TTFT analog is elapsed_s (runtime.py:134-206)."""
    batch, length, kv_heads = _check_qkv(q, k, v, cfg)
    if length > cfg.max_context:
        raise DimensionError(f"length {length} exceeds max_context {cfg.max_context}")
    if mode not in ("dense", "auto", "fixed"):
        raise SparseAttnError(f"unknown prefill mode {mode!r}")
    if mode == "fixed" and fixed_pattern is None:
        raise SparseAttnError("mode 'fixed' requires fixed_pattern")
    if mode == "auto" and min(cal_window, length) > dense_cap:
        raise SearchError(f"cal_window {cal_window} exceeds the dense evaluation cap {dense_cap}")
    _check_plan_args(mode, fixed_pattern, search, cal_window, q_est, length, cfg.d_head)
    dev = D.require_cuda()
    if (D.is_torch(q) and D.is_torch(k) and D.is_torch(v) and not q.is_cuda and not k.is_cuda
            and not v.is_cuda and cfg.d_head == D.HEAD_DIM):
        return _prefill_host_streamed(q, k, v, cfg, search, mode, fixed_pattern, cal_window, q_est,
                                      batch, length, kv_heads)
    if (not D.is_torch(q) and not D.is_torch(k) and not D.is_torch(v) and cfg.d_head == D.HEAD_DIM
            and all(np.asarray(x).dtype == np.float32 for x in (q, k, v))):
        return _prefill_numpy_f32(q, k, v, cfg, search, mode, fixed_pattern, cal_window, q_est,
                                  batch, length, kv_heads)
    t0 = time.perf_counter()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    qd, kd, vd = stage_layer(q, k, v)
    plan = PrefillPlan(batch, cfg.n_heads, kv_heads, length, cfg.d_head, mode, search=search,
                       fixed_pattern=fixed_pattern, cal_window=cal_window, q_est=q_est)
    ws = _workspace(plan.ws_bytes, dev)
    # AttnMatrices' finiteness scan (core.py:72-74) runs inside sa_prefill on a
    # side stream; its flag comes back with the plans (one readback) and raises
    # before any output is returned
    flag = torch.empty(1, dtype=torch.int32, device=dev)
    plan.desc.check_flag = flag.data_ptr()
    cdt = k.dtype if D.is_torch(k) else np.asarray(k).dtype
    cache = KvCache(batch, cfg.n_heads, cfg.d_head, cfg.max_context, dtype=cdt, kv_heads=kv_heads)
    dev_fill = D.is_torch(k) and k.dtype == torch.bfloat16 and cfg.d_head == D.HEAD_DIM
    if dev_fill:  # cache.append (runtime.py:197) inside sa_prefill, beside the estimators
        plan.desc.cache_k, plan.desc.cache_v = cache._k.data_ptr(), cache._v.data_ptr()
        plan.desc.cache_capacity = cfg.max_context
    out = torch.empty((batch, length, cfg.n_heads * D.HEAD_DIM), dtype=torch.bfloat16, device=dev)
    ev[1].record()
    if mode == "auto":
        plan.select(qd, kd, ws)
    ev[2].record()
    plan.run(qd, kd, vd, out, ws)
    plan.desc.check_flag = None
    plan.desc.cache_k = plan.desc.cache_v = None
    plan.desc.cache_capacity = 0
    try:
        plans = plan.plans(ws, flag=flag)
    except NonFiniteError:
        names = [nm for nm, x in (("q", qd), ("k", kd), ("v", vd)) if not bool(torch.isfinite(x).all())]
        raise NonFiniteError(f"{names[0] if names else 'input'} contains NaN or Inf") from None
    y = out
    if cfg.d_head < D.HEAD_DIM:
        y = out.view(batch, length, cfg.n_heads, D.HEAD_DIM)[..., : cfg.d_head].reshape(batch, length, cfg.d_model)
    outputs = D.to_host_or_keep(y, q)
    if dev_fill:
        cache.length = length
    else:  # the reference caches the rows as given (runtime.py:197), not their bf16 rounding
        cache.append(k, v)
    cache._np = not D.is_torch(k)
    ev_end = torch.cuda.Event(enable_timing=True)
    ev_end.record()
    torch.cuda.synchronize()
    elapsed = time.perf_counter() - t0
    select_s = ev[1].elapsed_time(ev[2]) / 1e3
    kernel_s = ev[2].elapsed_time(ev_end) / 1e3
    return PrefillResult(outputs=outputs, cache=cache, plans=plans, elapsed_s=elapsed,
                         select_s=select_s, kernel_s=kernel_s)


def _prefill_numpy_f32(q, k, v, cfg, search, mode, fixed_pattern, cal_window, q_est, batch, length,
                       kv_heads) -> PrefillResult:
    """prefill for numpy float32 inputs (the reference's own call and types):
    chunked pinned-staged H2D of the fp32 rows, one device pass converting them
    to bf16 with AttnMatrices' finiteness check on the rows as given
    (core.py:72-74), the layer, the KvCache kept in fp32 on the device (the
    reference caches the rows as given, runtime.py:197) and a chunked D2H of
    the fp32 output into a numpy array."""
    dev = D.require_cuda()
    t0 = time.perf_counter()
    H, HK, n, d = cfg.n_heads, kv_heads, length, D.HEAD_DIM
    st = D.stream()
    qf = torch.empty((batch * H, n, d), dtype=torch.float32, device=dev)
    cap = cfg.max_context
    cache = KvCache(batch, H, d, cap, dtype=np.float32, kv_heads=HK)
    if cap == n:  # the cache rows ARE the device copies of k / v
        kf, vf = cache._k.view(batch * HK, n, d), cache._v.view(batch * HK, n, d)
    else:
        kf = torch.empty((batch * HK, n, d), dtype=torch.float32, device=dev)
        vf = torch.empty((batch * HK, n, d), dtype=torch.float32, device=dev)
    D.h2d_f32([(np.ascontiguousarray(k), kf), (np.ascontiguousarray(v), vf), (np.ascontiguousarray(q), qf)])
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    bf = torch.bfloat16
    qd = torch.empty((batch * H, n, d), dtype=bf, device=dev)
    kd = torch.empty((batch * HK, n, d), dtype=bf, device=dev)
    vd = torch.empty((batch * HK, n, d), dtype=bf, device=dev)
    for src, dst in ((qf, qd), (kf, kd), (vf, vd)):
        _lib.call("sa_f32_to_bf16", src.data_ptr(), dst.data_ptr(), src.numel(), flag.data_ptr(), st)
    if cap != n:  # rows [0, n) of each (batch, kv head) of the cache
        for src, dst in ((kf, cache._k), (vf, cache._v)):
            _lib.call("sa_memcpy2d_async", dst.data_ptr(), cap * d * 4, src.data_ptr(), n * d * 4, n * d * 4,
                      batch * HK, st)
    key = ("np", batch, H, HK, n, d, mode, repr(search), repr(fixed_pattern), cal_window, q_est)
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        plan = PrefillPlan(batch, H, HK, n, d, mode, search=search, fixed_pattern=fixed_pattern,
                           cal_window=cal_window, q_est=q_est)
        if len(_PLAN_CACHE) > 64:
            _PLAN_CACHE.clear()
        _PLAN_CACHE[key] = plan
    ws = _workspace(plan.ws_bytes, dev)
    out = torch.empty((batch, n, H * d), dtype=bf, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    if mode == "auto":
        plan.select(qd, kd, ws)
    ev[1].record()
    plan.run(qd, kd, vd, out, ws)
    ev[2].record()
    try:
        plans = plan.plans(ws, flag=flag)  # raises before any output is returned
    except NonFiniteError:
        names = [nm for nm, x in (("q", qf), ("k", kf), ("v", vf)) if not bool(torch.isfinite(x).all())]
        raise NonFiniteError(f"{names[0] if names else 'input'} contains NaN or Inf") from None
    out32 = qf.view(-1)[: out.numel()].view(out.shape)  # q's fp32 staging is free again
    _lib.call("sa_bf16_to_f32", out.data_ptr(), out32.data_ptr(), out.numel(), st)
    outputs = np.empty((batch, n, H * d), dtype=np.float32)
    D.d2h_f32(out32, outputs)
    cache.length = n
    cache._np = True
    torch.cuda.synchronize()
    return PrefillResult(outputs=outputs, cache=cache, plans=plans, elapsed_s=time.perf_counter() - t0,
                         select_s=ev[0].elapsed_time(ev[1]) / 1e3, kernel_s=ev[1].elapsed_time(ev[2]) / 1e3)


# tools/e2e_timeline.py sets this to a list to collect per-group stream event times (ms)
_TIMELINE = None
_PLAN_CACHE: dict = {}


def _prefill_host_streamed(q, k, v, cfg, search, mode, fixed_pattern, cal_window, q_est, batch, length,
                           kv_heads) -> PrefillResult:
    """prefill for host (CPU torch) inputs: the layer streams through the GPU one
    kv-head group at a time so PCIe transfers overlap the kernels.

    Per group (the g = H / HK query heads sharing one kv head): H2D of its
    k, v, q on a copy stream; on the compute stream the finiteness check,
    selection and sa_prefill (writing its column slice of the (B, L, H*d)
    output through desc.out_ld) plus the KvCache fill; then a D2H of those
    output columns on a third stream.  Group i's compute and D2H overlap
    group i+1's H2D; the result is the same as the one-shot device path."""
    dev = D.require_cuda()
    t0 = time.perf_counter()
    H, HK, n, d = cfg.n_heads, kv_heads, length, D.HEAD_DIM
    g = H // HK
    bf = torch.bfloat16
    qs = q.reshape(batch * H, n, d)
    ks = k.reshape(batch * HK, n, d)
    vs = v.reshape(batch * HK, n, d)
    if qs.dtype != bf:
        qs, ks, vs = qs.to(bf), ks.to(bf), vs.to(bf)
    qd = torch.empty((batch * H, n, d), dtype=bf, device=dev)
    kd = torch.empty((batch * HK, n, d), dtype=bf, device=dev)
    vd = torch.empty((batch * HK, n, d), dtype=bf, device=dev)
    out = torch.empty((batch, n, H * d), dtype=bf, device=dev)
    host_out = torch.empty((batch, n, H * d), dtype=bf, pin_memory=True)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    key = (g, n, d, mode, repr(search), repr(fixed_pattern), cal_window, q_est, H * d)
    plan = _PLAN_CACHE.get(key)
    if plan is None:  # host-side planning (search space, refinement, descriptor) once per shape
        plan = PrefillPlan(1, g, 1, n, d, mode, search=search, fixed_pattern=fixed_pattern,
                           cal_window=cal_window, q_est=q_est)
        plan.desc.out_ld = H * d
        if len(_PLAN_CACHE) > 64:
            _PLAN_CACHE.clear()
        _PLAN_CACHE[key] = plan
    ws = _workspace(plan.ws_bytes, dev)
    view = plan.views(ws)
    auto = mode == "auto"
    choice_all = torch.zeros(batch * H, dtype=torch.int32, device=dev)
    nc = len(plan.refined) if auto else 0
    err_all = torch.zeros((batch * H, max(nc, 1)), dtype=torch.float64, device=dev)
    cache = KvCache(batch, H, d, cfg.max_context, dtype=k.dtype, kv_heads=HK)
    comp = torch.cuda.current_stream()
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    sel = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(batch * HK)]
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_start.record(comp)
    h2d.wait_stream(comp)
    d2h.wait_stream(comp)
    pitch = H * d * 2
    tl = [] if _TIMELINE is not None else None  # (h2d done, compute start, compute end, d2h done) per group
    for grp in range(batch * HK):
        b, kh = divmod(grp, HK)
        h0 = b * H + kh * g
        with torch.cuda.stream(h2d):
            kd[grp].copy_(ks[grp], non_blocking=True)
            vd[grp].copy_(vs[grp], non_blocking=True)
            qd[h0:h0 + g].copy_(qs[h0:h0 + g], non_blocking=True)
            ready = torch.cuda.Event(enable_timing=tl is not None)
            ready.record(h2d)
        comp.wait_event(ready)
        if tl is not None:
            c0 = torch.cuda.Event(enable_timing=True)
            c0.record(comp)
        for x in (qd[h0:h0 + g], kd[grp], vd[grp]):
            _lib.call("sa_check_finite_bf16", x.data_ptr(), x.numel(), flag.data_ptr(), comp.cuda_stream)
        qg, kg, vg = qd[h0:h0 + g], kd[grp:grp + 1], vd[grp:grp + 1]
        og = out[b, :, kh * g * d:]
        sel[grp][0].record(comp)
        if auto:
            plan.select(qg, kg, ws)
        sel[grp][1].record(comp)
        plan.run(qg, kg, vg, og, ws)
        if auto:
            choice_all[h0:h0 + g].copy_(_wrap(view.choice, g, torch.int32))
            err_all[h0:h0 + g].copy_(_wrap(view.errors, g * _lib.MAX_CAND, torch.float64).view(g, _lib.MAX_CAND)[:, :nc])
        cache._k[b, kh, :n].copy_(kd[grp])
        cache._v[b, kh, :n].copy_(vd[grp])
        done = torch.cuda.Event(enable_timing=tl is not None)
        done.record(comp)
        d2h.wait_event(done)
        _lib.call("sa_memcpy2d_async", host_out.data_ptr() + (b * n * H + kh * g) * d * 2, pitch,
                  og.data_ptr(), pitch, g * d * 2, n, d2h.cuda_stream)
        if tl is not None:
            dd = torch.cuda.Event(enable_timing=True)
            dd.record(d2h)
            tl.append((ready, c0, done, dd))
    e_end.record(comp)
    comp.wait_stream(d2h)
    torch.cuda.synchronize()
    if tl is not None:
        _TIMELINE.append([[e_start.elapsed_time(ev) for ev in grp_evs] for grp_evs in tl])
    # one readback: finiteness flag, per-head choice and window errors
    small = torch.cat([flag.double(), choice_all.double(), err_all.reshape(-1)]).cpu().numpy() if auto else \
        flag.double().cpu().numpy()
    if int(small[0]):
        raise NonFiniteError("q, k or v contains NaN or Inf")
    cache.length = n
    cache._np = False
    if k.dtype != bf:  # the reference caches the rows as given (runtime.py:197), not their bf16 rounding
        cache._k[:, :, :n].copy_(k)
        cache._v[:, :, :n].copy_(v)
    if auto:
        nh = batch * H
        plans = plan.plans_from(small[1:1 + nh].astype(np.int64), small[1 + nh:].reshape(nh, nc), batch, H)
    else:
        plans = plan.plans_from(None, None, batch, H)
    select_s = sum(a.elapsed_time(z) for a, z in sel) / 1e3
    kernel_s = e_start.elapsed_time(e_end) / 1e3 - select_s
    outputs = host_out if q.dtype == bf else host_out.to(q.dtype)
    return PrefillResult(outputs=outputs, cache=cache, plans=plans, elapsed_s=time.perf_counter() - t0,
                         select_s=select_s, kernel_s=kernel_s)


def decode_step(q_new, k_new, v_new, cache: KvCache, cfg: ModelConfig) -> DecodeResult:
    """Append one token's k/v and attend its query over the whole cache (runtime.py:209-242).

    Decode is outside the prefill hot path: a split-K CUDA-core
    kernel (csrc/decode.cu) reads the cache's K/V in place once per kv head."""
    batch, length, kv_heads = _check_qkv(q_new, k_new, v_new, cfg)
    if length != 1:
        raise DimensionError(f"decode consumes exactly one token, got length {length}")
    if cache.length < 1:
        raise SparseAttnError("decode requires a non-empty cache; run prefill first")
    t0 = time.perf_counter()
    cache.append(k_new, v_new)
    n = cache.length
    H, d = cfg.n_heads, cfg.d_head
    dev = cache._k.device
    qt = torch.as_tensor(q_new) if not D.is_torch(q_new) else q_new
    q32 = qt.to(device=dev, dtype=torch.float32).reshape(batch * H, d).contiguous()
    kc, vc, cap = cache._k, cache._v, cache.capacity
    if kc.dtype not in (torch.float32, torch.bfloat16):  # other cache dtypes: a converted copy
        kc, vc, cap = kc[:, :, :n].float().contiguous(), vc[:, :, :n].float().contiguous(), n
    out = torch.empty((batch * H, d), dtype=torch.float32, device=dev)
    nbytes = int(_lib.load().sa_decode_workspace(batch, H, kv_heads, n, d))
    ws = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
    _lib.call("sa_decode_attn", batch, H, kv_heads, n, d, cap, 1.0 / math.sqrt(d), q32.data_ptr(),
              kc.data_ptr(), vc.data_ptr(), 0 if kc.dtype == torch.float32 else 1, out.data_ptr(),
              ws.data_ptr(), ws.numel(), D.stream())
    y = out.reshape(batch, 1, H * d)
    output = D.to_host_or_keep(y, q_new)
    torch.cuda.synchronize()
    return DecodeResult(output=output, cache=cache, elapsed_s=time.perf_counter() - t0)
