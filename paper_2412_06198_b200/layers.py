"""Multi-layer prefill: L attention layers of one prompt back to back (SURVEY
§8(f)1, the C4 TTFT analog of BASELINE.json configs[3]).

The reference has one layer per ``runtime.prefill`` call (runtime.py:134-206),
each filling its KvCache (runtime.py:57-90, 197) inside the timed region.  A
TTFT over L layers is L such calls; here they run as one stream-ordered
sequence (one CUDA graph on a single GPU) sharing one prefill workspace: every
layer runs AttnMatrices' finiteness scan and fills its own device-resident
KvCache inside ``sa_prefill`` (side stream beside the estimators), its
per-head choice and window errors are kept per layer, and everything is read
back once at the end.  Like the reference (runtime.py:1-10) the
projections between layers are not part of the path: each layer takes its
own q / k / v.

With N > 1 ranks each rank runs its GQA group of every layer
(multigpu.shard_heads) and layer l's output all-gather (NCCL, a second
stream) overlaps layer l + 1's compute.
"""

from __future__ import annotations

import time
import numpy as np
import torch

from . import _device as D
from . import _lib
from .errors import DimensionError, NonFiniteError
from .runtime import KvCache, ModelConfig, PrefillPlan, PrefillResult, _check_qkv

__all__ = ["LayerStack", "prefill_layers"]


class LayerStack:
    """L layers of (batch, heads, length) attention on this rank's heads.

    ``run(q_layers, k_layers, v_layers)`` takes per-layer device tensors of
    shape (batch, heads, length, 128) bf16 (k / v with kv_heads heads) and
    writes ``outputs[l]`` = (batch, length, heads * 128); ``caches[l]`` hold
    the layer's k / v rows.  ``graph()`` captures ``run`` for fixed input
    buffers (single rank)."""

    def __init__(self, n_layers: int, cfg: ModelConfig, kv_heads: int, length: int, batch: int = 1,
                 mode: str = "auto", search=None, fixed_pattern=None, cal_window: int = 64, q_est: int = 64,
                 world: int = 1, group=None, device=None):
        if n_layers < 1:
            raise DimensionError(f"need at least one layer, got {n_layers}")
        if cfg.d_head != D.HEAD_DIM:
            raise DimensionError(f"LayerStack runs d_head = {D.HEAD_DIM} layers, got {cfg.d_head}")
        if length > cfg.max_context:
            raise DimensionError(f"length {length} exceeds max_context {cfg.max_context}")
        self.L, self.cfg, self.batch, self.n = n_layers, cfg, batch, length
        self.world, self.group = world, group
        if world > 1 and (kv_heads % world or cfg.n_heads % world):
            raise DimensionError(f"world={world} must divide kv_heads={kv_heads}")
        self.heads = cfg.n_heads // world  # this rank's heads (GQA-group aligned)
        self.kv_heads = kv_heads // world
        dev = D.require_cuda() if device is None else device
        self.dev = dev
        self.plan = PrefillPlan(batch, self.heads, self.kv_heads, length, cfg.d_head, mode, search=search,
                                fixed_pattern=fixed_pattern, cal_window=cal_window, q_est=q_est)
        self.ws = torch.empty(self.plan.ws_bytes, dtype=torch.uint8, device=dev)
        self.view = self.plan.views(self.ws)
        hh = self.plan.hh
        self.outputs = [torch.empty((batch, length, self.heads * D.HEAD_DIM), dtype=torch.bfloat16, device=dev)
                        for _ in range(n_layers)]
        self.finals = None
        if world > 1:
            self.finals = [torch.empty((batch, length, cfg.n_heads * D.HEAD_DIM), dtype=torch.bfloat16,
                                       device=dev) for _ in range(n_layers)]
        self.caches = [KvCache(batch, self.heads, cfg.d_head, cfg.max_context, dtype=torch.bfloat16,
                               kv_heads=self.kv_heads) for _ in range(n_layers)]
        self.flags = torch.zeros(n_layers, dtype=torch.int32, device=dev)
        # per-layer copy of the selection (choice, window errors) of the shared workspace
        self.choice = torch.zeros((n_layers, hh), dtype=torch.int32, device=dev)
        self.errors = torch.zeros((n_layers, hh * _lib.MAX_CAND), dtype=torch.float64, device=dev)
        self._comm = torch.cuda.Stream(device=dev) if world > 1 else None
        self._events = [torch.cuda.Event() for _ in range(n_layers)] if world > 1 else None

    def _layer(self, l: int, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> None:
        p, d = self.plan, self.plan.desc
        c = self.caches[l]
        d.check_flag = self.flags[l:l + 1].data_ptr()
        d.cache_k, d.cache_v, d.cache_capacity = c._k.data_ptr(), c._v.data_ptr(), c.capacity
        if p.mode == "auto":
            p.select(q, k, self.ws)
        p.run(q, k, v, self.outputs[l], self.ws)
        d.check_flag = d.cache_k = d.cache_v = None
        d.cache_capacity = 0
        if p.mode == "auto":
            hh = p.hh
            self.choice[l].copy_(self._ws_view(self.view.choice, hh, torch.int32))
            nc = len(p.refined)  # only the written columns of the error table
            self.errors[l].view(hh, _lib.MAX_CAND)[:, :nc].copy_(
                self._ws_view(self.view.errors, hh * _lib.MAX_CAND, torch.float64).view(hh, _lib.MAX_CAND)[:, :nc])

    def _ws_view(self, ptr: int, count: int, dtype) -> torch.Tensor:
        off = ptr - self.ws.data_ptr()
        esize = torch.empty(0, dtype=dtype).element_size()
        return self.ws[off: off + count * esize].view(dtype)

    def run(self, q_layers, k_layers, v_layers) -> None:
        """Stream-ordered L layers (no host synchronisation)."""
        from .multigpu import gather_heads

        if not (len(q_layers) == len(k_layers) == len(v_layers) == self.L):
            raise DimensionError(f"expected {self.L} layers of q / k / v")
        cur = torch.cuda.current_stream(self.dev)
        for l in range(self.L):
            q, k, v = (x.reshape(-1, self.n, D.HEAD_DIM) for x in (q_layers[l], k_layers[l], v_layers[l]))
            self._layer(l, q, k, v)
            if self.world > 1:  # layer l's all-gather beside layer l + 1's compute
                self._events[l].record(cur)
                self._comm.wait_event(self._events[l])
                with torch.cuda.stream(self._comm):
                    for b in range(self.batch):
                        gather_heads(self.outputs[l][b], self.world, group=self.group, out=self.finals[l][b])
        if self.world > 1:
            cur.wait_stream(self._comm)

    def graph(self, q_layers, k_layers, v_layers) -> torch.cuda.CUDAGraph:
        """CUDA graph of ``run`` on these input buffers (single rank)."""
        if self.world > 1:
            raise DimensionError("LayerStack.graph is single-rank; N > 1 runs eagerly")
        side = torch.cuda.Stream(device=self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            self.run(q_layers, k_layers, v_layers)  # warm the lazy per-kernel attributes
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=side):
                self.run(q_layers, k_layers, v_layers)
        torch.cuda.current_stream(self.dev).wait_stream(side)
        return g

    def finish(self):
        """One readback (finiteness flags, every layer's choice and errors):
        raises NonFiniteError for a layer with NaN / Inf inputs, else returns
        the per-layer plans ([batch][heads] HeadPlan lists)."""
        parts = [self.flags.double()]
        if self.plan.mode == "auto":
            parts += [self.choice.double().reshape(-1), self.errors.reshape(-1)]
        small = torch.cat(parts).cpu().numpy()
        bad = np.nonzero(small[: self.L])[0]
        if len(bad):
            raise NonFiniteError(f"layer {int(bad[0])}: q, k or v contains NaN or Inf")
        for c in self.caches:
            c.length = self.n
            c._np = False
        hh = self.plan.hh
        plans = []
        for l in range(self.L):
            if self.plan.mode == "auto":
                ch = small[self.L + l * hh: self.L + (l + 1) * hh].astype(np.int64)
                base = self.L + self.L * hh + l * hh * _lib.MAX_CAND
                er = small[base: base + hh * _lib.MAX_CAND].reshape(hh, _lib.MAX_CAND)
                plans.append(self.plan.plans_from(ch, er, self.batch, self.heads))
            else:
                plans.append(self.plan.plans_from(None, None, self.batch, self.heads))
        return plans


def prefill_layers(q_layers, k_layers, v_layers, cfg: ModelConfig, search=None, mode: str = "dense", *,
                   fixed_pattern=None, cal_window: int = 64, q_est: int = 64) -> list[PrefillResult]:
    """``runtime.prefill`` for L layers of one prompt, back to back on the
    device (one result per layer; every result's ``elapsed_s`` is the whole
    stack's wall time, the TTFT analog).  Inputs: sequences of per-layer
    (batch, heads, length, d_head) arrays or tensors (k / v may have
    n_heads / g heads); device bf16 tensors are used in place, anything else
    is staged to bf16 on the GPU first."""
    from .runtime import prefill, stage_layer

    if not (len(q_layers) == len(k_layers) == len(v_layers)) or not q_layers:
        raise DimensionError("need the same positive number of q, k and v layers")
    batch, length, kv_heads = _check_qkv(q_layers[0], k_layers[0], v_layers[0], cfg)
    if length > cfg.max_context:
        raise DimensionError(f"length {length} exceeds max_context {cfg.max_context}")
    if cfg.d_head != D.HEAD_DIM:  # the fused stack fills 128-wide bf16 caches; narrower heads go layer by layer
        t0 = time.perf_counter()
        res = [prefill(q, k, v, cfg, search, mode, fixed_pattern=fixed_pattern, cal_window=cal_window,
                       q_est=q_est) for q, k, v in zip(q_layers, k_layers, v_layers)]
        for r in res:
            r.elapsed_s = time.perf_counter() - t0
        return res
    for l in range(1, len(q_layers)):
        if _check_qkv(q_layers[l], k_layers[l], v_layers[l], cfg) != (batch, length, kv_heads):
            raise DimensionError(f"layer {l} has a different shape from layer 0")
    t0 = time.perf_counter()
    staged = [stage_layer(q, k, v) for q, k, v in zip(q_layers, k_layers, v_layers)]
    stack = LayerStack(len(q_layers), cfg, kv_heads, length, batch=batch, mode=mode, search=search,
                       fixed_pattern=fixed_pattern, cal_window=cal_window, q_est=q_est)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    stack.run([s[0] for s in staged], [s[1] for s in staged], [s[2] for s in staged])
    e1.record()
    plans = stack.finish()
    torch.cuda.synchronize()
    elapsed = time.perf_counter() - t0
    kernel_s = e0.elapsed_time(e1) / 1e3
    like = q_layers[0]
    results = []
    keep_bf16 = D.is_torch(k_layers[0]) and k_layers[0].dtype == torch.bfloat16
    for l in range(len(q_layers)):
        if not keep_bf16:  # the reference caches the rows as given (runtime.py:197)
            kl = k_layers[l]
            cdt = kl.dtype if D.is_torch(kl) else np.asarray(kl).dtype
            stack.caches[l] = KvCache(batch, cfg.n_heads, cfg.d_head, cfg.max_context, dtype=cdt,
                                      kv_heads=kv_heads)
            stack.caches[l].append(k_layers[l], v_layers[l])
        y = stack.outputs[l]
        if cfg.d_head < D.HEAD_DIM:
            y = y.view(batch, length, cfg.n_heads, D.HEAD_DIM)[..., : cfg.d_head].reshape(batch, length,
                                                                                        cfg.d_model)
        results.append(PrefillResult(outputs=D.to_host_or_keep(y, like), cache=stack.caches[l], plans=plans[l],
                                     elapsed_s=elapsed, select_s=0.0, kernel_s=kernel_s))
    return results
