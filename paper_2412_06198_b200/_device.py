"""Device plumbing for the host mirror: CUDA checks, staging to bf16 head tiles,
streams and result conversion.  PyTorch is used only for device memory and
streams; all compute runs in the C-ABI library (``_lib``)."""

from __future__ import annotations

import numpy as np
import torch

from .errors import DimensionError

HEAD_DIM = 128


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2412_06198_b200 runs on a CUDA B200 only (sm_100a); no CPU fallback exists"
        )
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def shape_of(x):
    return tuple(x.shape)


def stage_heads(x, name: str = "x") -> torch.Tensor:
    """(G, n, d) numpy/torch -> contiguous bf16 cuda (G, n, 128), zero-padded in d.

    Zero columns leave every logit unchanged; the caller passes the original
    1/sqrt(d) as the scale and slices the output back to d."""
    dev = require_cuda()
    t = torch.as_tensor(x) if not is_torch(x) else x
    if t.dim() != 3:
        raise DimensionError(f"{name} must be (heads, n, d), got {tuple(t.shape)}")
    g, n, d = t.shape
    if d > HEAD_DIM:
        raise DimensionError(f"head_dim {d} exceeds the {HEAD_DIM} supported by the B200 kernels")
    t = t.to(device=dev, dtype=torch.bfloat16, non_blocking=True)
    if d < HEAD_DIM:
        t = torch.nn.functional.pad(t, (0, HEAD_DIM - d))
    return t.contiguous()


def to_host_or_keep(t: torch.Tensor, like, dtype=None):
    """Return numpy if the caller passed numpy (dtype preserved), else a torch tensor."""
    if is_torch(like):
        return t.to(dtype=like.dtype if dtype is None else dtype)
    out = t.detach().float().cpu().numpy()
    want = np.asarray(like).dtype if dtype is None else dtype
    if np.issubdtype(np.dtype(want), np.floating):
        out = out.astype(want, copy=False)
    return out


def all_finite(x) -> bool:
    if is_torch(x):
        return bool(torch.isfinite(x).all().item())
    return bool(np.isfinite(np.asarray(x)).all())


# ---------------------------------------------------------------- host copies
# numpy (pageable) <-> device in chunks through a small pool of pinned buffers:
# the host-side copy of chunk i (torch's multi-threaded copy_, GIL released)
# overlaps the DMA of chunk i - 1.  Pageable cudaMemcpy of the whole array
# measured 47 ms for 537 MB; staged, the DMA runs at the PCIe rate.
_CHUNK = 8 << 20  # float32 elements per staging buffer (32 MB)
_PINNED: list = []
_COPY_STREAM = {}


def _pinned(i: int) -> torch.Tensor:
    while len(_PINNED) <= i:
        _PINNED.append(torch.empty(_CHUNK, dtype=torch.float32, pin_memory=True))
    return _PINNED[i]


def _copy_stream() -> torch.cuda.Stream:
    d = torch.cuda.current_device()
    if d not in _COPY_STREAM:
        _COPY_STREAM[d] = torch.cuda.Stream()
    return _COPY_STREAM[d]


def h2d_f32(pairs) -> None:
    """[(numpy float32 C-contiguous array, device float32 tensor of the same
    size), ...]: chunked, double-buffered copies on a copy stream; the current
    stream waits for them."""
    cs = _copy_stream()
    cs.wait_stream(torch.cuda.current_stream())
    ev = [None, None]
    i = 0
    for src, dst in pairs:
        s = torch.from_numpy(src.reshape(-1))
        d = dst.reshape(-1)
        for lo in range(0, s.numel(), _CHUNK):
            hi = min(s.numel(), lo + _CHUNK)
            slot = i & 1
            if ev[slot] is not None:
                ev[slot].synchronize()  # the DMA that last read this buffer is done
            buf = _pinned(slot)[: hi - lo]
            buf.copy_(s[lo:hi])
            with torch.cuda.stream(cs):
                d[lo:hi].copy_(buf, non_blocking=True)
                e = torch.cuda.Event()
                e.record(cs)
            ev[slot] = e
            i += 1
    torch.cuda.current_stream().wait_stream(cs)


def d2h_f32(src: torch.Tensor, out: np.ndarray) -> None:
    """device float32 tensor -> preallocated numpy float32 array (same size):
    chunked D2H into pinned buffers on a copy stream, each chunk copied out on
    the host while the next one is in flight."""
    cs = _copy_stream()
    cs.wait_stream(torch.cuda.current_stream())
    s = src.reshape(-1)
    o = torch.from_numpy(out.reshape(-1))
    bounds = [(lo, min(s.numel(), lo + _CHUNK)) for lo in range(0, s.numel(), _CHUNK)]
    ev = []
    for i, (lo, hi) in enumerate(bounds[:2]):
        with torch.cuda.stream(cs):
            _pinned(i & 1)[: hi - lo].copy_(s[lo:hi], non_blocking=True)
            e = torch.cuda.Event()
            e.record(cs)
        ev.append(e)
    for i, (lo, hi) in enumerate(bounds):
        ev[i].synchronize()
        o[lo:hi].copy_(_pinned(i & 1)[: hi - lo])
        if i + 2 < len(bounds):
            lo2, hi2 = bounds[i + 2]
            with torch.cuda.stream(cs):
                _pinned(i & 1)[: hi2 - lo2].copy_(s[lo2:hi2], non_blocking=True)
                e = torch.cuda.Event()
                e.record(cs)
            ev.append(e)
