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
