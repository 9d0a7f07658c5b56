"""Head-parallel prefill across ranks.

Heads have no cross-head math (runtime.py:174-195), so a layer shards by GQA
group: rank r of N owns kv heads [r*HK/N, (r+1)*HK/N) and their query heads.
The only collective is one all-gather of the per-rank outputs, permuted into
the reference's (B, n, H*d) layout (runtime.py:194).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_heads(rank: int, world: int, heads: int, kv_heads: int):
    """(q-head slice, kv-head slice) owned by `rank` (GQA-group aligned)."""
    if kv_heads % world or heads % kv_heads:
        raise ValueError(f"world={world} must divide kv_heads={kv_heads} (and kv_heads | heads)")
    hk = kv_heads // world
    g = heads // kv_heads
    return slice(rank * hk * g, (rank + 1) * hk * g), slice(rank * hk, (rank + 1) * hk)


def gather_heads(local: torch.Tensor, world: int, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather per-rank outputs (n, H_local*d) into (n, world*H_local*d),
    rank-major head order == global head order."""
    n, w = local.shape
    if world == 1:
        return local
    if out is None:
        out = torch.empty((n, world * w), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        buf = torch.empty((world, n, w), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(buf, local.contiguous(), group=group)
        out.view(n, world, w).copy_(buf.permute(1, 0, 2))
    else:  # gloo (CPU tests)
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local.contiguous(), group=group)
        out.view(n, world, w).copy_(torch.stack(parts, 1))
    return out
