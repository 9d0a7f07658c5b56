"""World-size-2 gloo test of the head-parallel path's host logic: GQA-aligned
head sharding plus the all-gather into the reference (n, H*d) layout, with the
CPU oracle standing in for each rank's per-head compute."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sparse_oracle as O
        from paper_2412_06198_b200.multigpu import gather_heads, shard_heads

        H, HK, n, d = 8, 4, 96, 16
        q, k, v = (O.bf16_round(x) for x in O.synth_qkv_gqa(3, n, H, HK, d))
        qs, ks = shard_heads(rank, world, H, HK)
        out, _ = O.prefill(q[:, qs], k[:, ks], v[:, ks], "fixed", O.Tri(24, 2))
        full = gather_heads(torch.from_numpy(out[0]), world)
        if rank == 0:
            want, _ = O.prefill(q, k, v, "fixed", O.Tri(24, 2))
            result_q.put(float(np.abs(full.numpy() - want[0]).max()))
    finally:
        dist.destroy_process_group()


def test_two_rank_head_parallel_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=5) == 0.0


def test_shard_heads_layout():
    from paper_2412_06198_b200.multigpu import shard_heads

    assert shard_heads(0, 8, 32, 8) == (slice(0, 4), slice(0, 1))
    assert shard_heads(3, 4, 32, 8) == (slice(24, 32), slice(6, 8))
    with pytest.raises(ValueError):
        shard_heads(0, 3, 32, 8)
