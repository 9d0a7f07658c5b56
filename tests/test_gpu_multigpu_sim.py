"""The balanced head-parallel layer (multigpu.BalancedLayer) with
every rank played in turn on one GPU and the two all-gathers emulated by
stacking: the assembled output must equal the single-GPU layer bit for bit
(each (head, query tile) is computed from the same realised index by the same
kernel), and the item deal must be a partition of all items with balanced
executed tiles."""
import re
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

H, HK, D = 32, 8, 128


def _inputs(n, seed=4):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return [(torch.rand((h, n, D), generator=g, device="cuda") * 2 - 1).bfloat16() for h in (H, HK, HK)]


@pytest.mark.parametrize("n,world,mode", [(4096, 2, "auto"), (4096, 8, "auto"), (3000, 4, "dense"),
                                          (32768, 8, "auto"), (2500, 8, "fixed")])
def test_balanced_layer_matches_single_gpu(n, world, mode):
    from paper_2412_06198_b200 import runtime as R
    from paper_2412_06198_b200.multigpu import BalancedLayer
    from paper_2412_06198_b200.patterns import VerticalSlash

    fixed = VerticalSlash(200, 150) if mode == "fixed" else None
    q, k, v = _inputs(n)
    plan = R.PrefillPlan(1, H, HK, n, D, mode, fixed_pattern=fixed)
    ws = R._workspace(plan.ws_bytes, q.device)
    want = torch.empty((1, n, H * D), dtype=torch.bfloat16, device="cuda")
    if mode == "auto":
        plan.select(q, k, ws)
    plan.run(q, k, v, want, ws)
    ranks = [BalancedLayer(r, world, H, HK, n, D, mode, fixed_pattern=fixed) for r in range(world)]
    packed = torch.stack([rk.estimate(q, k, v) for rk in ranks])
    for rk in ranks:
        rk.load_index(packed)
    blocks = torch.stack([rk.attend(q, k, v) for rk in ranks])
    got = ranks[0].assemble(blocks)
    torch.cuda.synchronize()
    assert torch.equal(got, want[0])
    # the deal is a partition of every (head, query tile) item, heaviest-first balanced
    items = torch.cat(ranks[0].owner_items).cpu().numpy()
    np.testing.assert_array_equal(np.sort(items), np.arange(H * ranks[0].nqt))
    cnt = R._wrap(plan.views(ws).tile_cnt, H * ranks[0].nqt, torch.int32).cpu().numpy()
    loads = [cnt[o.cpu().numpy()].sum() for o in ranks[0].owner_items]
    assert max(loads) <= 1.05 * cnt.sum() / world + cnt.max()


@pytest.mark.parametrize("exchange", ["nccl", "peer"])
def test_bench_two_ranks_share_one_gpu(exchange):
    """Dry run of `bench.py --gpus 2` under torchrun: two ranks on the one GPU
    with gloo collectives (SA_DIST_BACKEND=gloo) through the balanced layer
    (output exchange by all-gather, or fused into the attention epilogue over
    CUDA IPC: SA_MG_EXCHANGE=peer), ending in one JSON line from rank 0."""
    import json
    import os
    import socket
    import subprocess
    import sys

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SA_DIST_BACKEND="gloo", SA_MG_EXCHANGE=exchange)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--ctx", "8192", "--steps", "3",
           "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-ttft"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2
    assert lines[0]["details"]["parallelism"].startswith("balanced head-parallel x2")
    assert ("fused all-gather" in lines[0]["details"]["parallelism"]) == (exchange == "peer")


@pytest.mark.parametrize("world,n,mode", [(2, 4096, "auto"), (4, 2500, "fixed")])
def test_fused_peer_exchange(world, n, mode):
    """The fused output all-gather: `world` ranks share the GPU, map each
    other's output buffers over CUDA IPC and store their rows into all of them
    from the attention epilogue; every rank's buffer must equal the
    single-GPU layer bit for bit (twice: the mappings are reused)."""
    import json
    import os
    import socket
    import subprocess
    import sys

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(port), "tests/peer_worker.py", str(n), mode]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    # ranks share one stdout pipe: their lines can arrive concatenated
    lines = [json.loads(x) for x in re.findall(r"\{[^{}]*\}", r.stdout)]
    assert sorted(x["rank"] for x in lines) == list(range(world))
    assert all(x["ok"] == [True, True] for x in lines), lines
