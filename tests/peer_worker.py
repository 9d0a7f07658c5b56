"""Worker for tests/test_gpu_multigpu_sim.py::test_fused_peer_exchange: one
rank of a torchrun job whose ranks all share cuda:0 (gloo for the small
collectives).  It runs multigpu.BalancedLayer.step_peers (output all-gather
fused into the attention epilogue over CUDA IPC mappings, ordered by the
device-side peer barrier) and prints whether its output equals the
single-GPU layer bit for bit."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_06198_b200 import runtime as R  # noqa: E402
from paper_2412_06198_b200.multigpu import BalancedLayer, PeerOutputs  # noqa: E402
from paper_2412_06198_b200.patterns import VerticalSlash  # noqa: E402

H, HK, D = 32, 8, 128


def main():
    n, mode = int(sys.argv[1]), sys.argv[2]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    q, k, v = ((torch.rand((h, n, D), generator=g, device="cuda") * 2 - 1).bfloat16() for h in (H, HK, HK))
    fixed = VerticalSlash(200, 150) if mode == "fixed" else None
    plan = R.PrefillPlan(1, H, HK, n, D, mode, fixed_pattern=fixed)
    ws = R._workspace(plan.ws_bytes, q.device)
    want = torch.empty((1, n, H * D), dtype=torch.bfloat16, device="cuda")
    if mode == "auto":
        plan.select(q, k, ws)
    plan.run(q, k, v, want, ws)
    layer = BalancedLayer(rank, world, H, HK, n, D, mode, fixed_pattern=fixed)
    peer = PeerOutputs(rank, world, n, H * D)
    ok = []
    for _ in range(2):  # the mapped buffers are reused across layers
        # no host barrier: step_peers' device-side entry barrier orders this
        # clear before any peer stores into the buffer
        peer.local.fill_(float("nan"))
        got = layer.step_peers(q, k, v, peer)
        ok.append(bool(torch.equal(got, want[0])))
    peer.close()
    print(json.dumps({"rank": rank, "world": world, "ok": ok, "peers": world - 1}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
