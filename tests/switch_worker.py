"""Worker for tests/test_gpu_switches.py: one prefill per fixed pattern and one
auto layer on seeded inputs; prints a SHA-256 of every output (bf16 bytes), so
runs under different SA_* scheduling switches can be compared bit for bit."""
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_06198_b200 import runtime as R  # noqa: E402
from paper_2412_06198_b200.patterns import BlockSparse, Triangular, VerticalSlash  # noqa: E402

H, HK, D, N = 8, 2, 128, 4100


def main():
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    q, k, v = ((torch.rand((h, N, D), generator=g, device="cuda") * 2 - 1).bfloat16() for h in (H, HK, HK))
    out = {}
    cases = {"block8": ("fixed", BlockSparse(8, 2)), "block64": ("fixed", BlockSparse(64, 5)),
             "vs": ("fixed", VerticalSlash(300, 200)), "tri": ("fixed", Triangular(500, 16)),
             "dense": ("dense", None), "auto": ("auto", None)}
    for name, (mode, pat) in cases.items():
        plan = R.PrefillPlan(1, H, HK, N, D, mode, fixed_pattern=pat)
        ws = R._workspace(plan.ws_bytes, q.device)
        y = torch.empty((1, N, H * D), dtype=torch.bfloat16, device="cuda")
        if mode == "auto":
            plan.select(q, k, ws)
        plan.run(q, k, v, y, ws)
        torch.cuda.synchronize()
        out[name] = hashlib.sha256(y.view(torch.int16).cpu().numpy().tobytes()).hexdigest()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
