#!/usr/bin/env python
"""numpy float32 e2e phases (tool only): times prefill(numpy f32) at 32K and
its pieces in isolation (pinned-staged H2D of q/k/v, D2H of the output, the
np.empty first touch)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_06198_b200 import _device as D  # noqa: E402
from paper_2412_06198_b200 import runtime as R  # noqa: E402

n, H, HK, d = 32768, 32, 8, 128
rng = np.random.default_rng(0)
q = rng.uniform(-1, 1, (1, H, n, d)).astype(np.float32)
k = rng.uniform(-1, 1, (1, HK, n, d)).astype(np.float32)
v = rng.uniform(-1, 1, (1, HK, n, d)).astype(np.float32)
cfg = R.ModelConfig(n_heads=H, d_model=H * d, d_head=d, max_context=n)
dev = torch.device("cuda")


def t(f, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return sorted(ts)[len(ts) // 2]


for _ in range(2):
    R.prefill(q, k, v, cfg, mode="auto")
print("prefill numpy f32 e2e %.1f ms" % t(lambda: R.prefill(q, k, v, cfg, mode="auto"), 5))
qf = torch.empty((H, n, d), dtype=torch.float32, device=dev)
kf = torch.empty((HK, n, d), dtype=torch.float32, device=dev)
vf = torch.empty((HK, n, d), dtype=torch.float32, device=dev)
print("h2d_f32 q+k+v       %.1f ms" % t(lambda: D.h2d_f32([(k, kf), (v, vf), (q, qf)])))
out = np.empty((1, n, H * d), dtype=np.float32)
print("d2h_f32 (warm out)  %.1f ms" % t(lambda: D.d2h_f32(qf, out)))
print("d2h_f32 (fresh out) %.1f ms" % t(lambda: D.d2h_f32(qf, np.empty((1, n, H * d), dtype=np.float32))))
print("np.empty + fill     %.1f ms" % t(lambda: np.empty((1, n, H * d), dtype=np.float32).fill(0)))
print("torch threads", torch.get_num_threads())
# one kv group's output columns (n x 512 floats, 2 KB rows, row stride 16 KB)
pin = D.pinned_out(0, n * 512)
ot = torch.from_numpy(out)
print("strided group copy pinned->numpy (warm) %.2f ms" % t(lambda: ot[0, :, 0:512].copy_(pin.view(n, 512))))
fresh = lambda: torch.from_numpy(np.empty((1, n, H * d), dtype=np.float32))[0, :, 0:512].copy_(pin.view(n, 512))
print("strided group copy pinned->numpy (fresh) %.2f ms" % t(fresh))
print("contiguous 67 MB copy pinned->numpy (warm) %.2f ms" % t(lambda: ot.view(-1)[: n * 512].copy_(pin)))
import time as _t
for _ in range(2):
    torch.cuda.synchronize(); t0 = _t.perf_counter(); R.prefill(q, k, v, cfg, mode="auto"); torch.cuda.synchronize()
    print("prefill again %.1f ms" % (1e3 * (_t.perf_counter() - t0)))
