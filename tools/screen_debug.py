#!/usr/bin/env python
"""Debug (tool only): run sa_block_index_bf16 once and dump the screen's tracked
values / bounds from the workspace: mode counts and sample rows."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_06198_b200 import _lib  # noqa: E402

n, b, k_b = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 8, 1)))
H = int(sys.argv[4]) if len(sys.argv) > 4 else 1
T = 4 if k_b <= 1 else 5 if k_b == 2 else 7 if k_b <= 4 else 11
lib = _lib.load()
rng = np.random.default_rng(11)
q = torch.from_numpy(rng.uniform(-1, 1, (H, n, 128)).astype(np.float32)).cuda().bfloat16()
rng = np.random.default_rng(12)
k = torch.from_numpy(rng.uniform(-1, 1, (1, n, 128)).astype(np.float32)).cuda().bfloat16()
nb = -(-n // b)
idx = torch.empty((H, nb, k_b + 1), dtype=torch.int32, device="cuda")
ro = torch.empty((H, nb + 1), dtype=torch.int32, device="cuda")
wsb = int(lib.sa_block_index_workspace(1, H, 1, n, b, k_b))
ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(3):
    ev[0].record()
    _lib.call("sa_block_index_bf16", 1, H, 1, n, b, k_b, q.data_ptr(), k.data_ptr(), idx.data_ptr(), ro.data_ptr(),
              ws.data_ptr(), wsb, st)
    ev[1].record()
    torch.cuda.synchronize()
    print("time us", ev[0].elapsed_time(ev[1]) * 1e3)
print("rows/head", nb)
al = lambda x: (x + 255) & ~255
def pool_bytes(G):
    gb = G * nb
    return gb * 256 + gb * 512 + al(gb * 8) + al(G * 8)
base = (ws.data_ptr() + 1023) & ~1023
o = base - ws.data_ptr() + pool_bytes(H) + pool_bytes(1)
rows = H * nb
o += al(rows * T * 4) * 3 + al(rows * 4) * 2
w = ws[o: o + 4 * (rows + 1)].view(torch.int32).cpu().numpy()
cnt = int(w[0])
print("rescan rows", cnt, "of", rows)
if cnt:
    rr = np.sort(w[1: 1 + cnt])
    print("  sample (head, gq):", [(int(x) // nb, int(x) % nb) for x in rr[:12]])
