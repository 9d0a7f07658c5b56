#!/usr/bin/env python
"""Debug (tool only): the wide_range case of tests/test_gpu_block_screen.py —
dump the screen's tracked values / U / E for a few rows and the rescan list."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import sparse_oracle as O  # noqa: E402
from paper_2412_06198_b200 import _lib  # noqa: E402

n, b, k_b = 2048, 8, int(sys.argv[1]) if len(sys.argv) > 1 else 3
T = 4 if k_b <= 1 else 5 if k_b == 2 else 7 if k_b <= 4 else 11
rng = np.random.default_rng(40)
q = O.bf16_round(rng.uniform(-1, 1, (1, n, 128)).astype(np.float32))[0]
rng = np.random.default_rng(41)
k = O.bf16_round(rng.uniform(-1, 1, (1, n, 128)).astype(np.float32))[0]
q = O.bf16_round(q * 1e5)
mag = 10.0 ** np.repeat(np.random.default_rng(3).uniform(-6, 2, n // b), b)
k = O.bf16_round(k * mag[:, None].astype(np.float32))
lib = _lib.load()
nb = n // b
qd = torch.from_numpy(q[None]).cuda().bfloat16().contiguous()
kd = torch.from_numpy(k[None]).cuda().bfloat16().contiguous()
idx = torch.empty((nb, k_b + 1), dtype=torch.int32, device="cuda")
ro = torch.empty(nb + 1, dtype=torch.int32, device="cuda")
wsb = int(lib.sa_block_index_workspace(1, 1, 1, n, b, k_b))
ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
_lib.call("sa_block_index_bf16", 1, 1, 1, n, b, k_b, qd.data_ptr(), kd.data_ptr(), idx.data_ptr(), ro.data_ptr(),
          ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
al = lambda x: (x + 255) & ~255
pb = nb * 256 + nb * 512 + al(nb * 8) + al(8)
base = ((ws.data_ptr() + 1023) & ~1023) - ws.data_ptr()
w = ws.cpu().numpy()
so = base + 2 * pb
rows = nb
tv = w[so: so + rows * T * 4].view(np.float32).reshape(rows, T)
o2 = so + al(rows * T * 4)
ti = w[o2: o2 + rows * T * 4].view(np.int32).reshape(rows, T)
o3 = o2 + al(rows * T * 4)
te = w[o3: o3 + rows * 4].view(np.float32)
o4 = o3 + al(rows * 4)
tu = w[o4: o4 + rows * 4].view(np.float32)
o5 = o4 + al(rows * 4)
cnt = int(w[o5: o5 + 4].view(np.int32)[0])
lst = w[o5 + 4: o5 + 4 + 4 * cnt].view(np.int32)
print("rescan count", cnt, sorted(lst.tolist())[:20])
qb, kb = O.block_mean(q.astype(np.float64), b), O.block_mean(k.astype(np.float64), b)
logit = qb @ kb.T
got = idx.cpu().numpy()
for g in (0, 1, 2, 5, 8, 9, 40, 100):
    order = np.argsort(-logit[g, : g + 1], kind="stable")[:5]
    print(g, "tv", tv[g], "ti", ti[g], "E", te[g], "U", tu[g], "| got", got[g], "exact top", order,
          logit[g, order])
