#!/usr/bin/env python
"""Debug (tool only): k_b = 1 block index (block_top1_kernel + refine) on
uniform data: time, refine / rescan row counts, candidates-per-row histogram.
    python tools/top1_debug.py [n] [b] [heads] [kv_heads]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_06198_b200 import _lib  # noqa: E402

n, b, H, HK = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (32768, 8, 8, 2)))
k_b, T = 1, 16
lib = _lib.load()
rng = np.random.default_rng(11)
q = torch.from_numpy(rng.uniform(-1, 1, (H, n, 128)).astype(np.float32)).cuda().bfloat16()
k = torch.from_numpy(rng.uniform(-1, 1, (HK, n, 128)).astype(np.float32)).cuda().bfloat16()
nb = -(-n // b)
idx = torch.empty((H, nb, 2), dtype=torch.int32, device="cuda")
ro = torch.empty((H, nb + 1), dtype=torch.int32, device="cuda")
wsb = int(lib.sa_block_index_workspace(1, H, HK, n, b, k_b))
ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(4):
    ev[0].record()
    _lib.call("sa_block_index_bf16", 1, H, HK, n, b, k_b, q.data_ptr(), k.data_ptr(), idx.data_ptr(), ro.data_ptr(),
              ws.data_ptr(), wsb, st)
    ev[1].record()
    torch.cuda.synchronize()
    print("time us", round(ev[0].elapsed_time(ev[1]) * 1e3, 1))
al = lambda x: (x + 255) & ~255
def pool_bytes(G):
    gb = G * nb
    return gb * 256 + gb * 512 + al(gb * 8) + al(G * 8)
base = (ws.data_ptr() + 1023) & ~1023
o = base - ws.data_ptr() + pool_bytes(H) + pool_bytes(HK)
rows = H * nb
w = lambda off, cnt: ws[off: off + 4 * cnt].view(torch.int32).cpu().numpy()
o_ti = o + al(rows * T * 4)
o_resc = o + al(rows * T * 4) * 3 + al(rows * 4) * 2
print("rows", rows, "refine", int(w(o_ti, 1)[0]), "rescan", int(w(o_resc, 1)[0]))
