#!/usr/bin/env python
"""Per-CTA timeline of the VS estimator kernel (globaltimer stamps through
sa_vs_trace_buffer): pass-1 span, wait for the unit's merged statistics,
pass-2 span, per wave.   python tools/vs_trace.py [n] [heads] [kv_heads]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_06198_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
H = int(sys.argv[2]) if len(sys.argv) > 2 else 32
HK = int(sys.argv[3]) if len(sys.argv) > 3 else 8
g = torch.Generator(device="cuda")
g.manual_seed(1)
q = (torch.rand((H, n, 128), generator=g, device="cuda") * 2 - 1).bfloat16()
k = (torch.rand((HK, n, 128), generator=g, device="cuda") * 2 - 1).bfloat16()
col = torch.empty((H, n), dtype=torch.float32, device="cuda")
diag = torch.empty((H, n), dtype=torch.float32, device="cuda")
lib = _lib.load()
wsb = int(lib.sa_score_tail_workspace(1, H, n, n))
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count
tr = torch.zeros((sms + 4, 64), dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def run():
    _lib.call("sa_score_tail", 1, H, HK, n, 1 / np.sqrt(128), q.data_ptr(), k.data_ptr(), n - 64, n,
              col.data_ptr(), diag.data_ptr(), 0, None, 0, ws.data_ptr(), wsb, st)


for _ in range(3):
    run()
lib.sa_vs_trace_buffer(ctypes.c_void_p(tr.data_ptr()))
tr.zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
lib.sa_vs_trace_buffer(None)
print(f"n={n} H={H} HK={HK}: launch {e0.elapsed_time(e1) * 1e3:.1f} us (events, incl. build_units)")
trh = tr.cpu().numpy()
t = trh[:sms].reshape(sms, 8, 8).astype(np.float64)
tt = trh[sms:].reshape(-1, 8)[:32].astype(np.float64)  # CTA 0 wave 0 pass 1 per tile (clock64)
c0 = tt[0, 4]
print("CTA0 wave0 pass1 per tile (clk from first K ready): K ready | SE done (MMA) | SF seen | S loaded | computed")
for r in tt:
    if r[0] == 0:
        break
    print("   ", "  ".join(f"{x - c0:8.0f}" for x in (r[4], r[3], r[0], r[1], r[2])))
base = t[t > 0].min()
for v in range(8):
    w = t[:, v, :]
    act = w[:, 0] > 0
    if not act.any():
        break
    p1s, p1e, rdy, p2e = w[act, 0] - base, w[act, 1] - base, w[act, 3] - base, w[act, 4] - base
    mrel = w[:, 2][w[:, 2] > 0] - base
    sys.stdout.flush()
    print(f"wave {v}: CTAs {act.sum():3d}  P1 start {p1s.min() / 1e3:7.1f}..{p1s.max() / 1e3:7.1f}  "
          f"P1 end {p1e.min() / 1e3:7.1f}..{p1e.max() / 1e3:7.1f}  released {np.sort(mrel / 1e3).round(1)}  "
          f"ready seen {rdy[rdy > -base].min() / 1e3 if (rdy > -base).any() else 0:7.1f}..{rdy.max() / 1e3:7.1f}  "
          f"P2 end {p2e.min() / 1e3:7.1f}..{p2e.max() / 1e3:7.1f} us")
