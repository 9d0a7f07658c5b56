#!/usr/bin/env python
"""Top-k lab (tool only): the VS score rows of an all-VS layer (the bench's
estimator_roofline inputs) -> time sa_topk_stable_f32 over all 2H rows, check
the result against numpy's stable argsort on a few rows and save a sample of
rows for offline study.

  python tools/topk_lab.py [n ...] [--save gpurun_out/topk_rows.npz]
"""
import argparse
import math
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_06198_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("ns", type=int, nargs="*", default=[32768, 131072])
ap.add_argument("--save", default=None)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--trace", action="store_true", help="per-CTA phase stamps (globaltimer) of one launch")
args = ap.parse_args()
H, HK, D = 32, 8, 128
dev = torch.device("cuda")
lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
saved = {}
for n in args.ns:
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    q = (torch.rand((H, n, D), generator=g, device=dev) * 2 - 1).bfloat16()
    k = (torch.rand((HK, n, D), generator=g, device=dev) * 2 - 1).bfloat16()
    scores = torch.empty((2, H, n), dtype=torch.float32, device=dev)
    wsb = int(lib.sa_score_tail_workspace(1, H, n, n))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _lib.call("sa_score_tail", 1, H, HK, n, 1 / math.sqrt(D), q.data_ptr(), k.data_ptr(), n - 64, n,
              scores[0].data_ptr(), scores[1].data_ptr(), 0, None, 0, ws.data_ptr(), wsb, st)
    kk = 3 * n // 64
    idx = torch.empty((2 * H, kk), dtype=torch.int32, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for it in range(args.reps + 3):
        ev[0].record()
        _lib.call("sa_topk_stable_f32", scores.data_ptr(), 2 * H, n, n, kk, idx.data_ptr(), kk, st)
        ev[1].record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
    if args.trace:
        import ctypes

        tr = torch.zeros((2 * H * 16, 16), dtype=torch.int64, device=dev)
        lib.sa_topk_trace_buffer(ctypes.c_void_p(tr.data_ptr()))
        _lib.call("sa_topk_stable_f32", scores.data_ptr(), 2 * H, n, n, kk, idx.data_ptr(), kk, st)
        torch.cuda.synchronize()
        lib.sa_topk_trace_buffer(ctypes.c_void_p(0))
        t = tr.cpu().numpy().astype(np.float64)
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        print(f"  trace: {len(t)} CTAs, start spread {(t[:, 0].max() - t0) / 1e3:.1f} us, "
              f"end {(t[:, 15].max() - t0) / 1e3:.1f} us")
        prev = t[:, 0]
        for e in range(1, 16):
            col = t[:, e]
            ok = col > 0
            if not ok.any():
                continue
            d = (col[ok] - prev[ok]) / 1e3
            print(f"    phase {e:2d}: median {np.median(d):6.2f} us  max {d.max():6.2f} us  (CTAs {ok.sum()})")
            prev = np.where(ok, col, prev)
    s = scores.reshape(2 * H, n).cpu().numpy()
    got = idx.cpu().numpy()
    bad = 0
    for r in (0, 1, H, 2 * H - 1):
        ref = np.sort(np.argsort(-s[r], kind="stable")[:kk])
        bad += int(not np.array_equal(ref, got[r]))
    print(f"n={n} rows={2 * H} k={kk} topk median {statistics.median(ts):.1f} us  min {min(ts):.1f}  mismatched rows {bad}")
    for r in (0, H):
        row = s[r]
        srt = np.sort(row)[::-1]
        print(f"  row {r}: min {row.min():.3e} max {row.max():.3e} kth {srt[kk - 1]:.3e} "
              f"median {np.median(row):.3e}  distinct {len(np.unique(row))}")
    saved[f"n{n}"] = s[[0, 1, H, H + 1]]
if args.save:
    np.savez_compressed(args.save, **saved)
