#!/usr/bin/env python
"""Decode-step (ITL analog) device time at the Llama-3-8B
attention shape: sa_decode_attn over an n-row bf16 KV cache, CUDA events on
the launching stream, L2 flushed between reps (tool only)."""
import argparse
import ctypes
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_06198_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, nargs="+", default=[4096, 32768, 131072])
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
H, HK, D = 32, 8, 128
lib = _lib.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = []
for n in args.ctx:
    cap = n + 64
    kc = (torch.rand((1, HK, cap, D), device="cuda") * 2 - 1).bfloat16()
    vc = (torch.rand((1, HK, cap, D), device="cuda") * 2 - 1).bfloat16()
    q = torch.rand((H, D), device="cuda") * 2 - 1
    out = torch.empty((H, D), device="cuda")
    nb = int(lib.sa_decode_workspace(1, H, HK, n, D))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def step():
        _lib.call("sa_decode_attn", 1, H, HK, n, D, cap, 1.0 / math.sqrt(D), q.data_ptr(), kc.data_ptr(),
                  vc.data_ptr(), 1, out.data_ptr(), ws.data_ptr(), nb, st)

    for _ in range(3):
        step()
    times = []
    for _ in range(args.reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    times.sort()
    us = times[len(times) // 2] * 1e3
    byts = 2 * HK * n * D * 2
    # reference check of one head
    s = (kc[0, 0, :n].float() @ q[0]) / math.sqrt(D)
    want = torch.softmax(s, 0) @ vc[0, 0, :n].float()
    err = (out[0] - want).abs().max().item()
    res.append({"n": n, "us": round(us, 2), "kv_bytes": byts, "GB/s": round(byts / us / 1e3, 1), "max_err_h0": err})
    print(json.dumps(res[-1]))
