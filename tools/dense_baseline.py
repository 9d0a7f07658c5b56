#!/usr/bin/env python
"""Dense causal prefill baselines on the same bf16 tensors:
flashinfer's sm100 FMHA and torch SDPA.  Library code, timed for comparison only."""
import argparse
import time

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, default=32768)
args = ap.parse_args()
n, H, HK, D = args.ctx, 32, 8, 128
q = torch.randn(n, H, D, dtype=torch.bfloat16, device="cuda")
k = torch.randn(n, HK, D, dtype=torch.bfloat16, device="cuda")
v = torch.randn(n, HK, D, dtype=torch.bfloat16, device="cuda")
flops = 4 * D * H * n * (n + 1) / 2


def bench(fn, name, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name}: {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s (causal-useful)")


try:
    import flashinfer

    for backend in ("cutlass", "trtllm-gen", "fa2", "auto"):
        try:
            fn = lambda: flashinfer.single_prefill_with_kv_cache(q, k, v, causal=True, backend=backend)  # noqa: E731
            bench(fn, f"flashinfer single_prefill backend={backend}")
        except Exception as e:  # noqa: BLE001
            print(f"flashinfer backend={backend}: {type(e).__name__}: {str(e)[:120]}")
except Exception as e:  # noqa: BLE001
    print("flashinfer unavailable:", e)
qt, kt, vt = (x.transpose(0, 1).unsqueeze(0) for x in (q, k, v))
try:
    fn = lambda: torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=True, enable_gqa=True)  # noqa: E731
    bench(fn, "torch sdpa")
except Exception as e:  # noqa: BLE001
    print("sdpa:", e)
