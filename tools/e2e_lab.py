#!/usr/bin/env python
"""Host<->device copy primitives for numpy float32 layers (tool only): pageable
copies, pinned staging (torch copy_ into a pinned pool), cudaHostRegister of
the numpy buffer in place.  Sizes: the 32K layer's q (536 MB) and the output."""
import os
import time

import numpy as np
import torch

dev = torch.device("cuda")
torch.ones(1, device=dev)
print("cpus", os.cpu_count(), "torch threads", torch.get_num_threads())
n = 32768
q = np.random.default_rng(0).random((1, 32, n, 128), dtype=np.float32)
nbytes = q.nbytes
out_np = np.empty_like(q)
dq = torch.empty(q.shape, dtype=torch.float32, device=dev)


def t(f, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


print(f"bytes {nbytes / 1e6:.0f} MB")
print("pageable H2D from_numpy copy_   %.1f ms" % t(lambda: dq.copy_(torch.from_numpy(q))))
print("pageable H2D .to(bf16) on device %.1f ms" % t(lambda: torch.from_numpy(q).to(dev, torch.bfloat16)))
pin = torch.empty(q.shape, dtype=torch.float32, pin_memory=True)
print("numpy -> pinned copy_ (host)     %.1f ms" % t(lambda: pin.copy_(torch.from_numpy(q))))
print("pinned H2D                      %.1f ms" % t(lambda: dq.copy_(pin, non_blocking=True)))
print("D2H pageable (numpy out)        %.1f ms" % t(lambda: torch.from_numpy(out_np).copy_(dq)))
print("D2H pinned                      %.1f ms" % t(lambda: pin.copy_(dq, non_blocking=True)))
print("pinned -> numpy copy_ (host)    %.1f ms" % t(lambda: torch.from_numpy(out_np).copy_(pin)))
print("np.copyto pinned->numpy         %.1f ms" % t(lambda: np.copyto(out_np, pin.numpy())))
cr = torch.cuda.cudart()


def reg():
    r = cr.cudaHostRegister(q.ctypes.data, nbytes, 0)
    assert int(r) == 0, r


def unreg():
    cr.cudaHostUnregister(q.ctypes.data)


for _ in range(2):
    t0 = time.perf_counter(); reg(); t1 = time.perf_counter()
    dq.copy_(torch.from_numpy(q), non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    unreg(); t3 = time.perf_counter()
    print(f"register {1e3 * (t1 - t0):.1f} ms  H2D {1e3 * (t2 - t1):.1f} ms  unregister {1e3 * (t3 - t2):.1f} ms")
# chunked staging with a thread pool: host copies overlap the DMA
import concurrent.futures as cf

CH = 32 << 20
nch = (nbytes + CH - 1) // CH
pool_bufs = [torch.empty(CH // 4, dtype=torch.float32, pin_memory=True) for _ in range(4)]
flat = torch.from_numpy(q).reshape(-1)
dflat = dq.reshape(-1)
ex = cf.ThreadPoolExecutor(4)
s = torch.cuda.Stream()


def staged():
    evs = [None] * 4
    futs = {}
    def fill(i):
        b = pool_bufs[i % 4]
        lo = i * (CH // 4); hi = min(flat.numel(), lo + CH // 4)
        b[: hi - lo].copy_(flat[lo:hi])
        return lo, hi
    for i in range(min(4, nch)):
        futs[i] = ex.submit(fill, i)
    for i in range(nch):
        lo, hi = futs.pop(i).result()
        with torch.cuda.stream(s):
            dflat[lo:hi].copy_(pool_bufs[i % 4][: hi - lo], non_blocking=True)
            e = torch.cuda.Event(); e.record(s)
        evs[i % 4] = e
        if i + 4 < nch:
            e.synchronize()
            futs[i + 4] = ex.submit(fill, i + 4)
    s.synchronize()


print("chunked staging 4 threads       %.1f ms" % t(staged))
torch.set_num_threads(os.cpu_count())
print("numpy -> pinned copy_ all thr   %.1f ms" % t(lambda: pin.copy_(torch.from_numpy(q))))
