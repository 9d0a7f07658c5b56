#!/usr/bin/env python
"""bench.py — one Llama-3-8B-shape sparse prefill attention layer on B200.

Workload (BASELINE.json configs[1]): 32 query / 8 kv heads, head_dim 128,
one layer at 32K tokens (``--ctx``), bf16, SparseAccelerate ``auto`` mode
(per-head windowed selection -> estimators -> index -> tcgen05 sparse
attention).  A "step" is one layer over one batch of synthetic inputs
(uniform [-1, 1], rng([seed, ctx]), GQA draw order of SURVEY §7.3).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--ctx 32768] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): heads shard GQA-group-aligned across
ranks (8/N kv heads each) and the per-head outputs are all-gathered over NCCL
into the reference's (B, L, H*d) layout; every rank times the same steps and
rank 0 reports the max.  ``value`` is ms per layer (lower is better) with
inputs resident in HBM; ``e2e`` is the same metric through the public
``prefill`` API with host inputs (H2D) and the output read back (D2H).
``--impl reference`` times the CPU oracle port of the reference algorithm
(oracle/sparse_oracle.py) on the box's host cores; it is the reference arm.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

H, HK, D = 32, 8, 128
METRIC = "TTFT & sparse-attn ms/layer at 32K/128K; tensor-pipe % of bf16 peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--mode", default="auto", help="auto | dense | triangular | vertical-slash | block-sparse")
    ap.add_argument("--pattern", default=None,
                    help="fixed pattern for every head, e.g. block:8:1, vs:1536:1536, tri:3072:0 (overrides --mode)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-128k", action="store_true", help="skip the 131072-token sub-record")
    ap.add_argument("--no-est", action="store_true", help="skip the all-VS estimator roofline block")
    ap.add_argument("--no-ttft", action="store_true", help="skip the 32-layer 64K TTFT sub-record")
    ap.add_argument("--no-c5", action="store_true", help="skip the 16K-128K context sweep against dense SDPA")
    ap.add_argument("--ttft-layers", type=int, default=32)
    ap.add_argument("--ttft-ctx", type=int, default=65536)
    return ap.parse_args()


def maybe_relaunch(args) -> int | None:
    """--gpus N without a torchrun environment: re-run this command under
    torch.distributed.run with N ranks (127.0.0.1 rendezvous) and return its
    exit code; with WORLD_SIZE set it must equal --gpus."""
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != args.gpus:
            raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}; they must match")
        return None
    if args.gpus <= 1:
        return None
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd[1:6])} ...", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def common_config(args, world: int) -> dict:
    """The workload description both arms report (identical keys and values)."""
    return {"workload": f"llama3-8b-attn-layer-{args.ctx // 1024}k-{args.mode}", "heads": H, "kv_heads": HK,
            "head_dim": D, "seq_len": args.ctx, "batch": 1, "mode": args.mode,
            "pattern": args.pattern, "seed": args.seed, "n_gpus": world}


def synth_inputs(seed: int, ctx: int):
    """bf16-rounded uniform q (H, n, d), k (HK, n, d), v (HK, n, d) as float32."""
    import torch

    from paper_2412_06198_b200.harness import synth_qkv_gqa

    q, k, v = synth_qkv_gqa(seed, ctx, H, HK, D)
    return tuple(torch.from_numpy(x[0]).bfloat16().float().numpy() for x in (q, k, v))


def l2_note(n: int) -> str:
    q_mb, kv_mb = H * n * D * 2 / 1e6, 2 * HK * n * D * 2 / 1e6
    fits = "exceed" if q_mb + kv_mb > 126 else "fit in"
    return f"inputs (Q {q_mb:.0f} MB + K/V {kv_mb:.0f} MB) {fits} the 126 MB L2; no flush"


def measured_peaks():
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j.get("bf16_tflops", 1628.9), j.get("bf16_tflops_sustained", 1400.1), j.get("hbm_gbs", 6531.6), "measured"
    # the driver-written file is per pod; SURVEY.md §6 recorded this pool's copy of it
    return 1628.9, 1400.1, 6531.6, "measured (SURVEY.md §6 record of MEASURED_PEAKS.json)"


_SAMPLER = r"""
import sys, time
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
while True:
    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    print(sm, mx, rs, flush=True)
    time.sleep(0.002)
"""


class ClockSampler:
    """SM clocks and throttle reasons sampled every ~2 ms by a separate NVML
    process (not a thread: the launching thread holds the GIL) during the
    timed region."""

    def __init__(self, gpu_index: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        self.idx = int(vis.split(",")[gpu_index]) if vis else gpu_index
        self.samples = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen([sys.executable, "-c", _SAMPLER, str(self.idx)], stdout=subprocess.PIPE,
                                       stderr=subprocess.DEVNULL, text=True)
            self._p.stdout.readline()  # sampler is up (one sample taken) before the region starts
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        self._p.terminate()
        out, _ = self._p.communicate(timeout=10)
        for line in out.splitlines():
            try:
                sm, mx, rs = line.split()
                self.samples.append((float(sm), float(mx), int(rs)))
            except ValueError:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        # NVML clocks-event reason bits (nvml.h): sw_power_cap 0x4, hw_slowdown 0x8,
        # sw_thermal 0x20, hw_thermal 0x40, hw_power_brake 0x80
        bits = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
                0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}
        reasons = sorted({name for _, _, r in self.samples for b, name in bits.items() if r & b})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml, 2 ms"}


# ----------------------------------------------------------------------------- CPU reference arm

def oracle_plan(q, k, v, ctx):
    """The oracle's own auto selection for every head (cheap: 64-token windows)."""
    from oracle import sparse_oracle as O

    cal = min(64, ctx)
    space = O.default_space(cal, D)
    g = H // HK
    pats = []
    for h in range(H):
        qh, kh, vh = (x.astype(np.float32) for x in (q[h], k[h // g], v[h // g]))
        pats.append(O.select_windowed(qh, kh, vh, space, cal)[0])
    return pats


def oracle_head_seconds(q, k, v, h, ctx):
    """Wall seconds of one head's full reference-algorithm prefill (select + index + kernel)."""
    from oracle import sparse_oracle as O

    g = H // HK
    qh, kh, vh = (x.astype(np.float32) for x in (q[h], k[h // g], v[h // g]))
    t = time.perf_counter()
    cal = min(64, ctx)
    pat = O.select_windowed(qh, kh, vh, O.default_space(cal, D), cal)[0]
    idx = O.build_index(qh, kh, pat, "estimated", min(64, ctx))
    O.sparse_attention(qh, kh, vh, idx)
    return time.perf_counter() - t, pat


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count() or 1


def stratified_cpu_ms(q, k, v, ctx, budget_steps=None):
    """The CPU baseline of our arm's line: one head per family of the
    reference's own auto plan through the reference package's per-head
    prefill body (the oracle port when the package is absent), extrapolated
    to the layer by the family counts."""
    ref = _reference_module()
    g = H // HK
    cal = min(64, ctx)
    if ref is not None:
        space = ref.default_search_space(cal, D)
        mats = lambda h: ref.AttnMatrices(q[h], k[h // g], v[h // g], causal=True)  # noqa: E731
        pats = [ref.select_pattern_windowed(mats(h), space, cal).chosen for h in range(H)]

        def head_s(h):
            t = time.perf_counter()
            m = mats(h)
            pat = ref.select_pattern_windowed(m, space, cal).chosen
            ref.sparse_attention(m, ref.build_index(m, pat, mode="estimated", q_est=min(64, ctx)),
                                 need_weights=False)
            return time.perf_counter() - t
        kind, what = "reference", "the reference package (baseline/_ref)"
    else:
        pats = oracle_plan(q, k, v, ctx)
        head_s = lambda h: oracle_head_seconds(q, k, v, h, ctx)[0]  # noqa: E731
        kind, what = "port", "the oracle port of the reference algorithm"
    fam_of = lambda p: type(p).__name__  # noqa: E731
    counts, first = {}, {}
    for h, p in enumerate(pats):
        counts[fam_of(p)] = counts.get(fam_of(p), 0) + 1
        first.setdefault(fam_of(p), h)
    per = {f: head_s(h) for f, h in first.items()}
    ms = 1e3 * sum(counts[f] * per[f] for f in counts)
    sample = (f"one full {ctx}-token head per family of the reference's own auto plan through {what}'s per-head "
              f"prefill body ({', '.join(f'{f}x{counts[f]}: {per[f]:.2f}s' for f in counts)}), "
              f"layer = sum(count * per-head seconds)")
    return ms, sample, kind


def _reference_module():
    """The unmodified reference package installed into baseline/_ref (pip
    --target), or None."""
    ref_dir = os.path.join(HERE, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "sparseattn")):
        return None
    sys.path.insert(0, ref_dir)
    try:
        import sparseattn
    except Exception:
        return None
    finally:
        sys.path.remove(ref_dir)
    return sparseattn


def run_reference(args):
    """Reference arm: the reference's own CPU path (runtime.prefill's per-head
    body, runtime.py:174-193: AttnMatrices -> select_pattern_windowed ->
    build_index(estimated) -> sparse_attention) on the box's host cores, one
    head per step; the layer time is the per-family mean times the family
    counts of the reference's own selection over all heads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", "1"))
    ref = _reference_module()
    q, k, v = synth_inputs(args.seed, args.ctx)
    g = H // HK
    cal = min(64, args.ctx)
    q_est = min(64, args.ctx)
    if ref is not None:
        kind = "reference"
        space = ref.default_search_space(cal, D)

        def mats(h):
            return ref.AttnMatrices(q[h], k[h // g], v[h // g], causal=True)

        def select(h):
            return ref.select_pattern_windowed(mats(h), space, cal).chosen

        def head(h):
            m = mats(h)
            pat = ref.select_pattern_windowed(m, space, cal).chosen
            idx = ref.build_index(m, pat, mode="estimated", q_est=q_est)
            ref.sparse_attention(m, idx, need_weights=False)
    else:  # no installed reference: the oracle port of the same algorithm
        from oracle import sparse_oracle as O

        kind = "port"
        ospace = O.default_space(cal, D)

        def select(h):
            return O.select_windowed(q[h], k[h // g], v[h // g], ospace, cal)[0]

        def head(h):
            oracle_head_seconds(q, k, v, h, args.ctx)
    pats = [select(h) for h in range(H)]
    fam_of = lambda p: type(p).__name__  # noqa: E731
    counts, heads = {}, {}
    for h, p in enumerate(pats):
        counts[fam_of(p)] = counts.get(fam_of(p), 0) + 1
        heads.setdefault(fam_of(p), []).append(h)
    fams = sorted(counts)
    cheapest = min(fams, key=lambda f: {"BlockSparse": 0, "Blk": 0}.get(f, 1))
    for _ in range(args.warmup):
        head(heads[cheapest][0])
    samples = {f: [] for f in fams}
    step_s = []
    t0 = time.perf_counter()
    for s_ in range(args.steps):
        f = fams[s_ % len(fams)]
        hsel = heads[f][(s_ // len(fams)) % len(heads[f])]
        ts = time.perf_counter()
        head(hsel)
        sec = time.perf_counter() - ts
        samples[f].append(sec)
        step_s.append(sec)
    wall = time.perf_counter() - t0
    known = {f: statistics.mean(x) for f, x in samples.items() if x}
    avg = statistics.mean(known.values())
    value = 1e3 * sum(counts[f] * known.get(f, avg) for f in fams)
    cores = cpu_cores()
    sample = (f"each step = one full {args.ctx}-token head through the {'reference package' if ref else 'oracle port'}'s "
              f"per-head prefill body (runtime.py:174-193), families round-robin "
              f"({', '.join(f'{f}x{counts[f]}: {known.get(f, avg):.2f}s' for f in fams)}); value = layer ms = "
              f"sum(count * mean per-head ms); ms_per_step = mean wall ms of one sampled head")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "ms/layer",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.mean(step_s), 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (uniform [-1,1], rng([seed, ctx]) GQA draw, bf16-rounded)",
        "config": common_config(args, world),
        "cpu_baseline": {"value": round(value, 3), "unit": "ms/layer", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "ms/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(wall, 1),
        "families": counts,
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm

def count_step_kernels(step):
    """Kernel launches of one step, from a CUPTI trace (torch.profiler)."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    names = {}
    for ev in prof.events():
        if ev.device_type is not None and "cuda" in str(ev.device_type).lower() and "memset" not in ev.name.lower() \
                and "memcpy" not in ev.name.lower():
            key = ev.name.split("(")[0].split("<")[0].replace("void ", "").replace("sa::", "")
            names[key] = names.get(key, 0) + 1
    return sum(names.values()), names


def layer_graph(plan, qd, kd, vd, out, ws, flag, cache_k, cache_v):
    """CUDA graph of the whole layer step: selection + sa_prefill, which also
    runs AttnMatrices' finiteness scan (core.py:72-74) and the KvCache fill
    (runtime.py:197) on a side stream beside the estimators."""
    plan.desc.check_flag = flag.data_ptr()
    plan.desc.cache_k, plan.desc.cache_v = cache_k.data_ptr(), cache_v.data_ptr()
    plan.desc.cache_capacity = cache_k.shape[1]
    return plan.graph(qd, kd, vd, out, ws)


def time_graph(graph, steps, dev_index, world=1, clocks=True):
    import torch
    import torch.distributed as dist

    for _ in range(2):
        graph.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev_index) if clocks else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if sampler:
        sampler.__enter__()
    e0.record()
    for _ in range(steps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    if sampler:
        sampler.__exit__()
    if world > 1:
        dist.barrier()
    return e0.elapsed_time(e1) / steps, sampler


def stage_breakdown(plan, qd, kd, vd, out, ws, steps):
    """Per-stage ms from eager steps with stage events (after the timed region)."""
    import torch

    evsets = []
    for _ in range(steps):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        for e in evs:
            e.record()
        evsets.append(evs)
    torch.cuda.synchronize()
    for evs in evsets:
        evs[0].record()
        if plan.mode == "auto":
            plan.select(qd, kd, ws)
        for i in range(5):
            plan.desc.stage_events[i] = evs[1 + i].cuda_event
        plan.run(qd, kd, vd, out, ws)
        for i in range(5):
            plan.desc.stage_events[i] = None
        evs[6].record()
    torch.cuda.synchronize()
    stage = np.array([[evs[i].elapsed_time(evs[i + 1]) for i in range(6)] for evs in evsets])
    return stage.mean(axis=0)  # select, vs-est, block-est, tiles, attention, (gather)


def attn_roofline(plan, ws, attn_ms, n):
    from paper_2412_06198_b200 import runtime as R
    import torch

    view = plan.views(ws)
    cnt = R._wrap(view.tile_cnt, plan.hh * view.nqt, torch.int32).cpu().numpy()
    exec_tiles = int(cnt.sum())
    exec_flops = exec_tiles * 4.0 * 128 ** 3
    peak, peak_sus, _, peak_kind = measured_peaks()
    achieved = exec_flops / (attn_ms * 1e-3) / 1e12
    traffic = None
    tp = os.path.join(HERE, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"attn_{n}_{plan.mode}")
    return {"bound": "tensor", "kernel": "attn_fwd_kernel", "achieved": round(achieved, 1), "peak": peak,
            "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "frac_sustained": round(achieved / peak_sus, 4),
            "peak_kind": peak_kind, "traffic": traffic, "exec_tiles": exec_tiles, "attn_ms": round(attn_ms, 4),
            "flops_per_launch": exec_flops,
            "flops_note": "executed (q-tile, k-tile) pairs x 4*128^3 (QK^T and PV of a 128x128 tile, d=128)"}


def e2e_host(R, q_h, k_h, v_h, cfg, mode, fixed, reps, world=1, dev=None):
    """prefill() on HOST tensors (the public API): H2D of q/k/v, the layer,
    D2H of the (1, n, H*d) output, all inside the wall-clock region."""
    import torch
    import torch.distributed as dist

    kw = {"fixed_pattern": fixed} if fixed is not None else {}
    res = None
    for _ in range(2):
        res = R.prefill(q_h, k_h, v_h, cfg, mode=mode, **kw)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    walls = []
    for _ in range(reps):
        t0 = time.perf_counter()
        res = R.prefill(q_h, k_h, v_h, cfg, mode=mode, **kw)
        walls.append((time.perf_counter() - t0) * 1e3)
    ms = statistics.median(walls)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    out = res.outputs
    nbytes = lambda x: int(x.numel() * x.element_size()) if hasattr(x, "element_size") else int(x.nbytes)  # noqa
    return ms, nbytes(q_h) + nbytes(k_h) + nbytes(v_h), nbytes(out), reps


def estimator_roofline(n, dev, reps=5):
    """The VS estimator chain of an all-VS layer (32 q / 8 kv heads, q_est = 64):
    sa_score_tail (both passes, one kernel) + the stable top-k of the 32 column
    and 32 diagonal rows (k = 3n/64, the auto VS pattern), timed with CUDA
    events.  Algorithmic bytes: K read once (2 * n * 128 * 8) +
    the Q tails (2 * 64 * 128 * 32) + fp32 column / diagonal scores written
    (8 * n * 32) = 2304 n + 0.5 MB."""
    import torch

    from paper_2412_06198_b200 import _lib

    g = torch.Generator(device=dev)
    g.manual_seed(5)
    q = (torch.rand((H, n, D), generator=g, device=dev) * 2 - 1).bfloat16()
    k = (torch.rand((HK, n, D), generator=g, device=dev) * 2 - 1).bfloat16()
    # column rows then diagonal rows in one buffer: one top-k launch over all
    # 2H rows, as sa_prefill's VS index step launches it
    scores = torch.empty((2, H, n), dtype=torch.float32, device=dev)
    col, diag = scores[0], scores[1]
    kk = 3 * n // 64
    idx = torch.empty((2 * H, kk), dtype=torch.int32, device=dev)
    lib = _lib.load()
    wsb = int(lib.sa_score_tail_workspace(1, H, n, n))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    scale = 1 / math.sqrt(D)

    def est():
        _lib.call("sa_score_tail", 1, H, HK, n, scale, q.data_ptr(), k.data_ptr(), n - 64, n, col.data_ptr(),
                  diag.data_ptr(), 0, None, 0, ws.data_ptr(), wsb, st)

    def topk():
        _lib.call("sa_topk_stable_f32", scores.data_ptr(), 2 * H, n, n, kk, idx.data_ptr(), kk, st)

    for _ in range(2):
        est()
        topk()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t_est, t_topk = [], []
    for _ in range(reps):
        ev[0].record()
        est()
        ev[1].record()
        topk()
        ev[2].record()
        torch.cuda.synchronize()
        t_est.append(ev[0].elapsed_time(ev[1]) * 1e3)
        t_topk.append(ev[1].elapsed_time(ev[2]) * 1e3)
    est_us, topk_us = statistics.median(t_est), statistics.median(t_topk)
    _, _, hbm, peak_kind = measured_peaks()
    alg = 2304 * n + 2 * 64 * D * H
    traffic = None
    tp = os.path.join(HERE, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"vs_est_{n}")
    chain = est_us + topk_us
    return {"n": n, "heads": H, "kv_heads": HK, "q_est": 64, "topk_k": kk, "algorithmic_bytes": alg,
            "estimator_us": round(est_us, 1), "topk_us": round(topk_us, 1), "chain_us": round(chain, 1),
            "achieved_gbs": round(alg / (chain * 1e-6) / 1e9, 1),
            "estimator_achieved_gbs": round(alg / (est_us * 1e-6) / 1e9, 1),
            "peak_gbs": hbm, "peak_kind": peak_kind, "frac": round(alg / (chain * 1e-6) / 1e9 / hbm, 4),
            "estimator_frac": round(alg / (est_us * 1e-6) / 1e9 / hbm, 4), "traffic": traffic,
            "traffic_note": "ncu dram__bytes_read+write of vs_estimator_kernel (profiles/traffic.json)",
            "floor_note": "two exact passes: 2 x 2*64*128*32*n bf16 MMA FLOP and 2 x 64*32*n exps; "
                          "DESIGN.md 'VS estimator roofline'"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: world size {world} != --gpus {args.gpus}")
    if world > 1:
        # SA_DIST_BACKEND=gloo lets ranks share one GPU (a dry run of the N > 1 path)
        backend = os.environ.get("SA_DIST_BACKEND", "nccl")
        torch.cuda.set_device(local % torch.cuda.device_count())
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        else:
            dist.init_process_group(backend)
        if dist.get_world_size() != args.gpus:
            raise SystemExit(f"bench.py: communicator has {dist.get_world_size()} ranks, --gpus {args.gpus}")
        print(f"bench.py: rank {rank}/{world} backend {dist.get_backend()} on cuda:{torch.cuda.current_device()}",
              file=sys.stderr, flush=True)
    dev = torch.device("cuda", torch.cuda.current_device())
    if HK % world != 0:
        raise SystemExit(f"--gpus {world} must divide the {HK} kv heads")

    from paper_2412_06198_b200 import runtime as R
    from paper_2412_06198_b200.multigpu import gather_heads, shard_heads
    from paper_2412_06198_b200.patterns import BlockSparse, Triangular, VerticalSlash

    def make_fixed(n):
        mode = args.mode
        fixed = None
        if args.pattern:
            fam, p1, p2 = args.pattern.split(":")
            fixed = {"tri": Triangular, "vs": VerticalSlash, "block": BlockSparse}[fam](int(p1), int(p2))
            mode = "fixed"
        elif mode not in ("auto", "dense"):
            from paper_2412_06198_b200.harness import fixed_pattern_for

            fixed = fixed_pattern_for(mode, n)
            mode = "fixed"
        return mode, fixed

    n = args.ctx
    hk_l = HK // world
    h_l = H // world
    q, k, v = synth_inputs(args.seed, n)
    q_sl, kv_sl = shard_heads(rank, world, H, HK)
    qs, ks, vs = q[q_sl], k[kv_sl], v[kv_sl]
    # pinned host copies (e2e) and resident device copies (value)
    q_h = torch.from_numpy(np.ascontiguousarray(qs)).bfloat16().pin_memory()
    k_h = torch.from_numpy(np.ascontiguousarray(ks)).bfloat16().pin_memory()
    v_h = torch.from_numpy(np.ascontiguousarray(vs)).bfloat16().pin_memory()
    qd, kd, vd = q_h.to(dev), k_h.to(dev), v_h.to(dev)
    mode, fixed = make_fixed(n)
    plan = R.PrefillPlan(1, h_l, hk_l, n, D, mode, fixed_pattern=fixed)
    ws = R._workspace(plan.ws_bytes, dev)
    out = torch.empty((1, n, h_l * D), dtype=torch.bfloat16, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    cache_k = torch.empty((hk_l, n, D), dtype=torch.bfloat16, device=dev)
    cache_v = torch.empty((hk_l, n, D), dtype=torch.bfloat16, device=dev)
    final = torch.empty((n, H * D), dtype=torch.bfloat16, device=dev) if world > 1 else None
    # N > 1: the load-balanced layer (multigpu.BalancedLayer) is the timed step;
    # SA_MG_BALANCED=0 times the plain GQA-group sharding + output all-gather
    balanced = world > 1 and os.environ.get("SA_MG_BALANCED", "1") != "0"
    layer = peer = None
    if balanced:
        from paper_2412_06198_b200.multigpu import BalancedLayer

        qf, kf, vf = (torch.from_numpy(np.ascontiguousarray(x)).bfloat16().to(dev) for x in (q, k, v))
        layer = BalancedLayer(rank, world, H, HK, n, D, mode, fixed_pattern=fixed, device=dev)
        layer.enable_checks(flag, cache_k, cache_v)
        if os.environ.get("SA_MG_EXCHANGE", "nccl") == "peer":
            from paper_2412_06198_b200.multigpu import PeerOutputs

            peer = PeerOutputs(rank, world, n, H * D)

    # warm-up steps (eager), then the timed step
    for _ in range(max(3, args.warmup)):
        if plan.mode == "auto":
            plan.select(qd, kd, ws)
        plan.run(qd, kd, vd, out, ws)
    torch.cuda.synchronize()
    if balanced:
        def gstep():
            if peer is not None:
                layer.step_peers(qf, kf, vf, peer)
            else:
                layer.step(qf, kf, vf)
        for _ in range(2):
            gstep()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        clocks = ClockSampler(torch.cuda.current_device())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with clocks:
            e0.record()
            for _ in range(args.steps):
                gstep()
            e1.record()
            torch.cuda.synchronize()
        dist.barrier()
        ms = e0.elapsed_time(e1) / args.steps
    else:
        graph = layer_graph(plan, qd, kd, vd, out, ws, flag, cache_k, cache_v)
        if world > 1:
            def gstep():
                graph.replay()
                gather_heads(out[0], world, out=final)
        else:
            gstep = graph.replay
        for _ in range(2):
            gstep()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clocks = ClockSampler(torch.cuda.current_device())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with clocks:
            e0.record()
            for _ in range(args.steps):
                gstep()
            e1.record()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = e0.elapsed_time(e1) / args.steps
    torch.cuda.synchronize()
    if int(flag.item()):
        raise SystemExit("bench.py: the synthetic inputs tripped the finiteness check")
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # cache fill check: the cache holds the layer's k / v rows
    if os.environ.get("SA_CHECK_MODE", "0") in ("0", "1"):
        assert torch.equal(cache_k[:, :64], kd[:, :64]) and torch.equal(cache_v[:, -64:], vd[:, -64:])
    plan.desc.check_flag = None
    plan.desc.cache_k = plan.desc.cache_v = None
    plan.desc.cache_capacity = 0

    stage_ms = stage_breakdown(plan, qd, kd, vd, out, ws, args.steps)
    attn_ms = float(stage_ms[4])
    if balanced:  # the attention launch of this rank's dealt items, CUDA events on its stream
        ts = []
        for _ in range(args.steps):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            if peer is not None:
                layer.attend_peers(qf, kf, vf, peer)
            else:
                layer.attend(qf, kf, vf)
            a1.record()
            torch.cuda.synchronize()
            ts.append(a0.elapsed_time(a1))
        attn_ms = float(np.mean(ts))
    roof = attn_roofline(plan, ws, attn_ms, n)
    if balanced:  # this rank's attention launch covers its dealt items of every head
        from paper_2412_06198_b200.multigpu import _view

        cf = _view(layer.ws_full, layer.vf.tile_cnt, layer.items, torch.int32)
        roof["exec_tiles"] = int(cf[layer.mine.long()].sum().item())
        roof["flops_per_launch"] = roof["exec_tiles"] * 4.0 * 128 ** 3
        roof["achieved"] = round(roof["flops_per_launch"] / (attn_ms * 1e-3) / 1e12, 1)
        roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
    plans = plan.plans(ws, with_search=False)
    fams = [type(hp.pattern).__name__ if hp.pattern is not None else "dense" for hp in plans[0]]
    # kernels per step, counted by CUPTI (torch.profiler) on one extra untimed step
    launches_per_step, kernel_names = count_step_kernels(gstep)

    cfg = R.ModelConfig(n_heads=h_l, d_model=h_l * D, d_head=D, max_context=n)
    e2e = e2e_np = None
    if not args.no_e2e:
        reps = max(3, min(args.steps, 5))
        ems, bi, bo, reps = e2e_host(R, q_h[None], k_h[None], v_h[None], cfg, plan.mode, fixed, reps, world, dev)
        e2e = {"value": round(ems, 3), "unit": "ms/layer", "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
               "reps": reps, "timer": "wall, median",
               "path": "paper_2412_06198_b200.prefill(pinned host bf16 torch tensors) -> host outputs "
                       "(per-kv-group H2D / kernels / D2H streams overlapped)"}
        if world == 1:
            # the reference's own input type: numpy float32 (pageable), numpy float32 out
            qn, kn, vn = (np.ascontiguousarray(x)[None] for x in (qs, ks, vs))
            nms, bi2, bo2, r2 = e2e_host(R, qn, kn, vn, cfg, plan.mode, fixed, 3)
            e2e_np = {"value": round(nms, 3), "unit": "ms/layer", "h2d_bytes_per_step": bi2,
                      "d2h_bytes_per_step": bo2, "reps": r2, "timer": "wall, median",
                      "path": "paper_2412_06198_b200.prefill(numpy float32 (1, H|HK, n, 128)) -> numpy float32 "
                              "outputs (the reference's own call and types)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cms, sample, ckind = stratified_cpu_ms(q, k, v, n)
        cpu = {"value": round(cms, 1), "unit": "ms/layer", "cores": cpu_cores(), "kind": ckind, "sample": sample}

    # north-star sub-records (single GPU): the 128K layer and the all-VS estimator chain
    sub128 = None
    est = None
    if world == 1 and n != 131072 and not args.no_128k:
        del qd, kd, vd, out, cache_k, cache_v, q_h, k_h, v_h
        torch.cuda.empty_cache()
        sub128 = run_sub_layer(args, R, make_fixed, 131072, dev)
    if world == 1 and not args.no_est:
        est = [estimator_roofline(nn, dev) for nn in sorted({n, 131072})]
    ttft = None
    if not args.no_ttft:
        ttft = run_ttft(args, world, rank, dev)
    c5 = None
    if world == 1 and not args.no_c5 and args.mode == "auto" and args.pattern is None:
        known = {n: round(ms, 4)}
        if sub128 is not None:
            known[131072] = sub128["value"]
        c5 = c5_sweep(args, R, make_fixed, dev, known)

    if rank == 0:
        fam_counts = {f: fams.count(f) for f in sorted(set(fams))}
        line = {
            "metric": METRIC, "value": round(ms, 4), "unit": "ms/layer", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms, 4),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (uniform [-1,1], rng([seed, ctx]) GQA draw, bf16)",
            "config": common_config(args, world),
            "details": {
                "parallelism": (f"balanced head-parallel x{world}: per-group estimation, index all-gather, "
                                f"heaviest-first (head, q-tile) deal, " +
                                ("output rows stored into every rank's IPC-mapped buffer by the attention "
                                 "epilogue (fused all-gather)" if peer is not None else "output-block all-gather"))
                if balanced else (f"head-parallel x{world} + NCCL all-gather" if world > 1 else "single GPU"),
                "l2": l2_note(n),
                "step": ("eager balanced steps (BalancedLayer.step)" if balanced else
                         "CUDA graph of selection + sa_prefill; the step includes AttnMatrices' finiteness scan of "
                         "q/k/v (core.py:72-74) and the KvCache fill (runtime.py:197), both on a side stream beside "
                         "the estimators"),
                "families_rank0": fam_counts,
                "stage_note": "stage_ms from eager steps with stage events; the VS and block estimator chains "
                              "overlap on two streams: vs_estimator = selection end -> VS chain end, "
                              "block_estimator = the rest of the block chain"},
            "roofline": roof,
            "stage_ms": {k2: round(float(x), 4) for k2, x in zip(
                ["select", "vs_estimator", "block_estimator", "tile_lists", "attention", "all_gather"], stage_ms)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_numpy_f32": e2e_np,
            "gpu_launches": int(launches_per_step * args.steps),
            "kernels_per_step": kernel_names,
            "clocks": clocks.summary(),
            "ctx_131072": sub128,
            "estimator_roofline": est,
            "ttft_c4": ttft,
            "c5_sweep": c5,
        }
        print(json.dumps(line), flush=True)
    if peer is not None:
        peer.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_ttft(args, world, rank, dev):
    """BASELINE configs[3]: a 32-layer Llama-3-8B-shape sparse prefill at 64K
    (attention path only, like runtime.py:1-10), head-parallel over the ranks:
    layers.LayerStack runs every layer's selection, estimators, attention,
    finiteness scan and KvCache fill back to back (one CUDA graph on one GPU;
    with N > 1 each layer's output all-gather overlaps the next layer).  TTFT =
    device time of the stack, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2412_06198_b200.layers import LayerStack
    from paper_2412_06198_b200.runtime import ModelConfig

    L, n = args.ttft_layers, args.ttft_ctx
    cfg = ModelConfig(n_heads=H, d_model=H * D, d_head=D, max_context=n)
    h_l, hk_l = H // world, HK // world
    g = torch.Generator(device=dev)
    g.manual_seed(1000 * args.seed + rank)

    def draw(heads):
        return (torch.rand((1, heads, n, D), generator=g, device=dev) * 2 - 1).bfloat16()

    qs = [draw(h_l) for _ in range(L)]
    ks = [draw(hk_l) for _ in range(L)]
    vs = [draw(hk_l) for _ in range(L)]
    stack = LayerStack(L, cfg, HK, n, mode="auto", world=world, device=dev)
    if world == 1:
        graph = stack.graph(qs, ks, vs)
        step = graph.replay
    else:
        def step():
            stack.run(qs, ks, vs)
    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    reps = 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    plans = stack.finish()
    fams = {}
    for p in plans:
        for hp in p[0]:
            f = type(hp.pattern).__name__
            fams[f] = fams.get(f, 0) + 1
    del stack, qs, ks, vs
    torch.cuda.empty_cache()
    return {"layers": L, "seq_len": n, "ttft_ms": round(ms, 2), "ms_per_layer": round(ms / L, 4), "reps": reps,
            "n_gpus": world, "families_rank0_all_layers": fams,
            "data": "synthetic uniform [-1,1] per layer (device RNG), bf16",
            "step": ("one CUDA graph of the 32-layer stack" if world == 1 else
                     "eager layers; layer l's NCCL output all-gather overlaps layer l+1") +
                    "; every layer includes the finiteness scan and its KvCache fill"}


def run_sub_layer(args, R, make_fixed, n, dev):
    """The north-star config on the same run: one 128K layer (BASELINE configs[2]
    shape, auto mode unless --mode/--pattern), graph-timed like the headline,
    with its stage breakdown, attention roofline and host e2e."""
    import torch

    mode, fixed = make_fixed(n)
    q, k, v = synth_inputs(args.seed, n)
    q_h = torch.from_numpy(q).bfloat16().pin_memory()
    k_h = torch.from_numpy(k).bfloat16().pin_memory()
    v_h = torch.from_numpy(v).bfloat16().pin_memory()
    del q, k, v
    qd, kd, vd = q_h.to(dev), k_h.to(dev), v_h.to(dev)
    plan = R.PrefillPlan(1, H, HK, n, D, mode, fixed_pattern=fixed)
    ws = R._workspace(plan.ws_bytes, dev)
    out = torch.empty((1, n, H * D), dtype=torch.bfloat16, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    cache_k = torch.empty((HK, n, D), dtype=torch.bfloat16, device=dev)
    cache_v = torch.empty((HK, n, D), dtype=torch.bfloat16, device=dev)
    for _ in range(2):
        if plan.mode == "auto":
            plan.select(qd, kd, ws)
        plan.run(qd, kd, vd, out, ws)
    graph = layer_graph(plan, qd, kd, vd, out, ws, flag, cache_k, cache_v)
    steps = max(3, min(args.steps, 5))
    ms, sampler = time_graph(graph, steps, torch.cuda.current_device())
    assert not int(flag.item())
    plan.desc.check_flag = None
    plan.desc.cache_k = plan.desc.cache_v = None
    plan.desc.cache_capacity = 0
    stage_ms = stage_breakdown(plan, qd, kd, vd, out, ws, 2)
    roof = attn_roofline(plan, ws, float(stage_ms[4]), n)
    plans = plan.plans(ws, with_search=False)
    fams = [type(hp.pattern).__name__ if hp.pattern is not None else "dense" for hp in plans[0]]
    del graph, qd, kd, vd, out, cache_k, cache_v
    torch.cuda.empty_cache()
    e2e = None
    if not args.no_e2e:
        cfg = R.ModelConfig(n_heads=H, d_model=H * D, d_head=D, max_context=n)
        ems, bi, bo, reps = e2e_host(R, q_h[None], k_h[None], v_h[None], cfg, plan.mode, fixed, 3)
        e2e = {"value": round(ems, 3), "unit": "ms/layer", "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
               "reps": reps, "timer": "wall, median"}
    return {"seq_len": n, "workload": f"llama3-8b-attn-layer-{n // 1024}k-{args.mode}", "value": round(ms, 4),
            "unit": "ms/layer", "steps": steps, "families": {f: fams.count(f) for f in sorted(set(fams))},
            "roofline": roof,
            "stage_ms": {k2: round(float(x), 4) for k2, x in zip(
                ["select", "vs_estimator", "block_estimator", "tile_lists", "attention"], stage_ms[:5])},
            "e2e": e2e, "clocks": sampler.summary() if sampler else None, "l2": l2_note(n)}


def sdpa_dense_ms(n, dev, reps=3):
    """Dense causal attention of the same shape by torch SDPA (cuDNN on B200, the
    best installed dense kernel here: profiles/r02/dense_baseline_32k.txt),
    library code timed for comparison only."""
    import torch

    g = torch.Generator(device=dev)
    g.manual_seed(7)
    q = torch.rand((1, H, n, D), generator=g, device=dev).bfloat16()
    k = torch.rand((1, HK, n, D), generator=g, device=dev).bfloat16()
    v = torch.rand((1, HK, n, D), generator=g, device=dev).bfloat16()
    f = lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)  # noqa: E731
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    del q, k, v
    torch.cuda.empty_cache()
    return e0.elapsed_time(e1) / reps


def c5_sweep(args, R, make_fixed, dev, known):
    """BASELINE configs[4] on one GPU: the auto layer at 16K-128K (graph replay,
    the same synthetic draw as the headline; 32K / 128K reuse the lines above)
    against dense causal SDPA, and the TTFT growth gradient (least-squares ms
    per 1K tokens over the sweep, reference bench.py:336-378)."""
    import torch

    rows = []
    for n in (16384, 32768, 65536, 131072):
        ms = known.get(n)
        if ms is None:
            mode, fixed = make_fixed(n)
            q, k, v = synth_inputs(args.seed, n)
            qd, kd, vd = (torch.from_numpy(x).bfloat16().to(dev) for x in (q, k, v))
            del q, k, v
            plan = R.PrefillPlan(1, H, HK, n, D, mode, fixed_pattern=fixed)
            ws = R._workspace(plan.ws_bytes, dev)
            out = torch.empty((1, n, H * D), dtype=torch.bfloat16, device=dev)
            flag = torch.zeros(1, dtype=torch.int32, device=dev)
            cache_k = torch.empty((HK, n, D), dtype=torch.bfloat16, device=dev)
            cache_v = torch.empty((HK, n, D), dtype=torch.bfloat16, device=dev)
            for _ in range(2):
                if plan.mode == "auto":
                    plan.select(qd, kd, ws)
                plan.run(qd, kd, vd, out, ws)
            graph = layer_graph(plan, qd, kd, vd, out, ws, flag, cache_k, cache_v)
            ms, _ = time_graph(graph, 5, torch.cuda.current_device(), clocks=False)
            plan.desc.check_flag = None
            plan.desc.cache_k = plan.desc.cache_v = None
            plan.desc.cache_capacity = 0
            del graph, qd, kd, vd, out, cache_k, cache_v
            torch.cuda.empty_cache()
            ms = round(ms, 4)
        dn = sdpa_dense_ms(n, dev)
        rows.append({"ctx": n, "auto_ms": ms, "dense_sdpa_ms": round(dn, 4), "speedup_vs_dense": round(dn / ms, 2)})
    xs = np.array([r["ctx"] / 1024 for r in rows])
    grad = lambda key: float(np.polyfit(xs, np.array([r[key] for r in rows]), 1)[0])  # noqa: E731
    return {"rows": rows, "gradient_auto_ms_per_1k_tokens": round(grad("auto_ms"), 4),
            "gradient_dense_ms_per_1k_tokens": round(grad("dense_sdpa_ms"), 4),
            "dense": "torch SDPA (cuDNN) causal, enable_gqa, same shape, bf16"}


def main():
    args = parse()
    rc = maybe_relaunch(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
