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
    return ap.parse_args()


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
    """Time one head per family present in the oracle plan; extrapolate the layer."""
    from oracle import sparse_oracle as O

    pats = oracle_plan(q, k, v, ctx)
    fam_of = lambda p: type(p).__name__  # noqa: E731
    counts = {}
    first = {}
    for h, p in enumerate(pats):
        counts[fam_of(p)] = counts.get(fam_of(p), 0) + 1
        first.setdefault(fam_of(p), h)
    per = {}
    for f, h in first.items():
        per[f] = oracle_head_seconds(q, k, v, h, ctx)[0]
    ms = 1e3 * sum(counts[f] * per[f] for f in counts)
    sample = (f"one full {ctx}-token head per family of the oracle's own auto plan "
              f"({', '.join(f'{f}x{counts[f]}: {per[f]:.2f}s' for f in counts)}), "
              f"layer = sum(count * per-head seconds); oracle port of the reference algorithm")
    del O
    return ms, sample


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    q, k, v = synth_inputs(args.seed, args.ctx)
    pats = oracle_plan(q, k, v, args.ctx)
    fam_of = lambda p: type(p).__name__  # noqa: E731
    counts, heads = {}, {}
    for h, p in enumerate(pats):
        counts[fam_of(p)] = counts.get(fam_of(p), 0) + 1
        heads.setdefault(fam_of(p), []).append(h)
    fams = sorted(counts)
    cheapest = "Blk" if "Blk" in heads else fams[0]
    for _ in range(args.warmup):
        oracle_head_seconds(q, k, v, heads[cheapest][0], args.ctx)
    samples = {f: [] for f in fams}
    step_ms = []
    t0 = time.perf_counter()
    for s in range(args.steps):
        f = fams[s % len(fams)]
        hsel = heads[f][(s // len(fams)) % len(heads[f])]
        sec, _ = oracle_head_seconds(q, k, v, hsel, args.ctx)
        samples[f].append(sec)
        known = {g: statistics.mean(x) for g, x in samples.items() if x}
        # extrapolate with the families measured so far (missing ones at the mean)
        avg = statistics.mean(known.values())
        step_ms.append(1e3 * sum(counts[g] * known.get(g, avg) for g in fams))
    wall = time.perf_counter() - t0
    value = step_ms[-1]
    cores = cpu_cores()
    sample = (f"each step = one full {args.ctx}-token head of the oracle's own auto plan, families round-robin "
              f"({', '.join(f'{g}x{counts[g]}' for g in fams)}); layer ms = sum(count * mean per-head ms)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "ms/layer",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value, 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (uniform [-1,1], rng([seed, ctx]), bf16-rounded)",
        "config": {"workload": f"llama3-8b-attn-layer-{args.ctx // 1024}k-auto", "heads": H, "kv_heads": HK,
                   "head_dim": D, "seq_len": args.ctx, "mode": "auto", "parallelism": "none (CPU)"},
        "cpu_baseline": {"value": round(value, 3), "unit": "ms/layer", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "ms/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(wall, 1),
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


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # SA_DIST_BACKEND=gloo lets ranks share one GPU (a dry run of the N > 1 path)
        backend = os.environ.get("SA_DIST_BACKEND", "nccl")
        torch.cuda.set_device(local % torch.cuda.device_count())
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", torch.cuda.current_device())
    if HK % world != 0:
        raise SystemExit(f"--gpus {world} must divide the {HK} kv heads")

    from paper_2412_06198_b200 import _lib, runtime as R
    from paper_2412_06198_b200.patterns import BlockSparse, Triangular, VerticalSlash

    from paper_2412_06198_b200.multigpu import gather_heads, shard_heads

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

    mode = args.mode
    fixed = None
    if args.pattern:
        fam, p1, p2 = args.pattern.split(":")
        fixed = {"tri": Triangular, "vs": VerticalSlash, "block": BlockSparse}[fam](int(p1), int(p2))
        mode = "fixed"
    elif mode != "auto" and mode != "dense":
        from paper_2412_06198_b200.harness import fixed_pattern_for

        fixed = fixed_pattern_for(mode, n)
        mode = "fixed"
    plan = R.PrefillPlan(1, h_l, hk_l, n, D, mode, fixed_pattern=fixed)
    ws = R._workspace(plan.ws_bytes, dev)
    out = torch.empty((1, n, h_l * D), dtype=torch.bfloat16, device=dev)
    final = torch.empty((n, H * D), dtype=torch.bfloat16, device=dev) if world > 1 else None
    # N > 1: the load-balanced layer (multigpu.BalancedLayer) is the timed step;
    # SA_MG_BALANCED=0 times the plain GQA-group sharding + output all-gather
    balanced = world > 1 and os.environ.get("SA_MG_BALANCED", "1") != "0"
    layer = None
    if balanced:
        from paper_2412_06198_b200.multigpu import BalancedLayer

        qf, kf, vf = (torch.from_numpy(np.ascontiguousarray(x)).bfloat16().to(dev) for x in (q, k, v))
        layer = BalancedLayer(rank, world, H, HK, n, D, mode, fixed_pattern=fixed, device=dev)
    # SA_MG_EXCHANGE=peer: the output all-gather fused into the attention epilogue
    # (stores into every rank's CUDA-IPC-mapped output; multigpu.PeerOutputs)
    peer = None
    if balanced and os.environ.get("SA_MG_EXCHANGE", "nccl") == "peer":
        from paper_2412_06198_b200.multigpu import PeerOutputs

        peer = PeerOutputs(rank, world, n, H * D)

    def step(events=None):
        if events is not None:
            events[0].record()
        if plan.mode == "auto":
            plan.select(qd, kd, ws)
        if events is not None:
            for i in range(5):
                plan.desc.stage_events[i] = events[1 + i].cuda_event
        plan.run(qd, kd, vd, out, ws)
        if events is not None:
            for i in range(5):
                plan.desc.stage_events[i] = None
        if world > 1 and not balanced:
            gather_heads(out[0], world, out=final)
        if events is not None:
            events[6].record()

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if balanced and peer is not None:
        def gstep():
            layer.step_peers(qf, kf, vf, peer)
    elif balanced:
        def gstep():
            layer.step(qf, kf, vf)
    else:
        # the timed steps replay a CUDA graph of selection + layer (PrefillPlan.graph)
        graph = plan.graph(qd, kd, vd, out, ws)

        def gstep():
            graph.replay()
            if world > 1:
                gather_heads(out[0], world, out=final)

    for _ in range(2):
        gstep()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(torch.cuda.current_device())
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    with clocks:
        t_start.record()
        for s in range(args.steps):
            gstep()
        t_end.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = t_start.elapsed_time(t_end)
    ms = total_ms / args.steps
    # per-stage breakdown (and the attention kernel time for the roofline) from
    # eager steps with stage events, after the timed region
    evsets = []
    for _ in range(args.steps):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
        for e in evs:
            e.record()
        evsets.append(evs)
    torch.cuda.synchronize()
    for s in range(args.steps):
        step(evsets[s])
    torch.cuda.synchronize()
    stage = np.array([[evs[i].elapsed_time(evs[i + 1]) for i in range(6)] for evs in evsets])
    stage_ms = stage.mean(axis=0)  # select, vs-est, block-est, tiles, attention, gather
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # executed-tile and realised FLOPs of this rank's attention launch
    view = plan.views(ws)
    nqt = view.nqt
    cnt = R._wrap(view.tile_cnt, plan.hh * nqt, torch.int32).cpu().numpy()
    exec_tiles = int(cnt.sum())
    if balanced:  # this rank's attention launch covers its dealt items of every head
        from paper_2412_06198_b200.multigpu import _view

        cf = _view(layer.ws_full, layer.vf.tile_cnt, layer.items, torch.int32)
        exec_tiles = int(cf[layer.mine.long()].sum().item())
    exec_flops = exec_tiles * 4.0 * 128 ** 3
    plans = plan.plans(ws, with_search=False)
    fams = [type(hp.pattern).__name__ if hp.pattern is not None else "dense" for hp in plans[0]]
    attn_ms = float(stage_ms[4])
    if balanced:  # the attention launch of this rank's dealt items, CUDA events on its stream
        ts = []
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if peer is not None:
                layer.attend_peers(qf, kf, vf, peer)
            else:
                layer.attend(qf, kf, vf)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        attn_ms = float(np.mean(ts))
    peak, peak_sus, hbm, peak_kind = measured_peaks()
    achieved = exec_flops / (attn_ms * 1e-3) / 1e12
    if world > 1:
        t = torch.tensor([exec_flops, attn_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    # kernels per step, counted by CUPTI (torch.profiler) on one extra untimed step
    launches_per_step, kernel_names = count_step_kernels(gstep)

    e2e = None
    if not args.no_e2e:
        # the public API on HOST tensors: prefill streams the layer through the GPU
        # (H2D of q/k/v, kernels, D2H of the (1, n, H*d) output) and returns host outputs
        cfg = R.ModelConfig(n_heads=h_l, d_model=h_l * D, d_head=D, max_context=n)
        qh4, kh4, vh4 = q_h[None], k_h[None], v_h[None]
        kw = {"fixed_pattern": fixed} if fixed is not None else {}
        for _ in range(2):
            res = R.prefill(qh4, kh4, vh4, cfg, mode=plan.mode, **kw)
        assert not res.outputs.is_cuda
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        reps = max(3, min(args.steps, 5))
        walls = []
        for _ in range(reps):
            t0 = time.perf_counter()
            res = R.prefill(qh4, kh4, vh4, cfg, mode=plan.mode, **kw)
            walls.append((time.perf_counter() - t0) * 1e3)
        e2e_ms = statistics.median(walls)
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": round(e2e_ms, 3), "unit": "ms/layer",
               "h2d_bytes_per_step": int(q_h.numel() * 2 + k_h.numel() * 2 + v_h.numel() * 2),
               "d2h_bytes_per_step": int(res.outputs.numel() * 2), "reps": reps, "timer": "wall, median",
               "path": "paper_2412_06198_b200.prefill(pinned host bf16 torch tensors) -> host outputs "
                       "(per-kv-group H2D / kernels / D2H streams overlapped)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cms, sample = stratified_cpu_ms(q, k, v, n)
        cpu = {"value": round(cms, 1), "unit": "ms/layer", "cores": cpu_cores(), "kind": "port", "sample": sample}

    if rank == 0:
        traffic = None
        tp = os.path.join(HERE, "profiles", "traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                tj = json.load(f)
            traffic = tj.get(f"attn_{n}_{plan.mode}")
        fam_counts = {f: fams.count(f) for f in sorted(set(fams))}
        line = {
            "metric": METRIC, "value": round(ms, 4), "unit": "ms/layer", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms, 4),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (uniform [-1,1], rng([seed, ctx]) GQA draw, bf16)",
            "config": {"workload": f"llama3-8b-attn-layer-{n // 1024}k-{args.mode}", "heads": H, "kv_heads": HK,
                       "head_dim": D, "seq_len": n, "batch": 1, "mode": args.mode,
                       "parallelism": (f"balanced head-parallel x{world}: per-group estimation, index all-gather, "
                                       f"heaviest-first (head, q-tile) deal, " +
                                       ("output rows stored into every rank's IPC-mapped buffer by the attention "
                                        "epilogue (fused all-gather)" if peer is not None else
                                        "output-block all-gather")) if balanced else
                                      (f"head-parallel x{world} + NCCL all-gather" if world > 1 else "single GPU"),
                       "l2": l2_note(n),
                       "launch": ("eager balanced steps (BalancedLayer.step); stage_ms from eager steps of this "
                                  "rank's GQA-group plan with stage events") if balanced else
                                 ("timed steps replay a CUDA graph of selection + layer (PrefillPlan.graph); "
                                  "stage_ms from eager steps with stage events"),
                       "families_rank0": fam_counts,
                       "stage_note": "the VS and block estimator chains overlap on two streams: vs_estimator = "
                                     "selection end -> VS chain end, block_estimator = the rest of the block chain"},
            "roofline": {"bound": "tensor", "kernel": "attn_fwd_kernel", "achieved": round(achieved, 1),
                         "peak": peak, "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                         "frac_sustained": round(achieved / peak_sus, 4), "peak_kind": peak_kind,
                         "traffic": traffic, "exec_tiles": exec_tiles, "attn_ms": round(attn_ms, 4),
                         "flops_per_launch": exec_flops},
            "stage_ms": {k2: round(float(x), 4) for k2, x in zip(
                ["select", "vs_estimator", "block_estimator", "tile_lists", "attention", "all_gather"], stage_ms)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches_per_step * args.steps),
            "kernels_per_step": kernel_names,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if peer is not None:
        peer.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
