#!/usr/bin/env python
"""Summarise `ncu --set full` reports (run here, no GPU needed).

  python tools/ncu_summary.py gpurun_out/TAG/attn.ncu-rep [...] [--traffic-key attn_32768_auto]

Prints one markdown table row per profiled launch (duration, DRAM bytes,
DRAM/L2/tensor/XU utilisation, registers, occupancy) and, with --traffic-key,
merges the first attn_fwd launch's dram read+write bytes into
profiles/traffic.json (read by bench.py for roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "dur",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0,
        "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, data = r[0], r[1], r[2:]
    res = []
    for d in data:
        rec = {"kernel": d[hdr.index("Kernel Name")].split("(")[0][:40]}
        for m, k in WANT.items():
            if m in hdr:
                i = hdr.index(m)
                v = d[i].replace(",", "")
                try:
                    x = float(v) * UNIT.get(units[i], 1.0)
                except ValueError:
                    x = None
                rec[k] = x
        res.append(rec)
    return res


def main():
    args = sys.argv[1:]
    key = None
    if "--traffic-key" in args:
        i = args.index("--traffic-key")
        key = args[i + 1]
        args = args[:i] + args[i + 2:]
    print("| kernel | us | DRAM MB (rd+wr) | DRAM % | L2 % | tensor % | XU % | warps % | regs | grid |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    first_attn = None
    for rep in args:
        for rec in rows_of(rep):
            mb = ((rec.get("dram_rd") or 0) + (rec.get("dram_wr") or 0)) / 1e6
            f = lambda k, fmt="{:.1f}": fmt.format(rec[k]) if rec.get(k) is not None else "-"  # noqa: E731
            print(f"| {rec['kernel']} | {f('dur')} | {mb:.1f} | {f('dram_pct')} | {f('l2_pct')} | {f('tensor_pct')} "
                  f"| {f('xu_pct')} | {f('occ_pct')} | {f('regs', '{:.0f}')} | {f('grid', '{:.0f}')} |")
            if first_attn is None and rec["kernel"].startswith("void sa::attn_fwd") or (
                    first_attn is None and "attn_fwd" in rec["kernel"]):
                first_attn = rec
    if key and first_attn is not None:
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
        tj = json.load(open(path)) if os.path.exists(path) else {}
        tj[key] = int((first_attn.get("dram_rd") or 0) + (first_attn.get("dram_wr") or 0))
        json.dump(tj, open(path, "w"), indent=1, sort_keys=True)
        print(f"traffic[{key}] = {tj[key]} bytes -> {path}")


if __name__ == "__main__":
    main()
