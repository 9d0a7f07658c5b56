#!/usr/bin/env python
"""Summarise an ncu --csv launch list: mean device time per kernel per step
(and mean DRAM MB / achieved GB/s when the list carries dram__bytes_* too)."""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read().splitlines()
i = [n for n, l in enumerate(txt) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(io.StringIO("\n".join(txt[i:]))))
per_launch = collections.OrderedDict()  # (kernel, launch id) -> {metric: value}
for r in rows:
    k = r["Kernel Name"].split("(")[0][:48]
    d = per_launch.setdefault((k, r["ID"]), {})
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    name = r["Metric Name"]
    if name == "gpu__time_duration.sum":
        v = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)  # -> us
    elif name.startswith("dram__bytes"):
        v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    d[name] = v
agg = collections.OrderedDict()
for (k, _), d in per_launch.items():
    agg.setdefault(k, []).append(d)
steps = max(1, len(agg.get("attn_fwd_kernel", agg.get(next(iter(agg)), [1]))))
tot = 0.0
for k, ds in agg.items():
    t = [d.get("gpu__time_duration.sum", 0.0) for d in ds]
    tot += sum(t)
    line = f"{k:48s} launches={len(ds):4d} mean={sum(t) / len(t):9.1f} us  per-step={sum(t) / steps:9.1f} us"
    if any("dram__bytes_read.sum" in d for d in ds):
        b = [d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0) for d in ds]
        mb = sum(b) / len(b) / 1e6
        line += f"  dram={mb:8.2f} MB  {mb / 1e3 / (sum(t) / len(t) / 1e6):7.1f} GB/s"
    print(line)
print(f"total per step (serialised, cold) {tot / steps:.1f} us over {steps} steps")
