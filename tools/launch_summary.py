#!/usr/bin/env python
"""Summarise an ncu --csv launch list: mean device time per kernel per step."""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read().splitlines()
i = [n for n, l in enumerate(txt) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(io.StringIO("\n".join(txt[i:]))))
agg = collections.OrderedDict()
for r in rows:
    k = r["Kernel Name"].split("(")[0][:48]
    agg.setdefault(k, []).append(float(r["Metric Value"]) / (1e3 if r["Metric Unit"] == "ns" else 1.0))
steps = max(1, len(agg.get("attn_fwd_kernel", agg.get(next(iter(agg)), [1]))))
tot = 0.0
for k, v in agg.items():
    tot += sum(v)
    print(f"{k:48s} launches={len(v):4d} mean={sum(v) / len(v):9.1f} us  per-step={sum(v) / steps:9.1f} us")
print(f"total per step (serialised, cold) {tot / steps:.1f} us over {steps} steps")
