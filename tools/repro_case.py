#!/usr/bin/env python
"""Re-run one parity_sweep case: python tools/repro_case.py H HK n d mode [fam p1 p2] [seed]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import sparse_oracle as O  # noqa: E402
import paper_2412_06198_b200 as sa  # noqa: E402

H, HK, n, d = (int(x) for x in sys.argv[1:5])
mode = sys.argv[5]
fixed = None
if mode == "fixed":
    fam, p1, p2 = sys.argv[6], int(sys.argv[7]), int(sys.argv[8])
    fixed = {"T": sa.Triangular, "V": sa.VerticalSlash, "B": sa.BlockSparse}[fam](p1, p2)
q, k, v = (O.bf16_round(x) for x in O.synth_qkv_gqa(123, n, H, HK, d))
cfg = sa.ModelConfig(n_heads=H, d_model=H * d, d_head=d, max_context=n)
res = sa.prefill(q, k, v, cfg, mode=mode, **({"fixed_pattern": fixed} if fixed else {}))
print("ok", np.asarray(res.outputs).shape, [type(p.pattern).__name__ for p in res.plans[0]])
