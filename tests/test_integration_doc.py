"""INTEGRATION.md's ctypes stub is code a maintainer would paste into the
reference: check that its struct layout matches the header's (CPU) and that,
run as written against the in-tree library, it produces exactly what the
drop-in package produces (GPU)."""

import ctypes
import os
import re

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _snippet_source():
    doc = open(os.path.join(REPO, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", doc, flags=re.S)
    src = [b for b in blocks if "ctypes.CDLL" in b]
    assert len(src) == 1
    return src[0]


def _load_snippet():
    from paper_2412_06198_b200 import _lib

    src = _snippet_source().replace('"/path/to/paper_2412_06198_b200/_sa_b200.so"', repr(_lib.LIB_PATH))
    ns: dict = {}
    exec(compile(src, "INTEGRATION.md", "exec"), ns)
    return ns


def _layout(t):
    out = []
    for name, ty in t._fields_:
        f = getattr(t, name)
        out.append((name, f.offset, f.size))
    return out, ctypes.sizeof(t)


def test_doc_struct_layout_matches_binding():
    from paper_2412_06198_b200 import _lib

    ns = _load_snippet()
    assert _layout(ns["Pattern"]) == _layout(_lib.sa_pattern)
    assert _layout(ns["PrefillDesc"]) == _layout(_lib.sa_prefill_desc)


@pytest.mark.gpu
@pytest.mark.parametrize("mode,fixed", [("dense", None), ("fixed", (0, 300, 4)), ("fixed", (1, 64, 96)),
                                        ("fixed", (2, 8, 1)), ("fixed", (2, 4, 2))])
def test_doc_stub_matches_package(mode, fixed):
    import torch

    import paper_2412_06198_b200 as sa
    from paper_2412_06198_b200.runtime import _pat

    ns = _load_snippet()
    B, H, HK, n, d = 1, 8, 2, 1500, 128
    g = torch.Generator().manual_seed(7)
    q, k, v = (torch.randn(B, h, n, d, generator=g).to(torch.bfloat16).cuda() for h in (H, HK, HK))
    cfg = sa.ModelConfig(n_heads=H, d_model=H * d, d_head=d, max_context=n)
    kw = {} if fixed is None else {"fixed_pattern": _pat(*fixed)}
    ref = sa.prefill(q, k, v, cfg, mode=mode, **kw).outputs
    got = ns["prefill_b200"](q, k, v, mode, fixed=fixed)
    torch.cuda.synchronize()
    assert got.shape == ref.shape
    assert torch.equal(got, ref)
