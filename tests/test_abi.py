"""C ABI boundary checks that need no GPU: the in-tree library loads and
exports every entry point include/sparseattn_b200.h declares, the Python
binding types all of them, and host-side (integer) logic matches the oracle."""

import ctypes
import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "sparseattn_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sa_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2412_06198_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(_lib.exported_symbols()) == names


def test_struct_sizes_match_header_layout():
    from paper_2412_06198_b200 import _lib

    assert ctypes.sizeof(_lib.sa_pattern) == 12
    assert ctypes.sizeof(_lib.sa_head_index) == 80
    lib = _lib.load()
    assert lib.sa_version() == 1


def test_workspace_query_and_status_mapping():
    from paper_2412_06198_b200 import _lib, errors

    d = _lib.sa_prefill_desc()
    d.batch, d.heads, d.kv_heads, d.n, d.scale, d.mode, d.q_est = 1, 32, 8, 32768, 0.088, 0, 64
    assert _lib.load().sa_prefill_workspace_size(d) > 0
    d.heads = 30  # not a multiple of kv_heads
    assert _lib.load().sa_prefill_workspace_size(d) == 0
    with pytest.raises(errors.DimensionError):
        _lib.check(1)
    with pytest.raises(errors.PatternParamError):
        _lib.check(4)


def test_host_search_math_matches_oracle():
    from oracle import sparse_oracle as O
    from paper_2412_06198_b200 import search as S

    for n, d in [(64, 128), (64, 4), (256, 8), (4096, 128), (40, 16), (7, 3)]:
        s = S.default_search_space(n, d)
        cands, target, eps, iters = O.default_space(n, d)
        assert s.target_flops == target
        for c, oc in zip(s.candidates, cands):
            rc = S.refine_candidate(c, n, d, s.target_flops, s.epsilon, s.max_refine_iters)
            orc = O.refine(oc, n, d, target, eps, iters)
            assert tuple(rc.pattern.__dict__.values()) == tuple(orc[0].__dict__.values())
            assert (rc.flops, rc.iterations, rc.converged) == orc[1:]
    # auto rescale at n
    for n, tri, vs in [(4096, 384, 192), (32768, 3072, 1536), (131072, 12288, 6144)]:
        assert S._rescale_to_full(S.Triangular(6, 0), n / 64, n).window == tri
        assert S._rescale_to_full(S.VerticalSlash(3, 3), n / 64, n).k_v == vs


def test_prefill_plan_descriptor():
    from paper_2412_06198_b200.runtime import PrefillPlan

    p = PrefillPlan(1, 32, 8, 32768, 128, "auto")
    d = p.desc
    assert (d.mode, d.ncand, d.cal, d.q_est, d.preselected) == (2, 3, 64, 64, 1)
    assert [(d.full[c].family, d.full[c].p1, d.full[c].p2) for c in range(3)] == \
        [(0, 3072, 0), (1, 1536, 1536), (2, 8, 1)]
    assert p.ws_bytes > 0


def test_device_index_encoding():
    from paper_2412_06198_b200 import device_index as DI

    b = DI.HostIndexBuilder(300, 2)
    b.set_vertical_slash(0, [0, 5, 299], [0, 3])
    bits = np.unpackbits(b.colbits[0].view(np.uint8), bitorder="little")
    assert list(np.flatnonzero(bits)) == [0, 5, 299]
    rbits = np.unpackbits(b.diagrev[0].view(np.uint8), bitorder="little")
    assert sorted(300 + 127 - np.flatnonzero(rbits)) == [0, 3]


def test_peer_barrier_argument_checks():
    """sa_peer_barrier rejects bad rank / world / pointers before touching the
    device (the barrier itself runs in tests/test_gpu_multigpu_sim.py)."""
    from paper_2412_06198_b200 import _lib

    lib = _lib.load()
    buf = (ctypes.c_int32 * 16)()
    peers = (ctypes.c_void_p * 1)(None)
    assert lib.sa_peer_barrier(buf, peers, 0, 0, 1000, None) == 1  # world 0
    assert lib.sa_peer_barrier(buf, peers, 2, 2, 1000, None) == 1  # rank >= world
    assert lib.sa_peer_barrier(buf, peers, 0, 9, 1000, None) == 1  # more than 8 ranks
    assert lib.sa_peer_barrier(buf, peers, 0, 2, 1000, None) == 1  # null peer buffer
    assert lib.sa_peer_barrier(None, peers, 0, 2, 1000, None) == 1
    assert lib.sa_peer_barrier(buf, peers, 0, 2, 0, None) == 1  # no timeout
