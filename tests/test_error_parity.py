"""Error behaviour parity with the reference package (CPU; skipped when the
reference sources are absent, e.g. on the GPU box): the same invalid calls
raise the same exception classes (the reference's `SparseAttnError`
hierarchy, core.py:15-25), checked before any device work; edge calls the
reference accepts are accepted too."""
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "sparseattn")),
                                reason="reference sources not present")


@pytest.fixture(scope="module")
def mods():
    sys.path.insert(0, REF)
    try:
        import sparseattn as ref
    finally:
        sys.path.remove(REF)
    import paper_2412_06198_b200 as ours

    return ref, ours


def _raised(fn, mod):
    try:
        fn(mod)
    except Exception as e:  # noqa: BLE001 - the class is the point
        return type(e).__name__
    return None


def _qkv(shape, bad=None):
    rng = np.random.default_rng(0)
    q, k, v = (rng.uniform(-1, 1, shape).astype(np.float32) for _ in range(3))
    if bad == "nan":
        q[..., 0, 0] = np.nan
    return q, k, v


def _cfg(m, H=2, d=8, ctx=16):
    return m.ModelConfig(n_heads=H, d_model=H * d, d_head=d, max_context=ctx)


def _m(m, n=16, d=8, bad=None):
    q, k, v = _qkv((n, d), bad)
    return m.AttnMatrices(q, k, v)


CASES = {
    "config_zero": lambda m: m.ModelConfig(0, 1, 1, 1),
    "config_dmodel": lambda m: m.ModelConfig(2, 10, 4, 8),
    "prefill_3d": lambda m: m.prefill(*_qkv((2, 16, 8)), _cfg(m)),
    "prefill_heads": lambda m: m.prefill(*_qkv((1, 3, 16, 8)), _cfg(m)),
    "prefill_dhead": lambda m: m.prefill(*_qkv((1, 2, 16, 4)), _cfg(m)),
    "prefill_too_long": lambda m: m.prefill(*_qkv((1, 2, 17, 8)), _cfg(m)),
    "prefill_mode": lambda m: m.prefill(*_qkv((1, 2, 16, 8)), _cfg(m), mode="bogus"),
    "prefill_fixed_none": lambda m: m.prefill(*_qkv((1, 2, 16, 8)), _cfg(m), mode="fixed"),
    "tri_window": lambda m: m.Triangular(0),
    "tri_sinks": lambda m: m.Triangular(3, -1),
    "vs_zero": lambda m: m.VerticalSlash(0, 1),
    "block_zero": lambda m: m.BlockSparse(0, 1),
    "block_kb": lambda m: m.BlockSparse(4, 0),
    "mats_shape": lambda m: m.AttnMatrices(*(_qkv((16, 8))[:2] + (np.zeros((15, 8), np.float32),))),
    "mats_ndim": lambda m: m.AttnMatrices(*_qkv((2, 16, 8))),
    "mats_nan": lambda m: m.AttnMatrices(*_qkv((16, 8), "nan")),
    "score_mode": lambda m: m.score_columns(_m(m), mode="bogus"),
    "score_qest": lambda m: m.score_diagonals(_m(m), mode="estimated", q_est=0),
    "score_qest_big": lambda m: m.score_columns(_m(m), mode="estimated", q_est=17),
    "vs_index_kv": lambda m: m.build_vertical_slash_index(_m(m), 0, 1),
    "vs_index_ks": lambda m: m.build_vertical_slash_index(_m(m), 1, 17),
    "block_index_b": lambda m: m.build_block_index(_m(m), 0, 1),
    "block_index_b_big": lambda m: m.build_block_index(_m(m), 17, 1),
    "block_index_kb": lambda m: m.build_block_index(_m(m), 4, 5),
    "block_mean_b": lambda m: m.block_mean(np.zeros((8, 4), np.float32), 0),
    "space_density": lambda m: m.default_search_space(64, 8, density=0.0),
    "space_n": lambda m: m.default_search_space(0, 8),
    "flops_unknown": lambda m: m.estimate_flops(object(), 64, 8),
    "flops_n": lambda m: m.estimate_flops(m.Triangular(4), 0, 8),
    "refine_eps": lambda m: m.refine_candidate(m.Triangular(4), 64, 8, 1000, -1.0, 8),
    "refine_iters": lambda m: m.refine_candidate(m.VerticalSlash(4, 4), 64, 8, 1000, 0.05, -1),
    "select_metric": lambda m: m.select_pattern(_m(m), m.default_search_space(16, 8), metric="bogus"),
    "select_scoring": lambda m: m.select_pattern(_m(m), m.default_search_space(16, 8), scoring="bogus"),
    "select_qest0": lambda m: m.select_pattern(_m(m), m.default_search_space(16, 8), scoring="estimated", q_est=0),
    "select_cap": lambda m: m.select_pattern(_m(m), m.default_search_space(16, 8), dense_cap=8),
    "windowed_cal0": lambda m: m.select_pattern_windowed(_m(m), m.default_search_space(16, 8), 0),
    "windowed_cal_big": lambda m: m.select_pattern_windowed(_m(m), m.default_search_space(16, 8), 17),
    "prefill_cal_cap": lambda m: m.prefill(*_qkv((1, 2, 16, 8)), _cfg(m), mode="auto", cal_window=16,
                                           dense_cap=8),
    "sparse_block_kernel_vs": lambda m: m.vertical_slash_attention(
        _m(m), m.SparseIndex(n=16, blocks=((0, 0),), block_size=16, always_diagonal=False)),
    "index_col_range": lambda m: m.SparseIndex(n=16, columns=(16,)),
    "index_causal": lambda m: m.SparseIndex(n=16, blocks=((0, 1),), block_size=8),
    "realized_n": lambda m: m.realized_size(m.SparseIndex(n=16, columns=(1,)), 15),
    # argument errors the reference meets inside its per-head loop
    "prefill_cal0": lambda m: m.prefill(*_qkv((1, 2, 16, 8)), _cfg(m), mode="auto", cal_window=0),
    "prefill_cal_neg": lambda m: m.prefill(*_qkv((1, 2, 16, 8)), _cfg(m), mode="auto", cal_window=-3),
    "prefill_qest0_fixed_vs": lambda m: m.prefill(*_qkv((1, 2, 16, 8)), _cfg(m), mode="fixed",
                                                  fixed_pattern=m.VerticalSlash(2, 2), q_est=0),
    "prefill_qest_neg_auto": lambda m: m.prefill(*_qkv((1, 2, 16, 8)), _cfg(m), mode="auto", q_est=-1),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_same_exception_class(mods, name):
    ref, ours = mods
    want = _raised(CASES[name], ref)
    got = _raised(CASES[name], ours)
    assert got == want, f"{name}: reference raises {want}, ours {got}"
