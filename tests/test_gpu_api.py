"""The drop-in API on a B200, mirroring the reference's own tests
(pkg/tests/test_patterns.py, test_search.py, test_runtime.py, test_acceptance.py)
with the bf16 tolerances of the north star, plus the reference-generated
golden prefill cases (tests/golden/)."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import sparse_oracle as O  # noqa: E402
from tests.golden_io import load, uniform  # noqa: E402

MAX_ABS, MEAN_ABS = 2e-2, 2e-3


@pytest.fixture(scope="module")
def sa():
    import paper_2412_06198_b200 as m

    return m


def bf(x):
    return O.bf16_round(np.asarray(x, np.float32)).astype(np.float64)


def mats(sa, seed, n, d=4):
    q, k, v = (bf(x) for x in uniform(seed, n, d))
    return sa.AttnMatrices(q, k, v), (q, k, v)


def close(a, b):
    err = np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))
    assert err.max() <= MAX_ABS and err.mean() <= MEAN_ABS, (err.max(), err.mean())


# ---- scoring / indices (test_patterns.py:44-127) -------------------------------

def test_zero_logit_scores(sa):
    z = np.zeros((2, 2))
    m = sa.AttnMatrices(z, z, z)
    np.testing.assert_allclose(sa.score_columns(m), [1.5, 0.5], atol=1e-6)
    np.testing.assert_allclose(sa.score_diagonals(m), [1.5, 0.5], atol=1e-6)
    z1 = np.zeros((1, 2))
    np.testing.assert_allclose(sa.score_diagonals(sa.AttnMatrices(z1, z1, z1)), [1.0], atol=1e-6)


def test_scores_match_oracle(sa):
    m, (q, k, _) = mats(sa, 6, 40, 8)
    cs, ds = O.vs_scores(q, k, "estimated", 9)
    np.testing.assert_allclose(sa.score_columns(m, "estimated", 9), cs, rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(sa.score_diagonals(m, "estimated", 9), ds, rtol=1e-5, atol=1e-7)


def test_bad_scoring_args(sa):
    m, _ = mats(sa, 8, 4)
    with pytest.raises(sa.PatternParamError):
        sa.score_columns(m, "bogus")
    with pytest.raises(sa.PatternParamError):
        sa.score_columns(m, "estimated", q_est=0)
    with pytest.raises(sa.PatternParamError):
        sa.score_columns(m, "estimated", q_est=5)


def test_vs_index_ties_and_zero_logits(sa):
    z = np.zeros((6, 3))
    idx = sa.build_vertical_slash_index(sa.AttnMatrices(z, z, z), 1, 1)
    assert idx.diagonals == (0,)
    z = np.zeros((4, 2))
    idx = sa.build_vertical_slash_index(sa.AttnMatrices(z, z, z), 2, 2)
    assert idx.columns == (0, 1) and idx.diagonals == (0, 1)


def test_vs_index_matches_oracle(sa):
    m, (q, k, _) = mats(sa, 11, 64, 8)
    idx = sa.build_vertical_slash_index(m, 5, 7)
    o = O.vs_index(q, k, 5, 7)
    assert list(idx.columns) == o.columns.tolist() and list(idx.diagonals) == o.diagonals.tolist()


def test_block_index_matches_oracle(sa):
    m, (q, k, _) = mats(sa, 24, 16, 4)
    idx = sa.build_block_index(m, 4, 2)
    o = O.block_index(q, k, 4, 2)
    want = [(g, int(x)) for g, r in enumerate(o.block_rows) for x in r]
    assert list(idx.blocks) == want
    z = np.zeros((4, 2))
    zi = sa.build_block_index(sa.AttnMatrices(z, z, z), 2, 1)
    assert (0, 0) in zi.blocks and (1, 1) in zi.blocks


def test_block_mean(sa):
    x = np.arange(8, dtype=float).reshape(4, 2)
    np.testing.assert_allclose(sa.block_mean(x, 2), [(x[0] + x[1]) / 2, (x[2] + x[3]) / 2])
    x = np.random.default_rng(21).random((5, 2))
    out = sa.block_mean(x, 2)
    assert out.shape == (3, 2)
    np.testing.assert_allclose(out[2], x[4], rtol=1e-6)


# ---- kernels (test_patterns.py:130-268, test_acceptance.py:87-183) -------------

@pytest.mark.parametrize("n", [1, 2, 3, 8, 33, 64])
def test_full_coverage_equals_dense(sa, n):
    m, (q, k, v) = mats(sa, 100 + n, n, 4)
    w_d, y_d = sa.dense_attention(m)
    idx = sa.build_vertical_slash_index(m, n, n)
    w, y = sa.vertical_slash_attention(m, idx)
    close(y, y_d)
    close(w, w_d)
    close(y_d, O.dense_attention(q, k, v)[1])


def test_diagonal_only_is_identity(sa):
    m, (q, k, v) = mats(sa, 14, 7)
    w, y = sa.vertical_slash_attention(m, sa.SparseIndex(n=7, always_diagonal=True))
    np.testing.assert_allclose(w, np.eye(7), atol=1e-6)
    np.testing.assert_allclose(y, v, atol=1e-2)


@pytest.mark.parametrize("seed", range(6))
def test_kernels_match_mask_then_dense(sa, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 65))
    m, (q, k, v) = mats(sa, 200 + seed, n, int(rng.integers(2, 9)))
    k_v, k_s = int(rng.integers(1, n + 1)), int(rng.integers(1, n + 1))
    b = int(rng.integers(1, n + 1))
    nb = -(-n // b)
    for idx, oidx in (
        (sa.build_vertical_slash_index(m, k_v, k_s), O.vs_index(q, k, k_v, k_s)),
        (sa.build_block_index(m, b, int(rng.integers(1, nb + 1))), None),
        (sa.build_triangular_index(n, max(1, n // 3), min(2, n)), O.tri_index(n, max(1, n // 3), min(2, n))),
    ):
        w, y = sa.sparse_attention(m, idx)
        if oidx is None:
            rows = [[] for _ in range(-(-n // idx.block_size))]
            for gq, gk in idx.blocks:
                rows[gq].append(gk)
            oidx = O.Index(n, np.zeros(0, np.int64), np.zeros(0, np.int64), idx.block_size,
                           [np.array(r) for r in rows])
        allowed = O.index_mask_rows(oidx, 0, n)
        assert (np.asarray(w)[~allowed] == 0).all()
        np.testing.assert_allclose(np.asarray(w).sum(axis=1), 1.0, atol=1e-5)
        close(y, O.masked_attention(q, k, v, oidx))
        assert sa.realized_size(idx, n) == int(allowed.sum())


def test_work_bound(sa):
    m, _ = mats(sa, 32, 17)
    idx = sa.build_vertical_slash_index(m, 3, 4)
    c = sa.MacCounter()
    sa.sparse_attention(m, idx, counter=c)
    assert c.logit_macs == sa.realized_size(idx, 17) * m.d_head == c.output_macs


def test_kernel_rejections(sa):
    m, _ = mats(sa, 17, 8)
    with pytest.raises(sa.PatternParamError):
        sa.vertical_slash_attention(m, sa.build_block_index(m, 4, 1))
    with pytest.raises(sa.PatternParamError):
        sa.block_sparse_attention(m, sa.build_triangular_index(8, 2, 1))
    with pytest.raises(sa.DimensionError):
        sa.vertical_slash_attention(m, sa.SparseIndex(n=5))
    bad = np.array([[np.nan, 0.0], [0.0, 0.0]])
    with pytest.raises(sa.NonFiniteError):
        sa.AttnMatrices(bad, bad, bad)


# ---- search (test_search.py) -----------------------------------------------------

def test_select_pattern_matches_oracle(sa):
    _, meta = load()
    for c in meta["cases"]["select"]:
        q, k, v = (bf(x) for x in uniform(c["seed"], c["n"], c["d"]))
        m = sa.AttnMatrices(q, k, v)
        res = sa.select_pattern(m, sa.default_search_space(c["n"], c["d"]))
        o = O.select(q, k, v, O.default_space(c["n"], c["d"]))
        assert type(res.chosen).__name__[0] == type(o[0]).__name__[0]
        assert abs(res.error - o[2]) <= 1e-3 * max(1.0, o[2])


def test_windowed_rescale(sa):
    """search.py:261-319: the window choice, its parameters rescaled by n/cal
    and its error equal the oracle's (reference test_search.py:255-273)."""
    m, (q, k, v) = mats(sa, 77, 256, 8)
    res = sa.select_pattern_windowed(m, sa.default_search_space(64, 8), 64)
    want, err, _ = O.select_windowed(q, k, v, O.default_space(64, 8), 64)
    assert (type(res.chosen).__name__[0], *res.chosen.__dict__.values()) == \
        (type(want).__name__[0], *want.__dict__.values())
    assert abs(res.error - err) <= 1e-4 * max(1.0, err)


def test_windowed_proportional_rescale(sa):
    """test_search.py:261-266: VS(4,4) chosen on a 64-row window of 256 -> VS(16,16)."""
    m, _ = mats(sa, 51, 256, 4)
    p = sa.VerticalSlash(4, 4)
    s = sa.SearchSpace([p], target_flops=sa.estimate_flops(p, 64, 4).total)
    assert sa.select_pattern_windowed(m, s, 64).chosen == sa.VerticalSlash(16, 16)


def test_windowed_block_geometry_kept(sa):
    """test_search.py:268-273: a block candidate keeps its geometry."""
    m, _ = mats(sa, 52, 128, 4)
    p = sa.BlockSparse(b=8, k_b=2)
    s = sa.SearchSpace([p], target_flops=sa.estimate_flops(p, 64, 4).total)
    assert sa.select_pattern_windowed(m, s, 64).chosen == p


# ---- runtime (test_runtime.py, golden prefill) -----------------------------------

def test_single_token_output_is_v(sa):
    rng = np.random.default_rng(60)
    cfg = sa.ModelConfig(n_heads=2, d_model=6, d_head=3, max_context=4)
    q, k, v = (rng.uniform(-1, 1, (1, 2, 1, 3)) for _ in range(3))
    for mode, kw in (("dense", {}), ("fixed", {"fixed_pattern": sa.Triangular(1)}), ("auto", {})):
        res = sa.prefill(q, k, v, cfg, mode=mode, **kw)
        np.testing.assert_allclose(res.outputs[0, 0], v[0, :, 0, :].reshape(6), atol=1e-2)
        assert res.cache.length == 1


def test_fixed_full_window_equals_dense(sa):
    rng = np.random.default_rng(61)
    cfg = sa.ModelConfig(n_heads=2, d_model=8, d_head=4, max_context=32)
    q, k, v = (rng.uniform(-1, 1, (1, 2, 32, 4)) for _ in range(3))
    dense = sa.prefill(q, k, v, cfg, mode="dense")
    fixed = sa.prefill(q, k, v, cfg, mode="fixed", fixed_pattern=sa.Triangular(window=32))
    np.testing.assert_allclose(fixed.outputs, dense.outputs, atol=1e-6)


def test_prefill_rejections(sa):
    cfg = sa.ModelConfig(n_heads=2, d_model=8, d_head=4, max_context=8)
    x = np.zeros((1, 2, 16, 4))
    with pytest.raises(sa.DimensionError):
        sa.prefill(x, x, x, cfg)
    x = np.zeros((1, 2, 8, 4))
    with pytest.raises(sa.SparseAttnError):
        sa.prefill(x, x, x, cfg, mode="fixed")
    with pytest.raises(sa.SparseAttnError):
        sa.prefill(x, x, x, cfg, mode="bogus")


def test_decode_consistent_with_prefill(sa):
    rng = np.random.default_rng(62)
    cfg = sa.ModelConfig(n_heads=2, d_model=16, d_head=8, max_context=40)
    q, k, v = (rng.uniform(-1, 1, (1, 2, 33, 8)) for _ in range(3))
    full = sa.prefill(q, k, v, cfg, mode="dense")
    part = sa.prefill(q[:, :, :32], k[:, :, :32], v[:, :, :32], cfg, mode="dense")
    dec = sa.decode_step(q[:, :, 32:], k[:, :, 32:], v[:, :, 32:], part.cache, cfg)
    close(dec.output[0, 0], full.outputs[0, 32])
    assert dec.cache.length == 33


def pat_from(js):
    fam, a, b = js
    return {"triangular": O.Tri, "vertical-slash": O.VS, "block-sparse": O.Blk}[fam](a, b)


@pytest.mark.parametrize("cid", range(8))
def test_golden_prefill(sa, cid):
    arr, meta = load()
    c = meta["cases"]["prefill"][cid]
    if c["H"] == c["HK"]:
        q, k, v = O.synth_qkv(c["seed"], c["ctx"], c["H"], 128)
    else:
        q, k, v = O.synth_qkv_gqa(c["seed"], c["ctx"], c["H"], c["HK"], 128)
    q, k, v = (O.bf16_round(x) for x in (q, k, v))
    cfg = sa.ModelConfig(n_heads=c["H"], d_model=c["H"] * 128, d_head=128, max_context=c["ctx"])
    kw = {}
    if c["mode"] == "fixed":
        p = O.fixed_pattern_for(c["fixed"], c["ctx"])
        kw["fixed_pattern"] = {O.Tri: sa.Triangular, O.VS: sa.VerticalSlash, O.Blk: sa.BlockSparse}[type(p)](
            *p.__dict__.values())
    res = sa.prefill(q, k, v, cfg, mode=c["mode"], **kw)
    got_plans = [hp.pattern for hp in res.plans[0]]
    want = [pat_from(p) if p else None for p in c["plans"]]
    conv = lambda p: None if p is None else (type(p).__name__[0], *p.__dict__.values())  # noqa: E731
    assert [conv(p) for p in got_plans] == [conv(p) for p in want]
    step = max(1, c["ctx"] // 64)
    close(res.outputs[0, ::step], arr[f"prefill_{cid}_rows"])


@pytest.mark.parametrize("mode,n", [("auto", 1000), ("auto", 2048), ("dense", 300), ("fixed", 777)])
def test_host_streamed_prefill_equals_device(sa, mode, n):
    """CPU torch inputs stream through the GPU one kv group at a time; the
    result (outputs, plans, cache) is identical to the device-input call."""
    H, HK = 8, 2
    q, k, v = O.synth_qkv_gqa(5, n, H, HK, 128)
    q, k, v = (torch.from_numpy(O.bf16_round(x)).bfloat16() for x in (q, k, v))
    cfg = sa.ModelConfig(n_heads=H, d_model=H * 128, d_head=128, max_context=n + 4)
    kw = {"fixed_pattern": sa.VerticalSlash(40, 50)} if mode == "fixed" else {}
    host = sa.prefill(q.pin_memory(), k.pin_memory(), v.pin_memory(), cfg, mode=mode, **kw)
    dev = sa.prefill(q.cuda(), k.cuda(), v.cuda(), cfg, mode=mode, **kw)
    assert not host.outputs.is_cuda and host.outputs.dtype == torch.bfloat16
    assert torch.equal(host.outputs, dev.outputs.cpu())
    assert [hp.pattern for hp in host.plans[0]] == [hp.pattern for hp in dev.plans[0]]
    assert host.cache.length == n
    assert torch.equal(host.cache.keys().cpu(), k.cuda().cpu())
    assert torch.equal(host.cache.values().cpu(), v)
    if mode == "auto":
        e1 = [hp.search.error for hp in host.plans[0]]
        e2 = [hp.search.error for hp in dev.plans[0]]
        np.testing.assert_allclose(e1, e2, rtol=0, atol=0)


def test_host_streamed_nonfinite(sa):
    H, HK, n = 4, 2, 256
    q, k, v = O.synth_qkv_gqa(6, n, H, HK, 128)
    q, k, v = (torch.from_numpy(O.bf16_round(x)).bfloat16() for x in (q, k, v))
    cfg = sa.ModelConfig(n_heads=H, d_model=H * 128, d_head=128, max_context=n)
    v[0, 1, 17, 3] = float("nan")
    with pytest.raises(sa.NonFiniteError):
        sa.prefill(q, k, v, cfg, mode="auto")
    v[0, 1, 17, 3] = 0.0
    k[0, 0, n - 1, 127] = float("inf")
    with pytest.raises(sa.NonFiniteError):
        sa.prefill(q, k, v, cfg, mode="dense")


# ---- runtime tests of the reference (test_runtime.py:74-148), device path ----

def _inputs(seed, B, H, L, d):
    rng = np.random.default_rng(seed)
    return tuple(bf(rng.uniform(-1, 1, (B, H, L, d))) for _ in range(3))


def test_auto_matches_manual_composition(sa):
    """test_runtime.py:82-92: prefill(auto) == per-head build_index + sparse_attention."""
    cfg = sa.ModelConfig(n_heads=2, d_model=8, d_head=4, max_context=64)
    q, k, v = _inputs(62, 1, 2, 64, 4)
    res = sa.prefill(q, k, v, cfg, mode="auto", cal_window=32, q_est=16)
    for plan in res.plans[0]:
        m = sa.AttnMatrices(q[0, plan.head], k[0, plan.head], v[0, plan.head])
        idx = sa.build_index(m, plan.pattern, mode="estimated", q_est=16)
        _, y = sa.sparse_attention(m, idx, need_weights=False)
        h0 = plan.head * 4
        close(res.outputs[0, :, h0:h0 + 4], y)


def test_head_permutation_permutes_outputs_and_plans(sa):
    """test_runtime.py:105-117 (exact equality: heads are independent on device too)."""
    cfg = sa.ModelConfig(n_heads=3, d_model=6, d_head=2, max_context=16)
    q, k, v = _inputs(64, 1, 3, 16, 2)
    perm = [2, 0, 1]
    base = sa.prefill(q, k, v, cfg, mode="auto", cal_window=8)
    pres = sa.prefill(q[:, perm], k[:, perm], v[:, perm], cfg, mode="auto", cal_window=8)
    for new_h, old_h in enumerate(perm):
        np.testing.assert_array_equal(pres.outputs[0, :, new_h * 2:new_h * 2 + 2],
                                      base.outputs[0, :, old_h * 2:old_h * 2 + 2])
        assert pres.plans[0][new_h].pattern == base.plans[0][old_h].pattern


@pytest.mark.parametrize("mode", ["dense", "auto"])
def test_batched_sequences_independent(sa, mode):
    """test_runtime.py:119-125, plus batch 3 x 4 heads x GQA against the oracle."""
    cfg = sa.ModelConfig(n_heads=1, d_model=4, d_head=4, max_context=8)
    q, k, v = _inputs(65, 2, 1, 8, 4)
    both = sa.prefill(q, k, v, cfg, mode=mode)
    solo = sa.prefill(q[1:], k[1:], v[1:], cfg, mode=mode)
    np.testing.assert_array_equal(both.outputs[1], solo.outputs[0])
    B, H, HK, n = 3, 4, 2, 700
    q, k, v = (bf(x) for x in O.synth_qkv_gqa(66, n, H, HK, 128))
    q, k, v = (np.concatenate([x, x[:, ::-1] * 0.5, -x], 0) for x in (q, k, v))
    cfg = sa.ModelConfig(n_heads=H, d_model=H * 128, d_head=128, max_context=n)
    res = sa.prefill(q, k, v, cfg, mode=mode)
    want, plans = O.prefill(q, k, v, mode)
    close(res.outputs, want)
    if mode == "auto":
        conv = lambda p: (type(p).__name__[0], *p.__dict__.values())  # noqa: E731
        assert [[conv(hp.pattern) for hp in row] for row in res.plans] == [[conv(p) for p in row] for row in plans]


def test_batched_host_streamed(sa):
    """CPU torch inputs with batch 2 stream per (batch, kv group); same result as device inputs."""
    B, H, HK, n = 2, 4, 2, 513
    q, k, v = (torch.from_numpy(bf(x).astype(np.float32)).bfloat16() for x in O.synth_qkv_gqa(67, n, H, HK, 128))
    q, k, v = (torch.cat([x, x.flip(2)], 0) for x in (q, k, v))
    cfg = sa.ModelConfig(n_heads=H, d_model=H * 128, d_head=128, max_context=n)
    host = sa.prefill(q, k, v, cfg, mode="auto")
    dev = sa.prefill(q.cuda(), k.cuda(), v.cuda(), cfg, mode="auto")
    assert torch.equal(host.outputs, dev.outputs.cpu())
    assert [[hp.pattern for hp in r] for r in host.plans] == [[hp.pattern for hp in r] for r in dev.plans]


def test_timing_decomposition(sa):
    """test_runtime.py:139-147."""
    cfg = sa.ModelConfig(n_heads=2, d_model=8, d_head=4, max_context=64)
    q, k, v = _inputs(67, 1, 2, 64, 4)
    res = sa.prefill(q, k, v, cfg, mode="auto", cal_window=32)
    assert res.elapsed_s >= res.kernel_s >= 0.0
    assert res.select_s >= 0.0
    assert res.elapsed_s > 0.0


def test_prefill_plan_graph_replay(sa):
    """PrefillPlan.graph: a CUDA-graph replay equals the eager layer, and recomputes
    for new contents of the same input buffers."""
    from paper_2412_06198_b200 import runtime as R

    H, HK, n = 8, 2, 1000
    q, k, v = (torch.from_numpy(O.bf16_round(x)[0]).cuda().bfloat16() for x in O.synth_qkv_gqa(71, n, H, HK, 128))
    plan = R.PrefillPlan(1, H, HK, n, 128, "auto")
    ws = R._workspace(plan.ws_bytes, q.device)
    out = torch.empty((1, n, H * 128), dtype=torch.bfloat16, device="cuda")
    plan.select(q, k, ws)
    plan.run(q, k, v, out, ws)
    eager = out.clone()
    g = plan.graph(q, k, v, out, ws)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager)
    q.mul_(-1)
    g.replay()
    plan.select(q, k, ws)
    ref = torch.empty_like(out)
    plan.run(q, k, v, ref, ws)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


@pytest.mark.parametrize("extra", [8, 16])
def test_out_ld_row_layouts(sa, extra):
    """desc.out_ld wider than heads * 128: rows 16-byte aligned only (extra = 8,
    16-byte stores) or 32-byte aligned (extra = 16, 256-bit stores) give the
    same columns as the packed layout; out_ld % 8 != 0 is rejected."""
    from paper_2412_06198_b200 import runtime as R

    H, HK, n = 4, 2, 700
    q, k, v = O.synth_qkv_gqa(9, n, H, HK, 128)
    q, k, v = (torch.from_numpy(O.bf16_round(x[0])).bfloat16().cuda() for x in (q, k, v))
    plan = R.PrefillPlan(1, H, HK, n, 128, "fixed", fixed_pattern=sa.VerticalSlash(40, 50))
    ws = R._workspace(plan.ws_bytes, q.device)
    ref = torch.empty((1, n, H * 128), dtype=torch.bfloat16, device="cuda")
    plan.run(q, k, v, ref, ws)
    ld = H * 128 + extra
    wide = torch.zeros((1, n, ld), dtype=torch.bfloat16, device="cuda")
    plan.desc.out_ld = ld
    try:
        plan.run(q, k, v, wide, ws)
        torch.cuda.synchronize()
        assert torch.equal(wide[..., : H * 128], ref)
        assert not wide[..., H * 128:].any()
        plan.desc.out_ld = ld + 4
        with pytest.raises(sa.SparseAttnError):
            plan.run(q, k, v, wide, ws)
    finally:
        plan.desc.out_ld = 0


@pytest.mark.parametrize("H,HK,d,n,dt,B", [(8, 2, 128, 3000, "bf16", 1), (4, 4, 5, 300, "f32", 1),
                                           (32, 8, 128, 9000, "bf16", 1), (16, 1, 64, 700, "f32", 1),
                                           (8, 4, 128, 1000, "bf16", 3)])
def test_decode_step_split_k(sa, H, HK, d, n, dt, B):
    """decode_step (split-K kernel over the cache, in place) equals dense
    attention of the last row: both GQA and MHA, bf16 and fp32 caches, odd
    head_dim, query heads per kv head above one pass (16)."""
    rng = np.random.default_rng(n + d)
    q, k, v = (rng.uniform(-1, 1, (B, h, n, d)).astype(np.float32) for h in (H, HK, HK))
    if dt == "bf16":
        q, k, v = (torch.from_numpy(x).bfloat16().cuda() for x in (q, k, v))
    else:
        q, k, v = (torch.from_numpy(x).cuda() for x in (q, k, v))
    cfg = sa.ModelConfig(n_heads=H, d_model=H * d, d_head=d, max_context=n + 8)
    part = sa.prefill(q[:, :, : n - 1], k[:, :, : n - 1], v[:, :, : n - 1], cfg, mode="dense")
    dec = sa.decode_step(q[:, :, n - 1:], k[:, :, n - 1:], v[:, :, n - 1:], part.cache, cfg)
    assert dec.cache.length == n
    g = H // HK
    kf, vf = k.float().repeat_interleave(g, 1), v.float().repeat_interleave(g, 1)
    s = torch.einsum("bhd,bhjd->bhj", q[:, :, n - 1].float(), kf) / math.sqrt(d)
    want = torch.einsum("bhj,bhjd->bhd", torch.softmax(s.double(), 2).float(), vf).reshape(B, 1, H * d)
    err = (dec.output.float() - want).abs()
    assert err.max().item() <= MAX_ABS and err.mean().item() <= MEAN_ABS, (err.max().item(), err.mean().item())


@pytest.mark.parametrize("kind", ["numpy", "cpu_torch", "cuda_f32"])
def test_prefill_cache_keeps_input_rows(sa, kind):
    """The reference caches k/v as given (runtime.py:197): fp32 inputs are not
    replaced by their bf16 rounding, so a following decode is fp32-exact."""
    import torch

    rng = np.random.default_rng(91)
    H, HK, n, d = 4, 2, 300, 128
    q, k, v = (rng.uniform(-1, 1, (1, h, n + 1, d)).astype(np.float32) for h in (H, HK, HK))
    conv = {"numpy": lambda x: x, "cpu_torch": lambda x: torch.from_numpy(np.ascontiguousarray(x)),
            "cuda_f32": lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()}[kind]
    cfg = sa.ModelConfig(n_heads=H, d_model=H * d, d_head=d, max_context=n + 1)
    res = sa.prefill(conv(q[:, :, :n]), conv(k[:, :, :n]), conv(v[:, :, :n]), cfg, mode="dense")
    keys = res.cache.keys()
    keys = keys.cpu().numpy() if hasattr(keys, "cpu") else np.asarray(keys)
    np.testing.assert_array_equal(keys, k[:, :, :n])
    dec = sa.decode_step(conv(q[:, :, n:]), conv(k[:, :, n:]), conv(v[:, :, n:]), res.cache, cfg)
    out = dec.output.cpu().numpy() if hasattr(dec.output, "cpu") else np.asarray(dec.output)
    kk, vv = np.repeat(k, H // HK, axis=1)[0].astype(np.float64), np.repeat(v, H // HK, axis=1)[0].astype(np.float64)
    s = np.einsum("hd,hnd->hn", q[0, :, n].astype(np.float64), kk) / np.sqrt(d)
    w = np.exp(s - s.max(-1, keepdims=True))
    w /= w.sum(-1, keepdims=True)
    np.testing.assert_allclose(out.reshape(H, d), np.einsum("hn,hnd->hd", w, vv), atol=1e-5)


def test_decode_and_cache_errors(sa):
    """Decode / KvCache error classes as the reference raises them
    (runtime.py:222-225 decode_step, runtime.py:69-78 KvCache.append)."""
    rng = np.random.default_rng(93)
    H, d, n = 2, 8, 16
    cfg = sa.ModelConfig(n_heads=H, d_model=H * d, d_head=d, max_context=n)
    q, k, v = (rng.uniform(-1, 1, (1, H, n, d)).astype(np.float32) for _ in range(3))
    res = sa.prefill(q, k, v, cfg, mode="dense")
    one = (rng.uniform(-1, 1, (1, H, 1, d)).astype(np.float32) for _ in range(3))
    with pytest.raises(sa.CacheOverflowError):  # capacity max_context = n is full
        sa.decode_step(*one, res.cache, cfg)
    two = [rng.uniform(-1, 1, (1, H, 2, d)).astype(np.float32) for _ in range(3)]
    with pytest.raises(sa.DimensionError):
        sa.decode_step(*two, res.cache, cfg)
    empty = sa.KvCache(1, H, d, 8)
    with pytest.raises(sa.SparseAttnError):
        sa.decode_step(*(x[:, :, :1] for x in two), empty, cfg)
    with pytest.raises(sa.DimensionError):
        empty.append(two[1], two[2][:, :, :1])
    with pytest.raises(sa.DimensionError):
        empty.append(two[1][:, :1], two[2][:, :1])


def test_decode_past_prefill_limit(sa):
    """A cache filled to the prefill limit (262144 rows) keeps decoding: the
    split-K kernel takes up to 8M cached rows (1024-key chunks)."""
    H, HK, d, n = 4, 1, 128, 262144 + 1000
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    k, v = ((torch.rand((1, HK, n, d), generator=g, device="cuda") * 2 - 1).bfloat16() for _ in range(2))
    q = (torch.rand((1, H, 1, d), generator=g, device="cuda") * 2 - 1).bfloat16()
    cfg = sa.ModelConfig(n_heads=H, d_model=H * d, d_head=d, max_context=n + 1)
    cache = sa.KvCache(1, H, d, n + 1, dtype=torch.bfloat16, kv_heads=HK)
    cache.append(k, v)
    kn, vn = ((torch.rand((1, HK, 1, d), generator=g, device="cuda") * 2 - 1).bfloat16() for _ in range(2))
    dec = sa.decode_step(q, kn, vn, cache, cfg)
    kf = torch.cat([k, kn], 2).float().repeat_interleave(H // HK, 1)[0]
    vf = torch.cat([v, vn], 2).float().repeat_interleave(H // HK, 1)[0]
    s = torch.einsum("hd,hjd->hj", q[0, :, 0].float(), kf) / math.sqrt(d)
    want = torch.einsum("hj,hjd->hd", torch.softmax(s.double(), 1).float(), vf).reshape(1, 1, H * d)
    err = (dec.output.float() - want).abs()
    assert dec.cache.length == n + 1
    assert err.max().item() <= MAX_ABS and err.mean().item() <= MEAN_ABS


# ---- wide calibration windows and long candidate lists ---------------

@pytest.mark.parametrize("cal", [128, 200])
def test_prefill_wide_calibration_window(sa, cal):
    """cal_window > 64 takes the composed selection (fp32 weights): the per-head
    choice AND its window error equal the oracle's (search.py:276-319)."""
    q, k, v = O.synth_qkv_gqa(21, 600, 4, 2, 128)
    q, k, v = (O.bf16_round(x) for x in (q, k, v))
    cfg = sa.ModelConfig(n_heads=4, d_model=4 * 128, d_head=128, max_context=600)
    res = sa.prefill(q, k, v, cfg, mode="auto", cal_window=cal)
    kx, vx = O.expand_kv(k, 4), O.expand_kv(v, 4)
    space = O.default_space(cal, 128)
    for h, hp in enumerate(res.plans[0]):
        want, err, _ = O.select_windowed(q[0, h], kx[0, h], vx[0, h], space, cal)
        assert (type(hp.pattern).__name__[0], *hp.pattern.__dict__.values()) == \
            (type(want).__name__[0], *want.__dict__.values())
        assert abs(hp.search.error - err) <= 1e-4 * max(1.0, err), (h, hp.search.error, err)
    want_out, _ = O.prefill(q, k, v, "auto", cal_window=cal)
    close(res.outputs, want_out)


def test_prefill_many_candidates(sa):
    """A search space with more than 3 candidates (repeated families, as the
    reference accepts): the device selects among all of them with the
    reference's refinement and strict-< argmin (earlier wins ties)."""
    q, k, v = O.synth_qkv_gqa(22, 512, 4, 2, 128)
    q, k, v = (O.bf16_round(x) for x in (q, k, v))
    cfg = sa.ModelConfig(n_heads=4, d_model=4 * 128, d_head=128, max_context=512)
    target = O.default_space(64, 128)[1]
    cands = [sa.Triangular(16), sa.VerticalSlash(2, 2), sa.BlockSparse(8, 1), sa.Triangular(8),
             sa.VerticalSlash(4, 1), sa.BlockSparse(8, 2), sa.Triangular(16)]
    ocands = [O.Tri(16, 0), O.VS(2, 2), O.Blk(8, 1), O.Tri(8, 0), O.VS(4, 1), O.Blk(8, 2), O.Tri(16, 0)]
    res = sa.prefill(q, k, v, cfg, sa.SearchSpace(cands, target_flops=target), mode="auto")
    kx, vx = O.expand_kv(k, 4), O.expand_kv(v, 4)
    for h, hp in enumerate(res.plans[0]):
        want, err, _ = O.select_windowed(q[0, h], kx[0, h], vx[0, h], (ocands, target, 0.05, 8), 64)
        assert (type(hp.pattern).__name__[0], *hp.pattern.__dict__.values()) == \
            (type(want).__name__[0], *want.__dict__.values()), h
        assert abs(hp.search.error - err) <= 1e-4 * max(1.0, err)


# ---- non-causal dense attention (core.py:138-154; test_core.py:55-61) ------------

def _naive_attention(q, k, v, causal):
    """float64 three-loop restatement (reference tests/oracles.py:12-30)."""
    n, d = q.shape
    s = (q.astype(np.float64) @ k.astype(np.float64).T) / np.sqrt(d)
    if causal:
        s = np.where(np.tri(n, dtype=bool), s, -np.inf)
    w = np.exp(s - s.max(axis=1, keepdims=True))
    w /= w.sum(axis=1, keepdims=True)
    return w, w @ v.astype(np.float64)


@pytest.mark.parametrize("n,d", [(5, 3), (128, 128), (300, 64), (1000, 128)])
def test_dense_non_causal(sa, n, d):
    m, (q, k, v) = mats(sa, 70 + n, n, d)
    m = sa.AttnMatrices(m.q, m.k, m.v, causal=False)
    w, y = sa.dense_attention(m)
    ow, oy = _naive_attention(q, k, v, causal=False)
    close(y, oy)
    np.testing.assert_allclose(w, ow, atol=2e-3)
    np.testing.assert_allclose(np.asarray(w).sum(axis=1), 1.0, atol=1e-5)
    assert (np.asarray(w)[np.triu_indices(n, 1)] > 0).all()  # keys after the row do count


def test_sparse_rejects_non_causal(sa):
    """test_patterns.py:168-172: the sparse kernels stay causal-only."""
    m, _ = mats(sa, 18, 4, 2)
    m = sa.AttnMatrices(m.q, m.k, m.v, causal=False)
    with pytest.raises(sa.PatternParamError):
        sa.vertical_slash_attention(m, sa.SparseIndex(n=4))


@pytest.mark.parametrize("target", ["q_block_head", "q_other_head", "k", "v"])
@pytest.mark.parametrize("value", [float("nan"), float("inf")])
def test_device_nonfinite_every_writer(sa, target, value):
    """Device inputs: a Block-Cluster head's q rows are checked by its query
    pooling, every other q row and k / v by the scan beside the attention
    (prefill.cu); a NaN or Inf anywhere must raise (core.py:72-74)."""
    H, HK, n = 32, 8, 4096
    q, k, v = (torch.from_numpy(O.bf16_round(x)).bfloat16().cuda() for x in O.synth_qkv_gqa(0, n, H, HK, 128))
    cfg = sa.ModelConfig(n_heads=H, d_model=H * 128, d_head=128, max_context=n)
    fams = [type(hp.pattern).__name__ for hp in sa.prefill(q, k, v, cfg, mode="auto").plans[0]]
    assert "BlockSparse" in fams and any(f != "BlockSparse" for f in fams), fams
    if target == "q_block_head":
        x, idx = q, (0, fams.index("BlockSparse"), 1234, 5)
    elif target == "q_other_head":
        x, idx = q, (0, next(i for i, f in enumerate(fams) if f != "BlockSparse"), n - 1, 127)
    else:
        x, idx = (k if target == "k" else v), (0, 3, 17, 64)
    x[idx] = value
    with pytest.raises(sa.NonFiniteError):
        sa.prefill(q, k, v, cfg, mode="auto")
    x[idx] = 0.0
    sa.prefill(q, k, v, cfg, mode="auto")  # clean again: no stale flag
