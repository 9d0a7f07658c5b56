"""Pin the CPU oracle to the reference: golden vectors produced by running the
reference (tests/golden/make_golden.py) plus the reference tests' known answers."""

import numpy as np
import pytest

from oracle import sparse_oracle as O
from tests.golden_io import load, uniform

ARR, META = load()


def pat_from(js):
    if js is None:
        return None
    fam, a, b = js
    return {"triangular": O.Tri, "vertical-slash": O.VS, "block-sparse": O.Blk}[fam](a, b)


def index_from(js):
    n = js["n"]
    if js["blocks"]:
        b = js["block_size"]
        nb = -(-n // b)
        rows = [[] for _ in range(nb)]
        for gq, gk in js["blocks"]:
            rows[gq].append(gk)
        return O.Index(n, np.zeros(0, np.int64), np.zeros(0, np.int64), b,
                       [np.array(sorted(r), np.int64) for r in rows])
    return O.Index(n, np.array(js["columns"], np.int64), np.array(js["diagonals"], np.int64))


@pytest.mark.parametrize("cid", range(len(META["cases"]["scores"])))
def test_scores_match_reference(cid):
    seed, n, d, mode, qe = META["cases"]["scores"][cid]
    q, k, _ = uniform(seed, n, d)
    cs, ds = O.vs_scores(q, k, mode, qe)
    np.testing.assert_allclose(cs, ARR[f"score_{cid}_col"], atol=1e-12)
    np.testing.assert_allclose(ds, ARR[f"score_{cid}_diag"], atol=1e-12)


@pytest.mark.parametrize("cid", range(len(META["cases"]["topk"])))
def test_topk_bit_exact(cid):
    k = META["cases"]["topk"][cid]
    got = O.top_k_stable(ARR[f"topk_{cid}_scores"], k)
    np.testing.assert_array_equal(got, ARR[f"topk_{cid}_idx"])


@pytest.mark.parametrize("cid", range(len(META["cases"]["indices"])))
def test_indices_and_kernels(cid):
    c = META["cases"]["indices"][cid]
    q, k, v = uniform(c["seed"], c["n"], c["d"])
    kind, a, b = c["pat"]
    if kind == "vs":
        idx = O.vs_index(q, k, a, b, c["mode"], c["q_est"])
    elif kind == "block":
        idx = O.block_index(q, k, a, b)
    else:
        idx = O.tri_index(c["n"], a, b)
    want = index_from(c["index"])
    if want.is_block:
        assert idx.block_size == want.block_size
        assert [r.tolist() for r in idx.block_rows] == [r.tolist() for r in want.block_rows]
    else:
        assert idx.columns.tolist() == want.columns.tolist()
        assert idx.diagonals.tolist() == want.diagonals.tolist()
    assert O.realized_size(idx) == c["realized"]
    w, y = O.sparse_attention(q, k, v, idx, need_weights=True)
    np.testing.assert_allclose(w, ARR[f"index_{cid}_w"], atol=1e-12)
    np.testing.assert_allclose(y, ARR[f"index_{cid}_y"], atol=1e-12)
    # independent brute-force mask path agrees too
    np.testing.assert_allclose(O.masked_attention(q, k, v, idx), y, atol=1e-9)
    assert int(sum(O.index_mask_rows(idx, 0, c["n"]).sum(axis=1))) == c["realized"]


@pytest.mark.parametrize("cid", range(len(META["cases"]["block_mean"])))
def test_block_mean(cid):
    seed, n, d, b = META["cases"]["block_mean"][cid]
    x = np.random.default_rng(seed).random((n, d))
    np.testing.assert_allclose(O.block_mean(x, b), ARR[f"bmean_{cid}"], atol=1e-14)


@pytest.mark.parametrize("cid", range(len(META["cases"]["space"])))
def test_search_space_and_refinement(cid):
    c = META["cases"]["space"][cid]
    cands, target, eps, iters = O.default_space(c["n"], c["d"], c["density"])
    assert [pat_from(x) for x in c["candidates"]] == cands
    assert target == c["target"]
    for cand, (p, fl, it, conv) in zip(cands, c["refined"]):
        got = O.refine(cand, c["n"], c["d"], target, eps, iters)
        assert got == (pat_from(p), fl, it, conv)


@pytest.mark.parametrize("cid", range(len(META["cases"]["select"])))
def test_selection(cid):
    c = META["cases"]["select"][cid]
    q, k, v = uniform(c["seed"], c["n"], c["d"])
    if c["d"] == 128:
        q, k, v = (O.bf16_round(x.astype(np.float32)) for x in (q, k, v))
    res = O.select(q, k, v, O.default_space(c["n"], c["d"]))
    assert res[0] == pat_from(c["chosen"])
    assert abs(res[2] - c["error"]) <= 1e-5 * max(1.0, abs(c["error"]))
    qw, kw, vw = uniform(c["seed"] + 50, 4 * c["n"], c["d"])
    pat, err, _ = O.select_windowed(qw, kw, vw, O.default_space(c["n"], c["d"]), c["n"])
    assert pat == pat_from(c["windowed_chosen"])
    assert abs(err - c["windowed_error"]) <= 1e-9 * max(1.0, abs(err))


@pytest.mark.parametrize("cid", range(len(META["cases"]["prefill"])))
def test_prefill(cid):
    c = META["cases"]["prefill"][cid]
    if c["H"] == c["HK"]:
        q, k, v = O.synth_qkv(c["seed"], c["ctx"], c["H"], 128)
    else:
        q, k, v = O.synth_qkv_gqa(c["seed"], c["ctx"], c["H"], c["HK"], 128)
    q, k, v = (O.bf16_round(x) for x in (q, k, v))
    fixed = O.fixed_pattern_for(c["fixed"], c["ctx"]) if c["fixed"] else None
    out, plans = O.prefill(q, k, v, c["mode"], fixed)
    assert [pat_from(p) for p in c["plans"]] == plans[0]
    step = max(1, c["ctx"] // 64)
    np.testing.assert_allclose(out[0, ::step], ARR[f"prefill_{cid}_rows"], atol=2e-5)
    np.testing.assert_allclose(out[0].astype(np.float64).sum(axis=1), ARR[f"prefill_{cid}_rowsum"],
                               atol=2e-3)


# ---- known answers from the reference's own tests ---------------------------

def test_zero_logit_scores():  # test_patterns.py:45-56
    z = np.zeros((2, 2))
    cs, ds = O.vs_scores(z, z)
    np.testing.assert_allclose(cs, [1.5, 0.5])
    np.testing.assert_allclose(ds, [1.5, 0.5])
    z1 = np.zeros((1, 2))
    np.testing.assert_allclose(O.vs_scores(z1, z1)[1], [1.0])


def test_zero_logits_pick_offset_zero_and_ties():  # test_patterns.py:102-107, 122-127
    z = np.zeros((6, 3))
    assert O.vs_index(z, z, 1, 1).diagonals.tolist() == [0]
    z = np.zeros((4, 2))
    idx = O.vs_index(z, z, 2, 2)
    assert idx.columns.tolist() == [0, 1] and idx.diagonals.tolist() == [0, 1]


def test_partial_block_example():  # n=13, b=4, k_b=2
    q, k, _ = uniform(29, 13, 4)
    idx = O.block_index(q, k, 4, 2)
    assert sum(len(r) for r in idx.block_rows) in (8, 9, 10, 11, 12)
    assert all(g in r.tolist() for g, r in enumerate(idx.block_rows))


def test_band_sink_row():  # test_patterns.py:280-283
    m = O.index_mask_rows(O.tri_index(6, 2, 1), 0, 6)
    assert set(np.flatnonzero(m[4])) == {0, 3, 4}


def test_realized_examples():  # test_patterns.py:295-298
    assert O.realized_size(O.Index(4, np.zeros(0, np.int64), np.zeros(0, np.int64))) == 4
    assert O.realized_size(O.Index(4, np.array([0]), np.array([0]))) == 7


def test_flops_examples():  # test_search.py:35-57
    assert O.estimate_flops(O.Tri(64, 0), 64, 4)[1] == 16384
    assert O.estimate_flops(O.VS(2, 2), 64, 4)[1:] == (1024, 1024)
    assert O.estimate_flops(O.VS(2, 2), 64, 4, q_est=16)[0] == 16 * 64 * 4
    assert O.estimate_flops(O.Blk(8, 2), 64, 4)[0] == 2 * 64 * 4 + 8 * 8 * 4


def test_refine_examples():  # test_search.py:122-146
    target = sum(O.estimate_flops(O.VS(16, 16), 64, 4)) // 2
    p, fl, it, conv = O.refine(O.VS(16, 16), 64, 4, target, 0.05, 8)
    assert p == O.VS(8, 8) and it == 1 and conv
    p, fl, it, conv = O.refine(O.VS(2, 2), 64, 4, 1, 0.05, 8)
    assert p == O.VS(1, 1) and it == 8 and not conv


def test_rescale_example():  # test_search.py:261-273
    assert O.rescale_to_full(O.VS(4, 4), 4.0, 256) == O.VS(16, 16)
    assert O.rescale_to_full(O.Blk(8, 1), 4.0, 256) == O.Blk(8, 1)


def test_half_even_round():
    assert O.py_round(0.5) == 0 and O.py_round(2.5) == 2 and O.py_round(6553.6) == 6554
    assert O.fixed_pattern_for("vertical-slash", 131072) == O.VS(6554, 6554)
    assert O.fixed_pattern_for("block-sparse", 131072) == O.Blk(64, 205)


def test_bf16_round():
    x = np.array([1.0, 1.00390625, 1.005859375, -3.3, 0.0], np.float32)
    import torch

    np.testing.assert_array_equal(O.bf16_round(x), torch.from_numpy(x).bfloat16().float().numpy())
