"""Kernel-level parity on a B200: every CUDA stage of the path against the CPU
oracle (oracle/sparse_oracle.py) on identical bf16-rounded inputs.

Tolerances: bit-exact for index/top-k work given identical fp32 scores;
max-abs <= 2e-2 and mean-abs <= 2e-3 for attention outputs (north star);
1e-5 relative for fp32 estimator scores against the float64 oracle."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import sparse_oracle as O  # noqa: E402

MAX_ABS, MEAN_ABS = 2e-2, 2e-3


@pytest.fixture(scope="module")
def sa():
    import paper_2412_06198_b200 as m

    from paper_2412_06198_b200 import _lib

    _lib.load()
    return m


def rand_heads(seed, g, n, d=128):
    rng = np.random.default_rng(seed)
    return O.bf16_round(rng.uniform(-1, 1, (g, n, d)).astype(np.float32))


def to_dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda().bfloat16().contiguous()


def run_index(sa, q, k, v, builder, H, HK):
    from paper_2412_06198_b200 import _lib, device_index as DI

    n = q.shape[1]
    idx = builder.upload("cuda")
    off, cnt, tiles = DI.build_tiles(idx)
    out = torch.empty(n, H * 128, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(H, n, dtype=torch.float32, device="cuda")
    qd, kd, vd = to_dev(q), to_dev(k), to_dev(v)  # keep alive across the async launch
    _lib.call("sa_attn_sparse", 1, H, HK, n, 1 / np.sqrt(128), qd.data_ptr(), kd.data_ptr(),
              vd.data_ptr(), out.data_ptr(), idx.view(), off.data_ptr(), cnt.data_ptr(),
              tiles.data_ptr(), lse.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return out.float().cpu().numpy().reshape(n, H, 128).transpose(1, 0, 2), cnt


@pytest.mark.parametrize("n", [1, 127, 128, 300, 1000, 2049])
def test_attention_all_families_vs_oracle(sa, n):
    from paper_2412_06198_b200 import device_index as DI

    H, HK = 8, 2
    q, k, v = rand_heads(1, H, n), rand_heads(2, HK, n), rand_heads(3, HK, n)
    rng = np.random.default_rng(n)
    b = DI.HostIndexBuilder(n, H)
    idxs = []
    for h in range(H):
        kind = h % 4
        if kind == 0:
            b.set_dense(h)
            ix = O.tri_index(n, n, 0)
        elif kind == 1:
            w, s = int(rng.integers(1, n + 1)), int(rng.integers(0, n // 3 + 1)) * (h % 2)
            b.set_triangular(h, w, s)
            ix = O.tri_index(n, w, s)
        elif kind == 2:
            cols = np.sort(rng.choice(n, max(1, n // 9), replace=False))
            offs = np.sort(rng.choice(n, max(1, n // 11), replace=False))
            b.set_vertical_slash(h, cols, offs)
            ix = O.Index(n, cols, offs)
        else:
            bs = [1, 7, 8, 64, 200][h % 5]
            bs = min(bs, n)
            qq, kk = q[h].astype(np.float64), k[h // 4].astype(np.float64)
            ix = O.block_index(qq, kk, bs, max(1, (-(-n // bs)) // 4))
            b.set_block(h, bs, [r.astype(np.int32) for r in ix.block_rows])
        idxs.append(ix)
    got, _ = run_index(sa, q, k, v, b, H, HK)
    for h in range(H):
        want = O.masked_attention(q[h].astype(np.float64), k[h // 4].astype(np.float64),
                                  v[h // 4].astype(np.float64), idxs[h])
        err = np.abs(got[h] - want)
        assert err.max() <= MAX_ABS and err.mean() <= MEAN_ABS, (h, err.max(), err.mean())


def test_executed_tiles_equal_touched_tiles(sa):
    """The tile list holds exactly the (q-tile, k-tile) pairs the index touches."""
    from paper_2412_06198_b200 import device_index as DI

    n, H = 1000, 4
    q = k = v = rand_heads(4, H, n)
    rng = np.random.default_rng(5)
    b = DI.HostIndexBuilder(n, H)
    masks = []
    b.set_triangular(0, 200, 3)
    masks.append(O.index_mask_rows(O.tri_index(n, 200, 3), 0, n))
    cols, offs = np.sort(rng.choice(n, 5, replace=False)), np.sort(rng.choice(n, 4, replace=False))
    b.set_vertical_slash(1, cols, offs)
    masks.append(O.index_mask_rows(O.Index(n, cols, offs), 0, n))
    ix = O.block_index(q[2].astype(np.float64), k[2].astype(np.float64), 16, 3)
    b.set_block(2, 16, [r.astype(np.int32) for r in ix.block_rows])
    masks.append(O.index_mask_rows(ix, 0, n))
    b.set_dense(3)
    masks.append(np.tri(n, dtype=bool))
    _, cnt = run_index(sa, q, k, v, b, H, H)
    cnt = cnt.cpu().numpy().reshape(H, -1)
    nqt = -(-n // 128)
    for h in range(H):
        pad = np.zeros((nqt * 128, nqt * 128), bool)
        pad[:n, :n] = masks[h]
        touched = pad.reshape(nqt, 128, nqt, 128).any(axis=(1, 3)).sum(axis=1)
        if h == 2:  # Block-Cluster b=16: gather mode wherever it executes fewer tiles
            touched = np.minimum(touched, gather_tiles(ix.block_rows, 16, n))
        np.testing.assert_array_equal(cnt[h], touched)


def gather_tiles(rows, b, n):
    """Tiles per query tile in Block-Cluster gather mode: max off-diagonal blocks
    over the tile's 128/b query blocks, plus the diagonal tile (sa_types.h TK_GATHER)."""
    nqt = -(-n // 128)
    per = 128 // b
    out = np.zeros(nqt, np.int64)
    for qt in range(nqt):
        g = [int(np.sum(np.asarray(rows[gq]) < gq)) for gq in range(qt * per, min((qt + 1) * per, len(rows)))]
        out[qt] = max(g) + 1
    return out


@pytest.mark.parametrize("n,b,k_b", [(1000, 8, 1), (4096, 8, 1), (4100, 8, 2), (2049, 16, 3), (3000, 32, 2),
                                     (4096, 64, 4), (777, 8, 5), (300, 16, 1), (4100, 64, 3), (2000, 64, 1),
                                     (8192, 64, 20)])
def test_block_gather_vs_oracle(sa, n, b, k_b):
    """Block-Cluster heads through the gathered-tile path: outputs against the
    oracle's block kernel, and the tile counts the gather cost model implies."""
    from paper_2412_06198_b200 import device_index as DI

    H, HK = 4, 2
    q, k, v = rand_heads(20 + n, H, n), rand_heads(21 + n, HK, n), rand_heads(22 + n, HK, n)
    bld = DI.HostIndexBuilder(n, H)
    idxs = []
    for h in range(H):
        ix = O.block_index(q[h].astype(np.float64), k[h // 2].astype(np.float64), b, k_b)
        bld.set_block(h, b, [r.astype(np.int32) for r in ix.block_rows])
        idxs.append(ix)
    got, cnt = run_index(sa, q, k, v, bld, H, HK)
    cnt = cnt.cpu().numpy().reshape(H, -1)
    nqt = -(-n // 128)
    for h in range(H):
        want = O.masked_attention(q[h].astype(np.float64), k[h // 2].astype(np.float64),
                                  v[h // 2].astype(np.float64), idxs[h])
        err = np.abs(got[h] - want)
        assert err.max() <= MAX_ABS and err.mean() <= MEAN_ABS, (h, err.max(), err.mean())
        m = O.index_mask_rows(idxs[h], 0, n)
        pad = np.zeros((nqt * 128, nqt * 128), bool)
        pad[:n, :n] = m
        touched = pad.reshape(nqt, 128, nqt, 128).any(axis=(1, 3)).sum(axis=1)
        np.testing.assert_array_equal(cnt[h], np.minimum(touched, gather_tiles(idxs[h].block_rows, b, n)))


def device_topk(scores32: np.ndarray, k: int) -> np.ndarray:
    from paper_2412_06198_b200 import _lib

    rows, n = scores32.shape
    s = torch.from_numpy(np.ascontiguousarray(scores32)).cuda()
    out = torch.empty(rows, k, dtype=torch.int32, device="cuda")
    _lib.call("sa_topk_stable_f32", s.data_ptr(), rows, n, n, k, out.data_ptr(), k,
              torch.cuda.current_stream().cuda_stream)
    return out.cpu().numpy()


@pytest.mark.parametrize("n,k", [(1, 1), (7, 3), (300, 300), (4096, 205), (49153, 2000), (131072, 6144),
                                 (131072, 1), (131075, 131074), (262144, 9000)])
def test_topk_bit_exact(sa, n, k):
    rng = np.random.default_rng(n + k)
    rows = np.stack([
        rng.random(n).astype(np.float32),
        (rng.integers(0, 4, n) * 0.5).astype(np.float32),  # massive ties
        np.where(rng.random(n) < 0.3, np.float32(-0.0), rng.standard_normal(n).astype(np.float32)),
        np.zeros(n, np.float32),
    ])
    got = device_topk(rows, k)
    for r in range(rows.shape[0]):
        np.testing.assert_array_equal(got[r], O.top_k_stable(rows[r], k))


@pytest.mark.parametrize("n,k,nrows", [(32768, 1536, 48), (131072, 6144, 48), (20000, 777, 40)])
def test_topk_many_rows_bit_exact(sa, n, k, nrows):
    """More rows than one wave of clusters: rows that fit one CTA's shared
    memory go one CTA per row, longer ones to clusters in two waves
    (csrc/topk.cu launch_topk); both must stay bit-exact."""
    rng = np.random.default_rng(n + nrows)
    rows = []
    for r in range(nrows):
        kind = r % 4
        if kind == 0:
            rows.append(rng.random(n).astype(np.float32))
        elif kind == 1:
            rows.append((rng.integers(0, 6, n) * 0.25).astype(np.float32))
        elif kind == 2:
            rows.append((rng.random(n) ** 8 * 1e-3).astype(np.float32))
        else:
            rows.append(np.where(rng.random(n) < 0.5, np.float32(0.0), rng.standard_normal(n).astype(np.float32)))
    rows = np.stack(rows)
    got = device_topk(rows, k)
    for r in range(nrows):
        np.testing.assert_array_equal(got[r], O.top_k_stable(rows[r], k), err_msg=f"row {r}")


def test_topk_golden_vectors(sa):
    from tests.golden_io import load

    arr, meta = load()
    for cid, k in enumerate(meta["cases"]["topk"]):
        s = arr[f"topk_{cid}_scores"].astype(np.float32)
        # the golden scores are exact in fp32 (multiples of 0.25 plus tiny noise rounded once)
        got = device_topk(s[None], k)[0]
        np.testing.assert_array_equal(got, O.top_k_stable(s, k))


def device_scores(q, k, rows):
    from paper_2412_06198_b200 import _lib

    n = q.shape[0]
    qd, kd = to_dev(q[None]), to_dev(k[None])
    col = torch.empty(n, dtype=torch.float32, device="cuda")
    diag = torch.empty(n, dtype=torch.float32, device="cuda")
    lib = _lib.load()
    wsb = int(lib.sa_score_tail_workspace(1, 1, n, n))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    r_hi, g = n, 0
    while r_hi > n - rows:
        r_lo = max(n - rows, r_hi - 128)
        _lib.call("sa_score_tail", 1, 1, 1, n, 1 / np.sqrt(128), qd.data_ptr(), kd.data_ptr(), r_lo, r_hi,
                  col.data_ptr(), diag.data_ptr(), int(g > 0), None, 0, ws.data_ptr(), wsb,
                  torch.cuda.current_stream().cuda_stream)
        r_hi, g = r_lo, g + 1
    torch.cuda.synchronize()
    return col.cpu().numpy(), diag.cpu().numpy()


@pytest.mark.parametrize("n,rows", [(1, 1), (64, 64), (100, 64), (300, 300), (1000, 64), (5000, 64), (777, 200)])
def test_vs_estimator_scores(sa, n, rows):
    q, k = rand_heads(7, 1, n)[0], rand_heads(8, 1, n)[0]
    cs, ds = device_scores(q, k, rows)
    w, first = O.tail_weights(q.astype(np.float64), k.astype(np.float64), rows)
    ocs, ods = O.column_mass(w), O.diagonal_mass(w, first, n)
    tol = 2e-5 * max(1.0, rows / 64)
    np.testing.assert_allclose(cs, ocs, rtol=tol, atol=1e-7)
    np.testing.assert_allclose(ds, ods, rtol=tol, atol=1e-7)


@pytest.mark.parametrize("B,H,HK,n,rows,sel", [
    (1, 16, 4, 3000, 64, [0, 1, 2, 3, 5, 8, 9, 10, 15]),   # units of 4, 1, 3, 1 heads
    (2, 16, 2, 1500, 64, list(range(16))),                 # 8 heads per kv group: 2 units each
    (1, 4, 4, 700, 64, [1, 3]),                            # one head per kv group
    (1, 8, 2, 2049, 100, [0, 2, 4, 5, 6, 7]),              # 100 rows: 64 + 36 accumulated
    (1, 8, 2, 129, 128, [3, 4]),                           # n < 2 tiles
    (1, 8, 2, 40, 40, [0, 1, 2, 3, 4, 5, 6, 7]),           # n < 64: rows below the box
])
def test_vs_estimator_gqa_units(sa, B, H, HK, n, rows, sel):
    """The estimator over device-gated GQA units (up to 4 heads of one kv head
    share each K tile) equals the float64 tail weights of every selected head
    (patterns.py:165-202); unselected heads are not written."""
    from paper_2412_06198_b200 import _lib

    q, k = rand_heads(31, B * H, n), rand_heads(32, B * HK, n)
    qd, kd = to_dev(q), to_dev(k)
    gate = torch.full((B * H,), 9, dtype=torch.int32, device="cuda")
    for b in range(B):
        gate[torch.tensor(sel) + b * H] = 1
    col = torch.full((B * H, n), -7.0, dtype=torch.float32, device="cuda")
    diag = torch.full((B * H, n), -7.0, dtype=torch.float32, device="cuda")
    wsb = int(_lib.load().sa_score_tail_workspace(B, H, n, n))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    r_hi, g = n, 0
    while r_hi > n - rows:
        r_lo = max(n - rows, r_hi - 128)
        _lib.call("sa_score_tail", B, H, HK, n, 1 / np.sqrt(128), qd.data_ptr(), kd.data_ptr(), r_lo, r_hi,
                  col.data_ptr(), diag.data_ptr(), int(g > 0), gate.data_ptr(), 1, ws.data_ptr(), wsb, st)
        r_hi, g = r_lo, g + 1
    cs, ds = col.cpu().numpy(), diag.cpu().numpy()
    tol = 2e-5 * max(1.0, rows / 64)
    for hh in range(B * H):
        if hh % H not in sel:
            assert (cs[hh] == -7.0).all() and (ds[hh] == -7.0).all(), hh
            continue
        kvh = (hh // H) * HK + (hh % H) // (H // HK)
        w, first = O.tail_weights(q[hh].astype(np.float64), k[kvh].astype(np.float64), rows)
        np.testing.assert_allclose(cs[hh], O.column_mass(w), rtol=tol, atol=1e-7, err_msg=f"col {hh}")
        np.testing.assert_allclose(ds[hh], O.diagonal_mass(w, first, n), rtol=tol, atol=1e-7, err_msg=f"diag {hh}")


def test_vs_estimator_deterministic(sa):
    """Two runs give bit-identical scores (fixed merge order; <= 2 atomic terms per diagonal)."""
    q, k = rand_heads(33, 8, 20000), rand_heads(34, 2, 20000)
    from paper_2412_06198_b200 import _lib

    qd, kd = to_dev(q), to_dev(k)
    wsb = int(_lib.load().sa_score_tail_workspace(1, 8, 20000, 20000))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(2):
        col = torch.empty((8, 20000), dtype=torch.float32, device="cuda")
        diag = torch.empty((8, 20000), dtype=torch.float32, device="cuda")
        _lib.call("sa_score_tail", 1, 8, 2, 20000, 1 / np.sqrt(128), qd.data_ptr(), kd.data_ptr(), 20000 - 64,
                  20000, col.data_ptr(), diag.data_ptr(), 0, None, 0, ws.data_ptr(), wsb,
                  torch.cuda.current_stream().cuda_stream)
        outs.append((col.cpu(), diag.cpu()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_vs_index_same_scores_bit_exact(sa):
    """North-star contract: fed the same fp32 scores, the index sets match exactly."""
    n = 8192
    q, k = rand_heads(9, 1, n)[0], rand_heads(10, 1, n)[0]
    cs, ds = O.vs_scores(q.astype(np.float64), k.astype(np.float64), "estimated", 64)
    cs32, ds32 = cs.astype(np.float32), ds.astype(np.float32)
    kv = ks = round(0.05 * n)
    np.testing.assert_array_equal(device_topk(cs32[None], kv)[0], O.top_k_stable(cs32, kv))
    np.testing.assert_array_equal(device_topk(ds32[None], ks)[0], O.top_k_stable(ds32, ks))
    # end to end (device scores): near-total agreement with the float64 oracle
    dcs, dds = device_scores(q, k, 64)
    agree_c = len(set(device_topk(dcs[None], kv)[0]) & set(O.top_k_stable(cs, kv))) / kv
    agree_d = len(set(device_topk(dds[None], ks)[0]) & set(O.top_k_stable(ds, ks))) / ks
    assert agree_c >= 0.995 and agree_d >= 0.995, (agree_c, agree_d)


def device_block_rows(q, k, b, k_b):
    from paper_2412_06198_b200 import _lib

    n = q.shape[0]
    nb = -(-n // b)
    st = torch.cuda.current_stream().cuda_stream
    qd, kd = to_dev(q[None]), to_dev(k[None])
    qp = torch.empty((1, nb, 384), dtype=torch.bfloat16, device="cuda")
    kp = torch.empty((1, nb, 256), dtype=torch.bfloat16, device="cuda")
    _lib.call("sa_block_pool", 1, n, b, 0, qd.data_ptr(), qp.data_ptr(), None, st)
    _lib.call("sa_block_pool", 1, n, b, 1, kd.data_ptr(), kp.data_ptr(), None, st)
    idx = torch.empty((nb, k_b + 1), dtype=torch.int32, device="cuda")
    ro = torch.empty(nb + 1, dtype=torch.int32, device="cuda")
    wsb = max(256, int(_lib.load().sa_block_select_workspace(n, b, k_b)))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.call("sa_block_select", 1, 1, 1, n, b, k_b, 1 / np.sqrt(128), qp.data_ptr(), kp.data_ptr(),
              idx.data_ptr(), ro.data_ptr(), ws.data_ptr(), wsb, st)
    rows = idx.cpu().numpy()
    return [[int(x) for x in r if x != 2**31 - 1] for r in rows]


@pytest.mark.parametrize("n,b,k_b", [(13, 4, 2), (1000, 8, 1), (4096, 8, 1), (4096, 64, 6), (3000, 7, 3),
                                     (4096, 64, 13), (2000, 128, 2), (600, 200, 1),
                                     (2564, 16, 60), (1001, 8, 9)])  # materialized rows, nb % 4 != 0
def test_block_estimator(sa, n, b, k_b):
    q, k = rand_heads(11, 1, n)[0], rand_heads(12, 1, n)[0]
    got = device_block_rows(q, k, b, k_b)
    want = O.block_index(q.astype(np.float64), k.astype(np.float64), b, k_b).block_rows
    # pooled logits in split-bf16 precision (~16 mantissa bits of each pooled
    # mean: |logit error| <= ~2^-16 * sum|q||k| * scale ~ 1e-6 here): rows whose
    # top-k margin is below that bound may differ; everything else is exact
    qb, kb = O.block_mean(q.astype(np.float64), b), O.block_mean(k.astype(np.float64), b)
    logit = qb @ kb.T / np.sqrt(128)
    mism = 0
    for g, (r_got, r_want) in enumerate(zip(got, want)):
        if r_got == r_want.tolist():
            continue
        row = np.sort(logit[g, : g + 1])[::-1]
        keff = min(k_b, g + 1)
        margin = row[keff - 1] - row[keff] if keff < g + 1 else np.inf
        assert margin < 1e-5, (g, r_got, r_want.tolist(), margin)
        mism += 1
    assert mism <= max(1, len(got) // 200)


def test_selector_vs_oracle(sa):
    from paper_2412_06198_b200 import search as S

    n, H = 64, 32
    q, k = rand_heads(13, H, n), rand_heads(14, H, n)
    space = S.default_search_space(n, 128)
    refined = S.refined_candidates(space, n, 128, 0)
    choice, errs = S._device_select(to_dev(q), to_dev(k), H, H, n, 1 / np.sqrt(128), refined)
    choice, errs = choice.cpu().numpy(), errs.cpu().numpy()
    ospace = O.default_space(n, 128)
    for h in range(H):
        qh, kh = q[h].astype(np.float64), k[h].astype(np.float64)
        res = O.select(qh, kh, kh, ospace)
        assert refined[choice[h]].pattern.__class__.__name__[0] == {O.Tri: "T", O.VS: "V", O.Blk: "B"}[type(res[0])]
        np.testing.assert_allclose(errs[h, : len(res[5])], res[5], rtol=1e-4)


@pytest.mark.parametrize("items,max_cnt", [(1, 0), (1000, 7), (8192, 256), (20000, 2048)])
def test_order_work_is_heaviest_first_permutation(sa, items, max_cnt):
    """sa_order_work: a permutation of the items, tile counts non-increasing
    (exact below 1023 distinct counts, else within one count bucket), empty
    items last."""
    from paper_2412_06198_b200 import _lib

    rng = np.random.default_rng(items)
    cnt = torch.from_numpy(rng.integers(0, max_cnt + 1, items).astype(np.int32)).cuda()
    work = torch.empty(items, dtype=torch.int32, device="cuda")
    _lib.call("sa_order_work", cnt.data_ptr(), items, max_cnt, work.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    w = work.cpu().numpy()
    np.testing.assert_array_equal(np.sort(w), np.arange(items))
    c = cnt.cpu().numpy()[w]
    shift = 0
    while (max_cnt >> shift) >= 1023:
        shift += 1
    key = np.where(c > 0, np.minimum(c >> shift, 1022) + 1, 0)
    assert np.all(np.diff(key) <= 0)


@pytest.mark.parametrize("case", ["zeros", "repeated_keys", "two_level"])
def test_block_top1_ties_and_overflow(sa, case):
    """k_b = 1 filter/refine path on degenerate inputs: exact ties everywhere
    (every row overflows the candidate list and takes the exact scan) must
    still pick the lowest block id, like the reference's stable top-k."""
    n, b = 2048, 8
    rng = np.random.default_rng(31)
    q = rand_heads(40, 1, n)[0]
    k = rand_heads(41, 1, n)[0]
    if case == "zeros":
        q = np.zeros_like(q)
    elif case == "repeated_keys":
        k = np.tile(k[:b], (n // b, 1))
    else:  # many near-ties: two distinct key blocks repeated
        k = np.tile(np.concatenate([k[:b], k[b:2 * b]]), (n // (2 * b), 1))
    got = device_block_rows(q, k, b, 1)
    want = O.block_index(q.astype(np.float64), k.astype(np.float64), b, 1).block_rows
    for g, (r_got, r_want) in enumerate(zip(got, want)):
        assert r_got == r_want.tolist(), (g, r_got, r_want.tolist())


@pytest.mark.parametrize("gain", [6.0, 25.0])
def test_attention_large_logits(sa, gain):
    """Logits far from O(1) (q, k scaled up: row maxima jump by hundreds in
    log2 units within a row): the lazy rescale (stale max until it grows by
    > 2^8) must keep every family within tolerance of the fp64 oracle."""
    from paper_2412_06198_b200 import device_index as DI

    H, HK, n = 4, 1, 700
    q = O.bf16_round(rand_heads(71, H, n) * gain)
    k = O.bf16_round(rand_heads(72, HK, n) * gain)
    v = rand_heads(73, HK, n)
    b = DI.HostIndexBuilder(n, H)
    rng = np.random.default_rng(9)
    cols = np.sort(rng.choice(n, 60, replace=False))
    offs = np.sort(rng.choice(n, 50, replace=False))
    idxs = [O.tri_index(n, n, 0), O.tri_index(n, 97, 5), O.Index(n, cols, offs),
            O.block_index(q[3].astype(np.float64), k[0].astype(np.float64), 8, 3)]
    b.set_dense(0)
    b.set_triangular(1, 97, 5)
    b.set_vertical_slash(2, cols, offs)
    b.set_block(3, 8, [r.astype(np.int32) for r in idxs[3].block_rows])
    got, _ = run_index(sa, q, k, v, b, H, HK)
    for h in range(H):
        want = O.masked_attention(q[h].astype(np.float64), k[0].astype(np.float64), v[0].astype(np.float64), idxs[h])
        err = np.abs(got[h] - want)
        assert np.isfinite(got[h]).all()
        assert err.max() <= MAX_ABS and err.mean() <= MEAN_ABS, (h, err.max(), err.mean())


def test_select_family_on_given_errors(sa):
    """sa_select_family: strict-< argmin, earlier candidate wins ties, NaN never
    wins (search.py:245-250), on identical fp64 errors."""
    from paper_2412_06198_b200 import _lib

    rng = np.random.default_rng(5)
    err = rng.integers(0, 4, (500, 3)).astype(np.float64) * 0.25  # many exact ties
    err[7] = np.nan
    err[8, 0] = np.nan
    err[9, 1:] = np.inf
    want = np.zeros(500, np.int32)
    for r in range(500):
        best, bc = np.inf, 0
        for c in range(3):
            if err[r, c] < best:
                best, bc = err[r, c], c
        want[r] = bc
    d = torch.from_numpy(err).cuda()
    out = torch.empty(500, dtype=torch.int32, device="cuda")
    _lib.call("sa_select_family", d.data_ptr(), 3, 500, 3, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    np.testing.assert_array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("nb,k_b,ties", [(1, 1, False), (37, 3, True), (300, 1, False), (300, 8, True), (2000, 51, True)])
def test_block_topk_on_given_weights(sa, nb, k_b, ties):
    """sa_block_topk_f32: the Block-Cluster row selection of build_block_index
    (patterns.py:309-321) on identical fp32 weights, bit-exact."""
    from paper_2412_06198_b200 import _lib

    rng = np.random.default_rng(nb + k_b)
    w = (rng.integers(0, 5, (nb, nb)) * 0.5 if ties else rng.standard_normal((nb, nb))).astype(np.float32)
    want = np.full((nb, k_b + 1), np.iinfo(np.int32).max, np.int64)
    for gq in range(nb):
        top = np.argsort(-w[gq, : gq + 1], kind="stable")[: min(k_b, gq + 1)]
        sel = sorted(set(top.tolist()) | {gq})
        want[gq, : len(sel)] = sel
    d = torch.from_numpy(w).cuda()
    out = torch.empty((nb, k_b + 1), dtype=torch.int32, device="cuda")
    lib = _lib.load()
    ws = torch.empty(int(lib.sa_block_topk_workspace(nb, k_b)), dtype=torch.uint8, device="cuda")
    _lib.call("sa_block_topk_f32", d.data_ptr(), nb, nb, k_b, out.data_ptr(), ws.data_ptr(), ws.numel(),
              torch.cuda.current_stream().cuda_stream)
    np.testing.assert_array_equal(out.cpu().numpy().astype(np.int64), want)
