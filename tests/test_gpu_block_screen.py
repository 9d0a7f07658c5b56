"""The Block-Cluster index for k_b <= 8 (csrc/block_screen.cu: fp16 screen +
exact refine, the path sa_prefill takes) against the float64 oracle
(patterns.py:279-321 via oracle.block_index).

The refine re-scores every near-cut candidate with fp64 products of the fp32
pooled means, so a row may differ from the float64 oracle only where its
top-k margin is at fp32 pooling resolution (asserted < 2e-6 here, 5x tighter
than the split-bf16 bound of test_gpu_kernels.test_block_estimator); exact
ties (zeros, repeated key blocks) must pick the lowest ids."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import sparse_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    from paper_2412_06198_b200 import _lib

    return _lib.load()


def rand_heads(seed, g, n, d=128, scale=1.0):
    rng = np.random.default_rng(seed)
    return O.bf16_round((rng.uniform(-1, 1, (g, n, d)) * scale).astype(np.float32))


def screen_rows(q, k, b, k_b, heads=1, kv_heads=1):
    """(heads, n, 128) q, (kv_heads, n, 128) k -> per head the list of block rows."""
    from paper_2412_06198_b200 import _lib

    lib = _lib.load()
    n = q.shape[1]
    nb = -(-n // b)
    st = torch.cuda.current_stream().cuda_stream
    qd = torch.from_numpy(np.ascontiguousarray(q)).cuda().bfloat16().contiguous()
    kd = torch.from_numpy(np.ascontiguousarray(k)).cuda().bfloat16().contiguous()
    idx = torch.full((heads, nb, k_b + 1), -7, dtype=torch.int32, device="cuda")
    ro = torch.empty((heads, nb + 1), dtype=torch.int32, device="cuda")
    wsb = int(lib.sa_block_index_workspace(1, heads, kv_heads, n, b, k_b))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.call("sa_block_index_bf16", 1, heads, kv_heads, n, b, k_b, qd.data_ptr(), kd.data_ptr(), idx.data_ptr(),
              ro.data_ptr(), ws.data_ptr(), wsb, st)
    rows = idx.cpu().numpy()
    offs = ro.cpu().numpy()
    for h in range(heads):
        np.testing.assert_array_equal(offs[h], h * nb * (k_b + 1) + np.arange(nb + 1) * (k_b + 1))
    return [[[int(x) for x in r if x != 2**31 - 1] for r in rows[h]] for h in range(heads)]


def check_rows(got, q, k, b, k_b, tol=2e-6):
    want = O.block_index(q.astype(np.float64), k.astype(np.float64), b, k_b).block_rows
    qb, kb = O.block_mean(q.astype(np.float64), b), O.block_mean(k.astype(np.float64), b)
    logit = qb @ kb.T / np.sqrt(128)
    mism = 0
    for g, (r_got, r_want) in enumerate(zip(got, want)):
        if r_got == r_want.tolist():
            continue
        row = np.sort(logit[g, : g + 1])[::-1]
        keff = min(k_b, g + 1)
        margin = row[keff - 1] - row[keff] if keff < g + 1 else np.inf
        assert margin < tol, (g, r_got, r_want.tolist(), margin)
        mism += 1
    assert mism <= max(1, len(got) // 1000), mism


@pytest.mark.parametrize("n,b,k_b", [(13, 4, 2), (1000, 8, 1), (4096, 8, 1), (4096, 64, 6), (3000, 7, 3),
                                     (2000, 128, 2), (600, 200, 1), (1001, 8, 8), (20000, 8, 1),
                                     (16390, 16, 4), (32768, 8, 1), (8200, 16, 1), (129, 1, 1)])
def test_block_screen_vs_oracle(lib, n, b, k_b):
    q, k = rand_heads(11, 1, n), rand_heads(12, 1, n)
    got = screen_rows(q, k, b, k_b)[0]
    check_rows(got, q[0], k[0], b, k_b)


def test_block_screen_gqa_heads(lib):
    """4 query heads over 2 kv heads: head h reads kv head h // 2."""
    n, b, k_b = 3000, 8, 2
    q, k = rand_heads(21, 4, n), rand_heads(22, 2, n)
    got = screen_rows(q, k, b, k_b, heads=4, kv_heads=2)
    for h in range(4):
        check_rows(got[h], q[h], k[h // 2], b, k_b)


@pytest.mark.parametrize("case", ["zeros", "repeated_keys", "two_level", "pairs", "zero_keys", "wide_range", "tiny"])
@pytest.mark.parametrize("k_b", [1, 3])
def test_block_screen_ties_and_ranges(lib, case, k_b):
    """Exact ties everywhere (every row re-scored in full), repeated blocks,
    and magnitudes fp16 cannot hold directly (per-block power-of-two scaling)."""
    n, b = 2048, 8
    q, k = rand_heads(40, 1, n)[0], rand_heads(41, 1, n)[0]
    if case == "zeros":
        q = np.zeros_like(q)
    elif case == "repeated_keys":
        k = np.tile(k[:b], (n // b, 1))
    elif case == "two_level":
        k = np.tile(np.concatenate([k[:b], k[b:2 * b]]), (n // (2 * b), 1))
    elif case == "pairs":  # every key block twice in a row: each row's best block ties with its twin
        k = np.repeat(k.reshape(n // b, b, -1)[::2], 2, axis=0).reshape(n, -1)
    elif case == "zero_keys":
        k = np.zeros_like(k)
    elif case == "wide_range":  # 30x queries, key blocks spanning 1e-6 .. 1e1 (logits stay where the
        # reference's softmax keeps every weight nonzero: it selects on weights, ties at 0 to low ids)
        q = O.bf16_round(q * 30)
        mag = 10.0 ** np.repeat(np.random.default_rng(3).uniform(-6, 1, n // b), b)
        k = O.bf16_round(k * mag[:, None].astype(np.float32))
    else:  # pooled values below fp16's normal range (logits still resolvable after the softmax)
        q, k = O.bf16_round(q * 1e-4), O.bf16_round(k * 3e-5)
    got = screen_rows(q[None], k[None], b, k_b)[0]
    if case in ("zeros", "repeated_keys", "two_level", "pairs", "zero_keys"):
        want = O.block_index(q.astype(np.float64), k.astype(np.float64), b, k_b).block_rows
        for g, (r_got, r_want) in enumerate(zip(got, want)):
            assert r_got == r_want.tolist(), (g, r_got, r_want.tolist())
    else:
        scale = float(np.abs(O.block_mean(q.astype(np.float64), b)).max() *
                      np.abs(O.block_mean(k.astype(np.float64), b)).max())
        check_rows(got, q, k, b, k_b, tol=1e-5 * scale)


def test_block_screen_matches_split_path_in_prefill(lib):
    """sa_prefill with a fixed Block(8, 1) layer: the two-pass fp16 top-1
    (SA_BLOCK_SCREEN=1) and the default split-bf16 GEMM (unset / =0;
    separate processes) give the same block rows except at split-bf16
    near-ties."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, json, numpy as np, torch; sys.path.insert(0, '.');"
        "from paper_2412_06198_b200 import runtime as R, patterns as P;"
        "rng = np.random.default_rng(5); n = 4096;"
        "q = torch.from_numpy(rng.uniform(-1, 1, (4, n, 128)).astype(np.float32)).cuda().bfloat16();"
        "k = torch.from_numpy(rng.uniform(-1, 1, (2, n, 128)).astype(np.float32)).cuda().bfloat16();"
        "plan = R.PrefillPlan(1, 4, 2, n, 128, 'fixed', fixed_pattern=P.BlockSparse(8, 1));"
        "ws = R._workspace(plan.ws_bytes, torch.device('cuda'));"
        "out = torch.empty((1, n, 512), dtype=torch.bfloat16, device='cuda');"
        "plan.run(q, k, k, out, ws); torch.cuda.synchronize();"
        "v = plan.views(ws); off = v.index.blk_idx - ws.data_ptr(); st = v.blk_head_stride;"
        "rows = ws[off: off + 4 * 4 * st].view(torch.int32).reshape(4, st)[:, : 512 * 2].cpu().numpy();"
        "print(json.dumps(rows.tolist()))"
    )
    outs = []
    for env in (None, "1", "0"):
        e = dict(os.environ)
        e.pop("SA_BLOCK_SCREEN", None)
        if env is not None:
            e["SA_BLOCK_SCREEN"] = env
        r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300, env=e)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    dflt, scr, split = (np.array(o).reshape(4, 512, 2) for o in outs)
    np.testing.assert_array_equal(dflt, split)  # the split GEMM is the default
    diff = int((scr != split).any(axis=2).sum())
    assert diff <= 4, diff
