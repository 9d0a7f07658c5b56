"""Multi-layer prefill (layers.py): L layers back to back equal
L independent runtime.prefill calls (same kernels, deterministic), fill one
device KvCache per layer, replay as one CUDA graph, and raise the
reference's NonFiniteError for a layer with NaN inputs."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import sparse_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def sa():
    import paper_2412_06198_b200 as m

    return m


def _layers(L, n, H, HK, seed=0):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    mk = lambda h: (torch.rand((1, h, n, 128), generator=g, device="cuda") * 2 - 1).bfloat16()  # noqa: E731
    return [mk(H) for _ in range(L)], [mk(HK) for _ in range(L)], [mk(HK) for _ in range(L)]


@pytest.mark.parametrize("mode", ["auto", "dense"])
def test_layers_equal_per_layer_prefill(sa, mode):
    L, n, H, HK = 3, 1500, 8, 2
    qs, ks, vs = _layers(L, n, H, HK)
    cfg = sa.ModelConfig(n_heads=H, d_model=H * 128, d_head=128, max_context=n + 100)
    res = sa.prefill_layers(qs, ks, vs, cfg, mode=mode)
    for l in range(L):
        one = sa.prefill(qs[l], ks[l], vs[l], cfg, mode=mode)
        assert torch.equal(res[l].outputs, one.outputs), l
        conv = lambda p: None if p is None else (type(p).__name__, *p.__dict__.values())  # noqa: E731
        assert [conv(h.pattern) for h in res[l].plans[0]] == [conv(h.pattern) for h in one.plans[0]]
        if mode == "auto":
            assert [h.search.error for h in res[l].plans[0]] == [h.search.error for h in one.plans[0]]
        assert res[l].cache.length == n
        assert torch.equal(res[l].cache.keys(), ks[l]) and torch.equal(res[l].cache.values(), vs[l])


def test_layer_stack_graph_replay(sa):
    from paper_2412_06198_b200.layers import LayerStack

    L, n, H, HK = 4, 777, 8, 2
    qs, ks, vs = _layers(L, n, H, HK, seed=3)
    cfg = sa.ModelConfig(n_heads=H, d_model=H * 128, d_head=128, max_context=n)
    stack = LayerStack(L, cfg, HK, n, mode="auto")
    stack.run(qs, ks, vs)
    eager = [o.clone() for o in stack.outputs]
    plans_e = stack.finish()
    for o in stack.outputs:
        o.zero_()
    g = stack.graph(qs, ks, vs)
    for o in stack.outputs:
        o.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(eager, stack.outputs))
    assert [[h.pattern for h in p[0]] for p in stack.finish()] == [[h.pattern for h in p[0]] for p in plans_e]


def test_layers_nonfinite_layer(sa):
    L, n, H, HK = 3, 600, 4, 2
    qs, ks, vs = _layers(L, n, H, HK, seed=5)
    vs[1][0, 1, 17, 3] = float("nan")
    cfg = sa.ModelConfig(n_heads=H, d_model=H * 128, d_head=128, max_context=n)
    with pytest.raises(sa.NonFiniteError, match="layer 1"):
        sa.prefill_layers(qs, ks, vs, cfg, mode="auto")


def test_layers_numpy_inputs_match_oracle(sa):
    """numpy float32 layers (the reference's types): outputs within the
    north-star tolerance of the oracle, fp32 caches holding the rows as given."""
    L, n, H = 2, 300, 4
    rng = np.random.default_rng(9)
    qs, ks, vs = ([O.bf16_round(rng.uniform(-1, 1, (1, H, n, 128)).astype(np.float32)) for _ in range(L)]
                  for _ in range(3))
    cfg = sa.ModelConfig(n_heads=H, d_model=H * 128, d_head=128, max_context=n)
    res = sa.prefill_layers(qs, ks, vs, cfg, mode="auto")
    for l in range(L):
        want, _ = O.prefill(qs[l], ks[l], vs[l], "auto")
        err = np.abs(res[l].outputs.astype(np.float64) - want)
        assert err.max() <= 2e-2 and err.mean() <= 2e-3
        assert res[l].cache.keys().dtype == np.float32
        np.testing.assert_array_equal(res[l].cache.keys(), ks[l])
