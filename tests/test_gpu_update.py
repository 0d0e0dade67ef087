"""GPU parity of the model update (arc_topk_apply_update; SURVEY §8(f) row 4,
DESIGN.md R23/R24): bit-exact against the oracle's orc_apply_sgd /
orc_apply_adam on the same seeded inputs, through the C ABI."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def api():
    from paper_2510_26709_b200 import api as A
    return A


def _inputs(d, seed, special=False):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(d).astype(np.float32)
    gb = (rng.standard_normal(d) * 10.0 ** rng.integers(-6, 3, d)).astype(np.float32)
    m = (rng.standard_normal(d) * 0.01).astype(np.float32)
    v = (rng.random(d) * 1e-4).astype(np.float32)
    if special and d >= 16:
        gb[:8] = [0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -3e-39, 3e38]
        v[8:12] = [0.0, 1e-45, np.inf, 0.0]
        m[12:16] = [-0.0, np.nan, 1e-44, 0.0]
    return x, gb, m, v


def _same(a, b):
    """Bit equality, NaNs compared as NaN (payloads may differ)."""
    a, b = np.asarray(a), np.asarray(b)
    na, nb = np.isnan(a), np.isnan(b)
    return np.array_equal(na, nb) and np.array_equal(a[~na].view(np.uint32), b[~nb].view(np.uint32))


def _dev(a):
    return torch.from_numpy(a).to(DEV)


SIZES = [1, 3, 4, 5, 1023, 262_147, 148 * 8 * 256 * 4 * 2 + 4 * 37 + 3]


@pytest.mark.parametrize("d", SIZES)
def test_sgd_bit_exact(orc, api, d):
    x, gb, _, _ = _inputs(d, 100 + d, special=True)
    want = orc.apply_sgd(x, gb, 0.0375)
    xd, gd = _dev(x), _dev(gb)
    api.apply_update(xd, gd, 0.0375)
    torch.cuda.synchronize()
    assert _same(xd.cpu().numpy(), want)
    assert _same(gd.cpu().numpy(), gb)   # gbar untouched


@pytest.mark.parametrize("d", SIZES)
def test_adam_bit_exact_several_steps(orc, api, d):
    x, gb, m, v = _inputs(d, 200 + d, special=True)
    xd, md, vd = _dev(x), _dev(m), _dev(v)
    for t in range(1, 5):
        gbt = (gb * np.float32(1.0 + 0.25 * t)).astype(np.float32)
        x, m, v = orc.apply_adam(x, m, v, gbt, t, 1e-3, 0.9, 0.999, 1e-8)
        api.apply_update(xd, _dev(gbt), 1e-3, optimizer="adam", t=t, m=md, v=vd, beta1=0.9, beta2=0.999,
                         eps=1e-8)
    torch.cuda.synchronize()
    assert _same(xd.cpu().numpy(), x)
    assert _same(md.cpu().numpy(), m)
    assert _same(vd.cpu().numpy(), v)


def test_adam_late_step_and_hyperparameters(orc, api):
    # a large step count (bias corrections ~ 1) and other betas / eps
    d = 100_001
    x, gb, m, v = _inputs(d, 7)
    want = orc.apply_adam(x, m, v, gb, 10_000, 3e-4, 0.8, 0.95, 1e-6)
    xd, md, vd = _dev(x), _dev(m), _dev(v)
    api.apply_update(xd, _dev(gb), 3e-4, optimizer="adam", t=10_000, m=md, v=vd, beta1=0.8, beta2=0.95, eps=1e-6)
    torch.cuda.synchronize()
    for got, w in zip((xd, md, vd), want):
        assert _same(got.cpu().numpy(), w)


def test_full_size_c3(orc, api):
    """BASELINE.json's C3 size (d = 124,439,808) in bench.py's launch
    configuration (one wave of 148 x 8 CTAs, grid-stride)."""
    d = 124_439_808
    x, gb, m, v = _inputs(d, 11)
    xd, gd, md, vd = _dev(x), _dev(gb), _dev(m), _dev(v)
    api.apply_update(xd, gd, 0.01)
    want = orc.apply_sgd(x, gb, 0.01)
    torch.cuda.synchronize()
    assert _same(xd.cpu().numpy(), want)
    xd.copy_(_dev(x))
    api.apply_update(xd, gd, 1e-3, optimizer="adam", t=3, m=md, v=vd)
    torch.cuda.synchronize()
    wx, wm, wv = orc.apply_adam(x, m, v, gb, 3, 1e-3)
    assert _same(xd.cpu().numpy(), wx) and _same(md.cpu().numpy(), wm) and _same(vd.cpu().numpy(), wv)


def test_after_step_on_same_stream(orc, api):
    """Chained after ArcTopK.step on a side stream: the update reads the
    step's gbar (eq:ef21m-3 after eq:ef21m-2)."""
    from paper_2510_26709_b200 import ArcTopK, flat_layout
    d, n = 40_000, 64
    blocks = flat_layout(d, n, K=20)
    rng = np.random.default_rng(3)
    s = torch.cuda.Stream()
    ctx = ArcTopK(d, blocks, N=1, eta=0.1, device=DEV)
    h = torch.zeros(d, device=DEV)
    g = torch.zeros(d, device=DEV)
    gbar = torch.zeros(d, device=DEV)
    x0 = rng.standard_normal(d).astype(np.float32)
    x = _dev(x0)
    with torch.cuda.stream(s):
        grad = _dev(rng.standard_normal(d).astype(np.float32))
        s.wait_stream(torch.cuda.default_stream())
        ctx.step(0, [grad], [h], [g], gbar, stream=s)
        api.apply_update(x, gbar, 0.5, stream=s)
    s.synchronize()
    assert _same(x.cpu().numpy(), orc.apply_sgd(x0, gbar.cpu().numpy(), 0.5))
    assert int((gbar != 0).sum()) > 0
    ctx.close()


def test_step_and_update_in_one_cuda_graph(orc, api):
    """Step + SGD update captured together in one CUDA graph (the launch-bound
    small-d case): one replay gives the oracle's x_{t+1} bit for bit."""
    from paper_2510_26709_b200 import ArcTopK, flat_layout
    d, n, N = 30_011, 50, 2
    blocks = flat_layout(d, n, K=9)
    rng = np.random.default_rng(21)
    grads_np = [rng.standard_normal(d).astype(np.float32) for _ in range(N)]
    x0 = rng.standard_normal(d).astype(np.float32)
    ctx = ArcTopK(d, blocks, N=N, eta=0.1, seed=5)
    h = [torch.zeros(d, device=DEV) for _ in range(N)]
    g = [torch.zeros(d, device=DEV) for _ in range(N)]
    gbar = torch.zeros(d, device=DEV)
    grads = [_dev(a) for a in grads_np]
    x = _dev(x0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            ctx.step(0, grads, h, g, gbar, stream=s)
            api.apply_update(x, gbar, 0.125, stream=s)
    graph.replay()
    torch.cuda.synchronize()
    ref = orc.OracleEF21M(d, [orc.Block(b.offset, b.len, b.m, b.n, b.K, b.kind) for b in blocks], N=N, eta=0.1,
                          r=4, seed=5)
    ref.step(0, grads_np)
    assert gbar.cpu().numpy().tobytes() == ref.gbar.tobytes()
    assert _same(x.cpu().numpy(), orc.apply_sgd(x0, ref.gbar, 0.125))
    ctx.close()
