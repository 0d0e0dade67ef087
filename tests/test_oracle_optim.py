"""Pins of the oracle's model update (R23, R24).

SGD is eq:ef21m-3, x_{t+1} = x_t - gamma * gbar_t.  Adam is the
"standard Adam" of the paper's experiments, Kingma & Ba's
Algorithm 1 without weight decay, driven by gbar.  Each pin is fixed by
something other than the oracle: exact dyadic arithmetic, closed forms, and
torch.optim.Adam (an independent implementation) in float64.
"""
import numpy as np
import pytest
import torch


def test_sgd_dyadic_exact(orc):
    # every value and product is a small dyadic rational: the result is exact
    x = np.array([1.0, -2.0, 0.5, 0.0, 3.25], np.float32)
    gb = np.array([4.0, -1.0, 0.25, 8.0, 0.0], np.float32)
    out = orc.apply_sgd(x, gb, 0.25)
    assert np.array_equal(out, np.array([0.0, -1.75, 0.4375, -2.0, 3.25], np.float32))


def test_sgd_random_within_two_roundings(orc):
    rng = np.random.default_rng(7)
    x = rng.standard_normal(10_000).astype(np.float32)
    gb = rng.standard_normal(10_000).astype(np.float32)
    gamma = 0.0375
    out = orc.apply_sgd(x, gb, gamma).astype(np.float64)
    exact = x.astype(np.float64) - np.float64(np.float32(gamma)) * gb.astype(np.float64)
    bound = 2.0 ** -24 * (np.abs(exact) + gamma * np.abs(gb.astype(np.float64))) * 1.0001
    assert np.all(np.abs(out - exact) <= bound)
    # gamma = 0 leaves x untouched
    assert np.array_equal(orc.apply_sgd(x, gb, 0.0), x)


def test_adam_sign_descent_exact(orc):
    # beta1 = beta2 = 0, eps = 0: m = gbar, v = fl(gbar^2), sqrt(fl(g^2)) = |g|
    # exactly (correctly rounded sqrt), so every step is x - gamma * sign(gbar)
    x = np.array([1.0, 2.0, -0.5, 4.0], np.float32)
    m = np.zeros(4, np.float32)
    v = np.zeros(4, np.float32)
    rng = np.random.default_rng(3)
    expect = x.copy()
    for t in range(1, 6):
        gb = (rng.standard_normal(4) * 10.0 ** rng.integers(-3, 3, 4)).astype(np.float32)
        x, m, v = orc.apply_adam(x, m, v, gb, t, 0.25, 0.0, 0.0, 0.0)
        expect = (expect - np.float32(0.25) * np.sign(gb)).astype(np.float32)
        assert np.array_equal(x, expect)
        assert np.array_equal(m, gb)


def test_adam_constant_direction_closed_form(orc):
    # constant gbar = c: m_t = c (1 - b1^t), v_t = c^2 (1 - b2^t) in exact
    # arithmetic, so mhat = c, vhat = c^2 and x_T = x_0 - T gamma c / (|c| + eps):
    # a wrong bias correction (power, beta) moves x far from this
    c = np.array([0.3, -2.0, 1e-3, 5.0], np.float32)
    x = np.zeros(4, np.float32)
    m = np.zeros(4, np.float32)
    v = np.zeros(4, np.float32)
    T, gamma, eps = 40, 0.01, 1e-8
    for t in range(1, T + 1):
        x, m, v = orc.apply_adam(x, m, v, c, t, gamma, 0.9, 0.999, eps)
    c64 = c.astype(np.float64)
    expect = -T * gamma * c64 / (np.abs(c64) + eps)
    np.testing.assert_allclose(x, expect, rtol=2e-5, atol=0)


def test_adam_matches_torch_optim_adam_float64(orc):
    rng = np.random.default_rng(11)
    d, T = 4096, 30
    x0 = rng.standard_normal(d).astype(np.float32)
    p = torch.nn.Parameter(torch.tensor(x0, dtype=torch.float64))
    # the hyper-parameters as the fp32 values the oracle receives (1 - b2 is
    # then exact in both; 0.999 itself is not an fp32 number)
    f = lambda z: float(np.float32(z))
    opt = torch.optim.Adam([p], lr=f(1e-2), betas=(f(0.9), f(0.999)), eps=f(1e-8), weight_decay=0.0)
    x, m, v = x0.copy(), np.zeros(d, np.float32), np.zeros(d, np.float32)
    for t in range(1, T + 1):
        gb = (rng.standard_normal(d) * 0.1).astype(np.float32)
        p.grad = torch.tensor(gb, dtype=torch.float64)
        opt.step()
        x, m, v = orc.apply_adam(x, m, v, gb, t, 1e-2, 0.9, 0.999, 1e-8)
    ref = p.detach().numpy()
    # fp32 state against float64: the per-step move is gamma-sized, the
    # accumulated rounding a few fp32 ulps of x
    np.testing.assert_allclose(x, ref, rtol=0, atol=2e-5)
    st = opt.state[p]
    np.testing.assert_allclose(m, st["exp_avg"].numpy(), rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(v, st["exp_avg_sq"].numpy(), rtol=1e-5, atol=1e-10)


@pytest.mark.parametrize("bad", ["swap_betas", "no_bias_correction"])
def test_adam_pin_sensitivity(orc, bad):
    """The torch pin above would catch these mistakes: recomputing them in
    float64 lands far outside its tolerance."""
    rng = np.random.default_rng(5)
    d = 512
    gb_seq = [(rng.standard_normal(d) * 0.1) for _ in range(10)]
    def run(b1, b2, correct):
        x = np.zeros(d); m = np.zeros(d); v = np.zeros(d)
        for t, gb in enumerate(gb_seq, 1):
            m = b1 * m + (1 - b1) * gb
            v = b2 * v + (1 - b2) * gb * gb
            mh = m / (1 - b1 ** t) if correct else m
            vh = v / (1 - b2 ** t) if correct else v
            x = x - 1e-2 * mh / (np.sqrt(vh) + 1e-8)
        return x
    good = run(0.9, 0.999, True)
    wrong = run(0.999, 0.9, True) if bad == "swap_betas" else run(0.9, 0.999, False)
    assert np.max(np.abs(good - wrong)) > 1e-3
    x, m, v = np.zeros(d, np.float32), np.zeros(d, np.float32), np.zeros(d, np.float32)
    for t, gb in enumerate(gb_seq, 1):
        x, m, v = orc.apply_adam(x, m, v, gb.astype(np.float32), t, 1e-2, 0.9, 0.999, 1e-8)
    assert np.max(np.abs(x - good)) < 2e-5


def test_adam_eps_outside_sqrt_and_bias_correction_dyadic(orc):
    # beta1 = beta2 = 0.5, t = 1: bc1 = bc2 = 0.5, m = 0.5 g, v = 0.5 g^2, so
    # mhat = g and vhat = g^2 exactly; with eps = 1 the step is g / (|g| + 1)
    # (eps OUTSIDE the square root, Kingma & Ba Alg. 1): for g = 3 that is
    # 3/4, and x = 1 - 0.5 * 0.75 = 0.625 exactly (inside it would be 3/sqrt(10))
    x, m, v = orc.apply_adam(np.array([1.0, 1.0], np.float32), np.zeros(2, np.float32), np.zeros(2, np.float32),
                             np.array([3.0, -1.0], np.float32), 1, 0.5, 0.5, 0.5, 1.0)
    assert np.array_equal(x, np.array([0.625, 1.25], np.float32))
    assert np.array_equal(m, np.array([1.5, -0.5], np.float32))
    assert np.array_equal(v, np.array([4.5, 0.5], np.float32))
    # t = 2 with the same g: m = 0.75 g, v = 0.75 g^2, bc = 0.75: mhat = g, vhat = g^2 again
    x2, m2, v2 = orc.apply_adam(x, m, v, np.array([3.0, -1.0], np.float32), 2, 0.5, 0.5, 0.5, 1.0)
    assert np.array_equal(x2, np.array([0.25, 1.5], np.float32))
