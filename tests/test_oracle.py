"""Pins for the CPU oracle (``oracle/arc_oracle.c``) against what the paper and
the mathematics fix — never against the oracle itself.

Citations: P:n = /root/reference/PAPER.md line n (LaTeX label given too);
S:n = SPEC.md line n (test ideas only).  All tests here are CPU-only.
"""
import itertools
import math
import os

import numpy as np
import pytest

from synth import Block, adversarial, flat_blocks

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
U32 = 2.0 ** -24


def _all_uniforms():
    i = np.arange(2 ** 23, dtype=np.float64)
    return ((2 * i + 1) * U32).astype(np.float32)      # every value the generator can emit


def _ulp_err(approx, exact64):
    ulp = np.spacing(np.abs(exact64).astype(np.float32)).astype(np.float64)
    return np.abs(approx.astype(np.float64) - exact64) / ulp


# ---------------------------------------------------------------- generator (R8)

def test_philox_known_answers(orc):
    """Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    n = 0
    for line in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        out = orc.philox4x32_10(w[0:4], w[4:6])
        assert [int(x) for x in out] == w[6:10]
        n += 1
    assert n == 3


def test_uniform_is_exact_odd_multiple(orc):
    """u = (2i+1) 2^-24 exactly, i = x >> 9: in (0,1), never 0 or 1."""
    for x in [0, 1, 511, 512, 0xFFFFFFFF, 0x80000000, 0x12345678]:
        u = orc.uniform(x)
        assert u == (2 * (x >> 9) + 1) * U32
        assert 0.0 < u < 1.0


def test_ln_exhaustive_within_2ulp(orc):
    """ln over every generator value vs libm log in binary64: <= 2 ulp."""
    u = _all_uniforms()
    err = _ulp_err(orc.ln_array(u), np.log(u.astype(np.float64)))
    assert err.max() <= 2.0, err.max()


def test_sincos_exhaustive_within_2ulp(orc):
    """sin(2 pi u), cos(2 pi u) over every generator value vs libm (binary64): <= 2 ulp."""
    u = _all_uniforms()
    s, c = orc.sincos2pi_array(u)
    th = 2.0 * np.pi * u.astype(np.float64)
    assert _ulp_err(s, np.sin(th)).max() <= 2.0
    assert _ulp_err(c, np.cos(th)).max() <= 2.0
    # sin^2 + cos^2 = 1 within a few ulp, quadrant signs correct
    assert np.abs(s.astype(np.float64) ** 2 + c.astype(np.float64) ** 2 - 1).max() < 4e-7
    assert np.all(np.sign(s[(u > 0.01) & (u < 0.49)]) > 0) and np.all(np.sign(s[(u > 0.51) & (u < 0.99)]) < 0)


def test_gaussian_V_moments_spec_example(orc):
    """seed=7, n=64, r=64 -> mean within +-4/sqrt(4096), variance in [0.9, 1.1]."""
    V = orc.gaussian_V(7, 0, 0, 64, 64).astype(np.float64)
    assert abs(V.mean()) <= 0.0625
    assert 0.9 <= V.var() <= 1.1


def test_gaussian_V_is_standard_normal(orc):
    """vec(V) ~ N(0, I): KS test and near-zero cross-column correlation."""
    from scipy import stats
    V = orc.gaussian_V(20251030, 3, 1, 8192, 8).astype(np.float64)
    ks = stats.kstest(V.ravel(), "norm")
    assert ks.pvalue > 1e-3, ks
    C = np.corrcoef(V.T)
    assert np.abs(C - np.eye(8)).max() < 0.05
    # odd r: only the first r of each group of four are used
    V5 = orc.gaussian_V(1, 0, 0, 4096, 5).astype(np.float64)
    assert stats.kstest(V5.ravel(), "norm").pvalue > 1e-3


def test_gaussian_V_determinism_and_streams(orc):
    """same (seed,t,b) -> identical; any change of seed, t or block -> different."""
    a = orc.gaussian_V(42, 5, 2, 3, 2)
    assert np.array_equal(a, orc.gaussian_V(42, 5, 2, 3, 2))
    for other in [(43, 5, 2), (42, 6, 2), (42, 5, 3), (42 + (1 << 32), 5, 2), (42, 5 + (1 << 32), 2)]:
        assert not np.array_equal(a, orc.gaussian_V(other[0], other[1], other[2], 3, 2))


# ---------------------------------------------------------------- reshape / sketch

def test_row_major_reshape(orc):
    """S:48-50 / z72habsd00111, reading R1: g=[1..6], m=2 -> [[1,2,3],[4,5,6]];
    exact row norms 14 and 77 select row 1; the compact row is [4,5,6]."""
    out = orc.arc_round([np.arange(1, 7, dtype=np.float32)], n=3, K=1, exact=True, r=1)
    assert out["sigma"].tolist() == [14.0, 77.0]
    assert out["sel"].tolist() == [1]
    assert out["C"].tolist() == [[4.0, 5.0, 6.0]]
    # d not divisible by n (reading R14): virtual zero padding of the last row
    out = orc.arc_round([np.array([1, 2, 3], np.float32)], n=2, K=2, exact=True, r=1)
    assert out["sigma"].tolist() == [5.0, 9.0]
    assert out["C"].tolist() == [[1.0, 2.0], [3.0, 0.0]]


def test_sketch_spec_examples(orc):
    """S:130-132, P_i = (1/sqrt r) G_i V.  The oracle keeps P'_i = G_i V
    (reading R2); the reported P = P' * fl(1/sqrt r) * (1/N) matches S's values."""
    out = orc.arc_round([np.array([[1, 0], [0, 1]], np.float32)], n=2, K=1,
                        V=np.array([[2], [0]], np.float32))
    assert out["P_nodes"][0].tolist() == [[2.0], [0.0]]            # r = 1: P = P'
    out = orc.arc_round([np.array([[1, 1]], np.float32)], n=2, K=1,
                        V=np.array([[1, 1], [1, -1]], np.float32))
    assert out["S"].tolist() == [[2.0, 0.0]]
    P = (out["S"] * (np.float32(1) / np.sqrt(np.float32(2)))).astype(np.float64)
    assert abs(P[0, 0] - 2 / math.sqrt(2)) <= 2 * np.spacing(np.float32(1.41421356))
    assert P[0, 1] == 0.0
    out = orc.arc_round([np.zeros((3, 2), np.float32)], n=2, K=1, V=np.ones((2, 4), np.float32))
    assert not out["P_nodes"].any()


@pytest.mark.parametrize("N,m,n,r", [(1, 40, 300, 4), (3, 33, 129, 3), (4, 17, 1, 4), (2, 9, 1000, 1)])
def test_sketch_within_rounding_bound_of_exact_product(orc, N, m, n, r):
    """The fp32 sketch agrees with the binary64 matrix product (numpy) within the
    classical bound |fl(sum) - sum| <= gamma_k sum |terms|, gamma_k = k u / (1 - k u),
    k = n + 5 covering any O6 order (lane chain, butterfly, chunk sum).
    A dropped term, a wrong index or a transposed operand breaks it by orders of magnitude."""
    rng = np.random.default_rng(11 * m + n)
    G = [(rng.standard_normal((m, n)) * np.exp(rng.standard_normal((m, 1)))).astype(np.float32) for _ in range(N)]
    V = orc.gaussian_V(99, 1, 0, n, r)
    out = orc.arc_round(G, n=n, K=max(1, m // 4), V=V)
    u = 2.0 ** -24
    gam = lambda k: k * u / (1 - k * u)
    G64 = [x.astype(np.float64) for x in G]
    V64 = V.astype(np.float64)
    for i in range(N):
        exact = G64[i] @ V64
        bound = gam(n + 5) * (np.abs(G64[i]) @ np.abs(V64)) + 1e-300
        assert np.all(np.abs(out["P_nodes"][i] - exact) <= bound)
    S = sum(out["P_nodes"].astype(np.float64))
    absS = sum(np.abs(out["P_nodes"].astype(np.float64)))
    assert np.all(np.abs(out["S"] - S) <= gam(N + 1) * absS + 1e-300)
    sig = (out["S"].astype(np.float64) ** 2).sum(1)
    assert np.all(np.abs(out["sigma"] - sig) <= gam(r + 2) * sig + 1e-300)


def test_o6_order_is_the_lane_chunk_order(orc):
    """ARC-NUM v1 O6 pinned on a row where the order shows.  n = 1100
    (two chunks), V = 1.  Terms 2^25 at q = 0 (lane 0), 2 at q = 4 (lane 1) and 2 at
    q = 12 (lane 3): the butterfly pairs lanes 1 and 3 at o = 2 (2 + 2 = 4), then lane 0
    with lane 1 at o = 1: 2^25 + 4, exact.  A left-to-right sum rounds 2^25 + 2 to even
    twice and gives 2^25.  A term in chunk 1 is added after chunk 0's butterfly."""
    n = 1100
    x = np.zeros(n, np.float32)
    x[0], x[4], x[12] = 2.0 ** 25, 2.0, 2.0
    V = np.ones((n, 1), np.float32)
    assert orc.arc_round([x], n=n, K=1, V=V)["P_nodes"][0][0, 0] == np.float32(2.0 ** 25 + 4)
    lr = np.float32(0)
    for q in range(n):
        lr = np.float32(lr + x[q])
    assert lr == np.float32(2.0 ** 25)                     # the plain order differs
    x[1024] = -(2.0 ** 25)
    assert orc.arc_round([x], n=n, K=1, V=V)["P_nodes"][0][0, 0] == np.float32(4.0)
    # the lane chain is a fused multiply-add: the product (1 + 2^-12)(1 - 2^-12 + 2^-24) 2^-24
    # = 2^-24 (1 + 2^-36) rounds to 2^-24 on its own, and 1 + 2^-24 is a tie (-> 1.0);
    # fma rounds 1 + 2^-24 (1 + 2^-36) once, above the tie (-> 1 + 2^-23)
    y = np.zeros(8, np.float32)
    y[0], y[1] = 1.0, 1.0 + 2.0 ** -12
    W = np.ones((8, 1), np.float32)
    W[1, 0] = (1.0 - 2.0 ** -12 + 2.0 ** -24) * 2.0 ** -24
    assert np.float32(np.float32(y[1] * W[1, 0]) + np.float32(1.0)) == np.float32(1.0)
    got = orc.arc_round([y], n=8, K=1, V=W)["P_nodes"][0][0, 0]
    assert got == np.float32(1.0 + 2.0 ** -23)


# ---------------------------------------------------------------- selection (R5, R15)

def test_selection_spec_examples(orc):
    """S:139-141 / zn28373."""
    out = orc.arc_round([np.array([[1, 2], [0, 3]], np.float32)], n=2, K=1, V=np.eye(2, dtype=np.float32))
    # with V = I (r = 2): S = G, Sigma = [5, 9] (the paper's P = G/sqrt 2 halves both) -> I = {1}
    assert out["sel"].tolist() == [1]
    assert orc.argtop_k(np.array([5, 9], np.float32), 1).tolist() == [1]
    assert orc.argtop_k(np.array([1, 1], np.float32), 1).tolist() == [0]      # tie -> smaller index
    assert orc.argtop_k(np.array([25, 0, 1], np.float32), 2).tolist() == [0, 2]


def test_selection_brute_force_small(orc):
    """For m <= 9 and every K: I maximises sum of keys, and among maximisers it is the
    lexicographically smallest set (ties -> smaller indices); returned ascending."""
    rng = np.random.default_rng(5)
    for trial in range(60):
        m = int(rng.integers(1, 10))
        vals = rng.integers(0, 4, m).astype(np.float32)            # many ties
        if trial % 5 == 0:
            vals[rng.integers(0, m)] = np.inf
        keys = [orc.sigma_key(v) for v in vals]
        for K in range(1, m + 1):
            best = None
            for comb in itertools.combinations(range(m), K):       # lexicographic order
                s = sorted((keys[p] for p in comb), reverse=True)
                if best is None or s > best[0]:
                    best = (s, list(comb))
            assert orc.argtop_k(vals, K).tolist() == best[1]


def test_selection_equals_stable_sort(orc):
    """Any m: I = first K of a stable sort by key descending (numpy lexsort), incl.
    ties, +Inf and NaN (NaN ranks above +Inf, reading R15)."""
    rng = np.random.default_rng(8)
    for m in [1, 2, 100, 4097, 100_000]:
        v = np.abs(rng.standard_normal(m)).astype(np.float32)
        v[rng.integers(0, m, m // 3 + 1)] = 0.5
        v[rng.integers(0, m, m // 50 + 1)] = np.inf
        if m > 2:
            v[rng.integers(0, m, 2)] = np.nan
        keys = v.view(np.uint32).astype(np.int64)
        keys[np.isnan(v)] = 0xFFFFFFFF
        order = np.lexsort((np.arange(m), -keys))
        for K in sorted({1, m // 7 + 1, m // 2 + 1, m}):
            assert np.array_equal(orc.argtop_k(v, K), np.sort(order[:K]).astype(np.int32))


def test_selection_scale_invariance(orc):
    """scaling every row's sketch by c > 0 (exactly, a power of two) keeps I."""
    rng = np.random.default_rng(3)
    G = rng.standard_normal((64, 8)).astype(np.float32)
    V = orc.gaussian_V(1, 0, 0, 8, 4)
    a = orc.arc_round([G], n=8, K=9, V=V)["sel"]
    b = orc.arc_round([G * np.float32(8.0)], n=8, K=9, V=V)["sel"]
    assert np.array_equal(a, b)


# ---------------------------------------------------------------- statistical properties

def _monte_carlo_sigma(orc, G, r, seeds, N=1):
    n = G.shape[1]
    out = []
    for s in range(seeds):
        V = orc.gaussian_V(1000 + s, 0, 0, n, r)
        # reported Sigma = sigma / (r N^2) (reading R2/R3: selection-invariant factors)
        out.append(orc.arc_round([G] * N, n=n, K=1, V=V)["sigma"].astype(np.float64) / (r * N * N))
    return np.array(out)


def test_sketch_unbiased(orc):
    """z72ena: E[Sigma_p] = ||u_p||^2. G = [[3,4],[0,0],[1,0]], r = 1,
    10^4 seeds: mean within 5% of [25, 0, 1]."""
    sig = _monte_carlo_sigma(orc, np.array([[3, 4], [0, 0], [1, 0]], np.float32), 1, 10_000)
    mean = sig.mean(0)
    assert abs(mean[0] - 25) <= 0.05 * 25 and mean[1] == 0 and abs(mean[2] - 1) <= 0.05


def test_sketch_variance_falls_with_r(orc):
    """P:261 "larger values of r yielding smaller estimate variance"."""
    G = np.array([[3, 4], [0, 0], [1, 0]], np.float32)
    v1 = _monte_carlo_sigma(orc, G, 1, 3000).var(0)
    v16 = _monte_carlo_sigma(orc, G, 16, 3000).var(0)
    assert v16[0] < v1[0] and v16[2] < v1[2]
    # chi-square: Var[Sigma_p] = 2 ||u||^4 / r
    assert abs(v1[0] - 2 * 625) < 0.2 * 2 * 625 and abs(v16[0] - 2 * 625 / 16) < 0.2 * 2 * 625 / 16


def test_spec_full_round_seed_sweep(orc):
    """[[3,4],[0,0],[1,0]], K=1, r=32 -> row 0 selected in >= 990/1000 seeds, and the
    compression error when it is selected is ||[1,0]||^2 = 1."""
    G = np.array([[3, 4], [0, 0], [1, 0]], np.float32)
    hit = 0
    for s in range(1000):
        out = orc.arc_round([G], n=2, K=1, V=orc.gaussian_V(s, 0, 0, 2, 32))
        if out["sel"][0] == 0:
            hit += 1
            err = (G.astype(np.float64) ** 2).sum() - (out["C"].astype(np.float64) ** 2).sum()
            assert err == 1.0
    assert hit >= 990


@pytest.mark.parametrize("m,n,K,r", [(8, 4, 2, 2), (16, 8, 4, 1), (32, 16, 8, 4)])
def test_contraction_monte_carlo(orc, m, n, K, r):
    """Prop. 2: E||C(g) - g||^2 <= (1 - K/m) ||g||^2 with g the node average.
    Monte Carlo over 10^4 sketches, N = 2 heavy-tailed nodes; 3 standard errors + 1e-6."""
    rng = np.random.default_rng(m * 31 + r)
    G = [(rng.standard_normal((m, n)) * np.exp(1.5 * rng.standard_normal((m, 1)))).astype(np.float32) for _ in range(2)]
    gbar = (G[0].astype(np.float64) + G[1]) / 2
    tot = (gbar ** 2).sum()
    ratios = []
    for s in range(10_000):
        out = orc.arc_round(G, n=n, K=K, V=orc.gaussian_V(s, 0, 0, n, r))
        comp = np.zeros_like(gbar)
        comp[out["sel"]] = out["C"]
        ratios.append(((comp - gbar) ** 2).sum() / tot)
    ratios = np.array(ratios)
    se = ratios.std() / math.sqrt(len(ratios))
    assert ratios.mean() <= 1 - K / m + 3 * se + 1e-6


def test_contraction_exact_sketch_deterministic(orc):
    """With the exact sketch the top-K rows of the average carry at least the average
    mass, so ||C(g)-g||^2 <= (1-K/m)||g||^2 holds at every draw (Chebyshev step)."""
    rng = np.random.default_rng(4)
    for trial in range(50):
        m, n, N = int(rng.integers(2, 40)), int(rng.integers(1, 9)), int(rng.integers(1, 5))
        K = int(rng.integers(1, m + 1))
        G = [rng.standard_normal((m, n)).astype(np.float32) for _ in range(N)]
        out = orc.arc_round(G, n=n, K=K, exact=True, r=1)
        gbar = sum(x.astype(np.float64) for x in G) / N
        comp = np.zeros_like(gbar)
        comp[out["sel"]] = out["C"]
        assert ((comp - gbar) ** 2).sum() <= (1 - K / m) * (gbar ** 2).sum() * (1 + 1e-5) + 1e-12


# ---------------------------------------------------------------- special cases of north_star

def test_exact_sketch_N1_is_row_topk(orc):
    """north_star: "ARC-Top-K reduces to Top-K when N=1 with an exact sketch" — I equals
    the K rows of largest ||row||^2 (numpy, binary64, stable tie-break)."""
    rng = np.random.default_rng(12)
    for _ in range(20):
        m, n = int(rng.integers(5, 300)), int(rng.integers(1, 50))
        K = int(rng.integers(1, m + 1))
        G = rng.integers(-4, 5, (m, n)).astype(np.float32)       # exact sums: no rounding ties
        norms = (G.astype(np.float64) ** 2).sum(1)
        want = np.sort(np.lexsort((np.arange(m), -norms))[:K])
        assert np.array_equal(orc.arc_round([G], n=n, K=K, exact=True, r=1)["sel"], want)


def test_K_equals_m_is_identity(orc):
    """north_star "K=d gives the identity": with n = 1, K = m = d the compressor
    returns the node average of every row; with N = 1 bit for bit."""
    rng = np.random.default_rng(2)
    d = 257
    x = rng.standard_normal(d).astype(np.float32)
    out = orc.arc_round([x], n=1, K=d, V=orc.gaussian_V(1, 0, 0, 1, 4))
    assert out["sel"].tolist() == list(range(d))
    assert np.array_equal(out["C"].ravel(), x)
    xs = [rng.standard_normal(d).astype(np.float32) for _ in range(4)]
    out = orc.arc_round(xs, n=1, K=d, V=orc.gaussian_V(1, 0, 0, 1, 4))
    mean = sum(v.astype(np.float64) for v in xs) / 4
    mag = sum(np.abs(v.astype(np.float64)) for v in xs) / 4
    assert np.all(np.abs(out["C"].ravel() - mean) <= 4 * 2 ** -24 * mag)


def test_n1_is_coordinate_topk_of_node_sum(orc):
    """n = 1: Sigma_p = (S_p)^2 sum_j v_j^2 / (r N^2) is monotone in |S_p| (S_p = sum_i
    Delta_i[p]), so ARC selects the K largest |S_p| — classical Top-K of the average."""
    rng = np.random.default_rng(6)
    for trial in range(20):
        m, N = 200, 3
        K = int(rng.integers(1, 50))
        xs = [rng.integers(-50, 51, m).astype(np.float32) for _ in range(N)]
        S = np.abs(sum(x.astype(np.int64) for x in xs))
        order = np.lexsort((np.arange(m), -S))
        if K < m and S[order[K - 1]] == S[order[K]]:
            continue                      # boundary tie: several answers are correct
        out = orc.arc_round(xs, n=1, K=K, V=orc.gaussian_V(trial, 0, 0, 1, 4))
        assert set(out["sel"].tolist()) == set(order[:K].tolist())


def test_prop1_worked_example(orc):
    """Prop. 1, tests/golden/prop1_worked_example.txt: per-node Top-K (the
    baseline of Table I) gives C(g) = 0 and error ratio exactly 1; ARC-Top-K on the
    same nodes (n = 1) aligns on index 1 and the error is exactly 0."""
    gold = {}
    for line in open(os.path.join(GOLDEN, "prop1_worked_example.txt")):
        if "=" in line and not line.startswith("#"):
            k, v = line.split("=")
            gold[k.strip()] = [float(x) for x in v.split()]
    g1 = np.array(gold["g1"], np.float32)
    g2 = np.array(gold["g2"], np.float32)
    blocks = flat_blocks(2, 1, K=1)
    o = orc.OracleEF21M(2, blocks, N=2, eta=1.0, r=4, seed=1)
    res = o.step_topk(0, [g1, g2])
    assert res["values"][0].tolist() == [gold["topk_local_1"][0]] and res["sel"][0].tolist() == [0]
    assert res["values"][1].tolist() == [gold["topk_local_2"][0]] and res["sel"][1].tolist() == [0]
    assert o.gbar.tolist() == gold["topk_global"]
    g = (g1.astype(np.float64) + g2) / 2
    assert ((o.gbar - g) ** 2).sum() / (g ** 2).sum() == gold["topk_error_ratio"][0]
    a = orc.OracleEF21M(2, blocks, N=2, eta=1.0, r=4, seed=1)
    res = a.step(0, [g1, g2])
    assert res["sel"].tolist() == [1]
    assert a.gbar.tolist() == [0.0, np.float32(0.1)]       # C(g) = g exactly
    # and row Top-K with the EXACT sketch picks the same index
    assert orc.arc_round([g1, g2], n=1, K=1, exact=True, r=1)["sel"].tolist() == [1]


def test_symmetric_nodes_give_zero(orc):
    """nodes G and -G -> P = 0, Sigma = 0, I = {0..K-1} (tie-break), output 0."""
    xs = adversarial("symmetric", 96, 4, n=8)
    out = orc.arc_round(xs, n=8, K=5, V=orc.gaussian_V(3, 0, 0, 8, 4))
    assert not out["sigma"].any()
    assert out["sel"].tolist() == [0, 1, 2, 3, 4]
    assert not out["C"].any()


def test_compaction_is_row_gather_and_linear(orc):
    """2zn20: C_local_i = rows I of G_i; C = (1/N) sum_i C_local_i."""
    rng = np.random.default_rng(9)
    N, m, n = 3, 50, 7
    G = [rng.standard_normal((m, n)).astype(np.float32) for _ in range(N)]
    out = orc.arc_round(G, n=n, K=11, V=orc.gaussian_V(5, 0, 0, n, 4))
    for i in range(N):
        assert np.array_equal(out["C_local"][i], G[i][out["sel"]])
    mean = sum(x.astype(np.float64) for x in G)[out["sel"]] / N
    mag = sum(np.abs(x.astype(np.float64)) for x in G)[out["sel"]] / N
    assert np.all(np.abs(out["C"] - mean) <= 3 * 2 ** -24 * mag)


# ---------------------------------------------------------------- EF21M (eq:ef21m-1..3)

def test_momentum_eta_one_copies_gradient(orc):
    """eq:ef21m-1 with eta = 1: h_t = grad exactly."""
    rng = np.random.default_rng(1)
    d = 300
    o = orc.OracleEF21M(d, flat_blocks(d, 10, K=3), N=2, eta=1.0, r=4, seed=1,
                        h0=[rng.standard_normal(d)] * 2)
    gr = [rng.standard_normal(d).astype(np.float32) for _ in range(2)]
    o.step(0, gr)
    for i in range(2):
        assert np.array_equal(o.h[i], gr[i])


def test_momentum_closed_form(orc):
    """Constant gradient c: h_t = (1 - (1-eta)^(t+1)) c  (geometric series of eq:ef21m-1)."""
    d, eta = 64, 0.1
    c = np.linspace(-2, 3, d).astype(np.float32)
    o = orc.OracleEF21M(d, flat_blocks(d, 8, K=1), N=1, eta=eta, r=4, seed=1)
    for t in range(20):
        o.step(t, [c])
        want = (1 - (1 - eta) ** (t + 1)) * c.astype(np.float64)
        assert np.all(np.abs(o.h[0] - want) <= 1e-5 * np.abs(c) + 1e-30)


def test_ef21m_identity_compressor_tracks_gradient(orc):
    """K = m and eta = 1 -> g_i = grad_i (to an ulp: g + (h - g)) and
    gbar = mean of the gradients (gradient averaging), every step."""
    rng = np.random.default_rng(10)
    d, N = 120, 4
    blocks = flat_blocks(d, 12, K=10)
    o = orc.OracleEF21M(d, blocks, N=N, eta=1.0, r=4, seed=2)
    for t in range(5):
        gr = [rng.standard_normal(d).astype(np.float32) for _ in range(N)]
        g_prev = [x.copy() for x in o.g]
        res = o.step(t, gr)
        assert res["sel"].tolist() == list(range(10))
        for i in range(N):
            # g + (h - g), two roundings: within 1.5 ulp of max(|g_prev|, |h|)
            big = np.maximum(np.abs(g_prev[i]), np.abs(gr[i]))
            assert np.all(np.abs(o.g[i] - gr[i]) <= 1.5 * np.spacing(big))
        mean = sum(x.astype(np.float64) for x in gr) / N
        assert np.all(np.abs(o.gbar - mean) <= 1e-5 * (np.abs(mean) + sum(np.abs(x) for x in gr) / N))


def test_ef21m_gbar_is_mean_of_g(orc):
    """gbar is the replicated tracker (1/N) sum_i g_i consumed by eq:ef21m-3,
    reading R13: after T steps it equals the mean of the node trackers within tolerance."""
    from synth import GradientSource
    d, N = 4000, 4
    blocks = flat_blocks(d, 40, mu_bp=1000)
    src = GradientSource(d, blocks, N, seed=3)
    o = orc.OracleEF21M(d, blocks, N=N, eta=0.1, r=4, seed=3)
    for t in range(10):
        o.step(t, [x.numpy() for x in src.grads(t)])
    mean = sum(x.astype(np.float64) for x in o.g) / N
    mag = sum(np.abs(x.astype(np.float64)) for x in o.g) / N
    assert np.all(np.abs(o.gbar - mean) <= 1e-5 * mag + 1e-30)


def test_ef_rows_outside_selection_untouched(orc):
    """eq:ef21m-2: g changes only on the selected rows (C_local is zero elsewhere)."""
    rng = np.random.default_rng(13)
    d, n = 500, 10
    o = orc.OracleEF21M(d, flat_blocks(d, n, K=7), N=2, eta=0.5, r=4, seed=4,
                        g0=[rng.standard_normal(d)] * 2, gbar0=rng.standard_normal(d))
    g_before = [x.copy() for x in o.g]
    gb_before = o.gbar.copy()
    res = o.step(0, [rng.standard_normal(d) for _ in range(2)])
    mask = np.zeros(d // n, bool)
    mask[res["sel"]] = True
    rows = np.repeat(mask, n)
    for i in range(2):
        assert np.array_equal(o.g[i][~rows], g_before[i][~rows])
        assert not np.array_equal(o.g[i][rows], g_before[i][rows])
    assert np.array_equal(o.gbar[~rows], gb_before[~rows])


def test_multiblock_exact_sketch_is_per_block_topk(orc):
    """Per-tensor compression: each block b keeps its own K_b rows; with the
    exact sketch and integer data the choice equals numpy's per-block row Top-K."""
    rng = np.random.default_rng(14)
    shapes = [(7, 5, 2, 0), (12, 3, 12, 1), (20, 4, 6, 0), (1, 9, 1, 0)]
    blocks, off = [], 0
    for m, n, K, kind in shapes:
        blocks.append(Block(off, m * n, m, n, K, kind))
        off += m * n
    d = off
    N = 2
    gr = [rng.integers(-5, 6, d).astype(np.float32) for _ in range(N)]
    o = orc.OracleEF21M(d, blocks, N=N, eta=1.0, r=1, seed=5, exact=True)
    res = o.step(0, gr)
    pos = 0
    for B in blocks:
        x = sum(v[B.offset:B.offset + B.len].astype(np.int64) for v in gr).reshape(B.m, B.n)
        norms = (x.astype(np.float64) ** 2).sum(1)
        want = np.sort(np.lexsort((np.arange(B.m), -norms))[:B.K]) if B.kind == 0 else np.arange(B.m)
        got = res["sel"][pos:pos + B.K]
        # integer data with possible exact ties at the boundary: compare the unique part
        if B.kind == 0 and B.K < B.m:
            srt = np.sort(norms)[::-1]
            if srt[B.K - 1] == srt[B.K]:
                assert set(norms[got]) <= set(srt[:B.K])
                pos += B.K
                continue
        assert np.array_equal(got, want)
        pos += B.K


def test_determinism(orc):
    """same (seed, t, inputs) twice -> byte-identical outputs and state."""
    from synth import GradientSource
    d, N = 3000, 3
    blocks = flat_blocks(d, 30, mu_bp=500)
    src = GradientSource(d, blocks, N, seed=8)
    runs = []
    for _ in range(2):
        o = orc.OracleEF21M(d, blocks, N=N, eta=0.1, r=4, seed=8)
        outs = [o.step(t, [x.numpy() for x in src.grads(t)]) for t in range(3)]
        runs.append((outs, o))
    (a, oa), (b, ob) = runs
    for x, y in zip(a, b):
        assert np.array_equal(x["sel"], y["sel"]) and x["values"].tobytes() == y["values"].tobytes()
    assert oa.gbar.tobytes() == ob.gbar.tobytes()


# ---------------------------------------------------------------- Rand-K (Table I)

def test_randk_uniform_rows(orc):
    """m = 10, K = 3 over 10^5 draws: every row kept with frequency 0.3 +- 0.01,
    and the 120 possible 3-subsets are equally likely (chi-square)."""
    from scipy import stats
    m, K, T = 10, 3, 100_000
    counts = np.zeros(m)
    subsets = {}
    for t in range(T):
        sel = tuple(orc.argtop_k(orc.randk_keys(77, t, 0, m), K).tolist())
        counts[list(sel)] += 1
        subsets[sel] = subsets.get(sel, 0) + 1
    assert np.all(np.abs(counts / T - 0.3) <= 0.01)
    assert len(subsets) == 120
    assert stats.chisquare(list(subsets.values())).pvalue > 1e-3


def test_randk_shared_and_data_independent(orc):
    """Shared seed: identical on every node, independent of the data, K = m keeps every
    row; another seed or iteration gives another subset."""
    d, n, K = 4000, 40, 9
    blocks = flat_blocks(d, n, K=K)
    rng = np.random.default_rng(1)
    sels = []
    for data in (np.zeros(d, np.float32), rng.standard_normal(d).astype(np.float32)):
        o = orc.OracleEF21M(d, blocks, N=3, eta=0.5, r=4, seed=123, method="randk")
        sels.append(o.step(4, [data] * 3)["sel"])
    assert np.array_equal(sels[0], sels[1])
    keys = orc.randk_keys(123, 4, 0, d // n)
    assert np.array_equal(sels[0], orc.argtop_k(keys, K))
    assert not np.array_equal(orc.argtop_k(orc.randk_keys(124, 4, 0, 100), K), orc.argtop_k(keys, K))
    assert not np.array_equal(orc.argtop_k(orc.randk_keys(123, 5, 0, 100), K), orc.argtop_k(keys, K))
    o = orc.OracleEF21M(d, flat_blocks(d, n, K=d // n), N=2, eta=1.0, r=4, seed=1, method="randk")
    assert o.step(0, [rng.standard_normal(d)] * 2)["sel"].tolist() == list(range(d // n))


def test_randk_values_are_node_average_of_rows(orc):
    """C(g) = (1/N) sum_i [G_i]_{I,:} on the shared random rows (P:242 with Rand-K rows)."""
    rng = np.random.default_rng(2)
    d, n, K, N = 3000, 30, 7, 4
    o = orc.OracleEF21M(d, flat_blocks(d, n, K=K), N=N, eta=1.0, r=4, seed=5, method="randk")
    gr = [rng.standard_normal(d).astype(np.float32) for _ in range(N)]
    res = o.step(0, gr)
    rows = np.stack([x.reshape(-1, n) for x in gr])[:, res["sel"]].astype(np.float64)
    mean, mag = rows.mean(0), np.abs(rows).mean(0)
    assert np.all(np.abs(res["values"].reshape(K, n) - mean) <= N * 2 ** -24 * mag + 1e-30)


# ---------------------------------------------------------------- without EF (Table II, SPEC compressed_msgd_step)

def test_noef_identity_compressor_is_msgd(orc):
    """K = m: the compressor is the identity, so the step is heavy-ball momentum SGD on
    the node average (SPEC "K=m -> exact MSGD"): u_t = beta u_{t-1} + mean_i grad_i,
    checked against a plain numpy recursion in binary64 within the rounding of a few
    fp32 operations per step."""
    rng = np.random.default_rng(8)
    d, N, beta = 600, 3, 0.9
    o = orc.OracleEF21M(d, flat_blocks(d, 20, K=30), N=N, eta=beta, r=4, seed=2, method="noef_msgd")
    u = np.zeros(d)
    for t in range(12):
        gr = [rng.standard_normal(d).astype(np.float32) for _ in range(N)]
        o.step(t, gr)
        u = beta * u + sum(x.astype(np.float64) for x in gr) / N
        assert np.all(np.abs(o.gbar - u) <= 1e-5 * (np.abs(u) + 1))
        assert not any(x.any() for x in o.h) and not any(x.any() for x in o.g)   # no EF state


def test_noef_beta0_identity_is_gradient_average(orc):
    """beta = 0, K = m: plain (averaged) gradient descent direction (SPEC)."""
    rng = np.random.default_rng(9)
    d, N = 256, 4
    o = orc.OracleEF21M(d, flat_blocks(d, 16, K=16), N=N, eta=0.0, r=4, seed=3, method="noef_msgd")
    gr = [rng.integers(-8, 9, d).astype(np.float32) for _ in range(N)]   # exact sums
    o.step(0, gr)
    assert np.array_equal(o.gbar, (sum(x.astype(np.float64) for x in gr) / N).astype(np.float32))


def test_noef_prop1_shared_selection_keeps_signal(orc):
    """Prop. 1 inputs without EF: per-node Top-K would average to C(g) = 0,
    the shared ARC selection (n = 1) keeps index 1: u = [0, 0.1] exactly (beta = 0)."""
    g1 = np.array([-1.0, 0.1], np.float32)
    g2 = np.array([1.0, 0.1], np.float32)
    o = orc.OracleEF21M(2, flat_blocks(2, 1, K=1), N=2, eta=0.0, r=4, seed=1, method="noef_msgd")
    o.step(0, [g1, g2])
    assert o.gbar.tolist() == [0.0, np.float32(0.1)]


def test_noef_rows_outside_selection_only_decay(orc):
    """Rows outside I: u <- beta u exactly; rows in I: u <- beta u + values."""
    rng = np.random.default_rng(10)
    d, n, K, beta = 400, 10, 7, 0.75
    o = orc.OracleEF21M(d, flat_blocks(d, n, K=K), N=2, eta=beta, r=4, seed=4, method="noef_msgd")
    o.gbar[:] = rng.standard_normal(d).astype(np.float32)
    before = o.gbar.copy()
    out = o.step(0, [rng.standard_normal(d).astype(np.float32) for _ in range(2)])
    scaled = (np.float32(beta) * before).astype(np.float32)
    mask = np.zeros(d // n, bool)
    mask[out["sel"]] = True
    rows = o.gbar.reshape(-1, n)
    assert np.array_equal(rows[~mask], scaled.reshape(-1, n)[~mask])
    want = (scaled.reshape(-1, n)[mask] + out["values"].reshape(K, n)).astype(np.float32)
    assert np.array_equal(rows[mask], want)


def test_threads_are_bit_identical(orc):
    """The oracle's row-parallel loops (OpenMP) give bit-identical results to one
    thread: every row's arithmetic is the same sequence whichever thread runs it."""
    from synth import GradientSource
    blocks = [Block(0, 5000, 50, 100, 7, 0), Block(5000, 3001, 1001, 3, 40, 0), Block(8001, 999, 1, 1024, 1, 1),
              Block(9000, 20_000, 10, 2000, 2, 0)]
    d, N = 29_000, 3
    src = GradientSource(d, blocks, N, seed=4)
    outs = []
    for threads in (1, 8):
        orc.set_threads(threads)
        o = orc.OracleEF21M(d, blocks, N=N, eta=0.3, r=4, seed=2)
        res = [o.step(t, [x.numpy() for x in src.grads(t)], debug=True) for t in range(3)]
        outs.append((res, [x.copy() for x in o.h + o.g] + [o.gbar.copy()]))
    orc.set_threads(1)
    for a, b in zip(outs[0][0], outs[1][0]):
        for k in a:
            assert a[k].tobytes() == b[k].tobytes(), k
    for a, b in zip(outs[0][1], outs[1][1]):
        assert a.tobytes() == b.tobytes()
