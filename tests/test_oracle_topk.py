"""Pins for the oracle's All-Gather Top-K baseline (``orc_step_topk``): vanilla
EF21M with per-node row Top-K, Table I row "Top-K" (P:105-107,
P:212-218), inside eq:ef21m-1/2.

The reference here is written from the definitions with numpy, independently of
the oracle: node i keeps the K_b rows of ITS OWN residual Delta_i = h_i - g_i
with the largest ||row||^2 (ties -> smaller row, reading R5), its compact rows
C_i = Delta_i[sel_i], the EF update g_i[sel_i] += C_i (eq:ef21m-2, literal form
R12) and the tracker gbar[sel_j] += C_j / N for j = 0..N-1 (R13).

The inputs are small integers with eta = 1/2, so every value the baseline forms
(h, Delta, ||row||^2, C, g; gbar at N = 4) is a short dyadic fraction: the fp32
oracle must agree with the float64 reference EXACTLY, and a dropped term, a
doubled update or a wrong node index fails.
"""
import numpy as np
import pytest

from synth import Block


def _layout():
    # n = 1, 7 (short last row), 64, and a DENSE block (identity compressor, R20)
    blocks, off = [], 0
    for (m, n, length, K, kind) in [(40, 1, 40, 5, 0), (30, 7, 205, 4, 0), (12, 64, 768, 3, 0),
                                    (3, 16, 40, 3, 1), (9, 7, 63, 2, 0)]:
        blocks.append(Block(off, length, m, n, K, kind))
        off += length
    return off, blocks


def _numpy_topk_step(blocks, N, h, g, gbar, grads, eta):
    """One step of the baseline written from its definition (float64, exact here)."""
    h[:] = [(1 - eta) * h[i] + eta * grads[i] for i in range(N)]            # eq:ef21m-1
    sel_all, val_all = [[] for _ in range(N)], [[] for _ in range(N)]
    for B in blocks:
        pad = B.m * B.n - B.len
        C = []
        for i in range(N):
            D = np.concatenate([h[i][B.offset:B.offset + B.len] - g[i][B.offset:B.offset + B.len],
                                np.zeros(pad)]).reshape(B.m, B.n)         # residual rows, short row padded
            if B.kind == 0:
                norms = (D ** 2).sum(axis=1)
                order = np.lexsort((np.arange(B.m), -norms))                # norm desc, row asc (R5)
                sel = np.sort(order[:B.K])
            else:
                sel = np.arange(B.m)                                        # DENSE: every row
            sel_all[i].append(sel)
            val_all[i].append(D[sel].ravel())
            C.append((sel, D[sel]))
        for i, (sel, Ci) in enumerate(C):                                   # eq:ef21m-2, R12
            for k, p in enumerate(sel):
                nv = min(B.n, B.len - p * B.n)
                e = B.offset + p * B.n
                g[i][e:e + nv] += Ci[k, :nv]
        for j, (sel, Cj) in enumerate(C):                                   # gbar += C_j / N, node order
            for k, p in enumerate(sel):
                nv = min(B.n, B.len - p * B.n)
                e = B.offset + p * B.n
                gbar[e:e + nv] += Cj[k, :nv] / N
    return ([np.concatenate(s) for s in sel_all], [np.concatenate(v) for v in val_all])


@pytest.mark.parametrize("N", [3, 4])
def test_topk_baseline_matches_numpy_row_topk(orc, N):
    d, blocks = _layout()
    eta = 0.5
    rng = np.random.default_rng(100 + N)
    o = orc.OracleEF21M(d, blocks, N=N, eta=eta, r=4, seed=1)
    h = [np.zeros(d) for _ in range(N)]
    g = [np.zeros(d) for _ in range(N)]
    gbar = np.zeros(d)
    mag = np.zeros(d)                                       # sum over steps of (1/N) sum_i |C_i|
    for t in range(4):
        grads = [rng.integers(-8, 9, d).astype(np.float32) for _ in range(N)]
        # exact ties in ||row||^2 happen with small integers: the tie rule is exercised too
        g_prev = [x.copy() for x in g]
        sel_ref, val_ref = _numpy_topk_step(blocks, N, h, g, gbar, [x.astype(np.float64) for x in grads], eta)
        for i in range(N):
            mag += np.abs(g[i] - g_prev[i]) / N
        res = o.step_topk(t, grads)
        for i in range(N):
            assert np.array_equal(res["sel"][i], sel_ref[i]), f"node {i} selection differs at t={t}"
            assert np.array_equal(res["values"][i].astype(np.float64), val_ref[i]), f"node {i} C_i at t={t}"
            assert np.array_equal(o.h[i].astype(np.float64), h[i]), f"h[{i}] at t={t}"
            assert np.array_equal(o.g[i].astype(np.float64), g[i]), f"g[{i}] at t={t}"
        if N == 4:                                           # C / 4 exact: gbar exact too
            assert np.array_equal(o.gbar.astype(np.float64), gbar), f"gbar at t={t}"
        else:                                                # one rounding per C/3 and per add
            assert np.all(np.abs(o.gbar - gbar) <= 4 * (t + 1) * N * 2.0 ** -24 * mag), f"gbar at t={t}"
    # the EF invariant of the baseline: g_i moved exactly by what node i sent
    assert any(np.any(x != 0) for x in g)


def test_topk_baseline_rows_outside_selection_untouched(orc):
    """eq:ef21m-2 with C_local = per-node Top-K: rows node i did not select keep
    g_i unchanged, and gbar changes only on the union of the nodes' rows."""
    d, blocks = _layout()
    N = 3
    rng = np.random.default_rng(7)
    o = orc.OracleEF21M(d, blocks, N=N, eta=1.0, r=4, seed=1,
                        g0=[rng.integers(-4, 5, d).astype(np.float32) for _ in range(N)],
                        gbar0=rng.integers(-4, 5, d).astype(np.float32))
    g0 = [x.copy() for x in o.g]
    gb0 = o.gbar.copy()
    res = o.step_topk(0, [rng.integers(-8, 9, d).astype(np.float32) for _ in range(N)])
    union = np.zeros(d, bool)
    for i in range(N):
        touched = np.zeros(d, bool)
        pos = 0
        for B in blocks:
            for p in res["sel"][i][pos:pos + B.K]:
                e = B.offset + p * B.n
                touched[e:e + min(B.n, B.len - p * B.n)] = True
            pos += B.K
        assert np.array_equal(o.g[i][~touched], g0[i][~touched])
        union |= touched
    assert np.array_equal(o.gbar[~union], gb0[~union])
