"""Host model of the reduce="lsa" exchange protocol (arc_lsa.cu), CPU only.

The LSA kernels use per-CTA barriers only: CTA b of every rank owns sub-range b
of every rank's row slice (k_lsa_sigma), so the rows a CTA copies after barrier
2 are exactly the rows the same CTA index produced on their owner before it.
This checks that index math for many (M, G, grid) — every row of Σ produced
once, by its owner, and copied by the CTA that waited on its producer — and
that the node-ordered sum over peers' windows equals the ORDERED mode's sum
over the all-gathered payload (the same float32 additions in the same order).
"""
import numpy as np
import pytest

K_LSA_CTAS = 592   # arc_internal.cuh kLsaCtas


def lsa_grid(Ms):
    return max(1, min(K_LSA_CTAS, -(-Ms // 256)))


@pytest.mark.parametrize("M,G", [(1, 1), (7, 2), (1000, 3), (162031, 8), (5, 8), (76800, 4), (300_001, 7)])
def test_sigma_subrange_ownership(M, G):
    Ms = -(-M // G)
    grid = lsa_grid(Ms)
    chunk = -(-Ms // grid)
    produced = np.full(G * Ms, -1, dtype=np.int64)      # (rank, cta) that wrote row, encoded
    copied_ok = np.zeros(G * Ms, dtype=bool)
    for me in range(G):
        for b in range(grid):
            lo, hi = b * chunk, min(Ms, b * chunk + chunk)
            for p in range(lo, hi):
                row = me * Ms + p
                if row >= M:
                    break
                assert produced[row] == -1
                produced[row] = me * grid + b
    assert (produced[:M] >= 0).all() and (produced[M:] == -1).all()
    for me in range(G):
        for b in range(grid):
            lo, hi = b * chunk, min(Ms, b * chunk + chunk)
            for g in range(G):
                if g == me:
                    continue
                for p in range(lo, hi):
                    row = g * Ms + p
                    if row >= M:
                        break
                    assert produced[row] == g * grid + b     # same CTA index on the owner
                    copied_ok[row] = True
    if G > 1:
        # every rank holds every row: its own from phase A, the others copied
        assert copied_ok[:M].all()


@pytest.mark.parametrize("G,L", [(1, 1), (2, 3), (8, 1), (4, 2)])
def test_scatter_node_order_matches_ordered_mode(G, L):
    rng = np.random.default_rng(G * 10 + L)
    sum_Kn = 333
    win = [rng.standard_normal((L, sum_Kn)).astype(np.float32) for _ in range(G)]   # rank g's window
    N = G * L
    allg = np.concatenate([w.reshape(-1) for w in win])                             # ORDERED all-gather
    for o in range(sum_Kn):
        a_ord = allg[o]
        for i in range(1, N):
            a_ord = np.float32(a_ord + allg[i * sum_Kn + o])
        a_lsa = win[0][0, o]
        for i in range(1, N):
            g, l = divmod(i, L)
            a_lsa = np.float32(a_lsa + win[g][l, o])
        assert a_lsa.view(np.uint32) == a_ord.view(np.uint32)
