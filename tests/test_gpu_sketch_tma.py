"""GPU parity of the bulk-copy (TMA) fed streaming launch (arc_sketch_tma.cu).

By default it takes the EF21M blocks whose rows are not 16-byte aligned or whose
V_b^T is too wide for the main launch's stage; ARC_SKETCH_TMA=2 routes every ARC
block of more than 4 columns through it and ARC_SKETCH_TMA=0 none (read at
create).  Every case is bit-exact against the oracle (selection, values, Sigma,
V, h, g, gbar over several steps), so the h' bulk stores, the carried head of
each batch window, the scalar quads shared by neighbour rows, the rotated reads
and the O6 chain are all checked.
"""
import numpy as np
import pytest

from synth import Block

from test_gpu_parity import run_parity, _random_case  # noqa: F401  (module fixture _built runs on import use)
from test_gpu_parity import _built  # noqa: F401

pytestmark = pytest.mark.gpu


def _layout(shapes):
    blocks, off = [], 0
    for m, n, K, ragged in shapes:
        ln = m * n - ragged
        blocks.append(Block(off, ln, m, n, K, 0))
        off += ln
    return off, blocks


LAYOUTS = {
    # unaligned rows of every start offset mod 4, a ragged last row, a row shorter than a quad
    "unaligned_small": [(3, 5, 2, 0), (41, 7, 5, 3), (17, 127, 4, 0), (9, 2051, 3, 1000), (5, 6, 5, 4)],
    # the LLaMA down-projection row length, one batch window per 256 columns: 22 windows per row
    "n5461": [(1, 1, 1, 0), (33, 5461, 4, 0), (2, 3, 1, 0)],
    # aligned and unaligned wide rows next to an aligned narrow block; the buffer ends at d % 4 = 3
    "mixed_wide": [(40, 4100, 5, 0), (20, 1000, 3, 0), (9, 7777, 2, 0), (6, 4100, 2, 57), (1, 6, 1, 3)],
    # rows that fit in one window (lo/hi of the first and last batch at once)
    "one_window": [(50, 255, 7, 0), (50, 257, 7, 0), (60, 129, 9, 100)],
}


@pytest.mark.parametrize("tma", ["1", "2"])
@pytest.mark.parametrize("name", sorted(LAYOUTS))
@pytest.mark.parametrize("N,r", [(1, 4), (3, 4), (2, 8)])
def test_tma_feed_layouts(orc, monkeypatch, tma, name, N, r):
    monkeypatch.setenv("ARC_SKETCH_TMA", tma)
    d, blocks = _layout(LAYOUTS[name])
    run_parity(orc, d, blocks, N=N, steps=3, r=r)


@pytest.mark.parametrize("reduce", ["nccl", "ordered"])
def test_tma_feed_exchange_path(orc, monkeypatch, reduce):
    """Mode 1 (per-node sketches exported for the exchange) through the same launch."""
    monkeypatch.setenv("ARC_SKETCH_TMA", "2")
    d, blocks = _layout(LAYOUTS["mixed_wide"])
    run_parity(orc, d, blocks, N=2, steps=3, force_exchange=True, reduce=reduce)


@pytest.mark.parametrize("tma", ["0", "2"])
@pytest.mark.parametrize("case", range(8))
def test_tma_feed_randomized(orc, monkeypatch, tma, case):
    """The randomized layouts of test_gpu_parity with the launch forced on / off."""
    monkeypatch.setenv("ARC_SKETCH_TMA", tma)
    rng = np.random.default_rng(5000 + case)
    d, blocks = _random_case(rng)
    N = int(rng.integers(1, 5))
    r = int(rng.choice([1, 2, 4, 5, 8, 16]))
    eta = float(rng.choice([1.0, 0.5, 0.1, 0.01]))
    run_parity(orc, d, blocks, N=N, steps=2, eta=eta, r=r, seed=case, method="arc")


def test_tma_feed_exact_and_bf16(orc, monkeypatch):
    """The exact-sketch mode and the bf16 value wire over blocks of the TMA launch."""
    monkeypatch.setenv("ARC_SKETCH_TMA", "2")
    d, blocks = _layout(LAYOUTS["unaligned_small"])
    run_parity(orc, d, blocks, N=3, steps=3, method="exact")
    run_parity(orc, d, blocks, N=2, steps=3, wire="bf16")


def test_tma_kernels_per_step(monkeypatch):
    """The layout with unaligned rows launches the third sketch kernel (counted)."""
    import torch
    from paper_2510_26709_b200 import ArcTopK
    d, blocks = _layout(LAYOUTS["mixed_wide"])
    monkeypatch.setenv("ARC_SKETCH_TMA", "0")
    c0 = ArcTopK(d, blocks, N=1, eta=0.1, r=4, device=torch.device("cuda", 0))
    monkeypatch.setenv("ARC_SKETCH_TMA", "1")
    c1 = ArcTopK(d, blocks, N=1, eta=0.1, r=4, device=torch.device("cuda", 0))
    assert c1.kernels_per_step == c0.kernels_per_step + 1   # main + ranged + TMA vs main + ranged
    c0.close()
    c1.close()
