"""GPU parity of the selection kernel's two launch forms (arc_select.cu).

A selection of at most 16 slices runs as ONE thread-block cluster (hardware
cluster barriers, ordinary launch); larger ones as a cooperative grid (grid
barriers through global memory).  ARC_SELECT_CLUSTER (read at create) sets the
largest cluster, 0 forces the cooperative form.  Both must give the oracle's
result bit for bit: selection, values, h, g, gbar, over several steps, on the
early-gather path (no values requested) and the segment path (values
requested on alternate steps), with ties and several blocks.
"""
import pytest

from synth import ADVERSARIAL, Block  # noqa: F401

from test_gpu_parity import run_parity, _built  # noqa: F401

pytestmark = pytest.mark.gpu


def _layout(shapes):
    blocks, off = [], 0
    for m, n, K, kind in shapes:
        blocks.append(Block(off, m * n, m, n, K, kind))
        off += m * n
    return off, blocks


LAYOUTS = {
    "one_slice": [(200, 64, 7, 0)],
    "four_slices": [(977, 1024, 10, 0)],                       # C5 d = 1e6 shape
    "sixteen_slices": [(4096, 16, 41, 0)],                     # exactly 16 slices of 256 rows
    "blocks_and_dense": [(300, 33, 9, 0), (40, 100, 40, 1), (700, 8, 3, 0), (513, 5, 512, 0)],
    "seventeen_slices": [(4097, 16, 50, 0)],                   # one more: cooperative either way
}


@pytest.mark.parametrize("cluster", ["0", "16", "4"])
@pytest.mark.parametrize("name", sorted(LAYOUTS))
@pytest.mark.parametrize("N", [1, 3])
def test_selection_launch_forms(orc, monkeypatch, cluster, name, N):
    monkeypatch.setenv("ARC_SELECT_CLUSTER", cluster)
    d, blocks = _layout(LAYOUTS[name])
    run_parity(orc, d, blocks, N=N, steps=4)


@pytest.mark.parametrize("cluster", ["0", "16"])
@pytest.mark.parametrize("kind", ["dup_rows", "zeros", "nonfinite"])
def test_selection_launch_forms_ties(orc, monkeypatch, cluster, kind):
    """Massive ties (the candidate list overflows: digit-by-digit path) in both forms."""
    from synth import adversarial
    monkeypatch.setenv("ARC_SELECT_CLUSTER", cluster)
    d, blocks = _layout([(2000, 32, 300, 0)])
    run_parity(orc, d, blocks, N=2, steps=3,
               grads_fn=lambda t: adversarial(kind, d, 2, seed=t, n=32))


@pytest.mark.parametrize("reduce", ["nccl", "ordered"])
def test_selection_cluster_form_exchange_path(orc, monkeypatch, reduce):
    """Phase 0 (the kernel builds the digit-1 histogram from the exchanged Sigma) in the cluster form."""
    monkeypatch.setenv("ARC_SELECT_CLUSTER", "16")
    d, blocks = _layout(LAYOUTS["blocks_and_dense"])
    run_parity(orc, d, blocks, N=2, steps=3, force_exchange=True, reduce=reduce)
