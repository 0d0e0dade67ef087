"""GPU parity of the fused small-problem tail (arc_sketch.cu).

With one node on the GPU, no exchange and a small selection (every ARC block
of at most 8,192 rows, at most 8 ARC blocks, r <= 8), the LAST CTA of the
streaming launch runs S3 itself (a done counter, no grid barrier, no selection
kernel) and a small kernel launched behind it runs S4..S6.  ARC_TAIL (read at create) = 0 forces the selection
kernel.  Both must give the oracle's result bit for bit: selection, values,
h, g, gbar, V and Sigma over several steps (values requested on alternate
steps), with ties, K = m blocks, DENSE blocks, ragged rows, the Rand-K and
without-EF methods and the bf16 wire; at and just past the size limits.
"""
import numpy as np
import pytest
import torch

from synth import Block, adversarial

from test_gpu_parity import DEV, run_parity, _built  # noqa: F401

pytestmark = pytest.mark.gpu


def _layout(shapes):
    blocks, off = [], 0
    for m, n, K, kind in shapes:
        blocks.append(Block(off, m * n, m, n, K, kind))
        off += m * n
    return off, blocks


LAYOUTS = {
    "c5_1e6": [(977, 1024, 10, 0)],                              # C5 d = 1e6 shape (shape-2 launch)
    "c3_rows": [(131, 768, 13, 0)],                              # n = 768 (shape-0 launch)
    "c2_one_node": [(22831, 512, 229, 0)],                       # C2 with one node: selection kernel
    "one_row": [(1, 64, 1, 0)],
    "k_eq_m": [(64, 16, 64, 0)],                                 # identity block
    "blocks_and_dense": [(300, 33, 9, 0), (40, 100, 40, 1), (700, 8, 3, 0), (513, 5, 512, 0)],
    "eight_blocks": [(100 + 37 * i, 16 + 8 * i, 3 + i, 0) for i in range(8)],
    "nine_blocks": [(50 + 11 * i, 8, 2 + i, 0) for i in range(9)],   # one block too many: selection kernel
    "max_rows": [(8192, 16, 1024, 0)],                           # the largest block at the key limit (32 KB)
    "past_rows": [(8193, 8, 100, 0)],                            # one row more: selection kernel
    "crowded_bin": [(8000, 8, 4000, 0)],                         # K = m / 2: a crowded boundary bin
    "big_kn": [(600, 64, 513, 0)],                               # many selected rows (the update kernel)
    "unaligned_base": [(37, 12, 5, 0), (301, 20, 30, 0)],        # second block's Sigma not 16-byte aligned
    # blocks streamed by the other launches -- the TMA-fed launch (unaligned rows, n >= 256),
    # the ranged launch (V_b^T wider than the stage; n <= 4) -- take the selection kernel
    # (a tail behind those launches measured no faster on C4's DDP buckets: profiles/r02_tail.txt)
    "with_tma": [(300, 64, 9, 0), (200, 301, 5, 0)],               # n = 301: rows not 16-byte aligned
    "with_wide": [(300, 64, 9, 0), (40, 4100, 3, 0)],
    "with_n1": [(300, 64, 9, 0), (5000, 1, 50, 0)],
    "llama_bucket": [(5461, 2048, 6, 0), (2048, 5461, 3, 0), (2048, 2048, 3, 0)],   # a C4 DDP bucket
    "only_wide": [(40, 4100, 3, 0)],                             # no main-launch tile: selection kernel
}
TAILED = {"c5_1e6", "c3_rows", "crowded_bin", "one_row", "k_eq_m", "blocks_and_dense", "eight_blocks", "max_rows",
          "big_kn", "unaligned_base"}


def _plan(d, blocks):
    """ARC_Q_PLAN: [selection form (2 = the fused tail), selection CTAs, S1 launches, kernels per step]."""
    from paper_2510_26709_b200 import ArcTopK, _lib
    ctx = ArcTopK(d, blocks, N=1, eta=0.1, r=4, seed=5, nodes_local=1)
    plan = ctx.query(_lib.Q_PLAN).cpu().tolist()
    ctx.close()
    return plan


@pytest.mark.parametrize("name", sorted(LAYOUTS))
@pytest.mark.parametrize("tail", ["1", "0"])
def test_tail_parity(orc, monkeypatch, name, tail):
    monkeypatch.setenv("ARC_TAIL", tail)
    d, blocks = _layout(LAYOUTS[name])
    run_parity(orc, d, blocks, N=1, steps=5)


def test_tail_is_taken_exactly_where_eligible(monkeypatch):
    """ARC_TAIL=1 takes the tail exactly on the eligible layouts; ARC_TAIL=0 never.  The tail's
    step is the streaming launch + the update kernel (the same count as with the selection kernel)."""
    for name, shapes in LAYOUTS.items():
        d, blocks = _layout(shapes)
        monkeypatch.setenv("ARC_TAIL", "1")
        on = _plan(d, blocks)
        monkeypatch.setenv("ARC_TAIL", "0")
        off = _plan(d, blocks)
        assert (on[0] == 2) == (name in TAILED), (name, on)
        assert off[0] in (0, 1), (name, off)
        assert on[3] == off[3], (name, on, off)
        if name in TAILED:
            assert on[1] == 1 and on[2] == 1, (name, on)


@pytest.mark.parametrize("kind", ["dup_rows", "zeros", "nonfinite", "huge", "small_int", "subnormal"])
def test_tail_ties_and_nonfinite(orc, monkeypatch, kind):
    monkeypatch.setenv("ARC_TAIL", "1")
    d, blocks = _layout([(2000, 32, 300, 0)])
    run_parity(orc, d, blocks, N=1, steps=3, grads_fn=lambda t: adversarial(kind, d, 1, seed=t, n=32))


@pytest.mark.parametrize("method", ["randk", "noef_msgd"])
@pytest.mark.parametrize("name", ["c5_1e6", "blocks_and_dense"])
def test_tail_methods(orc, monkeypatch, method, name):
    monkeypatch.setenv("ARC_TAIL", "1")
    d, blocks = _layout(LAYOUTS[name])
    run_parity(orc, d, blocks, N=1, steps=4, method=method, check_debug=False)


@pytest.mark.parametrize("name", ["c5_1e6", "blocks_and_dense"])
def test_tail_bf16_wire(orc, monkeypatch, name):
    monkeypatch.setenv("ARC_TAIL", "1")
    d, blocks = _layout(LAYOUTS[name])
    run_parity(orc, d, blocks, N=1, steps=4, wire="bf16")


def test_tail_non_consecutive_t(orc, monkeypatch):
    """The speculative V of t + 1 drawn by the streaming launch is used only when the next t matches."""
    monkeypatch.setenv("ARC_TAIL", "1")
    d, blocks = _layout(LAYOUTS["c5_1e6"])
    run_parity(orc, d, blocks, N=1, ts=[0, 1, 2, 5, 6, 9, 3])


@pytest.mark.parametrize("r", [1, 3, 8])
def test_tail_sketch_widths(orc, monkeypatch, r):
    monkeypatch.setenv("ARC_TAIL", "1")
    d, blocks = _layout(LAYOUTS["blocks_and_dense"])
    run_parity(orc, d, blocks, N=1, steps=3, r=r)


def test_tail_graph_replays(orc, monkeypatch):
    """A captured step (device iteration counter) replayed at t = 0, 1, 2, 7, 8, 3, 4 equals
    the oracle's steps: the done counter returns to zero, t advances inside the tail, and
    the V drawn ahead by k_tail_update for the next t is used only when the counter matches."""
    from paper_2510_26709_b200 import ArcTopK
    from synth import GradientSource
    monkeypatch.setenv("ARC_TAIL", "1")
    d, blocks = _layout(LAYOUTS["c5_1e6"])
    src = GradientSource(d, blocks, 1, seed=9)
    ctx = ArcTopK(d, blocks, N=1, eta=0.1, r=4, seed=9, nodes_local=1, device_t=True)
    o = orc.OracleEF21M(d, blocks, N=1, eta=0.1, r=4, seed=9)
    h, g, gbar = (torch.zeros(d, device=DEV) for _ in range(3))
    grad = torch.zeros(d, device=DEV)
    sel = torch.empty(ctx.sum_K, dtype=torch.int32, device=DEV)
    graph = ctx.capture([grad], [h], [g], gbar, sel, None)
    ts = [0, 1, 2, 7, 8, 3, 4]   # jumps: the V drawn for the counter's next t is reused only when it matches
    for k, t in enumerate(ts):
        if k == 0 or t != ts[k - 1] + 1:
            ctx.set_iteration(t)
        gr = src.grads(t)[0]
        grad.copy_(gr.to(DEV))
        graph.replay()
        ref = o.step(t, [gr.numpy()])
        torch.cuda.synchronize()
        assert np.array_equal(sel.cpu().numpy(), ref["sel"]), t
    assert h.cpu().numpy().tobytes() == o.h[0].tobytes()
    assert g.cpu().numpy().tobytes() == o.g[0].tobytes()
    assert gbar.cpu().numpy().tobytes() == o.gbar.tobytes()
    ctx.close()
