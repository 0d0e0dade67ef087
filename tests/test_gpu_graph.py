"""GPU parity of ARC_FLAG_DEVICE_T: one step captured into a CUDA graph and
replayed is the step at t, t + 1, ... (the device iteration counter advances
with every replay), bit-exact against the oracle run eagerly at consecutive t
— V (ARC) and the Rand-K keys depend on t, so a replay at a stale t would
differ.  set_iteration moves the counter (also between replays)."""
import numpy as np
import pytest
import torch

from synth import Block, GradientSource

from test_gpu_parity import _built, assert_same_floats  # noqa: F401

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _layout():
    shapes = [(300, 96, 7, 0), (50, 20, 50, 1), (123, 517, 9, 0), (400, 3, 11, 0)]
    blocks, off = [], 0
    for m, n, K, kind in shapes:
        blocks.append(Block(off, m * n - (n // 2 if kind == 0 and n > 4 else 0), m, n, K, kind))
        off += blocks[-1].len
    return off, blocks


@pytest.mark.parametrize("method", ["arc", "randk", "noef_msgd"])
@pytest.mark.parametrize("N", [1, 3])
def test_replayed_graph_follows_consecutive_iterations(orc, method, N):
    from paper_2510_26709_b200 import ArcTopK
    d, blocks = _layout()
    eta = 0.5 if method == "noef_msgd" else 0.1
    src = GradientSource(d, blocks, N, seed=9)
    ctx = ArcTopK(d, blocks, N=N, eta=eta, r=4, seed=9, method=method, device_t=True)
    o = orc.OracleEF21M(d, blocks, N=N, eta=eta, r=4, seed=9, method=method)
    noef = method == "noef_msgd"
    grads = [torch.zeros(d, device=DEV) for _ in range(N)]
    h = None if noef else [torch.zeros(d, device=DEV) for _ in range(N)]
    g = None if noef else [torch.zeros(d, device=DEV) for _ in range(N)]
    gbar = torch.zeros(d, device=DEV)
    sel = torch.empty(ctx.sum_K, dtype=torch.int32, device=DEV)
    vals = torch.empty(ctx.sum_Kn, dtype=torch.float32, device=DEV)
    stream = torch.cuda.Stream()
    graph = ctx.capture(grads, h, g, gbar, sel, vals, stream=stream)
    ts = [3, 4, 5, 6, 40, 41, 42]          # set_iteration jumps to 40 after four replays
    for k, t in enumerate(ts):
        if k == 0 or t != ts[k - 1] + 1:
            ctx.set_iteration(t, stream=stream)
        gr = [x.numpy() for x in src.grads(t)]
        with torch.cuda.stream(stream):
            for i in range(N):
                grads[i].copy_(torch.from_numpy(gr[i]), non_blocking=False)
            graph.replay()
        ref = o.step(t, gr)
        torch.cuda.synchronize()
        assert np.array_equal(sel.cpu().numpy(), ref["sel"]), f"selection differs at t={t}"
        assert_same_floats(vals.cpu().numpy(), ref["values"], f"values (t={t})")
    if not noef:
        for i in range(N):
            assert_same_floats(h[i].cpu().numpy(), o.h[i], f"h[{i}]")
            assert_same_floats(g[i].cpu().numpy(), o.g[i], f"g[{i}]")
    assert_same_floats(gbar.cpu().numpy(), o.gbar, "gbar")
    ctx.close()


def test_device_t_eager_steps_ignore_the_argument(orc):
    """Eager steps of a device_t context use the counter (the t argument is ignored)."""
    from paper_2510_26709_b200 import ArcTopK
    d, blocks = _layout()
    src = GradientSource(d, blocks, 2, seed=4)
    ctx = ArcTopK(d, blocks, N=2, eta=0.1, r=4, seed=4, device_t=True)
    o = orc.OracleEF21M(d, blocks, N=2, eta=0.1, r=4, seed=4)
    h = [torch.zeros(d, device=DEV) for _ in range(2)]
    g = [torch.zeros(d, device=DEV) for _ in range(2)]
    gbar = torch.zeros(d, device=DEV)
    sel = torch.empty(ctx.sum_K, dtype=torch.int32, device=DEV)
    ctx.set_iteration(7)
    for t in (7, 8, 9):
        gr = [x.numpy() for x in src.grads(t)]
        ctx.step(12345, [torch.from_numpy(x).to(DEV) for x in gr], h, g, gbar, sel)
        ref = o.step(t, gr)
        torch.cuda.synchronize()
        assert np.array_equal(sel.cpu().numpy(), ref["sel"]), f"selection differs at t={t}"
    assert_same_floats(gbar.cpu().numpy(), o.gbar, "gbar")
    ctx.close()


def test_set_iteration_needs_the_flag():
    from paper_2510_26709_b200 import ArcTopK
    from paper_2510_26709_b200._lib import ArcError
    d, blocks = _layout()
    ctx = ArcTopK(d, blocks, N=1, eta=0.1, r=4)
    with pytest.raises(ArcError):
        ctx.set_iteration(3)
    with pytest.raises(ValueError):
        ctx.capture([torch.zeros(d, device=DEV)], [torch.zeros(d, device=DEV)], [torch.zeros(d, device=DEV)],
                    torch.zeros(d, device=DEV))
    ctx.close()
