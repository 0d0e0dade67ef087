"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.

With every node on one GPU (G = 1) the whole step follows the fixed order of
DESIGN.md R9 on both sides, so EVERYTHING is compared bit for bit: the
selection I, the compact values C, and the state h, g, gbar — over several
steps, so state feedback is covered too.
"""
import numpy as np
import pytest
import torch

from synth import ADVERSARIAL, Block, GradientSource, adversarial, config_blocks, flat_blocks

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__ as ge
    ge.build()
    torch.cuda.set_device(0)


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def assert_same_floats(gpu: np.ndarray, ref: np.ndarray, what: str):
    """Bit-identical, except that any two NaNs match (payloads are not specified)."""
    g, r = _bits(gpu.astype(np.float32)), _bits(ref.astype(np.float32))
    gn, rn = np.isnan(gpu), np.isnan(ref)
    assert np.array_equal(gn, rn), f"{what}: NaN positions differ"
    diff = (g != r) & ~gn
    if diff.any():
        i = int(np.flatnonzero(diff)[0])
        raise AssertionError(f"{what}: {int(diff.sum())} of {diff.size} differ; first at {i}: "
                             f"gpu={gpu.ravel()[i]!r} oracle={ref.ravel()[i]!r}")


def run_parity(orc, d, blocks, N, steps=3, eta=0.1, r=4, seed=5, grads_fn=None, reduce="nccl",
               force_exchange=False, check_debug=True, host=False, nodes_local=None, pg=None, ts=None,
               method="arc", wire="f32"):
    from paper_2510_26709_b200 import ArcTopK
    nl = N if nodes_local is None else nodes_local
    assert nl == N, "single-GPU parity: all nodes local"
    src = GradientSource(d, blocks, N, seed=seed) if grads_fn is None else None
    ctx = ArcTopK(d, blocks, N=N, eta=eta, r=r, seed=seed, nodes_local=nl, reduce=reduce,
                  debug_sketch=check_debug, force_exchange=force_exchange, host_staging=host, pg=pg,
                  method=method, wire=wire)
    o = orc.OracleEF21M(d, blocks, N=N, eta=eta, r=r, seed=seed, method="arc" if method == "exact" else method,
                        exact=method == "exact", wire=wire)
    noef = method == "noef_msgd"      # no (h, g) state: gbar is the momentum u
    h = [torch.zeros(d, device=DEV) for _ in range(N)]
    g = [torch.zeros(d, device=DEV) for _ in range(N)]
    gbar = torch.zeros(d, device=DEV)
    for t in (range(steps) if ts is None else ts):
        gr = [x.numpy() for x in src.grads(t)] if grads_fn is None else grads_fn(t)
        gr = [np.ascontiguousarray(x, dtype=np.float32) for x in gr]
        if host:
            gh = [torch.from_numpy(x).pin_memory() for x in gr]
            sel = torch.empty(ctx.sum_K, dtype=torch.int32).pin_memory()
            vals = torch.empty(ctx.sum_Kn, dtype=torch.float32).pin_memory()
            ctx.step_host(t, gh, None if noef else h, None if noef else g, gbar, sel, vals)
        else:
            # values are requested on every other step: without them the select
            # kernel takes its early-gather path (mode 0), with them the segment path
            sel = torch.empty(ctx.sum_K, dtype=torch.int32, device=DEV)
            vals = torch.empty(ctx.sum_Kn, dtype=torch.float32, device=DEV) if t % 2 else None
            ctx.step(t, [torch.from_numpy(x).to(DEV) for x in gr], None if noef else h, None if noef else g, gbar,
                     sel, vals)
        ref = o.step(t, gr, debug=check_debug)
        torch.cuda.synchronize()
        if check_debug and method == "arc":
            # the library keeps V_b transposed ([r][n_b], ARC_Q_V); the oracle row-major
            # (rows padded to ldv = round_up(n, 4); the padding is not compared)
            got, goff, off = ctx.query(0).cpu().numpy(), 0, 0
            for b in blocks:
                if b.kind == 0:
                    ldv = -(-b.n // 4) * 4
                    gb_ = got[goff:goff + r * ldv].reshape(r, ldv)[:, :b.n]
                    assert_same_floats(gb_, ref["V"][off:off + b.n * r].reshape(b.n, r).T, f"V (t={t})")
                    off += b.n * r
                    goff += r * ldv
        if check_debug:
            assert_same_floats(ctx.query(1).cpu().numpy(), ref["sigma"], f"Sigma (t={t})")
        assert np.array_equal(sel.cpu().numpy(), ref["sel"]), f"selection differs at t={t}"
        if vals is not None:
            assert_same_floats(vals.cpu().numpy(), ref["values"], f"values (t={t})")
    for i in range(N):
        assert_same_floats(h[i].cpu().numpy(), o.h[i], f"h[{i}]")
        assert_same_floats(g[i].cpu().numpy(), o.g[i], f"g[{i}]")
    assert_same_floats(gbar.cpu().numpy(), o.gbar, "gbar")
    st = ctx.status()
    ctx.close()
    return st


# ------------------------------------------------------------------ configs[0] (C1)

def test_c1_config0_bit_exact(orc):
    """BASELINE configs[0]: N = 4 simulated nodes, d = 65,536, K = 1 % (656) -> n = 1 (R6),
    20 steps (state feedback), everything bit-exact."""
    d, blocks = config_blocks("C1")
    assert blocks[0].K == 656
    run_parity(orc, d, blocks, N=4, steps=20, seed=20251030)


@pytest.mark.parametrize("n,K", [(128, 6), (256, 3)])
def test_c1_row_variants(orc, n, K):
    run_parity(orc, 65_536, flat_blocks(65_536, n, K=K), N=4, steps=5)


# ------------------------------------------------------------------ shapes, tails, r

@pytest.mark.parametrize("d,n,K", [
    (100_003, 768, 13),      # ragged last row (R14), several tiles
    (4_097, 3, 100),         # n % 4 != 0: scalar path, odd rows
    (5_461 * 70 + 11, 5_461, 7),   # LLaMA down-proj row length, unaligned rows
    (33, 33, 1),             # single row
    (1_000, 1, 1000),        # K = m (identity)
    (50_000, 40, 1),         # K = 1
    (64 * 129, 64, 64),      # exactly two tile heights
])
def test_shapes(orc, d, n, K):
    run_parity(orc, d, flat_blocks(d, n, K=K), N=2, steps=3)


@pytest.mark.parametrize("r", [1, 3, 4, 5, 8, 16, 32])
def test_sketch_widths(orc, r):
    run_parity(orc, 20_000, flat_blocks(20_000, 100, K=9), N=3, steps=2, r=r)


@pytest.mark.parametrize("eta", [1.0, 0.5, 1e-3])
def test_eta(orc, eta):
    run_parity(orc, 30_000, flat_blocks(30_000, 64, K=20), N=2, steps=3, eta=eta)


@pytest.mark.parametrize("N", [1, 2, 3, 8, 16])
def test_node_counts(orc, N):
    run_parity(orc, 12_345, flat_blocks(12_345, 50, K=11), N=N, steps=2)


# ------------------------------------------------------------------ adversarial sets

@pytest.mark.parametrize("kind", ADVERSARIAL)
@pytest.mark.parametrize("n", [1, 7, 64])
def test_adversarial(orc, kind, n):
    d, N = 9_000, 4
    blocks = flat_blocks(d, n, K=max(1, (d // n) // 10))
    fixed = adversarial(kind, d, N, n=n)
    st = run_parity(orc, d, blocks, N=N, steps=2, grads_fn=lambda t: fixed)
    if kind in ("nonfinite",):
        assert st & 1, "non-finite Sigma must raise the status flag"


def test_multi_block_with_dense(orc):
    """Per-tensor blocks with different n, aligned and unaligned, plus
    a DENSE block (R20)."""
    shapes = [(300, 128, 5, 0), (77, 5461 // 43, 3, 0), (64, 64, 64, 0), (1, 1000, 1, 0),
              (1000, 3, 17, 0), (13, 100, 13, 1), (129, 2048, 2, 0)]
    blocks, off = [], 0
    for m, n, K, kind in shapes:
        blocks.append(Block(off, m * n, m, n, K, kind))
        off += m * n
    run_parity(orc, off, blocks, N=3, steps=3)
    # the exchange path: DENSE rows through the streaming kernels and the payload
    run_parity(orc, off, blocks, N=3, steps=3, force_exchange=True, reduce="nccl")
    run_parity(orc, off, blocks, N=3, steps=3, force_exchange=True, reduce="ordered")


def test_llama_layout_small_mu(orc):
    """The C4 layout scaled down: one of each LLaMA tensor shape."""
    shapes = [(2048, 64), (5461, 64), (2048, 5461 // 64)]
    blocks, off = [], 0
    for m, n in shapes:
        blocks.append(Block(off, m * n, m, n, max(1, m // 100), 0))
        off += m * n
    blocks.append(Block(off, 4096, 4, 1024, 4, 1))
    off += 4096
    run_parity(orc, off, blocks, N=2, steps=2)


# ------------------------------------------------------------------ exchange path on 1 GPU

@pytest.mark.parametrize("reduce", ["nccl", "ordered"])
def test_exchange_kernels_single_gpu(orc, reduce):
    """The G > 1 kernel sequence (per-node sketch export, ordered node-sum reduce,
    wire gather, scatter) run with G = 1 (copies instead of NCCL): bit-exact."""
    run_parity(orc, 50_000, flat_blocks(50_000, 96, K=40), N=4, steps=3, reduce=reduce, force_exchange=True)


@pytest.mark.parametrize("wire", ["f32", "bf16"])
@pytest.mark.parametrize("reduce", ["nccl", "ordered", "lsa"])
def test_exchange_through_nccl_one_rank(orc, reduce, wire):
    """The exchange path with a real NCCL communicator borrowed from a 1-rank torch
    ProcessGroupNCCL (dlopen'd libnccl, ncclAllGather of the per-node sketches and
    of the ordered wire): bit-exact against the oracle."""
    import os
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        # (NCCL reduce + bf16 wire rounds the local pre-sum of several nodes to bf16 —
        # within the R25 tolerance, tested across emulated ranks in test_gpu_loopback.py;
        # with one node per rank the payload is each node's own bf16 rows: bit-exact)
        N = 1 if (reduce == "nccl" and wire == "bf16") else 2
        run_parity(orc, 30_000, flat_blocks(30_000, 128, K=21), N=N, steps=3, reduce=reduce, force_exchange=True,
                   pg=dist.group.WORLD, wire=wire)
    finally:
        pass


def _world_pg():
    import os
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    return dist.group.WORLD


@pytest.mark.parametrize("method", ["arc", "randk", "noef_msgd"])
def test_lsa_fused_scatter_multiblock(orc, method):
    """reduce="lsa" (exchange #2 fused with S6 over an NCCL symmetric window, LSA
    barriers, peer loads) through a real 1-rank communicator:
    per-tensor ARC blocks (aligned, unaligned, wide enough for the ranged launch), a
    DENSE block, several local nodes — gbar, g, h, selection and values bit-exact
    against the oracle, like the ORDERED mode it replaces."""
    pg = _world_pg()
    shapes = [(300, 128, 5, 0), (77, 127, 3, 0), (64, 64, 64, 0), (1000, 3, 17, 0), (13, 100, 13, 1),
              (9, 7777, 2, 0), (129, 2048, 2, 0)]
    blocks, off = [], 0
    for m, n, K, kind in shapes:
        blocks.append(Block(off, m * n, m, n, K, kind))
        off += m * n
    eta = 0.5 if method == "noef_msgd" else 0.1
    for N in (1, 3, 4):
        run_parity(orc, off, blocks, N=N, steps=3, eta=eta, method=method, force_exchange=True, reduce="lsa", pg=pg)


def test_lsa_flat_many_steps(orc):
    """The window and the LSA barrier epochs are reused step after step (the
    barrier that ends each scatter guards the next step's payload writes)."""
    pg = _world_pg()
    run_parity(orc, 200_000, flat_blocks(200_000, 768, K=3), N=2, steps=8, reduce="lsa", force_exchange=True, pg=pg)


def test_lsa_create_errors():
    """reduce="lsa" needs a communicator (INVALID_ARG without one) and is not offered
    for the All-Gather Top-K baseline (UNSUPPORTED); nothing is left allocated."""
    from paper_2510_26709_b200 import ArcTopK
    pg = _world_pg()
    blocks = flat_blocks(4096, 64, K=4)
    with pytest.raises(RuntimeError):
        ArcTopK(4096, blocks, N=2, eta=0.1, nodes_local=2, reduce="lsa", force_exchange=True, device=DEV)
    with pytest.raises(RuntimeError):
        ArcTopK(4096, blocks, N=2, eta=0.1, nodes_local=2, reduce="lsa", force_exchange=True, method="topk_allgather",
                pg=pg, device=DEV)


def test_nonconsecutive_steps(orc):
    """V for step t+1 is generated speculatively during step t; a caller that skips
    or repeats iteration numbers must still get V(seed, t) (R7)."""
    run_parity(orc, 30_000, flat_blocks(30_000, 96, K=15), N=2, ts=[0, 1, 5, 6, 6, 2, 3, 1 << 33, (1 << 33) + 1])


def test_host_staging_entry(orc):
    """arc_topk_step_host: gradients from pinned host memory, results copied back."""
    run_parity(orc, 40_000, flat_blocks(40_000, 80, K=25), N=2, steps=3, host=True, check_debug=False)


def test_determinism_and_graph_capture(orc):
    """Two runs give byte-identical state; the step can be captured in a CUDA graph
    and replayed with the same result."""
    from paper_2510_26709_b200 import ArcTopK
    d, N = 200_000, 2
    blocks = flat_blocks(d, 500, K=4)
    src = GradientSource(d, blocks, N, seed=3)
    grads = [x.to(DEV) for x in src.grads(0)]
    outs = []
    for mode in ("eager", "eager", "graph"):
        ctx = ArcTopK(d, blocks, N=N, eta=0.1, seed=3)
        h = [torch.zeros(d, device=DEV) for _ in range(N)]
        g = [torch.zeros(d, device=DEV) for _ in range(N)]
        gbar = torch.zeros(d, device=DEV)
        if mode == "graph":
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(graph, stream=s):
                    ctx.step(0, grads, h, g, gbar, stream=s)
            # capture does not execute: replay once
            graph.replay()
            torch.cuda.synchronize()
        else:
            ctx.step(0, grads, h, g, gbar)
        torch.cuda.synchronize()
        outs.append(gbar.cpu().numpy().tobytes() + b"".join(x.cpu().numpy().tobytes() for x in g))
        ctx.close()
    assert outs[0] == outs[1] == outs[2]


@pytest.mark.parametrize("kind", ["normal", "dup_rows"])
def test_graph_replayed_three_times_equals_three_eager_steps(kind):
    """A captured step replayed 3x gives exactly what 3 eager steps at the same t give
    (the selection's double-buffered candidate / boundary counters are switched by a
    device-side parity word, so replays of one graph never reuse a stale counter).
    dup_rows (every Sigma equal) overflows the candidate list: the boundary-row path."""
    from paper_2510_26709_b200 import ArcTopK
    from synth import adversarial
    d, N, n = 600_000, 2, 100
    blocks = flat_blocks(d, n, K=900)
    grads = [torch.from_numpy(x).to(DEV) for x in adversarial(kind, d, N, seed=4, n=n)]
    outs = []
    for mode in ("eager", "graph"):
        ctx = ArcTopK(d, blocks, N=N, eta=0.5, seed=3)
        h = [torch.zeros(d, device=DEV) for _ in range(N)]
        g = [torch.zeros(d, device=DEV) for _ in range(N)]
        gbar = torch.zeros(d, device=DEV)
        sel = torch.empty(ctx.sum_K, dtype=torch.int32, device=DEV)
        sels = []
        if mode == "graph":
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(graph, stream=s):
                    ctx.step(7, grads, h, g, gbar, sel, stream=s)
            for _ in range(3):
                graph.replay()
                torch.cuda.synchronize()
                sels.append(sel.cpu().numpy().copy())
        else:
            for _ in range(3):
                ctx.step(7, grads, h, g, gbar, sel)
                torch.cuda.synchronize()
                sels.append(sel.cpu().numpy().copy())
        outs.append((sels, gbar.cpu().numpy().tobytes() + b"".join(x.cpu().numpy().tobytes() for x in g + h)))
        ctx.close()
    for a, b in zip(outs[0][0], outs[1][0]):
        assert np.array_equal(a, b)
        assert np.all(np.diff(a) > 0) and a.min() >= 0 and a.max() < blocks[0].m
    assert outs[0][1] == outs[1][1]


# ------------------------------------------------------------------ bfloat16 value wire (R25)

@pytest.mark.parametrize("method", ["arc", "randk", "noef_msgd", "exact"])
@pytest.mark.parametrize("N", [1, 3])
def test_bf16_wire(orc, method, N):
    """The bf16 value wire (R25) with every node on one GPU: each sent entry
    rounded at the source, EF keeps the rest — bit-exact against the oracle's
    wire="bf16" (selection, values, h, g, gbar), early-gather and segment steps,
    mixed ARC (ragged, unaligned, K = m) and DENSE blocks."""
    shapes = [(300, 96, 5, 0), (77, 127, 3, 0), (64, 64, 64, 0), (13, 100, 13, 1), (1000, 3, 17, 0)]
    blocks, off = [], 0
    for m, n, K, kind in shapes:
        blocks.append(Block(off, m * n - (n // 2 if kind == 0 and m > 1 else 0), m, n, K, kind))
        off += blocks[-1].len
    eta = 0.9 if method == "noef_msgd" else 0.1
    run_parity(orc, off, blocks, N=N, steps=4, method=method, wire="bf16", eta=eta, check_debug=method == "arc")


@pytest.mark.parametrize("reduce", ["nccl", "ordered"])
def test_bf16_wire_exchange_kernels(orc, reduce):
    """The G > 1 kernel sequence on one GPU (no comm: collectives are copies) with
    bf16 payloads: k_dense payload, the gather's bf16 stores, k_scatter's reads."""
    shapes = [(300, 96, 5, 0), (13, 100, 13, 1), (1000, 3, 17, 0)]
    blocks, off = [], 0
    for m, n, K, kind in shapes:
        blocks.append(Block(off, m * n, m, n, K, kind))
        off += m * n
    # (NCCL + bf16 with several local nodes rounds their pre-sum: tolerance, test_gpu_loopback.py)
    run_parity(orc, off, blocks, N=3 if reduce == "ordered" else 1, steps=3, force_exchange=True, reduce=reduce,
               wire="bf16")


def test_bf16_wire_full_size_c3(orc):
    d, blocks = config_blocks("C3")
    run_parity(orc, d, blocks, N=1, steps=2, seed=20251030, wire="bf16", check_debug=False)


def test_query_node_sum_S(orc):
    """ARC_Q_S: S = P'_0 + P'_1 + ... (node order) equals the sum of the queried
    per-node sketches; Sigma = fma chain of S_j^2 (O8) equals the queried Sigma."""
    from paper_2510_26709_b200 import ArcTopK
    from paper_2510_26709_b200 import _lib as L
    d, N = 30_000, 3
    blocks = flat_blocks(d, 100, K=9)
    src = GradientSource(d, blocks, N, seed=8)
    ctx = ArcTopK(d, blocks, N=N, eta=0.1, r=4, seed=8, debug_sketch=True)
    h = [torch.zeros(d, device=DEV) for _ in range(N)]
    g = [torch.zeros(d, device=DEV) for _ in range(N)]
    gbar = torch.zeros(d, device=DEV)
    ctx.step(0, [x.to(DEV) for x in src.grads(0)], h, g, gbar)
    S = ctx.query(L.Q_S).cpu().numpy().reshape(-1, 4)
    Pn = ctx.query(L.Q_P_NODES).cpu().numpy().reshape(-1, N, 4)
    want = Pn[:, 0, :].copy()
    for i in range(1, N):
        want = (want + Pn[:, i, :]).astype(np.float32)
    assert S.tobytes() == want.tobytes()
    sig = ctx.query(L.Q_SIGMA).cpu().numpy()
    assert sig.tobytes() == orc.sigma_rows(S).tobytes()
    ctx.close()


# ------------------------------------------------------------------ persistent selection (several slices per CTA)

@pytest.fixture
def select_grid(monkeypatch):
    """Force the selection kernel onto fewer CTAs than slices (ARC_SELECT_GRID,
    read at create): every CTA then takes several slices (the persistent path)."""
    def set_grid(grid, slice_rows=256):
        monkeypatch.setenv("ARC_SELECT_GRID", str(grid))
        monkeypatch.setenv("ARC_SLICE_ROWS", str(slice_rows))
    return set_grid


@pytest.mark.parametrize("grid", [2, 3, 7])
def test_persistent_selection_multiblock(orc, select_grid, grid):
    """Several slices per CTA: mixed ARC blocks (ragged, unaligned, K = m, K = 1)
    and a DENSE block, early-gather steps and segment-gather steps alternating."""
    select_grid(grid)
    shapes = [(3000, 16, 31, 0), (700, 5461 // 43, 3, 0), (64, 64, 64, 0), (1, 1000, 1, 0),
              (5000, 3, 170, 0), (13, 100, 13, 1), (1300, 20, 2, 0)]
    blocks, off = [], 0
    for m, n, K, kind in shapes:
        blocks.append(Block(off, m * n, m, n, K, kind))
        off += m * n
    run_parity(orc, off, blocks, N=1, steps=4)
    run_parity(orc, off, blocks, N=3, steps=3)                     # phase 0: Sigma from the node sketches
    run_parity(orc, off, blocks, N=2, steps=3, force_exchange=True, reduce="ordered")


@pytest.mark.parametrize("kind", ["dup_rows", "zeros", "nonfinite"])
def test_persistent_selection_ties_overflow(orc, select_grid, kind):
    """Massive ties overflow the candidate list: the digit-by-digit path with
    several slices per CTA (and the early boundary-row list)."""
    select_grid(5)
    d, N, n = 40_000, 2, 4
    blocks = flat_blocks(d, n, K=700)
    fixed = adversarial(kind, d, N, n=n)
    run_parity(orc, d, blocks, N=N, steps=2, grads_fn=lambda t: fixed)


def test_persistent_selection_topk_baseline(orc, select_grid):
    """The All-Gather Top-K baseline (a selection block per node) on 4 CTAs."""
    select_grid(4)
    test_topk_allgather_baseline(orc, 4, 60_000, 96, 12)


def test_llama7b_shaped_table_creates_and_matches(orc):
    """A LLaMA-7B-shaped per-tensor table (226 ARC blocks, 1.42M rows: 368 slices of
    <= 4096 rows, more than the 296 co-resident CTAs) is accepted by create and
    is bit-exact against the oracle (rows scaled down to keep the oracle fast)."""
    from synth import llama7b_scaled_blocks
    d, blocks = llama7b_scaled_blocks()
    assert sum(1 for b in blocks if b.kind == 0) == 226
    assert sum(-(-b.m // 4096) for b in blocks if b.kind == 0) == 368
    run_parity(orc, d, blocks, N=1, steps=2, check_debug=False)


# ------------------------------------------------------------------ full-size configs

@pytest.mark.parametrize("name,N,steps", [("C2", 8, 2), ("C3", 1, 2)])
def test_full_size_configs(orc, name, N, steps):
    """BASELINE configs[1] (ResNet-18 d = 11.7M, N = 8 simulated) and configs[2] (GPT-2
    small d = 124M, one node per GPU, the bench workload): the whole step bit-exact
    against the oracle at full size."""
    d, blocks = config_blocks(name)
    run_parity(orc, d, blocks, N=N, steps=steps, seed=20251030, check_debug=True)


# ------------------------------------------------------------------ All-Gather Top-K baseline

@pytest.mark.parametrize("N,d,n,K", [(1, 50_000, 100, 7), (4, 60_000, 96, 12), (3, 4_097, 3, 40)])
def test_topk_allgather_baseline(orc, N, d, n, K):
    """The baseline of Table I row "Top-K": per-node exact row-norm Top-K,
    g_i += C_i, gbar += C_j / N in node order — bit-exact against the oracle's
    orc_step_topk, with overlapping supports across nodes."""
    from paper_2510_26709_b200 import ArcTopK
    blocks = flat_blocks(d, n, K=K)
    src = GradientSource(d, blocks, N, seed=17)
    ctx = ArcTopK(d, blocks, N=N, eta=0.3, seed=17, nodes_local=N, method="topk_allgather")
    o = orc.OracleEF21M(d, blocks, N=N, eta=0.3, r=4, seed=17)
    h = [torch.zeros(d, device=DEV) for _ in range(N)]
    g = [torch.zeros(d, device=DEV) for _ in range(N)]
    gbar = torch.zeros(d, device=DEV)
    for t in range(4):
        gr = [x.numpy() for x in src.grads(t)]
        ctx.step(t, [torch.from_numpy(x).to(DEV) for x in gr], h, g, gbar)
        o.step_topk(t, gr)
    torch.cuda.synchronize()
    for i in range(N):
        assert_same_floats(h[i].cpu().numpy(), o.h[i], f"h[{i}]")
        assert_same_floats(g[i].cpu().numpy(), o.g[i], f"g[{i}]")
    assert_same_floats(gbar.cpu().numpy(), o.gbar, "gbar")
    ctx.close()


def test_topk_allgather_multiblock_dense(orc):
    from paper_2510_26709_b200 import ArcTopK
    shapes = [(300, 64, 5, 0), (13, 100, 13, 1), (77, 33, 4, 0)]
    blocks, off = [], 0
    for m, n, K, kind in shapes:
        blocks.append(Block(off, m * n, m, n, K, kind))
        off += m * n
    N = 2
    src = GradientSource(off, blocks, N, seed=3)
    ctx = ArcTopK(off, blocks, N=N, eta=0.5, seed=3, nodes_local=N, method="topk_allgather")
    o = orc.OracleEF21M(off, blocks, N=N, eta=0.5, r=4, seed=3)
    h = [torch.zeros(off, device=DEV) for _ in range(N)]
    g = [torch.zeros(off, device=DEV) for _ in range(N)]
    gbar = torch.zeros(off, device=DEV)
    for t in range(3):
        gr = [x.numpy() for x in src.grads(t)]
        ctx.step(t, [torch.from_numpy(x).to(DEV) for x in gr], h, g, gbar)
        o.step_topk(t, gr)
    torch.cuda.synchronize()
    for i in range(N):
        assert_same_floats(g[i].cpu().numpy(), o.g[i], f"g[{i}]")
    assert_same_floats(gbar.cpu().numpy(), o.gbar, "gbar")
    ctx.close()


def test_full_size_c4_llama_per_tensor(orc):
    """BASELINE configs[3]: the 1.3B-parameter LLaMA-1B-shaped gradient with per-tensor
    compression (170 ARC blocks incl. unaligned n = 5461 rows, plus the DENSE block of
    1-D parameters), K = 0.1 % per tensor, one node per GPU (the bench launch
    configuration): selection, values and state bit-exact at full size, 2 steps."""
    d, blocks = config_blocks("C4")
    assert len(blocks) == 171 and d == 1_339_082_752
    run_parity(orc, d, blocks, N=1, steps=2, seed=20251030, check_debug=True)


# ------------------------------------------------------------------ Rand-K (Table I row "Rand-K")

@pytest.mark.parametrize("N,d,n,K", [(1, 50_000, 100, 7), (4, 60_000, 96, 12), (3, 4_097, 3, 40)])
def test_randk(orc, N, d, n, K):
    """Shared-seed Rand-K through the same path: the keys, the selection, values and
    state bit-exact against the oracle."""
    run_parity(orc, d, flat_blocks(d, n, K=K), N=N, steps=4, method="randk")


def test_randk_multiblock_and_exchange(orc):
    shapes = [(300, 64, 5, 0), (13, 100, 13, 1), (77, 33, 4, 0)]
    blocks, off = [], 0
    for m, n, K, kind in shapes:
        blocks.append(Block(off, m * n, m, n, K, kind))
        off += m * n
    run_parity(orc, off, blocks, N=2, steps=3, method="randk")
    run_parity(orc, off, blocks, N=2, steps=3, method="randk", force_exchange=True, reduce="ordered")


# ------------------------------------------------------------------ wide blocks (V staged in ranges)

@pytest.mark.parametrize("r,exchange", [(4, False), (8, False), (4, True)])
def test_wide_blocks_ranged_launch(orc, r, exchange):
    """Blocks whose V_b^T exceeds the streaming kernel's shared-memory stage (r n > 12288
    floats) go through the second, ranged launch (V staged in 1024-column ranges, P'
    carried across ranges); mixed with narrow blocks, a ragged wide last row and an
    unaligned row length."""
    shapes = [(37, 3500, 5), (20, 1000, 3), (9, 7777, 2)]
    blocks, off = [], 0
    for m, n, K in shapes:
        blocks.append(Block(off, m * n, m, n, K, 0))
        off += m * n
    last = Block(off, 6 * 4100 - 57, 6, 4100, 2, 0)            # ragged last row
    blocks.append(last)
    off += last.len
    run_parity(orc, off, blocks, N=2, steps=3, r=r, force_exchange=exchange,
               reduce="ordered" if exchange else "nccl")


@pytest.mark.parametrize("layout", [
    [(3, 5, 3, 0), (40, 4100, 5, 0)],                    # n % 4 == 0, block offset 14: every row s = 2
    [(1, 1, 1, 0), (33, 5461, 4, 0), (2, 3, 1, 0)],     # n = 5461: s cycles 1, 2, 3, 0 row by row
    [(2, 2, 2, 0), (9, 13001, 2, 0)],                    # V wider than the stage (ranges), s = 0, 1, 2, ...
    [(1, 6, 1, 0), (21, 5461, 21, 0)],                   # K = m, last block ends the buffer at d % 4 = 3
])
@pytest.mark.parametrize("r", [4, 8])
def test_wide_unaligned_rows_realigned(orc, layout, r):
    """Wide-row launch, rows that start off a 16-byte boundary: 16-byte loads of the
    aligned quads realigned with warp shuffles (arc_sketch.cu load_batch) — bit-exact,
    including the last row of the buffer (its aligned quad is never read past d)."""
    blocks, off = [], 0
    for m, n, K, kind in layout:
        blocks.append(Block(off, m * n - (n // 3 if m > 1 else 0), m, n, K, kind))
        off += blocks[-1].len
    run_parity(orc, off, blocks, N=2, steps=3, r=r)


@pytest.mark.parametrize("r", [4, 32])
def test_wide_blocks_beyond_the_full_stage(orc, r):
    """The second launch stages a wide block's whole V_b^T (up to 196 KB) once per
    block; wider ones (r = 4: n > 12288; r = 32: n > 1024) still go in ranges,
    next to fully staged wide blocks, narrow blocks and rows of <= 4 columns."""
    shapes = [(5, 13001, 2), (7, 5000, 1), (40, 300, 4), (6, 1100, 2), (90, 2, 9)]
    blocks, off = [], 0
    for m, n, K in shapes:
        blocks.append(Block(off, m * n, m, n, K, 0))
        off += m * n
    run_parity(orc, off, blocks, N=2, steps=3, r=r)


@pytest.mark.parametrize("method", ["arc", "randk", "noef_msgd"])
def test_rows_of_at_most_four_columns(orc, method):
    """Blocks of rows with n <= 4 (biases, norms) run one row per thread in the
    second launch (tiles of up to 512 rows); mixed with a normal block, several
    nodes and a ragged last row."""
    shapes = [(700, 1, 7), (301, 3, 5), (1000, 4, 9), (50, 200, 3)]
    blocks, off = [], 0
    for m, n, K in shapes:
        blocks.append(Block(off, m * n, m, n, K, 0))
        off += m * n
    last = Block(off, 3 * 129 - 2, 129, 3, 4, 0)                 # ragged last row
    blocks.append(last)
    off += last.len
    run_parity(orc, off, blocks, N=3, steps=3, method=method, eta=0.5 if method == "noef_msgd" else 0.1)


# ------------------------------------------------------------------ without EF (Table II)

@pytest.mark.parametrize("N,d,n,K,beta", [(1, 50_000, 100, 7, 0.9), (4, 60_000, 96, 12, 0.9), (3, 4_097, 3, 40, 0.0)])
def test_noef_msgd(orc, N, d, n, K, beta):
    """Compressed momentum SGD without error feedback (Table II "(without EF)"):
    the shared selection on the gradients, u = beta u + C; selection, values and u
    bit-exact against the oracle."""
    run_parity(orc, d, flat_blocks(d, n, K=K), N=N, steps=4, eta=beta, method="noef_msgd")


def test_noef_msgd_multiblock_and_exchange(orc):
    shapes = [(300, 64, 5, 0), (13, 100, 13, 1), (77, 33, 4, 0)]
    blocks, off = [], 0
    for m, n, K, kind in shapes:
        blocks.append(Block(off, m * n, m, n, K, kind))
        off += m * n
    run_parity(orc, off, blocks, N=2, steps=3, eta=0.5, method="noef_msgd")
    run_parity(orc, off, blocks, N=2, steps=3, eta=0.5, method="noef_msgd", force_exchange=True, reduce="ordered")
    run_parity(orc, off, blocks, N=2, steps=3, eta=0.5, method="noef_msgd", host=True, check_debug=False)


# ------------------------------------------------------------------ randomized sweep

def _random_case(rng):
    nb = int(rng.integers(1, 5))
    blocks, off = [], 0
    for _ in range(nb):
        n = int(rng.choice([1, 2, 3, 4, 5, 7, 31, 64, 96, 127, 128, 500, 768, 1024, 2051]))
        m = int(rng.integers(1, max(2, 60_000 // n)))
        ln = m * n - int(rng.integers(0, n)) if rng.random() < 0.4 else m * n   # ragged last row
        kind = 1 if rng.random() < 0.15 else 0
        K = m if kind == 1 else int(rng.integers(1, m + 1)) if rng.random() < 0.2 else max(1, m // int(rng.integers(2, 200)))
        blocks.append(Block(off, ln, m, n, K, kind))
        off += ln
    return off, blocks


@pytest.mark.parametrize("case", range(24))
def test_randomized_configurations(orc, case):
    """Seeded random layouts, sketch widths, node counts, momenta, methods and paths."""
    rng = np.random.default_rng(1000 + case)
    d, blocks = _random_case(rng)
    N = int(rng.integers(1, 6))
    r = int(rng.choice([1, 2, 4, 5, 8, 16]))
    eta = float(rng.choice([1.0, 0.5, 0.1, 0.01]))
    method = str(rng.choice(["arc", "arc", "arc", "randk"]))
    fx = bool(rng.random() < 0.3)
    reduce = str(rng.choice(["nccl", "ordered"]))
    run_parity(orc, d, blocks, N=N, steps=2, eta=eta, r=r, seed=case, method=method,
               force_exchange=fx, reduce=reduce)


# ------------------------------------------------------------------ selection vs torch.sort

@pytest.mark.parametrize("cfg,mu_bp", [("C5_1e8", 100), ("C5_1e8", 1000), ("C3", 10), ("C5_1e9", 100),
                                        ("C5_1e9", 1000), ("C5_1e9", 10)])
def test_selection_matches_torch_stable_sort(cfg, mu_bp):
    """the GPU selection against torch.sort(stable) of the same Sigma's
    order keys (larger key first, ties -> smaller row, NaN above +Inf) at full size,
    independently of the oracle."""
    from paper_2510_26709_b200 import ArcTopK
    from paper_2510_26709_b200 import _lib as L
    d, blocks = config_blocks(cfg, mu_bp)
    src = GradientSource(d, blocks, 1, seed=31, device=DEV)
    h, g, gbar = [torch.zeros(d, device=DEV)], [torch.zeros(d, device=DEV)], torch.zeros(d, device=DEV)
    ctx = ArcTopK(d, blocks, N=1, eta=0.1, r=4, seed=31, debug_sketch=True)
    for t in range(3):
        sel = torch.empty(ctx.sum_K, dtype=torch.int32, device=DEV)
        ctx.step(t, src.grads(t), h, g, gbar, sel)
    sig = ctx.query(L.Q_SIGMA)
    key = sig.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    key = torch.where(torch.isnan(sig), torch.full_like(key, 0xFFFFFFFF), key)
    base = 0
    for b in blocks:
        if b.kind != 0:
            continue
        kb = key[base:base + b.m]
        order = torch.sort(-kb, stable=True).indices           # stable: ties keep the smaller row first
        want = torch.sort(order[:b.K]).values.to(torch.int32)
        assert torch.equal(sel[sum(x.K for x in blocks[:blocks.index(b)]):][:b.K], want)
        base += b.m
    ctx.close()


# ------------------------------------------------------------------ selection valid in binary64

def _gamma(k):
    u = 2.0 ** -24
    return k * u / (1 - k * u)


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5_1e9"])
def test_selection_valid_in_binary64(cfg):
    """An order-independent check of the GPU selection at full size (not the O6
    order the oracle shares with the kernel): from the GPU's own residual
    Delta = h' (-) g_prev (one fp32 subtraction) and V, recompute S = Delta V and
    Sigma = sum_j S_j^2 in binary64 (zn28373 P:236-237, Alg. 1 l.4-6) with a
    rounding bound beta_p for ANY fp32 summation order: |S32_j - S64_j| <= E_j =
    gamma_{n+5} sum_q |Delta_q V_qj| (the dot products), then the squares and
    the r-term fma chain.  Asserts (a) the kernel's Sigma is within beta of the
    binary64 value on every row, and (b) every selected row's Sigma64 + beta is
    >= every unselected row's Sigma64 - beta (the K largest, up to rounding)."""
    from paper_2510_26709_b200 import ArcTopK
    from paper_2510_26709_b200 import _lib as L
    d, blocks = config_blocks(cfg)
    r = 4
    src = GradientSource(d, blocks, 1, seed=41, device=DEV)
    h, g, gbar = [torch.zeros(d, device=DEV)], [torch.zeros(d, device=DEV)], torch.zeros(d, device=DEV)
    ctx = ArcTopK(d, blocks, N=1, eta=0.1, r=r, seed=41, debug_sketch=True)
    sel = torch.empty(ctx.sum_K, dtype=torch.int32, device=DEV)
    for t in range(2):
        g_prev = g[0].clone()
        ctx.step(t, src.grads(t), h, g, gbar, sel)
    torch.cuda.synchronize()
    sig_gpu = ctx.query(L.Q_SIGMA).double()
    V_all = ctx.query(L.Q_V)
    goff = roff = soff = 0
    checked = 0
    for b in blocks:
        if b.kind != 0:
            soff += b.K
            continue
        ldv = -(-b.n // 4) * 4
        Vb = V_all[goff:goff + r * ldv].view(r, ldv)[:, :b.n].double().t().contiguous()      # n x r
        goff += r * ldv
        D = torch.zeros(b.m * b.n, device=DEV)
        D[:b.len] = h[0][b.offset:b.offset + b.len] - g_prev[b.offset:b.offset + b.len]    # fp32, as the kernel
        D = D.view(b.m, b.n)
        sig64 = torch.empty(b.m, dtype=torch.float64, device=DEV)
        beta = torch.empty(b.m, dtype=torch.float64, device=DEV)
        step = max(1, (1 << 27) // b.n)
        for p0 in range(0, b.m, step):
            D64 = D[p0:p0 + step].double()
            S = D64 @ Vb
            E = _gamma(b.n + 5) * (D64.abs() @ Vb.abs())
            sig64[p0:p0 + step] = (S * S).sum(1)
            beta[p0:p0 + step] = (2 * S.abs() * E + E * E).sum(1) + _gamma(r + 1) * ((S.abs() + E) ** 2).sum(1)
        sg = sig_gpu[roff:roff + b.m]
        assert torch.all((sg - sig64).abs() <= beta + 1e-300), f"{cfg} block at {b.offset}: Sigma outside the bound"
        chosen = torch.zeros(b.m, dtype=torch.bool, device=DEV)
        chosen[sel[soff:soff + b.K].long()] = True
        assert int(chosen.sum()) == b.K
        if b.K < b.m:
            lo = (sig64 + beta)[chosen].min()
            hi = (sig64 - beta)[~chosen].max()
            assert lo >= hi, f"{cfg} block at {b.offset}: a selected row is below an unselected one ({lo} < {hi})"
        checked += 1
        roff += b.m
        soff += b.K
    assert checked == sum(1 for b in blocks if b.kind == 0)
    ctx.close()


def test_misaligned_pointers_rejected():
    """T5: base pointers must be 16-byte aligned; a misaligned one is rejected before
    anything is enqueued (the state stays untouched)."""
    from paper_2510_26709_b200 import ArcTopK
    d, blocks = 4_000, flat_blocks(4_000, 40, K=3)
    ctx = ArcTopK(d, blocks, N=1, eta=0.1, r=4, seed=1)
    big = torch.zeros(d + 4, device=DEV)
    h, g, gbar = [torch.zeros(d, device=DEV)], [torch.zeros(d, device=DEV)], torch.zeros(d, device=DEV)
    grad = [torch.ones(d, device=DEV)]
    with pytest.raises(Exception):
        ctx.step(0, [big[1:d + 1]], h, g, gbar)           # 4-byte aligned only
    with pytest.raises(Exception):
        ctx.step(0, grad, [big[2:d + 2]], g, gbar)
    torch.cuda.synchronize()
    assert not h[0].any() and not g[0].any() and not gbar.any()
    ctx.step(0, grad, h, g, gbar)                        # aligned: fine
    torch.cuda.synchronize()
    assert h[0].any()
    ctx.close()


# ------------------------------------------------------------------ exact sketch (test mode)

@pytest.mark.parametrize("N,d,n,K,mixed", [
    (1, 100_003, 768, 13, False),      # N = 1: the exact sketch is row Top-K of Delta
    (4, 65_536, 1, 656, False),        # C1 shape (n = 1: coordinate Top-K of the node sum)
    (3, 40_000, 130, 17, False),       # n % 4 != 0, unaligned rows, ragged last row
    (2, 3_000 * 2_500 + 7, 2_500, 9, False),   # rows of several 1024-column chunks
    (4, 0, 0, 0, True),                # ARC blocks + a DENSE block
])
def test_exact_sketch_method(orc, N, d, n, K, mixed):
    """method="exact" (SURVEY §8(b) ARC_SKETCH_EXACT, §8(f) row 3): Sigma_p =
    ||sum_i Delta_i[p,:]||^2 with the squares in the O6 order — bit-exact
    against the oracle's exact mode (OracleEF21M(exact=True)): Sigma, the
    selection, values, h, g and gbar over several steps."""
    from paper_2510_26709_b200 import ArcTopK
    if mixed:
        blocks = [Block(0, 96 * 300 + 5, 301, 96, 11, 0), Block(96 * 300 + 5, 640, 10, 64, 10, 1),
                  Block(96 * 300 + 645, 50 * 77, 50, 77, 4, 0)]
        d = 96 * 300 + 645 + 50 * 77
    else:
        blocks = flat_blocks(d, n, K=K)
    src = GradientSource(d, blocks, N, seed=9)
    ctx = ArcTopK(d, blocks, N=N, eta=0.1, r=4, seed=9, nodes_local=N, method="exact")
    o = orc.OracleEF21M(d, blocks, N=N, eta=0.1, r=4, seed=9, exact=True)
    h = [torch.zeros(d, device=DEV) for _ in range(N)]
    g = [torch.zeros(d, device=DEV) for _ in range(N)]
    gbar = torch.zeros(d, device=DEV)
    for t in range(4):
        gr = [x.numpy() for x in src.grads(t)]
        sel = torch.empty(ctx.sum_K, dtype=torch.int32, device=DEV)
        vals = torch.empty(ctx.sum_Kn, dtype=torch.float32, device=DEV) if t % 2 else None
        ctx.step(t, [torch.from_numpy(x).to(DEV) for x in gr], h, g, gbar, sel, vals)
        ref = o.step(t, gr, debug=True)
        torch.cuda.synchronize()
        assert_same_floats(ctx.query(1).cpu().numpy(), ref["sigma"], f"exact Sigma (t={t})")
        assert np.array_equal(sel.cpu().numpy(), ref["sel"]), f"selection differs at t={t}"
        if vals is not None:
            assert_same_floats(vals.cpu().numpy(), ref["values"], f"values (t={t})")
    for i in range(N):
        assert_same_floats(h[i].cpu().numpy(), o.h[i], f"h[{i}]")
        assert_same_floats(g[i].cpu().numpy(), o.g[i], f"g[{i}]")
    assert_same_floats(gbar.cpu().numpy(), o.gbar, "gbar")
    ctx.close()


def test_exact_sketch_needs_all_nodes_local():
    from paper_2510_26709_b200 import ArcTopK
    from paper_2510_26709_b200._lib import ArcError
    blocks = flat_blocks(4096, 64, K=4)
    with pytest.raises(ArcError):
        ArcTopK(4096, blocks, N=2, eta=0.1, nodes_local=2, method="exact", force_exchange=True, device=DEV)


# ------------------------------------------------------------------ streaming-pass variants (round 2)

@pytest.mark.parametrize("shape", [None, "0", "2", "5"])
@pytest.mark.parametrize("layout", [
    [(9001, 768, 90)],                         # C3 row length, M past the fused tail's limit
    [(8300, 1024, 83), (300, 512, 9)],         # two blocks of full 128-column segments
])
def test_streaming_variants_with_ragged_rows(orc, monkeypatch, shape, layout):
    """Every streaming variant, including the predicate-free loop of variants 2 and 5 (full
    aligned rows) next to the generic loop (the short last row of each block), bit-exact;
    None = the variant the planner picks (5 for these one-node layouts)."""
    if shape is not None:
        monkeypatch.setenv("ARC_SKETCH_SHAPE", shape)
    blocks, off = [], 0
    for m, n, K in layout:
        ln = m * n - 36                        # a short last row (block offsets stay 16-byte aligned)
        blocks.append(Block(off, ln, m, n, K, 0))
        off += ln
    run_parity(orc, off, blocks, N=1, steps=3)
