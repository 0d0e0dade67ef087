"""The multi-GPU step (G > 1 ranks) executed on ONE GPU through the library's
in-process loopback communicator (arc_topk_loopback_*, ARC_FLAG_LOOPBACK_COMM):
G host threads, one context and one stream each, the collectives replaced by
stream-event-ordered device copies (no kernel waits on another rank).  Every
G > 1 kernel and offset of the library runs: exchange #1's all-to-all of row
slices of P'_i, k_sigma_slice on each rank's slice, the Sigma all-gather, the
per-rank selection from the gathered Sigma, the K-row payload, exchange #2
(all-reduce, or all-gather + node-ordered sum) and k_scatter.

Checked against the oracle (all N nodes simulated on the host), SURVEY §8(c5):
* I, h_i, g_i bit-exact on every rank, every step, every placement (G, L);
* gbar bit-exact with reduce="ordered";
* gbar within 1e-5 M with reduce="nccl" (the loopback all-reduce sums the ranks
  in descending order, not the oracle's order);
* placement invariance: (G, L) in {(1,8), (2,4), (4,2), (8,1)}
  give identical I, h, g;
* the ledger audit (Table I): the entries handed to each
  collective equal the closed forms.
"""
import threading

import numpy as np
import pytest
import torch

from synth import Block, GradientSource, flat_blocks

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__ as ge
    ge.build()
    torch.cuda.set_device(0)


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def run_ranks(d, blocks, N, L, grads, reduce="ordered", method="arc", eta=0.1, r=4, seed=5, want_values=False,
              wire="f32"):
    """Run every rank of G = N / L in its own thread; returns per-rank results."""
    from paper_2510_26709_b200 import ArcTopK, LoopbackGroup
    G = N // L
    grp = LoopbackGroup(G)
    steps = len(grads)
    out = [None] * G
    errs = []
    noef = method == "noef_msgd"

    def rank_fn(j):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctx = ArcTopK(d, blocks, N=N, eta=eta, r=r, seed=seed, nodes_local=L, rank=j, reduce=reduce,
                              method=method, loopback=grp, stream=s, wire=wire)
                h = [torch.zeros(d, device=DEV) for _ in range(L)]
                g = [torch.zeros(d, device=DEV) for _ in range(L)]
                gbar = torch.zeros(d, device=DEV)
                sels, vals = [], []
                for t in range(steps):
                    gr = [torch.from_numpy(grads[t][j * L + i]).to(DEV) for i in range(L)]
                    if method == "topk_allgather":
                        ctx.step(t, gr, h, g, gbar, stream=s)
                    else:
                        sel = torch.empty(ctx.sum_K, dtype=torch.int32, device=DEV)
                        v = torch.empty(ctx.sum_Kn, dtype=torch.float32, device=DEV) if want_values else None
                        ctx.step(t, gr, None if noef else h, None if noef else g, gbar, sel, v, stream=s)
                        sels.append(sel)
                        vals.append(v)
                s.synchronize()
                out[j] = dict(sel=[x.cpu().numpy() for x in sels],
                              values=[x.cpu().numpy() if x is not None else None for x in vals],
                              h=[x.cpu().numpy() for x in h], g=[x.cpu().numpy() for x in g],
                              gbar=gbar.cpu().numpy(), tally=ctx.comm_tally(), kernels=ctx.kernels_per_step)
                ctx.close()
        except Exception as e:  # re-raised in the main thread
            errs.append((j, e))

    ths = [threading.Thread(target=rank_fn, args=(j,)) for j in range(G)]
    for th in ths:
        th.start()
    for th in ths:
        th.join(timeout=600)
    grp.close()
    if errs:
        raise errs[0][1]
    assert all(o is not None for o in out)
    return out


def value_positions(blocks, sel):
    """Flat element of every entry of the values array (I order; -1 = padding)."""
    out, base = [], 0
    for b in blocks:
        for k in range(b.K):
            p = int(sel[base + k])
            q = np.arange(b.n)
            e = b.offset + p * b.n + q
            out.append(np.where(p * b.n + q < b.len, e, -1))
        base += b.K
    return np.concatenate(out)


def oracle_run(orc, d, blocks, N, grads, method="arc", eta=0.1, r=4, seed=5, wire="f32"):
    o = orc.OracleEF21M(d, blocks, N=N, eta=eta, r=r, seed=seed, method=method, wire=wire)
    sels, vals, mags = [], [], np.zeros(d)
    o.step_mags = []                                         # per step: (1/N) sum_i |C_i| per values entry
    for t, gr in enumerate(grads):
        g_prev = [x.astype(np.float64) for x in o.g]
        u_prev = o.gbar.astype(np.float64)
        if method == "topk_allgather":
            res = o.step_topk(t, gr)
        else:
            res = o.step(t, gr)
        if method == "noef_msgd":
            mags += np.abs(o.gbar - eta * u_prev) + np.abs(eta * u_prev)
        else:
            step_mag = sum(np.abs(o.g[i] - g_prev[i]) for i in range(N)) / N
            mags += step_mag
            if method != "topk_allgather":
                pos = value_positions(blocks, res["sel"])
                o.step_mags.append(np.where(pos >= 0, step_mag[np.maximum(pos, 0)], 0.0))
        sels.append(res["sel"])
        vals.append(res["values"])
    return o, sels, vals, mags


def make_grads(d, blocks, N, steps, seed=5):
    src = GradientSource(d, blocks, N, seed=seed)
    return [[np.ascontiguousarray(x.numpy()) for x in src.grads(t)] for t in range(steps)]


def check(orc, res, o, sels, vals, mags, N, L, reduce, method="arc", steps=None, rel=1e-5):
    G = N // L
    for j in range(G):
        rj = res[j]
        if method != "topk_allgather":
            for t, (a, b) in enumerate(zip(rj["sel"], sels)):
                assert np.array_equal(a, b), f"rank {j}: selection differs at t={t}"
            for t, (a, b) in enumerate(zip(rj["values"], vals)):
                if a is None:
                    continue
                if reduce == "ordered":
                    assert np.array_equal(_bits(a), _bits(b)), f"rank {j}: values differ at t={t}"
                else:
                    # per step: |A/N - oracle| <= rel (1/N) sum_i |C_i| (the contract proper is on gbar below)
                    err = np.abs(a.astype(np.float64) - b)
                    bad = np.flatnonzero(err > rel * o.step_mags[t] + 1e-37)
                    assert bad.size == 0, (f"values t={t}: {bad.size} entries, first {bad[:5]}: gpu {a[bad[:5]]} "
                                           f"oracle {b[bad[:5]]} mag {o.step_mags[t][bad[:5]]}")
        if method != "noef_msgd":
            for i in range(L):
                node = j * L + i
                assert np.array_equal(_bits(rj["h"][i]), _bits(o.h[node])), f"h[{node}] (rank {j})"
                assert np.array_equal(_bits(rj["g"][i]), _bits(o.g[node])), f"g[{node}] (rank {j})"
        if reduce == "ordered" or G == 1:
            assert np.array_equal(_bits(rj["gbar"]), _bits(o.gbar)), f"gbar (rank {j})"
        else:
            M = np.abs(o.gbar.astype(np.float64)) + mags
            err = np.abs(rj["gbar"].astype(np.float64) - o.gbar)
            assert np.all(err <= rel * M + 1e-37), f"gbar beyond {rel} M (rank {j}): {float((err / (M + 1e-300)).max())}"
        # replicated: every rank holds the same gbar, bit for bit
        assert np.array_equal(_bits(rj["gbar"]), _bits(res[0]["gbar"]))


@pytest.mark.parametrize("G,L", [(2, 4), (4, 2), (8, 1)])
@pytest.mark.parametrize("reduce", ["ordered", "nccl"])
def test_loopback_ranks_match_oracle(orc, G, L, reduce):
    """N = 8 nodes on G emulated ranks (ragged flat block + a DENSE block),
    4 steps: per-rank bit-exact I, h, g; gbar per the reduce mode."""
    N = 8
    d_arc = 96 * 1200 + 37
    blocks = [Block(0, d_arc, 1201, 96, 30, 0), Block(d_arc, 700, 7, 100, 7, 1)]
    d = d_arc + 700
    grads = make_grads(d, blocks, N, 4)
    res = run_ranks(d, blocks, N, L, grads, reduce=reduce, want_values=True)
    o, sels, vals, mags = oracle_run(orc, d, blocks, N, grads)
    check(orc, res, o, sels, vals, mags, N, L, reduce)


def test_placement_invariance(orc):
    """(G, L) in {(1,8), (2,4), (4,2), (8,1)} give identical I, h, g and
    (ORDERED) gbar — the node sums run in global node order on every placement."""
    N = 8
    d = 60_000
    blocks = flat_blocks(d, 64, K=20)
    grads = make_grads(d, blocks, N, 3, seed=9)
    outs = {}
    for (G, L) in [(1, 8), (2, 4), (4, 2), (8, 1)]:
        res = run_ranks(d, blocks, N, L, grads, reduce="ordered", seed=9)
        outs[(G, L)] = (res[0]["sel"], [x for j in range(G) for x in res[j]["h"]],
                        [x for j in range(G) for x in res[j]["g"]], res[0]["gbar"])
    ref = outs[(1, 8)]
    for k, v in outs.items():
        for a, b in zip(v[0], ref[0]):
            assert np.array_equal(a, b), k
        for a, b in zip(v[1] + v[2] + [v[3]], ref[1] + ref[2] + [ref[3]]):
            assert np.array_equal(_bits(a), _bits(b)), k


@pytest.mark.parametrize("method", ["randk", "noef_msgd", "topk_allgather"])
def test_loopback_baselines(orc, method):
    """Rand-K, compressed MSGD without EF and the All-Gather Top-K baseline on 4
    emulated ranks x 2 nodes, bit-exact (ordered) against the oracle."""
    N, L = 8, 2
    d = 40_000
    blocks = [Block(0, 30_000, 300, 100, 9, 0), Block(30_000, 10_000, 10, 1000, 10, 1)]
    eta = 0.9 if method == "noef_msgd" else 0.1
    grads = make_grads(d, blocks, N, 3)
    res = run_ranks(d, blocks, N, L, grads, reduce="ordered", method=method, eta=eta)
    o, sels, vals, mags = oracle_run(orc, d, blocks, N, grads, method=method, eta=eta)
    check(orc, res, o, sels, vals, mags, N, L, "ordered", method=method)


def test_ledger_audit_matches_table1():
    """Table I / P:318 ARC-Top-K row: per node per iteration the sketch
    All-Reduce carries m r entries and the value All-Reduce K n entries (the
    paper counts 2mr + 2Kn in the ring convention, R18).  The library hands
    exactly sum_b K_b n_b value entries to its all-reduce per step, and its
    sketch exchange moves every rank's m r entries once (each rank sends the
    (G-1)/G of its rows it does not own; the owner forms Sigma, and the
    all-gather returns ceil(m/G) Sigma entries per rank)."""
    from paper_2510_26709_b200.ledger import comm_entries
    N, L, steps = 4, 1, 3
    d = 50_000
    blocks = [Block(0, 48_000, 500, 96, 11, 0), Block(48_000, 2000, 2, 1000, 2, 1)]
    grads = make_grads(d, blocks, N, steps)
    res = run_ranks(d, blocks, N, L, grads, reduce="nccl")
    M = 500
    sumKn = 11 * 96 + 2 * 1000
    Ms = -(-M // N)
    for j, rj in enumerate(res):
        tl = rj["tally"]
        assert tl["steps"] == steps
        assert tl["values"] == steps * sumKn
        own = min(M, (j + 1) * Ms) - j * Ms
        assert tl["sketch"] == steps * (M - own) * L * 4          # r = 4 entries per row sent to the owner
        assert tl["sigma"] == steps * Ms
        assert tl["calls"] == steps * 3                          # all-to-all, Sigma all-gather, all-reduce
    # Table I's ARC row for the ARC block = 2 (K n + m r): payload counts x 2 (ring convention)
    assert comm_entries("arc", 500, 96, N, 11, 4) == 2 * (11 * 96) + 2 * (500 * 4)
    tot_sketch = sum(rj["tally"]["sketch"] for rj in res) // steps
    assert tot_sketch == (N - 1) * M * 4                          # every rank's m r entries, once


@pytest.mark.parametrize("G,L", [(2, 4), (8, 1)])
@pytest.mark.parametrize("reduce", ["ordered", "nccl"])
def test_loopback_bf16_wire(orc, G, L, reduce):
    """The bf16 value wire (R25) across emulated ranks: bf16 payloads in the
    all-gather (ORDERED: gbar bit-exact, the sums stay binary32) or a bf16
    all-reduce (NCCL: its partial sums are rounded to bf16.  bfloat16 keeps 8
    significand bits, so one rounding errs by <= u = 2^-8 relative; the loopback
    all-reduce rounds the rank pre-sums and the reduced sum once each, so per
    step |A - A_oracle| <= 2u sum_i |C_i| and gbar stays within 2^-7 M; NCCL's
    ring rounds up to G partial sums: (G + 1) u M, R25).  I, h, g
    bit-exact either way."""
    N = 8
    d_arc = 96 * 1200 + 37
    blocks = [Block(0, d_arc, 1201, 96, 30, 0), Block(d_arc, 700, 7, 100, 7, 1)]
    d = d_arc + 700
    grads = make_grads(d, blocks, N, 4)
    res = run_ranks(d, blocks, N, L, grads, reduce=reduce, want_values=True, wire="bf16")
    o, sels, vals, mags = oracle_run(orc, d, blocks, N, grads, wire="bf16")
    check(orc, res, o, sels, vals, mags, N, L, reduce, rel=2.0 ** -7)
