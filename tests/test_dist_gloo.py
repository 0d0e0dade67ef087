"""Multi-process (world_size 2, gloo, CPU) tests of the N > 1 host logic.

1. Parameter consistency across ranks (SPMD contract of arc_topk_create).
2. The exchange protocol of the multi-GPU path (reading R21):
   every rank exports its nodes' sketches P_i; an all-to-all of row slices
   gives rank j all nodes' sketches of its rows, which it sums in ascending
   GLOBAL node id into its slice of Sigma; an all-gather of the slices gives
   every rank all of Sigma.  The selection is then identical on every rank
   and equal to the single-process oracle's, bit for bit, for any placement of
   the N nodes on G ranks.  Exchange #2 in "ordered" mode (all-gather of the
   per-node rows) is bit-exact too; in "nccl" mode (an All-Reduce with
   unspecified order) gbar agrees within the 1e-5 tolerance.
   The per-node compute here uses the oracle's own functions; what is under
   test is the placement/exchange scheme the CUDA path implements.
3. Ledger closed forms (Table I).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_consistency(rank, world, port, q):
    _init(rank, world, port)
    from paper_2510_26709_b200.dist import check_consistent, params_digest
    from synth import flat_blocks
    ok = params_digest(1000, flat_blocks(1000, 10, K=3), 4, 2, 4, 0.1, 7, "nccl")
    check_consistent(dist.group.WORLD, ok)                       # identical: passes
    bad = params_digest(1000, flat_blocks(1000, 10, K=3 + rank), 4, 2, 4, 0.1, 7, "nccl")
    try:
        check_consistent(dist.group.WORLD, bad)
        q.put((rank, "no error"))
    except ValueError:
        q.put((rank, "raised"))
    dist.destroy_process_group()


def _f32_seq_sum(xs):
    s = xs[0].astype(np.float32).copy()
    for x in xs[1:]:
        s = (s + x.astype(np.float32)).astype(np.float32)
    return s


def _worker_protocol(rank, world, port, L, reduce, steps, q):
    _init(rank, world, port)
    import oracle
    from synth import GradientSource, flat_blocks
    N = world * L
    d, n, K, r, eta, seed = 6030, 30, 13, 4, 0.1, 9   # m = 201: uneven row slices
    blocks = flat_blocks(d, n, K=K)
    m = blocks[0].m
    src = GradientSource(d, blocks, N, seed=seed)
    nodes = list(range(rank * L, (rank + 1) * L))
    h = [np.zeros(d, np.float32) for _ in nodes]
    g = [np.zeros(d, np.float32) for _ in nodes]
    gbar = np.zeros(d, np.float32)
    ref = oracle.OracleEF21M(d, blocks, N=N, eta=eta, r=r, seed=seed)
    Nf = np.float32(N)
    out = []
    for t in range(steps):
        all_grads = [x.numpy() for x in src.grads(t)]
        ref_out = ref.step(t, all_grads)
        V = oracle.gaussian_V(seed, t, 0, n, r)
        Pi, D = [], []
        for l, i in enumerate(nodes):
            h[l] = oracle.momentum(h[l], all_grads[i], eta)
            D.append((h[l] - g[l]).astype(np.float32))
            Pi.append(oracle.arc_round([D[-1]], n=n, K=K, V=V)["P_nodes"][0])      # P'_i = Delta_i V
        # exchange #1: rank j owns rows [j Ms, (j+1) Ms); an
        # all-to-all (send/recv) brings it those rows' per-node sketches from every
        # rank, it sums them in global node order and forms its Sigma slice, and an
        # all-gather of the (padded) slices gives every rank all of Sigma
        Ms = -(-m // world)
        mine = np.zeros((world * Ms, L, r), np.float32)
        mine[:m] = np.stack(Pi, axis=1)                                              # [m][L][r]
        recv = [torch.empty((Ms, L, r)) for _ in range(world)]
        reqs = []
        for j in range(world):
            if j == rank:
                recv[j].copy_(torch.from_numpy(mine[j * Ms:(j + 1) * Ms]))
                continue
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(mine[j * Ms:(j + 1) * Ms])), j))
            reqs.append(dist.irecv(recv[j], j))
        for q_ in reqs:
            q_.wait()
        per_node = [recv[gr].numpy()[:, l, :] for gr in range(world) for l in range(L)]   # global node order
        S = _f32_seq_sum(per_node)
        sig_slice = oracle.sigma_rows(S)                                             # O8 on the slice
        got = [torch.empty(Ms) for _ in range(world)]
        dist.all_gather(got, torch.from_numpy(sig_slice))
        sig = np.concatenate([x.numpy() for x in got])[:m]
        I = oracle.argtop_k(sig, K)
        # compaction + local EF update
        C = [Dl.reshape(m, n)[I] for Dl in D]
        for l in range(L):
            gv = g[l].reshape(m, n)
            gv[I] = (gv[I] + C[l]).astype(np.float32)
        # exchange #2
        if reduce == "ordered":
            mine = torch.from_numpy(np.stack(C))
            got = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(got, mine)
            A = _f32_seq_sum([x.numpy()[l] for x in got for l in range(L)])
        else:
            A_loc = torch.from_numpy(_f32_seq_sum(C))
            dist.all_reduce(A_loc)
            A = A_loc.numpy()
        val = (A / Nf).astype(np.float32)
        gb = gbar.reshape(m, n)
        gb[I] = (gb[I] + val).astype(np.float32)
        # compare with the single-process oracle
        sel_same = bool(np.array_equal(I, ref_out["sel"]))
        state_same = all(h[l].tobytes() == ref.h[i].tobytes() and g[l].tobytes() == ref.g[i].tobytes()
                         for l, i in enumerate(nodes))
        mag = sum(np.abs(x.astype(np.float64)) for x in ref.g) / N + np.abs(ref.gbar)
        gbar_err = float(np.max(np.abs(gbar.astype(np.float64) - ref.gbar) / (mag + 1e-30)))
        out.append((sel_same, state_same, gbar.tobytes() == ref.gbar.tobytes(), gbar_err))
    # all ranks must hold the same selection / gbar
    gb_all = [torch.empty(d) for _ in range(world)]
    dist.all_gather(gb_all, torch.from_numpy(gbar))
    same_gbar_across_ranks = all(x.numpy().tobytes() == gb_all[0].numpy().tobytes() for x in gb_all)
    q.put((rank, out, same_gbar_across_ranks))
    dist.destroy_process_group()


def _spawn(fn, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    res, t0 = [], time.time()
    while len(res) < len(procs):
        try:
            res.append(q.get(timeout=1))
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            if dead or time.time() - t0 > 300:
                for p in procs:
                    p.kill()
                raise AssertionError(f"worker failed (exit codes {[p.exitcode for p in procs]})")
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


def test_params_consistency_gloo():
    res = _spawn(_worker_consistency, 2)
    assert [r[1] for r in res] == ["raised", "raised"]


@pytest.mark.parametrize("L,reduce", [(1, "ordered"), (2, "ordered"), (2, "nccl")])
def test_exchange_protocol_gloo(L, reduce):
    res = _spawn(_worker_protocol, 2, L, reduce, 4)
    for rank, steps, same_across in res:
        assert same_across
        for sel_same, state_same, gbar_exact, gbar_err in steps:
            assert sel_same and state_same
            if reduce == "ordered":
                assert gbar_exact
            else:
                assert gbar_err <= 1e-5


def test_ledger_closed_forms():
    """Table I / P:318 closed forms; SPEC S:283-285 worked numbers (m=4, n=3, N=2, K=1, r=1)."""
    from paper_2510_26709_b200 import comm_entries
    assert comm_entries("arc", 4, 3, 2, 1, r=1) == 14
    assert comm_entries("dense", 4, 3, 2, 1) == 24
    assert comm_entries("topk", 4, 3, 2, 1) == 4
    assert comm_entries("randk", 4, 3, 2, 1) == 6
    assert comm_entries("arc", 4, 3, 1, 1) == 0
    # r = 1 reduces ARC to 2Kn + 2m
    assert comm_entries("arc", 100, 8, 4, 5, r=1) == 2 * 5 * 8 + 2 * 100
    # this build's NVLink bytes per GPU: all-to-all of sketch row slices + Sigma
    # all-gather (G = 2, m = 10 -> slices of 5 rows), ring All-Reduce of K n values
    from paper_2510_26709_b200.ledger import arc_bus_bytes
    b = arc_bus_bytes(10, 30, r=4, G=2)
    assert b["sketch"] == 5 * 4 * 4 + 5 * 4 and b["values"] == 30 * 4
    assert arc_bus_bytes(10, 30, r=4, G=1)["total"] == 0


def test_node_placement():
    from paper_2510_26709_b200.dist import node_ids
    assert node_ids(0, 2) == [0, 1] and node_ids(3, 2) == [6, 7]
    allids = sum((node_ids(r, 4) for r in range(2)), [])
    assert allids == list(range(8))
