"""Benchmark of the EF21M + ARC-Top-K compression step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

One step = one pass of the whole hot path over one
batch of synthetic gradients: momentum + residual + sketch, exchange #1,
row importance, Top-K selection, compaction + EF update, exchange #2,
scatter into the replicated tracker.  One paper node per GPU (weak scaling:
the per-GPU gradient size is fixed as N grows).  Default workload: BASELINE
configs[2], the GPT-2-small-sized gradient (d = 124,439,808, n = 768, K = 1 %),
the config for which the north_star's roofline target (d >= 100M) is stated.

Prints ONE JSON line (rank 0).  `value` = whole-job gradient throughput
(4 bytes x d x N nodes / step time, GB/s); inputs are resident in HBM and far
larger than L2 (126 MB), so no L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ARC-Top-K step ms and grad GB/s at 1/2/4/8 B200; % of HBM/NVLink roofline"
PHASES = ["vgen", "ef_sketch", "exchange1_reduce", "select_gather", "exchange2_scatter", "copy_out"]


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index: int, period: float = 0.01):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self._thr = None
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - NVML missing
            self.nvml = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                fn = getattr(self.nvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    self.nvml.nvmlDeviceGetCurrentClocksThrottleReasons
                r = fn(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nvml is not None:
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thr is not None:
            self._thr.join()

    def summary(self):
        if self.nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "nvml")}
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def workload(name: str, nodes_per_gpu: int, world: int, mu_bp=None):
    from synth import config_blocks
    d, blocks = config_blocks(name, mu_bp)
    return d, blocks, nodes_per_gpu * world


def algorithmic_bytes(d, blocks, L, r):
    """HBM bytes the method must move per GPU per step:
    ef_sketch: 16 B per element per node of ARC blocks (read grad, h, g; write h)
               + 4 B per row (Sigma);
    gather/EF (+scatter at G = 1): per selected element 8 B (h, g) + 4 B (g) per
               node + 8 B (gbar RMW) (+ DENSE blocks also read grad and write h)."""
    d_arc = sum(b.len for b in blocks if b.kind == 0)
    M = sum(b.m for b in blocks if b.kind == 0)
    kn = sum(min(b.K * b.n, b.len) for b in blocks)
    kn_dense = sum(b.len for b in blocks if b.kind == 1)
    sketch = 16 * d_arc * L + 4 * M
    gather = 12 * kn * L + 8 * kn + 8 * kn_dense * L
    return {"ef_sketch": sketch, "gather_ef": gather, "total": sketch + gather + 8 * M}


def run_reference(args):
    """--impl reference: the CPU oracle (plain C, 1 thread) on the host cores,
    same workload, metric and unit; each step is a bounded sample of it (a
    contiguous range of whole rows), sized so the run ends within minutes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    from synth import Block, GradientSource
    d, blocks, _ = workload(args.config, args.nodes_per_gpu, 1)
    B = blocks[0]
    total_steps = args.steps + args.warmup
    budget_s = float(os.environ.get("ARC_REF_BUDGET_S", "90"))
    rate = 1.0e8                                        # elements/s, re-measured below
    rows = max(1, min(B.m, int(budget_s * rate / max(total_steps, 1) / B.n)))
    d_s = rows * B.n
    K_s = max(1, -(-rows * 100 // 10000))
    sb = [Block(0, d_s, rows, B.n, K_s, 0)]
    L = args.nodes_per_gpu
    src = GradientSource(d_s, sb, L, seed=20251030)
    gr = [x.numpy() for x in src.grads(0)]
    o = oracle.OracleEF21M(d_s, sb, N=L, eta=0.1, r=4, seed=20251030)
    for t in range(args.warmup):
        o.step(t, gr)
    t0 = time.perf_counter()
    for t in range(args.steps):
        o.step(args.warmup + t, gr)
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    value = 4.0 * d_s * L / dt / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config} sample: {rows} of {B.m} rows (n={B.n}), K=1% of sample",
                       "d_sample": d_s, "nodes": L},
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": f"{rows} rows x {B.n} cols of {args.config}, {L} node(s), per step"},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def cpu_baseline_leg(d, blocks, L, budget_s=20.0):
    """The oracle as it stands (1 thread), timed on this box's host cores on a
    bounded sample of the same workload (whole steps of the full config if they
    fit the budget, else a contiguous block of rows)."""
    import numpy as np

    import oracle
    from synth import Block, GradientSource
    B = blocks[0]
    if len(blocks) > 1 or B.kind != 0:
        rows, sample_blocks, d_s = None, blocks, d
    else:
        rows = B.m
        d_s = d
        sample_blocks = blocks
    src = GradientSource(d_s, sample_blocks, L, seed=20251030)
    gr = [x.numpy() for x in src.grads(0)]
    o = oracle.OracleEF21M(d_s, sample_blocks, N=L, eta=0.1, r=4, seed=20251030)
    t0 = time.perf_counter()
    steps = 0
    while True:
        o.step(steps, gr)
        steps += 1
        el = time.perf_counter() - t0
        if el > budget_s or steps >= 20:
            break
    dt = el / steps
    return {"value": 4.0 * d_s * L / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"{steps} full step(s) of the workload ({d_s} elements x {L} node(s)), single thread, "
                      f"{dt:.2f} s/step"}


def run_baselines(args, d, blocks, L, N, world, rank, pg, pool, pool_n, dev, stream, barrier):
    """Baselines measured in the same run, same gradients:
    * dense_ef21m: EF21M with the identity compressor (one DENSE block: every row
      kept, the value exchange is an All-Reduce of all d entries; "Dense 2mn");
    * nccl_allreduce_d (G > 1): a bare ncclAllReduce of d fp32 per GPU;
    * allgather_topk: vanilla EF21M with per-node row Top-K, whose
      exchange is an All-Gather of K values rows plus K indices per node;
    * randk_shared_seed: Rand-K — the same path with data-independent rows;
    * noef_msgd: Table II's "(without EF)" compressed momentum SGD on the same selection."""
    import torch
    import torch.distributed as dist

    from paper_2510_26709_b200 import ArcTopK, Block
    steps = max(3, min(args.steps, 50))
    out = {}

    def timed(fn):
        for t in range(3):
            fn(t)
        torch.cuda.synchronize()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for k in range(steps):
            fn(3 + k)
        b.record(stream)
        b.synchronize()
        barrier()
        ms = a.elapsed_time(b) / steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return {"ms_per_step": ms, "value": 4.0 * d * N / (ms * 1e-3) / 1e9, "unit": "GB/s", "steps": steps}

    nd = 1024
    md = -(-d // nd)
    dense = [Block(0, d, md, nd, md, 1)]
    hs = [torch.zeros(d, device=dev) for _ in range(L)]
    gs = [torch.zeros(d, device=dev) for _ in range(L)]
    gb = torch.zeros(d, device=dev)
    ctx = ArcTopK(d, dense, N=N, eta=0.1, r=4, seed=20251030, nodes_local=L, pg=pg, rank=rank, reduce=args.reduce)
    out["dense_ef21m"] = timed(lambda t: ctx.step(t, pool[t % pool_n], hs, gs, gb))
    out["dense_ef21m"]["note"] = "identity compressor through the same library (DENSE block), fp32 All-Reduce of d"
    ctx.close()
    del hs, gs, gb
    if world > 1:
        buf = torch.zeros(d, device=dev)
        out["nccl_allreduce_d"] = timed(lambda t: dist.all_reduce(buf))
        out["nccl_allreduce_d"]["bus_GBps"] = 2 * (world - 1) / world * 4 * d / (out["nccl_allreduce_d"]["ms_per_step"] * 1e-3) / 1e9
    try:
        hs = [torch.zeros(d, device=dev) for _ in range(L)]
        gs = [torch.zeros(d, device=dev) for _ in range(L)]
        gb = torch.zeros(d, device=dev)
        ctx = ArcTopK(d, blocks, N=N, eta=0.1, r=4, seed=20251030, nodes_local=L, pg=pg, rank=rank,
                      method="topk_allgather")
        out["allgather_topk"] = timed(lambda t: ctx.step(t, pool[t % pool_n], hs, gs, gb))
        out["allgather_topk"]["note"] = "per-node exact row-norm Top-K, All-Gather of K n values + K indices per node"
        ctx.close()
    except Exception as e:  # not built yet / unsupported layout
        out["allgather_topk"] = {"unavailable": str(e)[:200]}
    ctx = ArcTopK(d, blocks, N=N, eta=0.1, r=4, seed=20251030, nodes_local=L, pg=pg, rank=rank, method="randk")
    out["randk_shared_seed"] = timed(lambda t: ctx.step(t, pool[t % pool_n], hs, gs, gb))
    out["randk_shared_seed"]["note"] = "Rand-K rows from a shared seed (Table I row Rand-K), same EF21M path, no sketch"
    ctx.close()
    try:
        ctx = ArcTopK(d, blocks, N=N, eta=0.9, r=4, seed=20251030, nodes_local=L, pg=pg, rank=rank, method="noef_msgd")
        out["noef_msgd"] = timed(lambda t: ctx.step(t, pool[t % pool_n], None, None, gb))
        out["noef_msgd"]["note"] = ("compressed momentum SGD without EF (Table II rows without EF): the ARC selection "
                                    "on the gradients, u = 0.9 u + C; 12 B per element instead of 16")
        ctx.close()
    except Exception as e:
        out["noef_msgd"] = {"unavailable": str(e)[:200]}
    if world == 1:   # exact-sketch test mode (every node local): Sigma from exact row norms of the node sum
        try:
            ctx = ArcTopK(d, blocks, N=N, eta=0.1, r=4, seed=20251030, nodes_local=L, method="exact")
            out["exact_sketch"] = timed(lambda t: ctx.step(t, pool[t % pool_n], hs, gs, gb))
            out["exact_sketch"]["note"] = ("test mode (SURVEY 8(b) ARC_SKETCH_EXACT): the sketch pass plus "
                                           "k_exact_sigma (re-reads h', g) instead of the Gaussian estimate")
            ctx.close()
        except Exception as e:
            out["exact_sketch"] = {"unavailable": str(e)[:200]}
    # the model update that consumes gbar: not part of the
    # compression step, timed on its own against the HBM roofline
    try:
        from paper_2510_26709_b200 import apply_update
        peak, _ = _peaks()
        x = torch.zeros(d, device=dev)
        mom = torch.zeros(d, device=dev)
        var = torch.zeros(d, device=dev)
        gb = pool[0][0]
        for name, nbytes, fn in [
                ("update_sgd", 12, lambda t: apply_update(x, gb, 1e-3, stream=stream)),
                ("update_adam", 28, lambda t: apply_update(x, gb, 1e-3, optimizer="adam", t=t + 1, m=mom, v=var,
                                                           stream=stream))]:
            r = timed(fn)
            gbs = nbytes * d / (r["ms_per_step"] * 1e-3) / 1e9
            out[name] = {"ms_per_step": r["ms_per_step"], "value": gbs, "unit": "GB/s", "steps": r["steps"],
                         "frac_of_hbm_peak": gbs / peak, "bytes_per_element": nbytes,
                         "note": "k_apply_%s over d (eq:ef21m-3 / Adam on gbar), algorithmic bytes / CUDA-event time"
                                 % name.split("_")[1]}
        del x, mom, var
    except Exception as e:
        out["update"] = {"unavailable": str(e)[:200]}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--nodes-per-gpu", type=int, default=1)
    ap.add_argument("--reduce", default="nccl", choices=["nccl", "ordered", "lsa"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--pool", type=int, default=8, help="distinct gradient sets cycled in the timed loop")
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--mu-bp", type=int, default=None, help="override K/m in basis points (e.g. 10, 100, 1000)")
    ap.add_argument("--force-exchange", action="store_true",
                    help="diagnostic: run the multi-GPU kernel sequence on one GPU (collectives become copies)")
    args = ap.parse_args()
    assert args.warmup >= 3, "W >= 3 warm-up steps"
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import __graft_entry__
    __graft_entry__.build()
    from paper_2510_26709_b200 import ArcTopK
    from paper_2510_26709_b200.ledger import arc_bus_bytes
    from synth import GradientSource

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1 or (args.force_exchange and args.reduce == "lsa"):
        # (one GPU, lsa: a real 1-rank communicator owns the symmetric window)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
        pg = dist.group.WORLD
    L = args.nodes_per_gpu
    d, blocks, N = workload(args.config, L, world, args.mu_bp)
    src = GradientSource(d, blocks, N, seed=20251030, device=dev)
    nodes = list(range(rank * L, (rank + 1) * L))
    # A pool of distinct gradient sets cycled step by step, like a training
    # stream (re-using one set would drive h and g to a fixed point where every
    # residual row is exactly 0: an all-ties degenerate workload).
    pool_n = max(1, min(args.pool, int((torch.cuda.mem_get_info(dev)[0] * 0.5) // (4 * d * L))))
    pool = [src.grads(t, nodes) for t in range(pool_n)]
    grads = pool[0]
    h = [torch.zeros(d, device=dev) for _ in range(L)]
    g = [torch.zeros(d, device=dev) for _ in range(L)]
    gbar = torch.zeros(d, device=dev)
    ctx = ArcTopK(d, blocks, N=N, eta=0.1, r=4, seed=20251030, nodes_local=L, pg=pg, rank=rank,
                  reduce=args.reduce, host_staging=True, force_exchange=args.force_exchange)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    # ---------------------------------------------------------------- device-timed steps
    for t in range(args.warmup):
        ctx.step(t, pool[t % pool_n], h, g, gbar)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for k in range(args.steps):
            t = args.warmup + k
            ctx.step(t, pool[t % pool_n], h, g, gbar)
        e1.record(stream)
        e1.synchronize()
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    # second timed pass of K steps with CUDA events between the step's phases
    # (on the step's stream): per-kernel durations for the roofline.  Kept out of
    # the pass above because each event pair adds ~2-3 us to the step.
    ctx.read_timing()
    ctx.set_timing(True)
    for k in range(args.steps):
        t = args.warmup + args.steps + k
        ctx.step(t, pool[t % pool_n], h, g, gbar)
    phases_sum, nsteps = ctx.read_timing()
    ctx.set_timing(False)
    phase_ms = {k: v / max(nsteps, 1) for k, v in phases_sum.items()}
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = 4.0 * d * N / (ms * 1e-3) / 1e9

    # ---------------------------------------------------------------- end-to-end (host gradients)
    host = [x.cpu().pin_memory() for x in grads]
    sel_h = torch.empty(ctx.sum_K, dtype=torch.int32).pin_memory()
    val_h = torch.empty(ctx.sum_Kn, dtype=torch.float32).pin_memory()
    e2e_steps = max(1, min(args.e2e_steps, args.steps))
    for t in range(3):
        ctx.step_host(t, host, h, g, gbar, sel_h, val_h)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for k in range(e2e_steps):
        ctx.step_host(1000 + k, host, h, g, gbar, sel_h, val_h)
    f1.record(stream)
    f1.synchronize()
    barrier()
    e2e_ms = f0.elapsed_time(f1) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = 4.0 * d * N / (e2e_ms * 1e-3) / 1e9
    st = ctx.status()

    # ---------------------------------------------------------------- roofline
    peak, peak_src = _peaks()
    ab = algorithmic_bytes(d, blocks, L, 4)
    sk_ms = phase_ms["ef_sketch"]
    achieved = ab["ef_sketch"] / (sk_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_ef_sketch.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            if pj.get("workload") == args.config and pj.get("nodes_per_gpu", 1) == L:
                traffic = pj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    M = sum(b.m for b in blocks if b.kind == 0)
    kn = sum(b.K * b.n for b in blocks)
    bus = arc_bus_bytes(M, kn, 4, world, L, args.reduce)
    nvl_peak = 770.0  # GB/s per direction, measured peer copy (B200_PROFILING.md)
    t_roof = ab["total"] / (peak * 1e9) + bus["total"] / (nvl_peak * 1e9)
    launches = ctx.kernels_per_step * args.steps

    # ---------------------------------------------------------------- baselines (same run)
    baselines = {}
    if not args.no_baselines:
        try:
            baselines = run_baselines(args, d, blocks, L, N, world, rank, pg, pool, pool_n, dev, stream, barrier)
        except Exception as e:  # a baseline must never cost the headline line
            baselines = {"error": f"{type(e).__name__}: {str(e)[:300]}"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(d, blocks, L)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config}: GPT-2-small-sized gradient d={d}, n={blocks[0].n}, "
                                   f"K=1% ({blocks[0].K} rows), r=4, eta=0.1, one paper node per GPU"
                                   if args.config == "C3" and args.mu_bp is None else
                                   f"{args.config}: d={d}, {len(blocks)} block(s), sum K={sum(b.K for b in blocks)}, "
                                   f"mu_bp={args.mu_bp}, r=4, eta=0.1, {L} node(s) per GPU",
                       "d": d, "N_nodes": N, "nodes_per_gpu": L, "reduce": args.reduce,
                       "parallelism": f"dp{world}",
                       "l2": "no flush: per-step inputs (16 B x d = %.1f GB) exceed the 126 MB L2" % (16 * d / 1e9),
                       "gradient_pool": pool_n},
            "roofline": {"bound": "hbm", "kernel": "k_ef_sketch", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": ab["ef_sketch"], "peak_source": peak_src,
                         "launch_ms": sk_ms,
                         # also against the nominal HBM3e figure (HGX B200, 7.7 TB/s)
                         "nominal_peak": 7700.0, "nominal_frac": achieved / 7700.0},
            "step_roofline": {"t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms,
                              "hbm_bytes": ab["total"], "nvlink_bus_bytes": bus["total"]},
            "phases_ms": phase_ms,
            "baselines": baselines,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "GB/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": 4 * d * L, "d2h_bytes_per_step": 4 * ctx.sum_K + 4 * ctx.sum_Kn},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "status_flags": st,
        }
        print(json.dumps(line))
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
