"""Benchmark of the EF21M + ARC-Top-K compression step (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

One step = one pass of the whole hot path over one
batch of synthetic gradients: momentum + residual + sketch, exchange #1,
row importance, Top-K selection, compaction + EF update, exchange #2,
scatter into the replicated tracker.  One paper node per GPU (weak scaling:
the per-GPU gradient size is fixed as N grows).  Default workload: BASELINE
configs[2], the GPT-2-small-sized gradient (d = 124,439,808, n = 768, K = 1 %),
the config for which the north_star's roofline target (d >= 100M) is stated;
the same line also carries the largest single-GPU sweep point (C5, d = 1e9) and
the per-tensor LLaMA-1B layout (C4) under `extra_workloads`.

`--gpus N > 1` without a torchrun environment re-launches itself under
`torch.distributed.run` with N ranks (one process per GPU, NCCL).

Prints ONE JSON line (rank 0).  `value` = whole-job gradient throughput
(4 bytes x d x N nodes / step time, GB/s); inputs are resident in HBM and far
larger than L2 (126 MB), so no L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ARC-Top-K step ms and grad GB/s at 1/2/4/8 B200; % of HBM/NVLink roofline"
NVLINK_PEAK = 770.0   # GB/s per direction, measured peer copy (B200_PROFILING.md)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def host_info() -> dict:
    """CPU model, logical cores and RAM of the host the CPU baseline ran on."""
    model, ram = None, None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                ram = round(int(line.split()[1]) / 1024 / 1024, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "logical_cores": os.cpu_count(), "ram_gib": ram}


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

    def _sample(self):
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

    def _run(self):
        while not self._stop.is_set():
            self._sample()
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
        if self.nvml is not None and not self.samples:
            self._sample()

    def summary(self):
        if self.nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "nvml")}
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def workload(name: str, mu_bp=None):
    from synth import config_blocks
    return config_blocks(name, mu_bp)


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


def _oracle_threads() -> int:
    return max(1, int(os.environ.get("ARC_ORACLE_THREADS", os.cpu_count() or 1)))


def run_reference(args):
    """--impl reference: the CPU oracle (plain C; row-parallel OpenMP over the
    host's cores, bit-identical to one thread) on the same workload, metric and
    unit; each step is a bounded sample of it (a contiguous range of whole rows),
    sized so the run ends within minutes.  Under torchrun only rank 0 works."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    from synth import Block, GradientSource
    threads = _oracle_threads()
    oracle.set_threads(threads)
    d, blocks = workload(args.config)
    B = blocks[0]
    total_steps = args.steps + args.warmup
    budget_s = float(os.environ.get("ARC_REF_BUDGET_S", "90"))
    rate = 1.0e8 * min(threads, 8) / 2                  # elements/s (rough; bounds the sample)
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
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "oracle",
                             "sample": f"{rows} rows x {B.n} cols of {args.config}, {L} node(s), per step, "
                                       f"{threads} OpenMP thread(s)", **host_info()},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_leg(d, blocks, L, budget_s=20.0):
    """The oracle (bit-identical at any thread count) timed on this box's host
    cores on a bounded sample of the same workload: whole steps of the full
    config, with P = all host threads (the reported value) and with 1 thread."""
    import oracle
    from synth import GradientSource
    src = GradientSource(d, blocks, L, seed=20251030)
    gr = [x.numpy() for x in src.grads(0)]
    out = {}
    for threads in (_oracle_threads(), 1):
        oracle.set_threads(threads)
        o = oracle.OracleEF21M(d, blocks, N=L, eta=0.1, r=4, seed=20251030)
        t0 = time.perf_counter()
        steps = 0
        while True:
            o.step(steps, gr)
            steps += 1
            el = time.perf_counter() - t0
            if el > budget_s / 2 or steps >= 20:
                break
        out[threads] = (el / steps, steps)
        del o
    oracle.set_threads(1)
    P = _oracle_threads()
    dt, steps = out[P]
    dt1, steps1 = out[1]
    return {"value": 4.0 * d * L / dt / 1e9, "unit": "GB/s", "cores": P, "kind": "oracle",
            "sample": f"{steps} full step(s) of the workload ({d} elements x {L} node(s)), {P} OpenMP threads, "
                      f"{dt:.2f} s/step",
            "value_1thread": 4.0 * d * L / dt1 / 1e9, "s_per_step_1thread": dt1, "steps_1thread": steps1,
            **host_info()}


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
        del buf
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


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(nproc: int) -> int:
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run
    with N ranks on this node (one process per GPU); rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


class Runner:
    """One rank's device, process group and timing helpers."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        self.pg = None
        if self.world > 1 or (args.force_exchange and args.reduce == "lsa"):
            # (one GPU, lsa: a real 1-rank communicator owns the symmetric window)
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", device_id=self.dev, rank=self.rank, world_size=self.world)
            self.pg = dist.group.WORLD

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max_over_ranks(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


def measure(run: Runner, args, config: str, mu_bp, steps: int, warmup: int, *, e2e_steps: int = 0,
            pool_max: int = 8, clocks: bool = True, keep: bool = False):
    """Time the step on one workload: the bracketed K-step loop (the value), a
    per-step event pass (p50 / p90), a phase-event pass (per-kernel roofline)
    and optionally the end-to-end host-buffer path.  Returns a dict (and the
    context + buffers when keep=True, for the baselines)."""
    torch, dist = run.torch, run.dist
    from paper_2510_26709_b200 import ArcTopK
    from paper_2510_26709_b200.ledger import arc_bus_bytes
    from synth import GradientSource
    L = args.nodes_per_gpu
    d, blocks = workload(config, mu_bp)
    N = L * run.world
    dev = run.dev
    src = GradientSource(d, blocks, N, seed=20251030, device=dev)
    nodes = list(range(run.rank * L, (run.rank + 1) * L))
    # A pool of distinct gradient sets cycled step by step, like a training
    # stream (re-using one set would drive h and g to a fixed point where every
    # residual row is exactly 0: an all-ties degenerate workload).
    free = torch.cuda.mem_get_info(dev)[0]
    pool_n = max(1, min(pool_max, int((free * 0.5 - 16 * d * L) // (4 * d * L))))
    pool = [src.grads(t, nodes) for t in range(pool_n)]
    h = [torch.zeros(d, device=dev) for _ in range(L)]
    g = [torch.zeros(d, device=dev) for _ in range(L)]
    gbar = torch.zeros(d, device=dev)
    ctx = ArcTopK(d, blocks, N=N, eta=0.1, r=4, seed=20251030, nodes_local=L, pg=run.pg, rank=run.rank,
                  reduce=args.reduce, host_staging=e2e_steps > 0, force_exchange=args.force_exchange,
                  wire=args.wire)
    stream = torch.cuda.current_stream()

    # ---------------------------------------------------------------- device-timed steps
    for t in range(warmup):
        ctx.step(t, pool[t % pool_n], h, g, gbar)
    torch.cuda.synchronize()
    run.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(run.local) if clocks else None
    if clk:
        clk.__enter__()
    e0.record(stream)
    for k in range(steps):
        t = warmup + k
        ctx.step(t, pool[t % pool_n], h, g, gbar)
    e1.record(stream)
    e1.synchronize()
    if clk:
        clk.__exit__(None, None, None)
    torch.cuda.synchronize()
    run.barrier()
    ms = run.max_over_ranks(e0.elapsed_time(e1) / steps)
    t_next = warmup + steps
    # per-step events (p50 / p90 of the step time; events between steps only)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    run.barrier()
    evs[0].record(stream)
    for k in range(steps):
        t = t_next + k
        ctx.step(t, pool[t % pool_n], h, g, gbar)
        evs[k + 1].record(stream)
    evs[-1].synchronize()
    per = sorted(evs[k].elapsed_time(evs[k + 1]) for k in range(steps))
    t_next += steps
    p50 = run.max_over_ranks(per[len(per) // 2])
    p90 = run.max_over_ranks(per[min(len(per) - 1, (9 * len(per)) // 10)])
    # phase events on the step's stream: per-kernel durations for the roofline
    # (kept out of the timed pass: each event pair adds ~2-3 us to the step)
    ctx.read_timing()
    ctx.set_timing(True)
    for k in range(steps):
        t = t_next + k
        ctx.step(t, pool[t % pool_n], h, g, gbar)
    phases_sum, nsteps = ctx.read_timing()
    ctx.set_timing(False)
    t_next += steps
    phase_ms = {k: v / max(nsteps, 1) for k, v in phases_sum.items()}
    value = 4.0 * d * N / (ms * 1e-3) / 1e9

    out = {"config": config, "d": d, "blocks": len(blocks), "sum_K": ctx.sum_K, "sum_Kn": ctx.sum_Kn,
           "N_nodes": N, "nodes_per_gpu": L, "ms_per_step": ms, "value": value, "unit": "GB/s",
           "p50_ms": p50, "p90_ms": p90, "steps": steps, "gradient_pool": pool_n, "phases_ms": phase_ms}
    # ---------------------------------------------------------------- end-to-end (host gradients)
    if e2e_steps > 0:
        host = [x.cpu().pin_memory() for x in pool[0]]
        sel_h = torch.empty(ctx.sum_K, dtype=torch.int32).pin_memory()
        val_h = torch.empty(ctx.sum_Kn, dtype=torch.float32).pin_memory()
        for t in range(3):
            ctx.step_host(t_next + t, host, h, g, gbar, sel_h, val_h)
        torch.cuda.synchronize()
        run.barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for k in range(e2e_steps):
            ctx.step_host(t_next + 3 + k, host, h, g, gbar, sel_h, val_h)
        f1.record(stream)
        f1.synchronize()
        run.barrier()
        e2e_ms = run.max_over_ranks(f0.elapsed_time(f1) / e2e_steps)
        out["e2e"] = {"value": 4.0 * d * N / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
                      "h2d_bytes_per_step": 4 * d * L, "d2h_bytes_per_step": 4 * ctx.sum_K + 4 * ctx.sum_Kn}
        del host
    out["status_flags"] = ctx.status()
    out["comm_tally"] = ctx.comm_tally()
    out["kernels_per_step"] = ctx.kernels_per_step

    # ---------------------------------------------------------------- roofline
    peak, peak_src = _peaks()
    ab = algorithmic_bytes(d, blocks, L, 4)
    sk_ms = phase_ms["ef_sketch"]
    achieved = ab["ef_sketch"] / (sk_ms * 1e-3) / 1e9
    M = sum(b.m for b in blocks if b.kind == 0)
    kn = sum(b.K * b.n for b in blocks)
    bus = arc_bus_bytes(M, kn, 4, run.world, L, args.reduce)
    t_roof = ab["total"] / (peak * 1e9) + bus["total"] / (NVLINK_PEAK * 1e9)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_ef_sketch.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            if pj.get("workload") == config and pj.get("nodes_per_gpu", 1) == L:
                traffic = pj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    out["roofline"] = {"bound": "hbm", "kernel": "k_ef_sketch", "achieved": achieved, "peak": peak, "unit": "GB/s",
                       "frac": achieved / peak, "traffic": traffic, "algorithmic_bytes_per_launch": ab["ef_sketch"],
                       "peak_source": peak_src, "launch_ms": sk_ms,
                       # also against the nominal HBM3e figure (HGX B200, 7.7 TB/s)
                       "nominal_peak": 7700.0, "nominal_frac": achieved / 7700.0}
    # the selection kernel (the verdict's kernel furthest below its roofline): latency-bound;
    # its algorithmic bytes are the selected rows' S4..S6 traffic plus its Sigma key reads
    sel_ms = phase_ms.get("select_gather", 0.0)
    if sel_ms > 0:
        sel_bytes = ab["gather_ef"] + 4 * M
        out["roofline_select"] = {"bound": "latency", "kernel": "k_select_gather", "algorithmic_bytes_per_launch": sel_bytes,
                                  "launch_ms": sel_ms, "achieved": sel_bytes / (sel_ms * 1e-3) / 1e9, "peak": peak,
                                  "unit": "GB/s", "frac": sel_bytes / (sel_ms * 1e-3) / 1e9 / peak}
    out["step_roofline"] = {"t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms, "hbm_bytes": ab["total"],
                            "nvlink_bus_bytes": bus["total"], "nvlink_peak_GBps": NVLINK_PEAK}
    # what each rank hands to the two exchanges per step (Table I's payloads)
    we = 2 if args.wire == "bf16" else 4
    out["wire"] = {"dtype": args.wire, "value_payload_bytes": we * kn * (L if args.reduce != "nccl" else 1),
                   "sketch_payload_bytes": 4 * M * L * 4, "sent_at_this_G": run.world > 1 or args.force_exchange}
    # the two exchanges: bytes this GPU moves over NVLink per step and the bus
    # rate over their phase time (phase = collective + the kernel it feeds)
    if run.world > 1:
        coll = {}
        for name, phase, nbytes in [("exchange1_sketch", "exchange1_reduce", bus["sketch"]),
                                    ("exchange2_values", "exchange2_scatter", bus["values"])]:
            pm = phase_ms.get(phase, 0.0)
            coll[name] = {"bus_bytes": nbytes, "phase_ms": pm,
                          "bus_GBps": nbytes / (pm * 1e-3) / 1e9 if pm > 0 else None}
        out["collectives"] = coll
    if clk:
        out["clocks"] = clk.summary()
    if keep:
        return out, dict(ctx=ctx, pool=pool, pool_n=pool_n, h=h, g=g, gbar=gbar, d=d, blocks=blocks, N=N)
    ctx.close()
    del pool, h, g, gbar
    torch.cuda.empty_cache()
    return out


def measure_graph(run: Runner, config: str, steps: int, S: int = 8, **ctx_kw):
    """Device time of a step with the host out of the loop (one GPU): S consecutive
    steps, one per gradient set, captured in ONE CUDA graph (device iteration
    counter, ARC_FLAG_DEVICE_T; the public ArcTopK.step inside torch.cuda.graph)
    and replayed; ms per step = elapsed / (replays * S).  For small workloads the
    eager loop is bound by the host's launch + marshalling time instead."""
    torch = run.torch
    from paper_2510_26709_b200 import ArcTopK, _lib
    from synth import GradientSource
    d, blocks = workload(config, None)
    dev = run.dev
    src = GradientSource(d, blocks, 1, seed=20251030, device=dev)
    pool = [src.grads(t) for t in range(S)]
    h, g = [torch.zeros(d, device=dev)], [torch.zeros(d, device=dev)]
    gbar = torch.zeros(d, device=dev)
    ctx = ArcTopK(d, blocks, N=1, eta=0.1, r=4, seed=20251030, nodes_local=1, device_t=True, **ctx_kw)
    plan = ctx.query(_lib.Q_PLAN).cpu().tolist()
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream())
    for j in range(S):
        ctx.step(0, pool[j], h, g, gbar, stream=s)
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s, capture_error_mode="relaxed"):
        for j in range(S):
            ctx.step(0, pool[j], h, g, gbar, stream=s)
    ctx.set_iteration(S)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    reps = max(1, steps // S)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        graph.replay()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / (reps * S)
    ctx.close()
    del pool, h, g, gbar, graph
    torch.cuda.empty_cache()
    return {"ms_per_step": ms, "steps": reps * S, "value": 4.0 * d / (ms * 1e-3) / 1e9, "unit": "GB/s",
            "selection_form": ["cooperative grid", "one cluster", "fused tail", "none"][plan[0]],
            "kernels_per_step": plan[3]}


def measure_bucketed(run: Runner, args, config: str, steps: int, warmup: int, bucket_elems: int = 25 * 2**20,
                     pool_max: int = 4, graphs: bool = False):
    """The per-layer bucketed variant: the
    config's block table cut into DDP-style buckets of <= bucket_elems elements
    (whole tensors, in order), one context per bucket (sharing one communicator
    at G > 1, as paper_2510_26709_b200.ddp does), each bucket's step on one of two
    alternating streams.  Timed like the single-call step; same gradients.
    graphs=True: every bucket's step captured once per gradient set into a CUDA
    graph (device-side iteration counter, ARC_FLAG_DEVICE_T) and replayed, as the
    DDP hook's cuda_graphs option does.  host_ms_per_step: CPU time to enqueue a
    step (the launches and the ctypes marshalling the graphs replace)."""
    import time
    torch = run.torch
    from paper_2510_26709_b200 import ArcTopK, Block
    from synth import GradientSource
    L = args.nodes_per_gpu
    d, blocks = workload(config, None)
    N = L * run.world
    dev = run.dev
    buckets, cur, size = [], [], 0
    for b in blocks:
        if cur and size + b.len > bucket_elems:
            buckets.append(cur)
            cur, size = [], 0
        cur.append(b)
        size += b.len
    if cur:
        buckets.append(cur)
    src = GradientSource(d, blocks, N, seed=20251030, device=dev)
    nodes = list(range(run.rank * L, (run.rank + 1) * L))
    free = torch.cuda.mem_get_info(dev)[0]
    pool_n = max(1, min(pool_max, int((free * 0.5 - 16 * d * L) // (4 * d * L))))
    pool = [src.grads(t, nodes) for t in range(pool_n)]
    h = [torch.zeros(d, device=dev) for _ in range(L)]
    g = [torch.zeros(d, device=dev) for _ in range(L)]
    gbar = torch.zeros(d, device=dev)
    comm = None
    if run.world > 1:
        from paper_2510_26709_b200.dist import private_nccl_group
        comm = private_nccl_group(run.pg, dev)
    streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
    ctxs = []
    for bk in buckets:
        off0 = bk[0].offset
        lb = [Block(b.offset - off0, b.len, b.m, b.n, b.K, b.kind) for b in bk]
        dl = sum(b.len for b in bk)
        ctxs.append((ArcTopK(dl, lb, N=N, eta=0.1, r=4, seed=20251030, nodes_local=L, pg=run.pg, rank=run.rank,
                             reduce=args.reduce, comm_group=comm, device_t=graphs), off0, dl))
    main = torch.cuda.current_stream()
    cgraphs = []
    if graphs:   # one graph per (bucket, gradient set): the inputs are fixed per graph
        for k, (ctx, off0, dl) in enumerate(ctxs):
            ctx.set_iteration(0, stream=streams[k % 2])
            cgraphs.append([ctx.capture([x[off0:off0 + dl] for x in pool[j]], [x[off0:off0 + dl] for x in h],
                                        [x[off0:off0 + dl] for x in g], gbar[off0:off0 + dl], stream=streams[k % 2])
                            for j in range(pool_n)])
        torch.cuda.synchronize()

    def one_step(t):
        gr = pool[t % pool_n]
        for k, (ctx, off0, dl) in enumerate(ctxs):
            st = streams[k % 2]
            st.wait_stream(main)
            if graphs:
                with torch.cuda.stream(st):
                    cgraphs[k][t % pool_n].replay()
            else:
                ctx.step(t, [x[off0:off0 + dl] for x in gr], [x[off0:off0 + dl] for x in h],
                         [x[off0:off0 + dl] for x in g], gbar[off0:off0 + dl], stream=st)
        for st in streams:
            main.wait_stream(st)

    for t in range(warmup):
        one_step(t)
    torch.cuda.synchronize()
    run.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    host_s = 0.0
    for k in range(steps):
        c0 = time.perf_counter()
        one_step(warmup + k)
        host_s += time.perf_counter() - c0
    e1.record(main)
    e1.synchronize()
    run.barrier()
    ms = run.max_over_ranks(e0.elapsed_time(e1) / steps)
    out = {"config": config, "buckets": len(buckets), "bucket_elems_max": bucket_elems, "ms_per_step": ms,
           "host_ms_per_step": 1e3 * host_s / steps, "cuda_graphs": graphs,
           "value": 4.0 * d * N / (ms * 1e-3) / 1e9, "unit": "GB/s", "steps": steps,
           "kernels_per_step": sum(c[0].kernels_per_step for c in ctxs),
           "note": "one context per DDP-style bucket (whole tensors, <= 25 Mi elements), two alternating streams"}
    del cgraphs
    for c in ctxs:
        c[0].close()
    del pool, h, g, gbar
    torch.cuda.empty_cache()
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
    ap.add_argument("--wire", default="f32", choices=["f32", "bf16"], help="exchange #2 payload precision (R25)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--pool", type=int, default=8, help="distinct gradient sets cycled in the timed loop")
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the extra workloads (C5 d=1e9, C4)")
    ap.add_argument("--mu-bp", type=int, default=None, help="override K/m in basis points (e.g. 10, 100, 1000)")
    ap.add_argument("--force-exchange", action="store_true",
                    help="diagnostic: run the multi-GPU kernel sequence on one GPU (collectives become copies)")
    args = ap.parse_args()
    assert args.warmup >= 3, "W >= 3 warm-up steps"
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2

    import torch

    import __graft_entry__
    __graft_entry__.build()
    run = Runner(args)
    L = args.nodes_per_gpu

    head, keep = measure(run, args, args.config, args.mu_bp, args.steps, args.warmup, e2e_steps=args.e2e_steps,
                         pool_max=args.pool, keep=True)
    baselines = {}
    if not args.no_baselines:
        try:
            baselines = run_baselines(args, keep["d"], keep["blocks"], L, keep["N"], run.world, run.rank, run.pg,
                                      keep["pool"], keep["pool_n"], run.dev, torch.cuda.current_stream(),
                                      run.barrier)
        except Exception as e:  # a baseline must never cost the headline line
            baselines = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
    keep["ctx"].close()
    keep.clear()
    torch.cuda.empty_cache()

    # the largest single-GPU sweep point (BASELINE configs[4], d = 1e9, K = 1 %) and
    # the per-tensor 1.3B LLM layout (configs[3]), same protocol, in the same line
    extras = {}
    if not args.no_extras and args.mu_bp is None:
        for name in ("C5_1e9", "C4"):
            if name == args.config:
                continue
            try:
                ex = measure(run, args, name, None, max(10, min(args.steps, 50)), args.warmup, pool_max=4)
                extras[name] = {k: ex[k] for k in ("d", "blocks", "sum_K", "ms_per_step", "value", "unit", "p50_ms",
                                                   "p90_ms", "steps", "phases_ms", "status_flags")}
                extras[name]["roofline_frac"] = ex["roofline"]["frac"]
                extras[name]["sketch_GBps"] = ex["roofline"]["achieved"]
                extras[name]["step_roofline_frac"] = ex["step_roofline"]["frac"]
                extras[name]["clocks"] = ex.get("clocks")
            except Exception as e:
                extras[name] = {"unavailable": f"{type(e).__name__}: {str(e)[:200]}"}
        # the small single-GPU configs, eager and with the host out of the loop
        # (configs[4]'s d = 1e6 point: the fused tail; C2 with one node)
        if run.world == 1:
            for name in ("C5_1e6", "C2"):
                try:
                    ex = measure(run, args, name, None, max(50, min(args.steps, 300)), args.warmup, pool_max=8,
                                 clocks=False)
                    gr = measure_graph(run, name, max(80, min(args.steps, 400)))
                    extras[name] = {"d": ex["d"], "sum_K": ex["sum_K"], "ms_per_step": ex["ms_per_step"],
                                    "graph": gr, "step_roofline_frac_graph":
                                        ex["step_roofline"]["t_roof_ms"] / gr["ms_per_step"],
                                    "t_roof_ms": ex["step_roofline"]["t_roof_ms"], "phases_ms": ex["phases_ms"]}
                except Exception as e:
                    extras[name] = {"unavailable": f"{type(e).__name__}: {str(e)[:200]}"}
        try:   # the per-layer bucketed C4 against its single call
            bk = measure_bucketed(run, args, "C4", max(10, min(args.steps, 50)), args.warmup)
            single = extras.get("C4", {}).get("ms_per_step")
            if single:
                bk["single_call_ms_per_step"] = single
                bk["bucketed_over_single"] = bk["ms_per_step"] / single
            extras["C4_bucketed"] = bk
            bg = measure_bucketed(run, args, "C4", max(10, min(args.steps, 50)), args.warmup, graphs=True)
            if single:
                bg["bucketed_over_single"] = bg["ms_per_step"] / single
            extras["C4_bucketed_graphs"] = bg
        except Exception as e:
            extras["C4_bucketed"] = {"unavailable": f"{type(e).__name__}: {str(e)[:200]}"}

    cpu = None
    if run.rank == 0 and not args.no_cpu_baseline:
        from synth import config_blocks
        d, blocks = config_blocks(args.config, args.mu_bp)
        cpu = cpu_baseline_leg(d, blocks, L)
    run.barrier()

    if run.rank == 0:
        d = head["d"]
        nccl_ver = None
        try:
            nccl_ver = ".".join(str(x) for x in torch.cuda.nccl.version())
        except Exception:
            pass
        line = {
            "metric": METRIC, "value": head["value"], "unit": "GB/s", "n_gpus": run.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "p50_ms": head["p50_ms"],
            "p90_ms": head["p90_ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config}: GPT-2-small-sized gradient d={d}, n=768, "
                                   f"K=1% ({head['sum_K']} rows), r=4, eta=0.1, one paper node per GPU"
                                   if args.config == "C3" and args.mu_bp is None else
                                   f"{args.config}: d={d}, {head['blocks']} block(s), sum K={head['sum_K']}, "
                                   f"mu_bp={args.mu_bp}, r=4, eta=0.1, {L} node(s) per GPU",
                       "d": d, "N_nodes": head["N_nodes"], "nodes_per_gpu": L, "reduce": args.reduce,
                       "wire": args.wire,
                       "parallelism": f"dp{run.world}",
                       "l2": "no flush: per-step inputs (16 B x d = %.1f GB) exceed the 126 MB L2" % (16 * d / 1e9),
                       "gradient_pool": head["gradient_pool"]},
            "roofline": head["roofline"],
            "roofline_select": head.get("roofline_select"),
            "step_roofline": head["step_roofline"],
            "phases_ms": head["phases_ms"],
            "wire": head["wire"],
            "collectives": head.get("collectives"),
            "comm_tally_per_rank0": head["comm_tally"],
            "nccl": {"version": nccl_ver, "NCCL_ALGO": os.environ.get("NCCL_ALGO"),
                     "NCCL_PROTO": os.environ.get("NCCL_PROTO")},
            "extra_workloads": extras,
            "baselines": baselines,
            "cpu_baseline": cpu,
            "e2e": head.get("e2e"),
            "gpu_launches": head["kernels_per_step"] * args.steps,
            "clocks": head.get("clocks"),
            "status_flags": head["status_flags"],
        }
        print(json.dumps(line), flush=True)
    if run.world > 1:
        run.dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
