"""EF21M + ARC-Top-K as a PyTorch DDP communication hook.

Every DDP gradient bucket gets its own compression context (per-tensor blocks
in the bucket's order: each 2-D (or conv) tensor is an ARC block of rows =
output units, every other tensor a DENSE block — P:510 "we compress only
two-dimensional tensors"; per-tensor K).  The hook returns the
bucket's replicated tracker gbar = (1/N) sum_i g_i, so the optimizer that
follows applies x <- x - gamma gbar (eq:ef21m-3) — or Adam on gbar, as
in the paper's experiments.

For the first `warmup_steps` iterations the hook averages the gradients
densely (the paper starts compression after 1000 iterations).  The
EF21M state of a context is initialised at the first compressed iteration it
sees — h = g = the local gradient, gbar = their average (V_0 = 0, the Theorem 1
setting) — so a bucket that DDP rebuilds (it re-buckets once after its
first iteration) restarts from that state instead of from zeros.

Scaling (one process per GPU):
  * one library communicator for every bucket (made once per hook state with
    ``dist.private_nccl_group``) instead of one per bucket context;
  * two side streams, alternating by bucket index: bucket b+1's streaming pass
    (S1, HBM-bound) runs while bucket b's exchanges (S2, S5) wait on NVLink.
    NCCL keeps one communicator's operations in issue order, and every rank
    issues the buckets in the same order, as NCCL requires.
Each side stream first waits for the backward stream, so a bucket's
compression also overlaps the backward pass of the layers still to come; the
returned future carries the side stream's completion.

With ``cuda_graphs=True`` each bucket's step is captured once into a CUDA graph
and replayed every iteration (one host launch per bucket instead of the step's
kernel launches and argument marshalling); the iteration t lives in device
memory and advances with each replay (the library's ARC_FLAG_DEVICE_T).

    from paper_2510_26709_b200.ddp import ArcTopKHookState, arc_topk_hook
    state = ArcTopKHookState(mu_bp=100, eta=0.1, r=4, seed=1234, warmup_steps=1000)
    ddp_model.register_comm_hook(state, arc_topk_hook)
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .api import ArcTopK, Block
from . import _lib as L


def bucket_layout(shapes, mu_bp: int, dense_n: int = 1024) -> tuple[int, list[Block]]:
    """Blocks for tensors laid out back to back in this order."""
    blocks, off = [], 0
    for s in shapes:
        numel = 1
        for x in s:
            numel *= int(x)
        if len(s) >= 2 and numel > 0:
            m, n = int(s[0]), numel // int(s[0])
            K = max(1, min(m, -(-m * int(mu_bp) // 10000)))
            blocks.append(Block(off, numel, m, n, K, L.BLOCK_ARC))
        elif numel > 0:
            n = min(numel, dense_n)
            m = -(-numel // n)
            blocks.append(Block(off, numel, m, n, m, L.BLOCK_DENSE))
        off += numel
    return off, blocks


class ArcTopKHookState:
    """Hook state: compression settings, one context and EF21M state per bucket,
    the shared library communicator and the two side streams."""

    NUM_STREAMS = 2

    def __init__(self, mu_bp: int = 100, eta: float = 0.1, r: int = 4, seed: int = 20251030,
                 warmup_steps: int = 0, process_group=None, reduce: str = "nccl", cuda_graphs: bool = False):
        self.mu_bp, self.eta, self.r, self.seed = int(mu_bp), float(eta), int(r), int(seed)
        self.cuda_graphs = bool(cuda_graphs)
        self.warmup_steps = int(warmup_steps)
        self.pg = process_group
        self.reduce = reduce
        self.iteration = 0
        self.buckets: dict[int, dict] = {}
        self._streams: list[torch.cuda.Stream] = []
        self._comm = None
        self.contexts_created = 0

    def world(self) -> int:
        return dist.get_world_size(self.pg) if dist.is_initialized() else 1

    def stream(self, device, index: int) -> torch.cuda.Stream:
        if not self._streams:
            self._streams = [torch.cuda.Stream(device=device) for _ in range(self.NUM_STREAMS)]
        return self._streams[index % len(self._streams)]

    def comm_group(self, pg, device):
        """The one NCCL group every bucket's context uses (collective on first use:
        every rank reaches it at the same bucket of the same iteration)."""
        if self._comm is None:
            from .dist import private_nccl_group
            self._comm = private_nccl_group(pg, device)
        return self._comm

    def context(self, index: int, bucket) -> tuple[dict, bool]:
        """The bucket's context; fresh = True when it was (re)created now."""
        b = self.buckets.get(index)
        buf = bucket.buffer()
        shapes = [tuple(p.shape) for p in bucket.parameters()]
        if b is not None and b["shapes"] == shapes:
            return b, False
        # new bucket (DDP rebuilds its buckets once, early)
        if b is not None:
            b["ctx"].close()
        d, blocks = bucket_layout(shapes, self.mu_bp)
        assert d == buf.numel(), "bucket buffer does not match its parameters"
        N = self.world()
        pg = self.pg if self.pg is not None else (dist.group.WORLD if N > 1 else None)
        comm = self.comm_group(pg, buf.device) if pg is not None and N > 1 else None
        ctx = ArcTopK(d, blocks, N=N, eta=self.eta, r=self.r, seed=self.seed + 7919 * index, nodes_local=1,
                      pg=pg, rank=dist.get_rank(pg) if pg is not None else 0, reduce=self.reduce,
                      device=buf.device, comm_group=comm, device_t=self.cuda_graphs)
        b = {"d": d, "ctx": ctx, "h": torch.zeros_like(buf), "g": torch.zeros_like(buf),
             "gbar": torch.zeros_like(buf), "shapes": shapes, "blocks": blocks}
        self.buckets[index] = b
        self.contexts_created += 1
        return b, True


def arc_topk_hook(state: ArcTopKHookState, bucket) -> torch.futures.Future:
    """DDP comm hook: dense average during warm-up, then one EF21M + ARC-Top-K step
    per bucket; the bucket's gradient becomes gbar."""
    buf = bucket.buffer()
    device = buf.device
    idx = bucket.index()
    t = state.iteration
    if bucket.is_last():
        state.iteration += 1
    N = state.world()
    main = torch.cuda.current_stream(device)
    side = state.stream(device, idx)
    side.wait_stream(main)
    fut = torch.futures.Future(devices=[device])
    with torch.cuda.stream(side):
        buf.record_stream(side)
        if t < state.warmup_steps:
            if N > 1:
                dist.all_reduce(buf, group=state.pg)
                buf.div_(N)
        else:
            b, fresh = state.context(idx, bucket)
            if fresh:                             # EF21M start: h = g = local gradient, gbar = average
                b["h"].copy_(buf)
                b["g"].copy_(buf)
                b["gbar"].copy_(buf)
                if N > 1:
                    dist.all_reduce(b["gbar"], group=state.pg)
                    b["gbar"].div_(N)
            elif state.cuda_graphs:
                # one CUDA graph per bucket: the step is captured once (on the bucket's
                # buffer, which DDP keeps from iteration to iteration) and replayed, one
                # host launch per bucket; the context's device iteration counter advances
                # with every replay (ARC_FLAG_DEVICE_T)
                if b.get("graph_buf") != buf.data_ptr():
                    b["ctx"].set_iteration(t, stream=side)
                    b["graph"] = b["ctx"].capture([buf], [b["h"]], [b["g"]], b["gbar"], stream=side)
                    b["graph_buf"] = buf.data_ptr()
                b["graph"].replay()
            else:
                b["ctx"].step(t, [buf], [b["h"]], [b["g"]], b["gbar"], stream=side)
            buf.copy_(b["gbar"])
        fut.set_result(buf)
    return fut
