"""Python surface of the library: argument marshalling around the C ABI.

``ArcTopK(...).step(t, grads, h, g, gbar)`` runs one EF21M + ARC-Top-K
iteration (eq:ef21m-1/2 P:325-326 with Algorithm 1) for the nodes
this GPU holds.  All arithmetic happens in ``libarctopk.so``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import torch

from . import _lib as L


@dataclass(frozen=True)
class Block:
    """The m x n row-major view of flat elements [offset, offset + len);
    K rows are kept per step (K = m for DENSE blocks)."""
    offset: int
    len: int
    m: int
    n: int
    K: int
    kind: int = L.BLOCK_ARC


def flat_layout(d: int, n: int, K: int | None = None, mu_bp: int | None = None) -> list[Block]:
    """The whole vector as one block of rows of n (the last row may be short);
    K given directly or as ceil(mu * m) with mu in basis points (Alg. 1)."""
    m = -(-d // n)
    if K is None:
        if mu_bp is None:
            raise ValueError("give K or mu_bp")
        K = max(1, min(m, -(-m * int(mu_bp) // 10000)))
    return [Block(0, d, m, n, int(K), L.BLOCK_ARC)]


def per_tensor_layout(shapes: Sequence[tuple[int, ...]], mu_bp: int) -> tuple[int, list[Block]]:
    """Per-tensor blocks for a model's parameters: every 2-D
    tensor (out, in) is an ARC block of m = out rows of n = in; conv kernels are
    viewed as (out, in*kh*kw); all other tensors are packed into one DENSE block."""
    blocks, off, dense = [], 0, 0
    for s in shapes:
        if len(s) >= 2:
            m = int(s[0])
            n = 1
            for x in s[1:]:
                n *= int(x)
            K = max(1, min(m, -(-m * int(mu_bp) // 10000)))
            blocks.append(Block(off, m * n, m, n, K, L.BLOCK_ARC))
            off += m * n
        else:
            dense += int(s[0]) if len(s) else 1
    if dense:
        nd = 1024
        md = -(-dense // nd)
        blocks.append(Block(off, dense, md, nd, md, L.BLOCK_DENSE))
        off += dense
    return off, blocks


def nccl_comm_ptr(pg, device: torch.device) -> int:
    """The ncclComm_t behind a torch ProcessGroupNCCL (borrowed, not owned).

    The group must have created its communicator (``init_process_group(...,
    device_id=...)`` or one collective before)."""
    backend = pg._get_backend(device)
    ptr = int(backend._comm_ptr())
    if ptr == 0:
        raise RuntimeError("the process group has no NCCL communicator yet")
    return ptr


def _stream_handle(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _ptrs(ts) -> ctypes.Array | None:
    if ts is None:      # (NOEF_MSGD: no h / g state)
        return None
    return (ctypes.c_void_p * len(ts))(*[int(x.data_ptr()) for x in ts])


class ArcTopK:
    """One EF21M + ARC-Top-K context on the current CUDA device.

    Args:
      d: per-node vector length.  blocks: the block table (tiles [0, d)).
      N: nodes in the job.  nodes_local: nodes held by this GPU (simulated
      nodes when > 1).  eta: EF21M momentum.  r: sketch width.  seed: shared
      base seed.  pg: torch process group (NCCL) when N / nodes_local > 1.
      rank: this GPU's rank in pg.  reduce: "nccl" (All-Reduce of the K rows)
      or "ordered" (bit-exact node-ordered sum) or "lsa" (both exchanges
      fused into the library's kernels over NCCL symmetric windows, bit-exact).
      comm_group: an NCCL group over pg's ranks for the library's collectives
      (``dist.private_nccl_group(pg, device)``), shared by several contexts;
      default: a private group per context.
      wire: "f32" or "bf16" — exchange #2's payload precision (R25: each sent
      entry rounded to bfloat16 at the source, EF keeps the rounding error).
      blocks=None with n, K: the single-block shorthand (rows of n, K kept).
      loopback: a :class:`LoopbackGroup` of G = N / nodes_local emulated ranks
      (tests on one GPU; this context is rank ``rank`` of it, and must be
      created and stepped from its own host thread, concurrently with the
      other ranks'); no process group is used then.
    """

    def __init__(self, d: int, blocks: Sequence | None, N: int, eta: float, r: int = 4, seed: int = 20251030,
                 nodes_local: int | None = None, pg=None, rank: int = 0, reduce: str = "nccl",
                 host_staging: bool = False, debug_sketch: bool = False, force_exchange: bool = False,
                 method: str = "arc", device=None, stream=None, comm_group=None, loopback=None,
                 wire: str = "f32", n: int | None = None, K: int | None = None, device_t: bool = False):
        self.lib = L.lib()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.d, self.N = int(d), int(N)
        self.nodes_local = int(nodes_local if nodes_local is not None else N)
        self.G = self.N // self.nodes_local
        if blocks is None:                       # the ABI's single-block shorthand (n, K)
            if n is None or K is None:
                raise ValueError("give blocks, or n and K")
            blocks = [Block(0, int(d), -(-int(d) // int(n)), int(n), int(K), L.BLOCK_ARC)]
            nb = 0
        else:
            nb = len(blocks)
        self.blocks = list(blocks)
        self._cblocks = (L.ArcBlock * len(self.blocks))(*[
            L.ArcBlock(int(b.offset), int(b.len), int(b.m), int(b.n), int(b.K), int(b.kind), 0) for b in self.blocks])
        flags = (L.FLAG_HOST_STAGING if host_staging else 0) | (L.FLAG_DEBUG_SKETCH if debug_sketch else 0) | \
                (L.FLAG_FORCE_EXCHANGE if force_exchange else 0) | (L.FLAG_LOOPBACK_COMM if loopback is not None else 0) | \
                (L.FLAG_DEVICE_T if device_t else 0)
        self.device_t = bool(device_t)
        self.params = L.ArcParams(L.ABI_VERSION, self.N, self.nodes_local, int(rank), self.d, int(r),
                                  nb, self._cblocks if nb else None, float(eta),
                                  {"nccl": L.REDUCE_NCCL, "ordered": L.REDUCE_ORDERED, "lsa": L.REDUCE_LSA}[reduce],
                                  int(seed) & (2**64 - 1), flags,
                                  {"arc": L.METHOD_ARC, "topk_allgather": L.METHOD_TOPK_ALLGATHER,
                                   "randk": L.METHOD_RANDK, "noef_msgd": L.METHOD_NOEF_MSGD,
                                   "exact": L.METHOD_EXACT}[method],
                                  int(n or 0), int(K or 0), {"f32": L.WIRE_F32, "bf16": L.WIRE_BF16}[wire], 0)
        self.wire = wire
        self.method = method
        nbytes = ctypes.c_size_t()
        L.check(self.lib.arc_topk_workspace_bytes(ctypes.byref(self.params), ctypes.byref(nbytes)),
                "arc_topk_workspace_bytes")
        self.workspace = torch.empty(max(int(nbytes.value), 1), dtype=torch.uint8, device=self.device)
        comm = None
        self._pg = None
        if loopback is not None:
            if loopback.G != self.G:
                raise ValueError(f"loopback group has {loopback.G} ranks, N / nodes_local = {self.G}")
            comm = loopback.comm(int(rank))
        elif self.G > 1 or (pg is not None and force_exchange):
            if pg is None:
                raise ValueError("N / nodes_local > 1 needs an NCCL process group")
            from .dist import check_consistent, params_digest, private_nccl_group
            check_consistent(pg, params_digest(d, self.blocks, self.N, self.nodes_local, r, eta, seed, reduce,
                                               method, wire))
            # the library's collectives get a communicator of their own, so they can
            # never interleave with torch's collectives on the caller's group; several
            # contexts (e.g. one per DDP bucket) may share one: comm_group, made once
            # with dist.private_nccl_group (their steps are issued in the same order
            # on every rank, NCCL's rule for a shared communicator)
            self._pg = comm_group if comm_group is not None else private_nccl_group(pg, self.device)
            import torch.distributed as dist
            self.params.rank = dist.get_rank(self._pg)     # this GPU's rank in the library's communicator
            comm = nccl_comm_ptr(self._pg, self.device)
        ctx = ctypes.c_void_p()
        L.check(self.lib.arc_topk_create(ctypes.byref(self.params), comm, int(self.workspace.data_ptr()),
                                          int(nbytes.value), _stream_handle(stream), ctypes.byref(ctx)),
                "arc_topk_create")
        self.ctx = ctx
        sK, sKn, sM, sNR = (ctypes.c_int64() for _ in range(4))
        L.check(self.lib.arc_topk_sizes(self.ctx, ctypes.byref(sK), ctypes.byref(sKn), ctypes.byref(sM),
                                        ctypes.byref(sNR)), "arc_topk_sizes")
        self.sum_K, self.sum_Kn, self.sum_m_arc, self.sum_nr_arc = sK.value, sKn.value, sM.value, sNR.value
        self.r = int(r)

    # ------------------------------------------------------------------ step
    def _check_state(self, grads, h, g, gbar):
        nl = self.nodes_local
        if self.method == "noef_msgd" and h is None and g is None:   # no (h, g) state without EF
            h = g = []
            if len(grads) != nl:
                raise ValueError(f"expected {nl} gradient tensors")
        elif not (len(grads) == len(h) == len(g) == nl):
            raise ValueError(f"expected {nl} node tensors each")
        for x in list(h) + list(g) + [gbar]:
            if not (x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.numel() == self.d):
                raise ValueError("state tensors must be contiguous float32 CUDA tensors of length d")

    def step(self, t: int, grads, h, g, gbar, sel_out: torch.Tensor | None = None,
             values_out: torch.Tensor | None = None, stream=None) -> None:
        """One EF21M + ARC-Top-K step: updates h, g, gbar in place (async).  For
        method="noef_msgd" pass h = g = None; gbar is the momentum u."""
        self._check_state(grads, h, g, gbar)
        for x in grads:
            if not (x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.numel() == self.d):
                raise ValueError("grads must be contiguous float32 CUDA tensors of length d")
        if sel_out is not None and (sel_out.dtype != torch.int32 or sel_out.numel() < self.sum_K):
            raise ValueError("sel_out must be int32 with sum_K elements")
        if values_out is not None and (values_out.dtype != torch.float32 or values_out.numel() < self.sum_Kn):
            raise ValueError("values_out must be float32 with sum_Kn elements")
        L.check(self.lib.arc_topk_step(self.ctx, int(t), _ptrs(grads), _ptrs(h), _ptrs(g), int(gbar.data_ptr()),
                                       sel_out.data_ptr() if sel_out is not None else None,
                                       values_out.data_ptr() if values_out is not None else None,
                                       _stream_handle(stream)), "arc_topk_step")

    def set_iteration(self, t: int, stream=None) -> None:
        """device_t contexts: the iteration the next step uses (async on the stream);
        every step then advances the device counter by one."""
        L.check(self.lib.arc_topk_set_iteration(self.ctx, int(t), _stream_handle(stream)), "arc_topk_set_iteration")

    def capture(self, grads, h, g, gbar, sel_out: torch.Tensor | None = None,
                values_out: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None,
                pool=None) -> torch.cuda.CUDAGraph:
        """device_t contexts: capture one step on these tensors into a CUDA graph.
        Each ``replay()`` runs one whole step (one launch from the host) at the
        device iteration counter and advances it, so replays continue t, t + 1, ...
        Capturing enqueues no work; call :meth:`set_iteration` before the first
        replay."""
        if not self.device_t:
            raise ValueError("capture needs a context created with device_t=True")
        graph = torch.cuda.CUDAGraph()
        s = stream if stream is not None else torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.graph(graph, stream=s, pool=pool, capture_error_mode="relaxed"):
            self.step(0, grads, h, g, gbar, sel_out, values_out, stream=s)
        return graph

    def step_host(self, t: int, grads_host, h, g, gbar, sel_host: torch.Tensor | None = None,
                  values_host: torch.Tensor | None = None, stream=None) -> None:
        """The same step with the gradients in (pinned) host memory; the selection
        and values are copied back into host tensors (async on the stream)."""
        self._check_state(grads_host, h, g, gbar)
        for x in grads_host:
            if x.is_cuda or x.dtype != torch.float32 or not x.is_contiguous() or x.numel() != self.d:
                raise ValueError("grads_host must be contiguous float32 host tensors of length d")
        L.check(self.lib.arc_topk_step_host(self.ctx, int(t), _ptrs(grads_host), _ptrs(h), _ptrs(g),
                                            int(gbar.data_ptr()),
                                            sel_host.data_ptr() if sel_host is not None else None,
                                            values_host.data_ptr() if values_host is not None else None,
                                            _stream_handle(stream)), "arc_topk_step_host")

    # ------------------------------------------------------------------ debug
    def query(self, what: int, stream=None) -> torch.Tensor:
        shapes = {L.Q_V: (self.sum_nr_arc, torch.float32), L.Q_SIGMA: (self.sum_m_arc, torch.float32),
                  L.Q_SEL: (self.sum_K, torch.int32),
                  L.Q_P_NODES: (self.sum_m_arc * self.nodes_local * self.r, torch.float32),
                  L.Q_S: (self.sum_m_arc * self.r, torch.float32),
                  L.Q_CANDIDATES: (len(self.blocks) * (self.nodes_local if self.method == "topk_allgather" else 1),
                                   torch.int32),
                  L.Q_PLAN: (4, torch.int32)}
        n, dt = shapes[what]
        out = torch.empty(max(n, 1), dtype=dt, device=self.device)
        L.check(self.lib.arc_topk_query(self.ctx, int(what), int(out.data_ptr()), out.numel() * out.element_size(),
                                        _stream_handle(stream)), "arc_topk_query")
        return out[:n]

    def status(self) -> int:
        """Synchronises; returns the status word, raises on NCCL async errors."""
        f = ctypes.c_uint32()
        st = self.lib.arc_topk_get_status(self.ctx, ctypes.byref(f))
        if st not in (L.OK, L.ERR_NONFINITE):
            L.check(st, "arc_topk_get_status")
        return int(f.value)

    def set_timing(self, enable: bool) -> None:
        """Record CUDA events between the step's phases (not during graph capture)."""
        L.check(self.lib.arc_topk_set_timing(self.ctx, int(bool(enable))), "arc_topk_set_timing")

    def read_timing(self) -> tuple[dict, int]:
        """Synchronises; summed device milliseconds per phase since the last read."""
        ms = (ctypes.c_float * L.TIMING_PHASES)()
        steps = ctypes.c_int32()
        L.check(self.lib.arc_topk_read_timing(self.ctx, ms, L.TIMING_PHASES, ctypes.byref(steps)),
                "arc_topk_read_timing")
        return {name: float(ms[k]) for k, name in enumerate(L.PHASE_NAMES)}, int(steps.value)

    def comm_tally(self) -> dict:
        """Floats this rank handed to the step's collectives since create (Table I
        ledger audit): sketch (exchange #1), sigma, values (exchange #2), calls, steps."""
        out = (ctypes.c_int64 * 8)()
        L.check(self.lib.arc_topk_comm_tally(self.ctx, out, 8), "arc_topk_comm_tally")
        return {name: int(out[k]) for k, name in enumerate(L.TALLY_NAMES)}

    @property
    def kernels_per_step(self) -> int:
        return int(self.lib.arc_topk_kernels_per_step(self.ctx))

    def close(self) -> None:
        if getattr(self, "ctx", None):
            self.lib.arc_topk_destroy(self.ctx)
            self.ctx = None
        self._pg = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackGroup:
    """G ranks emulated in one process on the current GPU (arc_topk_loopback_*):
    the library's multi-GPU step sequence with stream-event-ordered copies in
    place of NCCL, for tests on one GPU.  Each rank's ArcTopK lives in its own
    host thread (ctypes releases the GIL during the library's calls)."""

    def __init__(self, G: int):
        self.lib = L.lib()
        self.G = int(G)
        h = ctypes.c_void_p()
        L.check(self.lib.arc_topk_loopback_create(self.G, ctypes.byref(h)), "arc_topk_loopback_create")
        self.handle = h

    def comm(self, rank: int) -> int:
        c = ctypes.c_void_p()
        L.check(self.lib.arc_topk_loopback_comm(self.handle, int(rank), ctypes.byref(c)), "arc_topk_loopback_comm")
        return int(c.value)

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.arc_topk_loopback_destroy(self.handle)
            self.handle = None


def apply_update(x: torch.Tensor, gbar: torch.Tensor, gamma: float, *, optimizer: str = "sgd",
                 t: int = 1, m: torch.Tensor | None = None, v: torch.Tensor | None = None,
                 beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, stream=None) -> None:
    """The model update that consumes the step's gbar (include/arc_topk.h
    ``arc_topk_apply_update``), in place on x (and m, v for Adam):

    * ``"sgd"``:  x <- x - gamma * gbar   (eq:ef21m-3; R23)
    * ``"adam"``: standard Adam on gbar, no weight decay (R24),
      t >= 1 its step count, m and v its moment buffers.

    Enqueued on ``stream`` (default: the current stream) — call it after
    ``ArcTopK.step`` on the same stream."""
    kind = {"sgd": L.OPT_SGD, "adam": L.OPT_ADAM}[optimizer]
    ts = [x, gbar] + ([m, v] if kind == L.OPT_ADAM else [])
    if any(u is None or u.dtype != torch.float32 or not u.is_cuda or not u.is_contiguous() for u in ts):
        raise ValueError("x, gbar (and m, v for adam) must be contiguous float32 CUDA tensors")
    if any(u.numel() != x.numel() for u in ts):
        raise ValueError("x, gbar, m, v must have the same number of elements")
    p = L.ArcOptParams(kind, float(gamma), float(beta1), float(beta2), float(eps))
    ptr = lambda u: ctypes.c_void_p(u.data_ptr()) if u is not None else None
    L.check(L.lib().arc_topk_apply_update(ctypes.byref(p), int(t), ptr(x), ptr(gbar), ptr(m), ptr(v),
                                          int(x.numel()), _stream_handle(stream)), "arc_topk_apply_update")
