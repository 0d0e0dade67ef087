"""ctypes binding of ``libarctopk.so`` (include/arc_topk.h).

Argument marshalling only: every step of the path runs in the library's CUDA
kernels.  There is no CPU fallback — if the library is missing or its calls
fail, these functions raise.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# ARC_LIB_PATH: an alternative build of the same library (A/B timing experiments)
LIB_PATH = os.environ.get("ARC_LIB_PATH") or os.path.join(_PKG, "libarctopk.so")

ABI_VERSION = 2
MAX_NODES_LOCAL = 16

# arc_status
OK, ERR_INVALID_ARG, ERR_UNSUPPORTED, ERR_PARAM_MISMATCH, ERR_CUDA, ERR_NCCL, ERR_NONFINITE = range(7)
# arc_block_kind
BLOCK_ARC, BLOCK_DENSE = 0, 1
# arc_reduce_mode
REDUCE_NCCL, REDUCE_ORDERED, REDUCE_LSA = 0, 1, 2
# flags
FLAG_HOST_STAGING, FLAG_DEBUG_SKETCH, FLAG_FORCE_EXCHANGE, FLAG_LOOPBACK_COMM, FLAG_DEVICE_T = 0x1, 0x2, 0x4, 0x8, 0x10
# arc_method
METHOD_ARC, METHOD_TOPK_ALLGATHER, METHOD_RANDK, METHOD_NOEF_MSGD, METHOD_EXACT = 0, 1, 2, 3, 4
# arc_opt_kind
OPT_SGD, OPT_ADAM = 0, 1
# arc_query
Q_V, Q_SIGMA, Q_SEL, Q_P_NODES, Q_CANDIDATES, Q_S, Q_PLAN = 0, 1, 2, 3, 4, 5, 6
# arc_wire
WIRE_F32, WIRE_BF16 = 0, 1

EXPORTED = [
    "arc_topk_workspace_bytes", "arc_topk_create", "arc_topk_step", "arc_topk_step_host",
    "arc_topk_set_iteration", "arc_topk_query", "arc_topk_sizes", "arc_topk_get_status", "arc_topk_kernels_per_step",
    "arc_topk_destroy", "arc_topk_status_string", "arc_topk_set_timing", "arc_topk_read_timing",
    "arc_topk_debug_stamps", "arc_topk_apply_update", "arc_topk_comm_tally",
    "arc_topk_loopback_create", "arc_topk_loopback_comm", "arc_topk_loopback_destroy",
]
TALLY_NAMES = ["sketch", "sigma", "values", "calls", "steps"]
TIMING_PHASES = 6
PHASE_NAMES = ["vgen", "ef_sketch", "exchange1_reduce", "select_gather", "exchange2_scatter", "copy_out"]


class ArcBlock(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_int64), ("len", ctypes.c_int64), ("m", ctypes.c_int64),
                ("n", ctypes.c_int64), ("K", ctypes.c_int64), ("kind", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class ArcParams(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_uint32), ("N", ctypes.c_int32), ("nodes_local", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("d", ctypes.c_int64), ("r", ctypes.c_int32),
                ("num_blocks", ctypes.c_int32), ("blocks", ctypes.POINTER(ArcBlock)),
                ("eta", ctypes.c_float), ("value_reduce", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("flags", ctypes.c_uint32), ("method", ctypes.c_uint32),
                ("n", ctypes.c_int64), ("K", ctypes.c_int64), ("wire", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class ArcOptParams(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_uint32), ("gamma", ctypes.c_float), ("beta1", ctypes.c_float),
                ("beta2", ctypes.c_float), ("eps", ctypes.c_float)]


class ArcError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {status_string(status)} ({status})")


_lib = None


def lib():
    """Load libarctopk.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                               "or python -m paper_2510_26709_b200._build")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        P = ctypes.POINTER
        L.arc_topk_workspace_bytes.argtypes = [P(ArcParams), P(ctypes.c_size_t)]
        L.arc_topk_create.argtypes = [P(ArcParams), vp, vp, ctypes.c_size_t, vp, P(vp)]
        L.arc_topk_step.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, vp]
        L.arc_topk_step_host.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, vp]
        if hasattr(L, "arc_topk_set_iteration"):   # (absent from older builds used in A/B runs)
            L.arc_topk_set_iteration.argtypes = [vp, i64, vp]
        L.arc_topk_query.argtypes = [vp, i32, vp, ctypes.c_size_t, vp]
        L.arc_topk_sizes.argtypes = [vp, P(i64), P(i64), P(i64), P(i64)]
        L.arc_topk_get_status.argtypes = [vp, P(ctypes.c_uint32)]
        L.arc_topk_kernels_per_step.argtypes = [vp]
        L.arc_topk_kernels_per_step.restype = i32
        L.arc_topk_set_timing.argtypes = [vp, i32]
        L.arc_topk_read_timing.argtypes = [vp, P(ctypes.c_float), i32, P(i32)]
        L.arc_topk_debug_stamps.argtypes = [vp, vp, i64, P(i32)]
        L.arc_topk_debug_stamps.restype = ctypes.c_int
        L.arc_topk_apply_update.argtypes = [P(ArcOptParams), i64, vp, vp, vp, vp, i64, vp]
        L.arc_topk_comm_tally.argtypes = [vp, P(i64), i32]
        L.arc_topk_loopback_create.argtypes = [i32, P(vp)]
        L.arc_topk_loopback_comm.argtypes = [vp, i32, P(vp)]
        L.arc_topk_loopback_destroy.argtypes = [vp]
        L.arc_topk_destroy.argtypes = [vp]
        L.arc_topk_status_string.argtypes = [ctypes.c_int]
        L.arc_topk_status_string.restype = ctypes.c_char_p
        for name in ["arc_topk_workspace_bytes", "arc_topk_create", "arc_topk_step", "arc_topk_step_host",
                     "arc_topk_set_iteration", "arc_topk_query", "arc_topk_sizes", "arc_topk_get_status", "arc_topk_destroy",
                     "arc_topk_set_timing", "arc_topk_read_timing", "arc_topk_apply_update",
                     "arc_topk_comm_tally", "arc_topk_loopback_create", "arc_topk_loopback_comm",
                     "arc_topk_loopback_destroy"]:
            if hasattr(L, name):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def status_string(status: int) -> str:
    return lib().arc_topk_status_string(int(status)).decode()


def check(status: int, what: str) -> None:
    if status != OK:
        raise ArcError(status, what)
