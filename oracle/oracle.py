"""ctypes wrapper around ``oracle/arc_oracle.c`` (TEST INFRASTRUCTURE ONLY).

Each function is a thin marshalling layer; the arithmetic lives in the C file,
whose header cites the paper passages it follows (PAPER.md = the paper's
LaTeX, "P:n" = line n).  Nothing here is imported by the product path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "arc_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libarc_oracle.so")

# Plain IEEE binary32: every operation rounded once, no contraction into FMA,
# no fast-math.  (The only FMAs are the explicit fmaf() calls ARC-NUM v1 and
# ARC-RNG v1 prescribe: the momentum, the O6 sketch order, Sigma, ln/sincos.)
CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
          "-fexcess-precision=standard", "-Wall", "-fopenmp"]


def build(force: bool = False) -> str:
    """Compile the oracle into ``oracle/libarc_oracle.so`` (gcc)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.run(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"], check=True)
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.POINTER
        L.orc_philox4x32_10.argtypes = [P(ctypes.c_uint32), P(ctypes.c_uint32), P(ctypes.c_uint32)]
        L.orc_uniform.argtypes = [ctypes.c_uint32]
        L.orc_uniform.restype = ctypes.c_float
        L.orc_ln.argtypes = [ctypes.c_float]
        L.orc_ln.restype = ctypes.c_float
        L.orc_sincos2pi.argtypes = [ctypes.c_float, P(ctypes.c_float), P(ctypes.c_float)]
        L.orc_gaussian_V.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64,
                                     ctypes.c_int32, ctypes.c_void_p]
        L.orc_sigma_key.argtypes = [ctypes.c_float]
        L.orc_sigma_key.restype = ctypes.c_uint32
        L.orc_argtop_k.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        L.orc_arc_round.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_int32, ctypes.c_int32] + [ctypes.c_void_p] * 6
        L.orc_bf16.argtypes = [ctypes.c_float]
        L.orc_bf16.restype = ctypes.c_float
        L.orc_randk_keys.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p]
        L.orc_ln_array.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.orc_sigma_rows.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p]
        L.orc_momentum.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_float]
        L.orc_sincos2pi_array.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_step.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 8
        L.orc_step.restype = ctypes.c_int
        L.orc_step_topk.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 6
        L.orc_step_topk.restype = ctypes.c_int
        L.orc_step_noef.argtypes = [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 6
        L.orc_step_noef.restype = ctypes.c_int
        L.orc_apply_sgd.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_float]
        L.orc_apply_adam.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_int64] + [ctypes.c_float] * 4
        L.orc_set_threads.argtypes = [ctypes.c_int32]
        L.orc_get_threads.restype = ctypes.c_int32
        # the plain oracle (1 thread) unless a caller asks for threads (bit-identical)
        L.orc_set_threads(int(os.environ.get("ARC_ORACLE_THREADS", "1")))
        _lib = L
    return _lib


class _Block(ctypes.Structure):
    _fields_ = [("offset", ctypes.c_int64), ("len", ctypes.c_int64), ("m", ctypes.c_int64),
                ("n", ctypes.c_int64), ("K", ctypes.c_int64), ("kind", ctypes.c_int32),
                ("pad_", ctypes.c_int32)]


class _Cfg(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("r", ctypes.c_int32), ("d", ctypes.c_int64),
                ("eta", ctypes.c_float), ("exact", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("num_blocks", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("blocks", ctypes.POINTER(_Block)), ("wire", ctypes.c_int32), ("pad2_", ctypes.c_int32)]


@dataclass(frozen=True)
class Block:
    """One m x n view of the flat vector: elements [offset, offset+len)."""
    offset: int
    len: int
    m: int
    n: int
    K: int
    kind: int = 0  # 0 ARC, 1 DENSE


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _f32(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


def set_threads(n: int) -> None:
    """Threads for the oracle's row-parallel loops (bit-identical to 1 thread)."""
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return int(lib().orc_get_threads())


def philox4x32_10(ctr, key) -> np.ndarray:
    c = (ctypes.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return np.array(list(o), dtype=np.uint32)


def uniform(x: int) -> float:
    return float(lib().orc_uniform(int(x) & 0xFFFFFFFF))


def ln(u: float) -> float:
    return float(lib().orc_ln(float(u)))


def sincos2pi(u: float):
    s = ctypes.c_float()
    c = ctypes.c_float()
    lib().orc_sincos2pi(float(u), ctypes.byref(s), ctypes.byref(c))
    return s.value, c.value


def ln_array(u) -> np.ndarray:
    u = _f32(u)
    out = np.empty_like(u)
    lib().orc_ln_array(_ptr(u), u.size, _ptr(out))
    return out


def sincos2pi_array(u):
    u = _f32(u)
    s = np.empty_like(u)
    c = np.empty_like(u)
    lib().orc_sincos2pi_array(_ptr(u), u.size, _ptr(s), _ptr(c))
    return s, c


def gaussian_V(seed: int, t: int, b: int, n: int, r: int) -> np.ndarray:
    V = np.empty((n, r), dtype=np.float32)
    lib().orc_gaussian_V(int(seed) & (2**64 - 1), int(t), int(b), int(n), int(r), _ptr(V))
    return V


def randk_keys(seed: int, t: int, b: int, m: int) -> np.ndarray:
    k = np.empty(m, dtype=np.float32)
    lib().orc_randk_keys(int(seed) & (2**64 - 1), int(t), int(b), int(m), _ptr(k))
    return k


def momentum(h, grad, eta: float) -> np.ndarray:
    """eq:ef21m-1 on one vector (returns the new h; the input is not modified)."""
    out = np.array(h, dtype=np.float32, copy=True)
    g = np.ascontiguousarray(grad, dtype=np.float32)
    lib().orc_momentum(_ptr(out), _ptr(g), out.size, float(eta))
    return out


def sigma_rows(S) -> np.ndarray:
    """O8: Sigma of each row of the node sums S [rows, r] (fma chain over j)."""
    S = np.ascontiguousarray(S, dtype=np.float32)
    out = np.zeros(S.shape[0], np.float32)
    lib().orc_sigma_rows(_ptr(S), S.shape[0], S.shape[1], _ptr(out))
    return out


def sigma_key(s: float) -> int:
    return int(lib().orc_sigma_key(float(s)))


def argtop_k(sigma, K: int) -> np.ndarray:
    s = _f32(sigma)
    sel = np.empty(int(K), dtype=np.int32)
    lib().orc_argtop_k(_ptr(s), s.size, int(K), _ptr(sel))
    return sel


def _ptr_array(arrs):
    return (ctypes.c_void_p * len(arrs))(*[_ptr(a) for a in arrs])


def bf16(x: float) -> float:
    """The binary32 value rounded to bfloat16 (ties to even) [R25]."""
    return float(lib().orc_bf16(float(x)))


def arc_round(G_nodes, n: int, K: int, V=None, r: int | None = None, exact: bool = False, m: int | None = None,
              wire: str = "f32"):
    """Algorithm 1 on N local flat blocks (each ``len`` floats viewed as m x n).

    Returns dict with P_nodes [N,m,r] (P'_i = G_i V, unscaled), S [m,r] (their
    node-order sum), sigma [m] (diag(S S^T)), sel [K], C_local [N,K,n], C [K,n].
    The paper's reported P = (1/N)(1/sqrt r) S and its Sigma = sigma / (r N^2)
    differ from these by selection-invariant factors (reading R2/R3)."""
    G = [_f32(x).ravel() for x in G_nodes]
    N = len(G)
    length = G[0].size
    if m is None:
        m = -(-length // n)
    if V is None:
        assert exact, "V required for the Gaussian sketch"
        V = np.zeros((n, r or 1), dtype=np.float32)
    V = _f32(V)
    r = V.shape[1]
    out = dict(P_nodes=np.zeros((N, m, r), np.float32), S=np.zeros((m, r), np.float32),
               sigma=np.zeros(m, np.float32), sel=np.zeros(K, np.int32),
               C_local=np.zeros((N, K, n), np.float32), C=np.zeros((K, n), np.float32))
    Gp = _ptr_array(G)
    lib().orc_arc_round(N, length, m, n, K, r, ctypes.cast(Gp, ctypes.c_void_p), _ptr(V), int(bool(exact)),
                        {"f32": 0, "bf16": 1}[wire],
                        _ptr(out["P_nodes"]), _ptr(out["S"]), _ptr(out["sigma"]), _ptr(out["sel"]),
                        _ptr(out["C_local"]), _ptr(out["C"]))
    return out


class OracleEF21M:
    """EF21M + ARC-Top-K state for N nodes (all nodes simulated on the host).

    State arrays are float32 numpy arrays owned by this object:
    ``h[i]``, ``g[i]`` (per node) and ``gbar`` (the replicated tracker)."""

    def __init__(self, d: int, blocks, N: int, eta: float, r: int, seed: int, exact: bool = False,
                 h0=None, g0=None, gbar0=None, method: str = "arc", wire: str = "f32"):
        self.d, self.N, self.eta, self.r, self.seed, self.exact = int(d), int(N), float(eta), int(r), int(seed), bool(exact)
        self.method = method
        self.blocks = list(blocks)
        self._cblocks = (_Block * len(self.blocks))(*[
            _Block(b.offset, b.len, b.m, b.n, b.K, b.kind, 0) for b in self.blocks])
        mode = 2 if method == "randk" else int(self.exact)
        self.wire = wire
        self._cfg = _Cfg(self.N, self.r, self.d, self.eta, mode, self.seed & (2**64 - 1),
                         len(self.blocks), 0, self._cblocks, {"f32": 0, "bf16": 1}[wire], 0)
        self.h = [np.zeros(d, np.float32) if h0 is None else _f32(h0[i]).copy() for i in range(N)]
        self.g = [np.zeros(d, np.float32) if g0 is None else _f32(g0[i]).copy() for i in range(N)]
        self.gbar = np.zeros(d, np.float32) if gbar0 is None else _f32(gbar0).copy()
        self.sum_K = sum(b.K for b in self.blocks)
        self.sum_Kn = sum(b.K * b.n for b in self.blocks)
        self.sum_m_arc = sum(b.m for b in self.blocks if b.kind == 0)
        self.sum_nr_arc = sum(b.n * self.r for b in self.blocks if b.kind == 0)

    def step(self, t: int, grads, debug: bool = False):
        if self.method == "noef_msgd":
            return self.step_noef(t, grads, debug)
        grads = [_f32(x).ravel() for x in grads]
        assert len(grads) == self.N and all(x.size == self.d for x in grads)
        sel = np.zeros(self.sum_K, np.int32)
        vals = np.zeros(self.sum_Kn, np.float32)
        V = np.zeros(self.sum_nr_arc, np.float32) if debug else None
        sig = np.zeros(self.sum_m_arc, np.float32) if debug else None
        rc = lib().orc_step(ctypes.byref(self._cfg), int(t),
                            ctypes.cast(_ptr_array(grads), ctypes.c_void_p),
                            ctypes.cast(_ptr_array(self.h), ctypes.c_void_p),
                            ctypes.cast(_ptr_array(self.g), ctypes.c_void_p),
                            _ptr(self.gbar), _ptr(sel), _ptr(vals),
                            _ptr(V) if debug else None, _ptr(sig) if debug else None)
        assert rc == 0
        out = dict(sel=sel, values=vals)
        if debug:
            out.update(V=V, sigma=sig)
        return out

    def step_noef(self, t: int, grads, debug: bool = False):
        """Compressed MSGD without EF (Table II "(without EF)"): gbar is the momentum
        u, eta is beta; h and g are untouched."""
        grads = [_f32(x).ravel() for x in grads]
        assert len(grads) == self.N and all(x.size == self.d for x in grads)
        sel = np.zeros(self.sum_K, np.int32)
        vals = np.zeros(self.sum_Kn, np.float32)
        V = np.zeros(self.sum_nr_arc, np.float32) if debug else None
        sig = np.zeros(self.sum_m_arc, np.float32) if debug else None
        rc = lib().orc_step_noef(ctypes.byref(self._cfg), int(t), ctypes.cast(_ptr_array(grads), ctypes.c_void_p),
                                 _ptr(self.gbar), _ptr(sel), _ptr(vals),
                                 _ptr(V) if debug else None, _ptr(sig) if debug else None)
        assert rc == 0
        out = dict(sel=sel, values=vals)
        if debug:
            out.update(V=V, sigma=sig)
        return out

    def step_topk(self, t: int, grads):
        """Vanilla EF21M with per-node row Top-K (the All-Gather baseline)."""
        grads = [_f32(x).ravel() for x in grads]
        sel = np.zeros(self.N * self.sum_K, np.int32)
        vals = np.zeros(self.N * self.sum_Kn, np.float32)
        rc = lib().orc_step_topk(ctypes.byref(self._cfg), int(t),
                                 ctypes.cast(_ptr_array(grads), ctypes.c_void_p),
                                 ctypes.cast(_ptr_array(self.h), ctypes.c_void_p),
                                 ctypes.cast(_ptr_array(self.g), ctypes.c_void_p),
                                 _ptr(self.gbar), _ptr(sel), _ptr(vals))
        assert rc == 0
        return dict(sel=sel.reshape(self.N, self.sum_K), values=vals.reshape(self.N, self.sum_Kn))


__all__ = ["Block", "OracleEF21M", "bf16", "get_threads", "set_threads", "apply_adam", "apply_sgd", "arc_round", "argtop_k", "build", "gaussian_V", "ln", "ln_array", "lib",
           "momentum", "philox4x32_10", "randk_keys", "sigma_key", "sigma_rows", "sincos2pi", "sincos2pi_array",
           "uniform"]


def apply_sgd(x, gbar, gamma: float) -> np.ndarray:
    """eq:ef21m-3: x - gamma * gbar, per element [R23]; returns the new x."""
    x = _f32(x).copy()
    gbar = _f32(gbar)
    lib().orc_apply_sgd(_ptr(x), _ptr(gbar), x.size, float(gamma))
    return x


def apply_adam(x, m, v, gbar, t: int, gamma: float, beta1: float = 0.9, beta2: float = 0.999,
               eps: float = 1e-8):
    """Adam step t >= 1 on the EF21M direction gbar [R24];
    returns the new (x, m, v)."""
    x, m, v = _f32(x).copy(), _f32(m).copy(), _f32(v).copy()
    gbar = _f32(gbar)
    lib().orc_apply_adam(_ptr(x), _ptr(m), _ptr(v), _ptr(gbar), x.size, int(t), float(gamma),
                         float(beta1), float(beta2), float(eps))
    return x, m, v
