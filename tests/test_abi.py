"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and validates arguments before touching the GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2510_26709_b200 import _build, _lib
    _build.build()
    return _lib


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "arc_topk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(arc_topk_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol(L):
    lib = L.lib()
    declared = _declared_functions()
    assert len(declared) >= 8
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(L.EXPORTED) == declared


def test_binding_fails_loudly_without_library(monkeypatch, L):
    monkeypatch.setattr(L, "_lib", None)
    monkeypatch.setattr(L, "LIB_PATH", "/nonexistent/libarctopk.so")
    with pytest.raises(RuntimeError):
        L.lib()


def _params(L, blocks, **kw):
    arr = (L.ArcBlock * len(blocks))(*[L.ArcBlock(*b, 0) for b in blocks])
    d = sum(b[1] for b in blocks)
    p = L.ArcParams(L.ABI_VERSION, kw.get("N", 2), kw.get("nodes_local", 2), kw.get("rank", 0), kw.get("d", d),
                    kw.get("r", 4), len(blocks), arr, kw.get("eta", 0.1), kw.get("reduce", 0), 7,
                    kw.get("flags", 0), 0)
    p._keep = arr
    return p


def _ws(L, p):
    n = ctypes.c_size_t()
    st = L.lib().arc_topk_workspace_bytes(ctypes.byref(p), ctypes.byref(n))
    return st, n.value


def test_workspace_bytes_valid(L):
    st, n = _ws(L, _params(L, [(0, 1000, 10, 100, 3, 0)]))
    assert st == L.OK and n > 0
    # staging adds nodes_local * d floats
    st2, n2 = _ws(L, _params(L, [(0, 1000, 10, 100, 3, 0)], flags=L.FLAG_HOST_STAGING))
    assert st2 == L.OK and n2 >= n + 2 * 1000 * 4


@pytest.mark.parametrize("blocks,kw", [
    ([(0, 1000, 10, 100, 0, 0)], {}),                 # K = 0
    ([(0, 1000, 10, 100, 11, 0)], {}),                # K > m
    ([(0, 1000, 9, 100, 3, 0)], {}),                  # len > m n
    ([(0, 1000, 11, 100, 3, 0)], {}),                 # len <= (m-1) n
    ([(0, 1000, 10, 100, 3, 1)], {}),                 # DENSE with K != m
    ([(0, 500, 5, 100, 3, 0), (600, 500, 5, 100, 3, 0)], {"d": 1100}),   # gap between blocks
    ([(0, 1000, 10, 100, 3, 0)], {"d": 1001}),        # blocks do not cover d
    ([(0, 1000, 10, 100, 3, 0)], {"N": 3}),           # N % nodes_local != 0
    ([(0, 1000, 10, 100, 3, 0)], {"r": 0}),
    ([(0, 1000, 10, 100, 3, 0)], {"r": 33}),
    ([(0, 1000, 10, 100, 3, 0)], {"eta": 0.0}),
    ([(0, 1000, 10, 100, 3, 0)], {"eta": 1.5}),
    ([(0, 1000, 10, 100, 3, 0)], {"reduce": 5}),
    ([(0, 1000, 10, 100, 3, 0)], {"flags": 0x100}),
    ([(0, 1000, 10, 100, 3, 0)], {"N": 4, "nodes_local": 2, "rank": 2}),
    ([(0, 1000, 10, 100, 3, 0)], {"nodes_local": 17, "N": 17}),
    ([(0, 1000, 10, 100, 3, 2)], {}),                 # unknown kind
])
def test_workspace_bytes_rejects_invalid(L, blocks, kw):
    st, _ = _ws(L, _params(L, blocks, **kw))
    assert st == L.ERR_INVALID_ARG


def test_workspace_bytes_multi_gpu_and_methods(L):
    """Host-only plan checks of the G > 1 layout (no GPU needed): the exchange buffers
    (all-to-all receive [G][ceil(M/G)][L][r], the K-row wire) appear once G > 1 and
    stay O(M r + K n) as G grows; the method-specific momentum ranges validate."""
    blocks = [(0, 100_000, 1000, 100, 10, 0)]
    st1, n1 = _ws(L, _params(L, blocks, N=1, nodes_local=1))
    st2, n2 = _ws(L, _params(L, blocks, N=2, nodes_local=1, rank=1))
    st8, n8 = _ws(L, _params(L, blocks, N=8, nodes_local=1, rank=7))
    assert st1 == st2 == st8 == L.OK
    M, r, Kn = 1000, 4, 10 * 100
    assert n2 > n1                                             # exchange buffers
    assert n8 - n1 <= 4 * (2 * 8 * (-(-M // 8)) * r + 8 * M + 2 * Kn) + 64 * 1024   # O(M r + K n)
    p = _params(L, blocks, N=1, nodes_local=1, eta=0.0)
    p.method = L.METHOD_NOEF_MSGD                               # beta = 0 is a valid heavy-ball constant
    assert _ws(L, p)[0] == L.OK
    p = _params(L, blocks, N=1, nodes_local=1, eta=1.0)
    p.method = L.METHOD_NOEF_MSGD                               # beta = 1 never decays: rejected
    assert _ws(L, p)[0] == L.ERR_INVALID_ARG
    p = _params(L, blocks, N=1, nodes_local=1)
    p.method = 9
    assert _ws(L, p)[0] == L.ERR_INVALID_ARG


def test_null_arguments_rejected(L):
    lib = L.lib()
    assert lib.arc_topk_workspace_bytes(None, None) == L.ERR_INVALID_ARG
    assert lib.arc_topk_step(None, 0, None, None, None, None, None, None, None) == L.ERR_INVALID_ARG
    assert lib.arc_topk_destroy(None) == L.ERR_INVALID_ARG
    assert lib.arc_topk_kernels_per_step(None) == -1
    for s in range(7):
        assert isinstance(L.status_string(s), str) and L.status_string(s) != "unknown status"


def test_sass_is_sm100a(L):
    """The library carries sm_100a SASS for every kernel."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_apply_update_validation(L):
    """arc_topk_apply_update validates before touching the GPU (host-only here)."""
    import math
    lib = L.lib()
    fake = ctypes.c_void_p(1 << 20)          # 16-byte aligned, never dereferenced
    odd = ctypes.c_void_p((1 << 20) + 4)     # not 16-byte aligned

    def call(p, t=1, x=fake, gb=fake, m=fake, v=fake, d=1024):
        return lib.arc_topk_apply_update(None if p is None else ctypes.byref(p), t, x, gb, m, v, d, None)

    sgd = L.ArcOptParams(L.OPT_SGD, 0.1, 0.9, 0.999, 1e-8)
    adam = L.ArcOptParams(L.OPT_ADAM, 0.1, 0.9, 0.999, 1e-8)
    assert call(None) == L.ERR_INVALID_ARG
    assert call(sgd, d=-1) == L.ERR_INVALID_ARG
    assert call(sgd, d=0) == L.OK and call(adam, d=0) == L.OK          # no-op, nothing enqueued
    assert call(sgd, x=None) == L.ERR_INVALID_ARG
    assert call(sgd, gb=odd) == L.ERR_INVALID_ARG
    assert call(adam, m=None) == L.ERR_INVALID_ARG
    assert call(adam, v=odd) == L.ERR_INVALID_ARG
    assert call(adam, t=0) == L.ERR_INVALID_ARG
    assert call(L.ArcOptParams(L.OPT_ADAM, 0.1, 1.0, 0.999, 1e-8)) == L.ERR_INVALID_ARG
    assert call(L.ArcOptParams(L.OPT_ADAM, 0.1, 0.9, -0.1, 1e-8)) == L.ERR_INVALID_ARG
    assert call(L.ArcOptParams(L.OPT_ADAM, 0.1, 0.9, 0.999, -1.0)) == L.ERR_INVALID_ARG
    assert call(L.ArcOptParams(L.OPT_SGD, math.inf, 0.9, 0.999, 1e-8)) == L.ERR_INVALID_ARG
    assert call(L.ArcOptParams(7, 0.1, 0.9, 0.999, 1e-8)) == L.ERR_UNSUPPORTED


def test_exact_method_validation(L):
    """ARC_METHOD_EXACT (test mode) needs every node on this GPU and no forced exchange."""
    blocks = [(0, 1000, 10, 100, 3, 0)]
    p = _params(L, blocks, N=2, nodes_local=2)
    p.method = L.METHOD_EXACT
    assert _ws(L, p)[0] == L.OK
    p = _params(L, blocks, N=4, nodes_local=2)
    p.method = L.METHOD_EXACT
    assert _ws(L, p)[0] == L.ERR_UNSUPPORTED
    p = _params(L, blocks, N=2, nodes_local=2, flags=L.FLAG_FORCE_EXCHANGE)
    p.method = L.METHOD_EXACT
    assert _ws(L, p)[0] == L.ERR_UNSUPPORTED


def test_product_never_touches_the_oracle():
    """The product package (Python and CUDA sources) never imports, links or
    names the oracle; the oracle includes nothing from the product."""
    import glob
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_2510_26709_b200")
    srcs = glob.glob(os.path.join(pkg, "*.py")) + glob.glob(os.path.join(pkg, "csrc", "*"))
    assert srcs
    for p in srcs:
        txt = open(p, encoding="utf-8", errors="replace").read()
        assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), p
        assert "arc_oracle" not in txt and "libarc_oracle" not in txt, p
    orc = open(os.path.join(root, "oracle", "arc_oracle.c")).read()
    for inc in re.findall(r'#include\s+[<"]([^>"]+)[>"]', orc):
        assert not inc.startswith("arc_") or inc == "arc_oracle.h", inc
    # the loaded product library does not depend on the oracle's shared object
    import subprocess
    from paper_2510_26709_b200 import _lib as L
    out = subprocess.run(["ldd", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "arc_oracle" not in out


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: with the library absent the binding raises on first use."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import paper_2510_26709_b200._lib as L\n"
            "try:\n    L.lib()\nexcept RuntimeError as e:\n    print('RAISED', 'missing' in str(e))\n")
    env = dict(os.environ, ARC_LIB_PATH=str(tmp_path / "absent.so"), PYTHONPATH=root)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=root)
    assert "RAISED True" in out.stdout, out.stderr


def test_single_block_shorthand_and_wire_validation(L):
    """ABI v2: num_blocks == 0 with blocks == NULL is the single-block shorthand
    (rows of n, K kept) — the same workspace as the explicit block;
    the wire field accepts ARC_WIRE_F32 / ARC_WIRE_BF16 only, and the bf16 wire is
    refused for the Top-K baseline (its payload carries indices); an ABI v1
    struct version is rejected."""
    d, n, K = 100_003, 768, 13
    explicit = _params(L, [(0, d, -(-d // n), n, K, 0)], N=1, nodes_local=1)
    st1, b1 = _ws(L, explicit)
    short = L.ArcParams(L.ABI_VERSION, 1, 1, 0, d, 4, 0, None, 0.1, 0, 7, 0, 0, n, K, 0, 0)
    st2, b2 = _ws(L, short)
    assert st1 == st2 == L.OK and b1 == b2
    bad_k = L.ArcParams(L.ABI_VERSION, 1, 1, 0, d, 4, 0, None, 0.1, 0, 7, 0, 0, n, -(-d // n) + 1, 0, 0)
    assert _ws(L, bad_k)[0] == L.ERR_INVALID_ARG
    bad_n = L.ArcParams(L.ABI_VERSION, 1, 1, 0, d, 4, 0, None, 0.1, 0, 7, 0, 0, 0, 1, 0, 0)
    assert _ws(L, bad_n)[0] == L.ERR_INVALID_ARG
    for wire, want in [(L.WIRE_F32, L.OK), (L.WIRE_BF16, L.OK), (2, L.ERR_INVALID_ARG)]:
        p = _params(L, [(0, 1000, 10, 100, 3, 0)])
        p.wire = wire
        assert _ws(L, p)[0] == want
    p = _params(L, [(0, 1000, 10, 100, 3, 0)])
    p.wire, p.method = L.WIRE_BF16, L.METHOD_TOPK_ALLGATHER
    assert _ws(L, p)[0] == L.ERR_UNSUPPORTED
    p = _params(L, [(0, 1000, 10, 100, 3, 0)])
    p.abi_version = 1
    assert _ws(L, p)[0] == L.ERR_INVALID_ARG
    # the bf16 wire halves exchange #2's workspace payload (ORDERED: [L][sum Kn] + [G][L][sum Kn])
    base = _params(L, [(0, 100_000, 1000, 100, 100, 0)], N=4, nodes_local=2, reduce=L.REDUCE_ORDERED)
    half = _params(L, [(0, 100_000, 1000, 100, 100, 0)], N=4, nodes_local=2, reduce=L.REDUCE_ORDERED)
    half.wire = L.WIRE_BF16
    s_f, s_h = _ws(L, base)[1], _ws(L, half)[1]
    assert s_f - s_h >= (2 * 100 * 100 * 2 + 2 * 2 * 100 * 100 * 2) - 1024


def test_query_kinds_match_the_header():
    """The binding's query constants are the header's arc_query values (ARC_Q_PLAN included)."""
    import re
    from paper_2510_26709_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "arc_topk.h")).read()
    vals = {m.group(1): int(m.group(2)) for m in re.finditer(r"\bARC_Q_([A-Z_]+)\s*=\s*(\d+)", hdr)}
    assert set(vals) >= {"V", "SIGMA", "SEL", "P_NODES", "S", "CANDIDATES", "PLAN"}
    for name, v in vals.items():
        assert getattr(_lib, "Q_" + name) == v, name
