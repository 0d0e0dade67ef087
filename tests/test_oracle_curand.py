"""The oracle's Philox4x32-10 (ARC-RNG v1, reading R8) against cuRAND's own
implementation (curand_philox4x32_x.h, compiled for the host with nvcc): a
library-routine pin beyond the Random123 known-answer vectors."""
import ctypes
import os
import shutil
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def curand_ref(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    out = tmp_path_factory.mktemp("curand") / "libcurand_ref.so"
    subprocess.run([nvcc, "-shared", "-Xcompiler", "-fPIC", "-O2", "-o", str(out),
                    os.path.join(HERE, "aux", "curand_philox_ref.cu")], check=True)
    lib = ctypes.CDLL(str(out))
    lib.curand_ref_philox.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_longlong]
    return lib


def test_oracle_philox_equals_curand(orc, curand_ref):
    rng = np.random.default_rng(2510)
    n = 20_000
    ctr = rng.integers(0, 2**32, (n, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, (n, 2), dtype=np.uint64).astype(np.uint32)
    ctr[:4] = [[0, 0, 0, 0], [0xFFFFFFFF] * 4, [1, 0, 0, 0], [0, 0, 0, 0x80000000]]
    key[:4] = [[0, 0], [0xFFFFFFFF] * 2, [0, 1], [7, 0]]
    ref = np.zeros((n, 4), np.uint32)
    curand_ref.curand_ref_philox(ctr.ctypes.data, key.ctypes.data, ref.ctypes.data, n)
    got = np.array([orc.philox4x32_10(list(map(int, c)), list(map(int, k))) for c, k in zip(ctr, key)], np.uint32)
    assert np.array_equal(got, ref)
