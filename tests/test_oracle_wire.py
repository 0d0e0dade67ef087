"""Pins for the oracle's bfloat16 value wire (reading R25):
each compact entry a node sends in exchange #2 is C_i = bf16(Delta_i[I]) (round
to nearest, ties to even); sums stay binary32 (A = sum_i C_i in node order,
gbar += A / N) and the EF update adds what was sent, g_i += bf16(Delta_i), so
the rounding error stays in the residual h_i - g_i (error feedback, eq:ef21m-2
P:326).  Pinned against torch's float32 -> bfloat16 conversion (a library
routine), hand-computed ties, and the f32 wire on inputs bf16 represents exactly.
"""
import numpy as np
import pytest
import torch

from synth import Block, flat_blocks


def _torch_bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float32).numpy()


def test_bf16_rounding_hand_cases(orc):
    f = orc.bf16
    assert f(1.0) == 1.0 and f(-2.5) == -2.5 and f(0.0) == 0.0
    assert f(1 + 2 ** -8) == 1.0                            # halfway, the even neighbour (1.0)
    assert f(1 + 3 * 2 ** -8) == 1 + 2 ** -6                # halfway, the even neighbour (1 + 2^-6)
    assert f(1 + 2 ** -8 + 2 ** -20) == 1 + 2 ** -7         # just above halfway: up
    assert f(float(np.float32(3.4028235e38))) == float("inf")   # max finite rounds to +Inf (RNE)
    assert f(float("inf")) == float("inf") and f(float("-inf")) == float("-inf")
    assert np.isnan(f(float("nan")))
    assert f(2.0 ** -133) == 2.0 ** -133                    # subnormal, exactly representable


def test_bf16_rounding_matches_torch(orc):
    """orc_bf16 on 200,000 binary32 patterns (all exponents, random mantissas, every
    low-half pattern class incl. exact ties) equals torch's float32 -> bfloat16."""
    rng = np.random.default_rng(0)
    hi = rng.integers(0, 1 << 16, 200_000, dtype=np.uint32)
    lo = rng.choice(np.array([0, 1, 0x7FFF, 0x8000, 0x8001, 0xFFFF], np.uint32), 200_000)
    lo = np.where(rng.random(200_000) < 0.5, lo, rng.integers(0, 1 << 16, 200_000, dtype=np.uint32))
    bits = (hi << 16) | lo
    x = bits.view(np.float32)
    x = x[~np.isnan(x)]
    want = _torch_bf16(x)
    got = np.array([orc.bf16(float(v)) for v in x], np.float32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_bf16_wire_equals_f32_wire_on_exact_inputs(orc):
    """Small integers (|Delta| < 256: exact in bfloat16), eta = 1, N = 4: every sent
    value is already bf16, so the bf16 wire must give the f32 wire's results bit for bit."""
    rng = np.random.default_rng(3)
    d, N = 3000, 4
    blocks = [Block(0, 2000, 200, 10, 17, 0), Block(2000, 1000, 10, 100, 10, 1)]
    runs = []
    for wire in ("f32", "bf16"):
        o = orc.OracleEF21M(d, blocks, N=N, eta=1.0, r=4, seed=2, wire=wire)
        rr = np.random.default_rng(3)
        res = [o.step(t, [rr.integers(-60, 61, d).astype(np.float32) for _ in range(N)]) for t in range(3)]
        runs.append((res, o))
    for a, b in zip(runs[0][0], runs[1][0]):
        assert np.array_equal(a["sel"], b["sel"])
        assert a["values"].tobytes() == b["values"].tobytes()
    for i in range(N):
        assert runs[0][1].g[i].tobytes() == runs[1][1].g[i].tobytes()
    assert runs[0][1].gbar.tobytes() == runs[1][1].gbar.tobytes()


@pytest.mark.parametrize("exact", [True, False])
def test_bf16_wire_rounds_what_is_sent_and_ef_keeps_the_rest(orc, exact):
    """One step from the zero state, N = 3, normal data.  The selection is the f32
    wire's (Sigma does not see the value wire); the selected rows of g_i become
    bf16(Delta_i) (torch's rounding of the f32 run's g_i = Delta_i); h_i - g_i there
    is Delta_i - bf16(Delta_i) exactly (the error EF feeds back); values = A / N with
    A the node-order binary32 sum of the rounded entries; rows outside I untouched."""
    rng = np.random.default_rng(11)
    d, N = 4000, 3
    blocks = flat_blocks(d, 40, K=9)
    grads = [rng.standard_normal(d).astype(np.float32) for _ in range(N)]
    out = {}
    for wire in ("f32", "bf16"):
        o = orc.OracleEF21M(d, blocks, N=N, eta=0.5, r=4, seed=5, exact=exact, wire=wire)
        out[wire] = (o.step(0, grads), o)
    (rf, of), (rb, ob) = out["f32"], out["bf16"]
    assert np.array_equal(rf["sel"], rb["sel"])
    rows = np.zeros(d, bool)
    for p in rf["sel"]:
        rows[p * 40:(p + 1) * 40] = True
    A = np.zeros(rows.sum(), np.float32)
    for i in range(N):
        delta = of.g[i][rows]                                  # f32 wire from zero state: g_i = Delta_i on I
        sent = _torch_bf16(delta)
        assert ob.g[i][rows].tobytes() == sent.tobytes()
        assert (ob.h[i] - ob.g[i])[rows].tobytes() == (delta - sent).astype(np.float32).tobytes()
        assert not ob.g[i][~rows].any()
        A = sent if i == 0 else (A + sent).astype(np.float32)
    assert rb["values"].tobytes() == (A / np.float32(N)).astype(np.float32).tobytes()
    assert ob.gbar[rows].tobytes() == (A / np.float32(N)).astype(np.float32).tobytes()
