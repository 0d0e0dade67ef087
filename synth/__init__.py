"""Seeded synthetic inputs shared by the tests, ``bench.py`` and ``smoke()``.

This module holds NONE of the method's arithmetic: it only builds block
tables (the m x n views and K per block, i.e. configuration) and draws
gradient tensors.  Both the CUDA path and the CPU oracle receive exactly the
arrays produced here.  See DESIGN.md §4 ("Input recipe").

Gradient recipe: for node i at step t, element (b, p, q)

    grad_i[b,p,q] = s_b * s_p * (rho * zc[b,p,q] + sqrt(1 - rho^2) * z_i[b,p,q])

with s_p = exp(xi_p) a persistent log-normal row scale (heavy-tailed row
importance, which ARC-Top-K exploits), s_b = exp(0.5 xi_b) a
per-block scale, rho = 0.5 coupling the nodes, and zc / z_i standard normals.
"""
from __future__ import annotations

import math
import zlib
from dataclasses import dataclass

import numpy as np
import torch

SEED = 20251030  # default base seed for every config


@dataclass(frozen=True)
class Block:
    """One m x n row-major view of the flat vector: elements [offset, offset+len)."""
    offset: int
    len: int
    m: int
    n: int
    K: int
    kind: int = 0  # 0 = ARC (compressed), 1 = DENSE (identity compressor)


def k_from_bp(m: int, mu_bp: int) -> int:
    """K = ceil(mu * m) with mu given in basis points, in integer arithmetic
    (Alg. 1 input line P:267: K = ceil(mu m))."""
    return max(1, min(m, -(-m * int(mu_bp) // 10000)))


def flat_blocks(d: int, n: int, mu_bp: int | None = None, K: int | None = None) -> list[Block]:
    """The whole vector as one m x n view, m = ceil(d/n); the last row may be short."""
    m = -(-d // n)
    if K is None:
        K = k_from_bp(m, mu_bp)
    return [Block(0, d, m, n, K, 0)]


def llama1b_blocks(mu_bp: int = 10) -> tuple[int, list[Block]]:
    """Per-tensor layout of a LLaMA-1B-shaped model (hidden 2048, FFN 5461,
    24 layers, vocab 32000): 170 ARC blocks (2-D tensors) + one DENSE block
    holding every 1-D (RMSNorm) parameter ("we compress only
    two-dimensional tensors"; per-tensor K)."""
    H, F, L, Vv = 2048, 5461, 24, 32000
    shapes = [(Vv, H)]
    for _ in range(L):
        shapes += [(H, H), (H, H), (H, H), (H, H), (F, H), (F, H), (H, F)]
    shapes += [(Vv, H)]
    blocks, off = [], 0
    for (m, n) in shapes:
        blocks.append(Block(off, m * n, m, n, k_from_bp(m, mu_bp), 0))
        off += m * n
    dense = (2 * L + 1) * H  # input/post-attn norms per layer + final norm
    nd = 1024
    md = -(-dense // nd)
    blocks.append(Block(off, dense, md, nd, md, 1))
    off += dense
    return off, blocks


def llama7b_scaled_blocks(mu_bp: int = 10, col_div: int = 512) -> tuple[int, list[Block]]:
    """A LLaMA-7B-shaped per-tensor table (hidden 4096, FFN 11008, 32 layers,
    vocab 32000: 226 ARC blocks + one DENSE block) with the true row counts m
    but every row length divided by `col_div` (scaled down so the CPU oracle
    finishes in seconds): the selection sees the full 7B block/row structure
    (1.42M rows, 368 slices of <= 4096 rows), the streaming pass a small d."""
    H, F, L, Vv = 4096, 11008, 32, 32000
    shapes = [(Vv, H)]
    for _ in range(L):
        shapes += [(H, H), (H, H), (H, H), (H, H), (F, H), (F, H), (H, F)]
    shapes += [(Vv, H)]
    blocks, off = [], 0
    for (m, n) in shapes:
        n = max(1, n // col_div)
        blocks.append(Block(off, m * n, m, n, k_from_bp(m, mu_bp), 0))
        off += m * n
    dense = (2 * L + 1) * H // col_div
    blocks.append(Block(off, dense, 1, dense, 1, 1))
    off += dense
    return off, blocks


# Named configurations (BASELINE.json "configs").
CONFIGS = {
    # configs[0]: N=4 simulated nodes on one GPU, d=65,536, K=1% -> n=1 (m=d, K=656)
    "C1": dict(d=65_536, n=1, mu_bp=100, N=4),
    # configs[1]: ResNet-18-sized gradient, K=1%, N=8
    "C2": dict(d=11_689_512, n=512, mu_bp=100, N=8),
    # configs[2]: GPT-2 small gradient, K=1%
    "C3": dict(d=124_439_808, n=768, mu_bp=100, N=1),
    # configs[3]: 1.3B-parameter LLM, K=0.1%, per-tensor blocks
    "C4": dict(llama=True, mu_bp=10, N=8),
    # configs[4]: sweep points, n=1024
    "C5_1e6": dict(d=1_000_000, n=1024, mu_bp=100, N=1),
    "C5_1e8": dict(d=100_000_000, n=1024, mu_bp=100, N=1),
    "C5_1e9": dict(d=1_000_000_000, n=1024, mu_bp=100, N=1),
    # probes (not BASELINE configs): one flat block with the LLaMA row lengths
    "P_n2048": dict(d=2048 * 48_828, n=2048, mu_bp=10, N=1),
    "P_n5461": dict(d=5461 * 18_311, n=5461, mu_bp=10, N=1),
    "P_n5460": dict(d=5460 * 18_315, n=5460, mu_bp=10, N=1),
}


def config_blocks(name: str, mu_bp: int | None = None) -> tuple[int, list[Block]]:
    c = CONFIGS[name]
    mu = c["mu_bp"] if mu_bp is None else mu_bp
    if c.get("llama"):
        return llama1b_blocks(mu)
    return c["d"], flat_blocks(c["d"], c["n"], mu)


def _row_index(d: int, blocks: list[Block]) -> tuple[np.ndarray, np.ndarray]:
    """(global row id, block id) of every flat element."""
    rows = np.empty(d, dtype=np.int64)
    bid = np.empty(d, dtype=np.int64)
    base = 0
    for b, B in enumerate(blocks):
        e = np.arange(B.len, dtype=np.int64)
        rows[B.offset:B.offset + B.len] = base + e // B.n
        bid[B.offset:B.offset + B.len] = b
        base += B.m
    return rows, bid


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed) & (2**63 - 1))
    return g


def _mix(*xs: int) -> int:
    h = 0x9E3779B97F4A7C15
    for x in xs:
        h ^= (int(x) + 0x9E3779B97F4A7C15 + ((h << 6) & (2**64 - 1)) + (h >> 2)) & (2**64 - 1)
        h &= 2**64 - 1
    return h


class GradientSource:
    """Seeded generator of the N per-node gradients of every step.

    ``grads(t, i)`` returns node i's fp32 gradient at step t on ``device``.
    Row scales are fixed per run (persistent importance)."""

    def __init__(self, d: int, blocks: list[Block], N: int, seed: int = SEED, rho: float = 0.5,
                 device="cpu"):
        self.d, self.blocks, self.N, self.seed, self.rho = d, blocks, N, seed, rho
        self.device = torch.device(device)
        m_tot = sum(B.m for B in blocks)
        g = _gen(_mix(seed, 1), "cpu")
        xi_rows = torch.randn(m_tot, generator=g, dtype=torch.float64)
        xi_blk = torch.randn(len(blocks), generator=g, dtype=torch.float64)
        row_scale = torch.exp(xi_rows)
        blk_scale = torch.exp(0.5 * xi_blk) if len(blocks) > 1 else torch.ones(1, dtype=torch.float64)
        # expand per element (float32), built block by block
        scale = torch.empty(d, dtype=torch.float32)
        base = 0
        for b, B in enumerate(blocks):
            s = (row_scale[base:base + B.m] * blk_scale[b]).to(torch.float32)
            scale[B.offset:B.offset + B.len] = s.repeat_interleave(B.n)[:B.len]
            base += B.m
        self.scale = scale.to(self.device)

    def common(self, t: int) -> torch.Tensor:
        return torch.randn(self.d, generator=_gen(_mix(self.seed, 2, t), self.device),
                           device=self.device, dtype=torch.float32)

    def grads(self, t: int, nodes=None) -> list[torch.Tensor]:
        """Gradients of step t for the given global node ids (default: all N)."""
        zc = self.common(t)
        a = float(self.rho)
        b = float(math.sqrt(1.0 - self.rho ** 2))
        out = []
        for i in (range(self.N) if nodes is None else nodes):
            zi = torch.randn(self.d, generator=_gen(_mix(self.seed, 3, t, i), self.device),
                             device=self.device, dtype=torch.float32)
            out.append(self.scale * (a * zc + b * zi))
        return out


# ---- adversarial input families -------------------------------

def adversarial(kind: str, d: int, N: int, seed: int = 7, n: int = 1) -> list[np.ndarray]:
    """Node gradients (float32 numpy) for the edge cases of DESIGN.md §4."""
    rng = np.random.default_rng(_mix(seed, zlib.crc32(kind.encode()), d, N, n) & (2**63 - 1))
    if kind == "zeros":
        return [np.zeros(d, np.float32) for _ in range(N)]
    if kind == "dup_rows":          # exact Sigma ties: every row identical
        m = -(-d // n)
        row = rng.standard_normal(n).astype(np.float32)
        base = np.tile(row, m)[:d]
        return [base.copy() for _ in range(N)]
    if kind == "symmetric":         # nodes G, -G interleaved (N even) -> P = 0 exactly
        half = [rng.standard_normal(d).astype(np.float32) for _ in range(N // 2)]
        out = []
        for x in half:
            out += [x, -x]
        return out
    if kind == "small_int":
        return [rng.integers(-3, 4, d).astype(np.float32) for _ in range(N)]
    if kind == "subnormal":
        return [(rng.standard_normal(d) * 1e-41).astype(np.float32) for _ in range(N)]
    if kind == "huge":              # Sigma overflows to +Inf, ties among Inf
        return [(rng.standard_normal(d) * 1e20).astype(np.float32) for _ in range(N)]
    if kind == "nonfinite":
        xs = [rng.standard_normal(d).astype(np.float32) for _ in range(N)]
        xs[0][d // 3] = np.nan
        xs[-1][(2 * d) // 3] = np.inf
        return xs
    if kind == "normal":
        return [rng.standard_normal(d).astype(np.float32) for _ in range(N)]
    raise ValueError(kind)


ADVERSARIAL = ["zeros", "dup_rows", "symmetric", "small_int", "subnormal", "huge", "nonfinite"]
