// arc_rng.cuh — ARC-RNG v1 (R8), device side: Philox4x32-10 and a
// Box–Muller transform whose ln / sin / cos use only exactly rounded operations,
// so every V entry is bit-identical wherever it is generated.
#pragma once
#include <cuda_runtime.h>

#include "arc_device.cuh"
#include "arc_internal.cuh"

namespace arc {
namespace rng {
using namespace dev;

// =============================================================================
// S0: ARC-RNG v1 (R8) — Philox4x32-10 + Box–Muller with portable
// ln / sincos(2 pi u) made of exactly rounded operations only.
// =============================================================================

static __device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        if (round != 0) {
            k.x += 0x9E3779B9u;
            k.y += 0xBB67AE85u;
        }
        const unsigned lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const unsigned lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

// (x >> 9) * 2^-23 + 2^-24: both operations exact, u = (2i+1) 2^-24 in (0,1)
static __device__ __forceinline__ float word_to_unit(unsigned x) {
    return fadd(fmul(__uint2float_rn(x >> 9), 0x1p-23f), 0x1p-24f);
}

// ln(u), u a positive normal float: u = f 2^e with f in [sqrt(1/2), sqrt(2)),
// x = f - 1 exact, Cephes logf minimax polynomial in Horner form with fma.
static __device__ __forceinline__ float ln_exact_ops(float u) {
    const unsigned bits = __float_as_uint(u);
    int e = static_cast<int>(bits >> 23) - 126;
    const float f = __uint_as_float((bits & 0x007FFFFFu) | 0x3F000000u);   // [0.5, 1)
    float x;
    if (f < 0x1.6a09e6p-1f) {            // sqrt(1/2) rounded to float
        e -= 1;
        x = fsub(fadd(f, f), 1.0f);
    } else {
        x = fsub(f, 1.0f);
    }
    const float z = fmul(x, x);
    float p = 0x1.204376p-4f;
    p = ffma(p, x, -0x1.d7a370p-4f);
    p = ffma(p, x, 0x1.de4a34p-4f);
    p = ffma(p, x, -0x1.fcba9ep-4f);
    p = ffma(p, x, 0x1.23d37ep-3f);
    p = ffma(p, x, -0x1.555ca0p-3f);
    p = ffma(p, x, 0x1.999d58p-3f);
    p = ffma(p, x, -0x1.fffff8p-3f);
    p = ffma(p, x, 0x1.555554p-2f);
    float y = fmul(fmul(p, x), z);
    const float fe = __int2float_rn(e);
    y = ffma(fe, -0x1.bd0106p-13f, y);   // ln2 low part
    y = ffma(-0.5f, z, y);
    const float res = fadd(x, y);
    return ffma(fe, 0x1.63p-1f, res);    // ln2 high part 0.693359375
}

// sin / cos of (pi/2) f for |f| <= 1/2: Taylor coefficients (pi/2)^k / k!
// correctly rounded to float.
static __device__ __forceinline__ void sincos_quarter_turn(float f, float& s, float& c) {
    const float f2 = fmul(f, f);
    float ps = 0x1.507834p-13f;
    ps = ffma(ps, f2, -0x1.32d2ccp-8f);
    ps = ffma(ps, f2, 0x1.466bc6p-4f);
    ps = ffma(ps, f2, -0x1.4abbcep-1f);
    ps = ffma(ps, f2, 0x1.921fb6p+0f);
    s = fmul(ps, f);
    float pc = -0x1.a6d1f2p-16f;
    pc = ffma(pc, f2, 0x1.e1f506p-11f);
    pc = ffma(pc, f2, -0x1.55d3c8p-6f);
    pc = ffma(pc, f2, 0x1.03c1f0p-2f);
    pc = ffma(pc, f2, -0x1.3bd3ccp+0f);
    c = ffma(pc, f2, 1.0f);
}

// 2 pi u = (pi/2)(k + f), k = rint(4u), f = 4u - k (exact); quadrant rotation.
static __device__ __forceinline__ void sincos_2pi(float u, float& s, float& c) {
    const float w = fmul(4.0f, u);
    const float kf = rintf(w);
    const float f = fsub(w, kf);
    float sq, cq;
    sincos_quarter_turn(f, sq, cq);
    switch (static_cast<int>(kf) & 3) {
        case 0: s = sq; c = cq; break;
        case 1: s = cq; c = -sq; break;
        case 2: s = -sq; c = -cq; break;
        default: s = -cq; c = sq; break;
    }
}

static __device__ __forceinline__ void box_muller(unsigned xa, unsigned xb, float& za, float& zb) {
    const float ua = word_to_unit(xa), ub = word_to_unit(xb);
    const float rho = __fsqrt_rn(fmul(-2.0f, ln_exact_ops(ua)));
    float s, c;
    sincos_2pi(ub, s, c);
    za = fmul(rho, c);
    zb = fmul(rho, s);
}


// Entries of V for step t: item it (in [0, sum_b n_b ceil(r/4)) over the ARC
// blocks in order) is Philox block (q, jj) of the block it falls in.
// item `it` of block b (b = the last ARC block whose first item is <= it)
static __device__ __forceinline__ void gen_V_item_in(const BlockDev* __restrict__ blocks, int b, int r, uint2 key,
                                                     unsigned t_lo, unsigned t_hi, long long it, float* __restrict__ V);

static __device__ __forceinline__ void gen_V_item(const BlockDev* __restrict__ blocks, int num_blocks, int r,
                                                  uint2 key, unsigned t_lo, unsigned t_hi, long long it,
                                                  float* __restrict__ V) {
    const int R4 = (r + 3) >> 2;
    int lo = 0, hi = num_blocks - 1, b = -1;
    while (lo <= hi) {   // last ARC block whose first item is <= it
        const int mid = (lo + hi) >> 1;
        const long long first = (blocks[mid].v_off / r) * R4;   // (v_off = sum of r * ldv)
        if (first <= it) { b = mid; lo = mid + 1; } else hi = mid - 1;
    }
    gen_V_item_in(blocks, b, r, key, t_lo, t_hi, it, V);
}

// the same with the blocks' first items in a (shared-memory) table: first[b] =
// (v_off_b / r) * ceil(r / 4) — no dependent global loads in the search
static __device__ __forceinline__ void gen_V_item_tab(const BlockDev* __restrict__ blocks, const long long* first,
                                                      int num_blocks, int r, uint2 key, unsigned t_lo, unsigned t_hi,
                                                      long long it, float* __restrict__ V) {
    int lo = 0, hi = num_blocks - 1, b = -1;
    while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        if (first[mid] <= it) { b = mid; lo = mid + 1; } else hi = mid - 1;
    }
    gen_V_item_in(blocks, b, r, key, t_lo, t_hi, it, V);
}

static __device__ __forceinline__ void gen_V_item_in(const BlockDev* __restrict__ blocks, int b, int r, uint2 key,
                                                     unsigned t_lo, unsigned t_hi, long long it, float* __restrict__ V) {
    const int R4 = (r + 3) >> 2;
    while (b >= 0 && blocks[b].kind != ARC_BLOCK_ARC) --b;   // DENSE blocks own no items
    if (b < 0) return;
    const long long local = it - (blocks[b].v_off / r) * R4;
    if (local >= static_cast<long long>(blocks[b].n) * R4) return;
    const uint4 x = philox4x32_10(make_uint4(static_cast<unsigned>(local), static_cast<unsigned>(b), t_lo, t_hi), key);
    float z[4];
    box_muller(x.x, x.y, z[0], z[1]);
    box_muller(x.z, x.w, z[2], z[3]);
    const long long q = local / R4;
    const int j0 = 4 * static_cast<int>(local - q * R4);
    const int ldv = (blocks[b].n + 3) & ~3;
    float* dst = V + blocks[b].v_off + q;   // V_b stored transposed: column j at j * ldv
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (j0 + k < r) dst[static_cast<long long>(j0 + k) * ldv] = z[k];
}

}  // namespace rng
}  // namespace arc
