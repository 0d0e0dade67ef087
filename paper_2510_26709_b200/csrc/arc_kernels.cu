// arc_kernels.cu — sm_100a kernels of the EF21M + ARC-Top-K step.
//
// Every floating-point operation on the path is an explicitly rounded IEEE
// binary32 intrinsic (__fadd_rn, __fmul_rn, ...) in the order DESIGN.md §3
// fixes (R9, R11), so results are bit-identical to the plain definition; the
// library is also built with -fmad=false -ftz=false -prec-div=true.
//
// Kernels (DESIGN.md §5 has the roofline of each):
//   k_vgen          S0  V_b = Gaussian(seed, t, b)                  P:229-230, Alg.1 l.3
//   k_ef_sketch     S1+S2  h' = (1-eta)h + eta grad; Delta = h' - g;  eq:ef21m-1 P:325,
//                      P_i = (1/sqrt r) Delta V; (G==1) P, Sigma      P:231-237, Alg.1 l.4-6
//   k_sketch_reduce S2 (G>1) ordered node sum of exchanged P_i, Sigma
//   k_select        S3  I_b = argtop_K(Sigma), cluster radix select  zn28373 P:236-237
//   k_gather_ef     S4 (+S5+S6 when G==1)                            2zn20 P:241-243, eq:ef21m-2
//   k_scatter       S6 (G>1)                                         eq:ef21m-3 P:327
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "arc_device.cuh"
#include "arc_internal.cuh"

namespace cg = cooperative_groups;

namespace arc {
namespace {
using namespace dev;

// =============================================================================
// S0: ARC-RNG v1 (R8) — Philox4x32-10 + Box–Muller with portable
// ln / sincos(2 pi u) made of exactly rounded operations only.
// =============================================================================

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
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
__device__ __forceinline__ float word_to_unit(unsigned x) {
    return fadd(fmul(__uint2float_rn(x >> 9), 0x1p-23f), 0x1p-24f);
}

// ln(u), u a positive normal float: u = f 2^e with f in [sqrt(1/2), sqrt(2)),
// x = f - 1 exact, Cephes logf minimax polynomial in Horner form with fma.
__device__ __forceinline__ float ln_exact_ops(float u) {
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
__device__ __forceinline__ void sincos_quarter_turn(float f, float& s, float& c) {
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
__device__ __forceinline__ void sincos_2pi(float u, float& s, float& c) {
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

__device__ __forceinline__ void box_muller(unsigned xa, unsigned xb, float& za, float& zb) {
    const float ua = word_to_unit(xa), ub = word_to_unit(xb);
    const float rho = __fsqrt_rn(fmul(-2.0f, ln_exact_ops(ua)));
    float s, c;
    sincos_2pi(ub, s, c);
    za = fmul(rho, c);
    zb = fmul(rho, s);
}

// V_b[q][j]: one thread per (q, jj) of block b = blockIdx.y; counter
// (q*R4 + jj, b, lo32 t, hi32 t), key (lo32 seed, hi32 seed).
__global__ void __launch_bounds__(256) k_vgen(const BlockDev* __restrict__ blocks, int r, uint2 key,
                                              unsigned t_lo, unsigned t_hi, float* __restrict__ V) {
    const int b = blockIdx.y;
    if (blocks[b].kind != ARC_BLOCK_ARC) return;
    const int n = blocks[b].n;
    const long long v_off = blocks[b].v_off;
    const int R4 = (r + 3) >> 2;
    const long long items = static_cast<long long>(n) * R4;
    for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < items;
         it += (long long)gridDim.x * blockDim.x) {
        const uint4 x = philox4x32_10(make_uint4(static_cast<unsigned>(it), static_cast<unsigned>(b), t_lo, t_hi), key);
        float z[4];
        box_muller(x.x, x.y, z[0], z[1]);
        box_muller(x.z, x.w, z[2], z[3]);
        const long long q = it / R4;
        const int j0 = 4 * static_cast<int>(it - q * R4);
        float* dst = V + v_off + q * r + j0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (j0 + k < r) dst[k] = z[k];
    }
}

__device__ __forceinline__ int row_valid_cols(const BlockDev& B, int p) {
    const long long rest = B.len - static_cast<long long>(p) * B.n;
    return rest < B.n ? static_cast<int>(rest) : B.n;
}

// =============================================================================
// S2 for G > 1: ordered node sum of the all-gathered P_i (R9, R21) and Sigma.
// xrecv layout [G][M][L][r]; global node id = g*L + l.
// =============================================================================
__global__ void __launch_bounds__(256) k_sketch_reduce(const float* __restrict__ xrecv, int M, int G, int L, int r,
                                                       float Nf, float* __restrict__ sigma, unsigned* status) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < M; p += gridDim.x * blockDim.x) {
        float sig = 0.0f;
        for (int j = 0; j < r; ++j) {
            float S = 0.0f;
            for (int g = 0; g < G; ++g)
                for (int l = 0; l < L; ++l) {
                    const float v = xrecv[((static_cast<long long>(g) * M + p) * L + l) * r + j];
                    S = (g == 0 && l == 0) ? v : fadd(S, v);
                }
            const float pv = __fdiv_rn(S, Nf);
            sig = fadd(sig, fmul(pv, pv));
        }
        sigma[p] = sig;
        if (!isfinite(sig)) atomicOr(status, kStatusNonfinite);
    }
}

// =============================================================================
// S3: I_b = argtop_{K_b}(Sigma_b) — one 8-CTA cluster per block.
// MSB-first radix select over the order keys (R15) with 8-bit digits: each CTA
// histograms its slice in shared memory, the cluster merges the histograms
// through distributed shared memory, and every CTA derives the same digit.
// After 4 passes the K-th key T and the number of keys == T still to take are
// known; a stable compaction then writes the selected rows in ascending order,
// taking the keys equal to T with the smallest indices (R5).
// =============================================================================
constexpr int kSelCluster = 8;
constexpr int kSelThreads = 1024;
constexpr int kSelItems = 8;

__device__ __forceinline__ unsigned order_key(float s) {
    return isnan(s) ? 0xFFFFFFFFu : __float_as_uint(s);
}

// exclusive scan of one int per thread over the CTA; returns the exclusive
// prefix and writes the CTA total to *total.
__device__ __forceinline__ int cta_exclusive_scan(int v, int* warp_sums, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        int w = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(kFull, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nw) warp_sums[lane] = w;       // inclusive
    }
    __syncthreads();
    const int excl = x - v + (warp > 0 ? warp_sums[warp - 1] : 0);
    *total = warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
    return excl;
}

__global__ void __cluster_dims__(kSelCluster, 1, 1) __launch_bounds__(kSelThreads)
k_select(const BlockDev* __restrict__ blocks, const float* __restrict__ sigma, int32_t* __restrict__ sel,
         int cache_cap) {
    cg::cluster_group cluster = cg::this_cluster();
    const int crank = static_cast<int>(cluster.block_rank());
    const int b = blockIdx.x / kSelCluster;
    const BlockDev B = blocks[b];
    const int m = B.m, K = B.K;
    const int tid = threadIdx.x, lane = tid & 31;
    const int lo = static_cast<int>((static_cast<long long>(m) * crank) / kSelCluster);
    const int hi = static_cast<int>((static_cast<long long>(m) * (crank + 1)) / kSelCluster);
    const int len = hi - lo;
    int32_t* __restrict__ out = sel + B.sel_base;

    if (B.kind != ARC_BLOCK_ARC || K >= m) {        // identity selection (DENSE, or K = m)
        for (int p = lo + tid; p < hi; p += kSelThreads) out[p] = p;
        return;                                     // uniform across the cluster: no DSMEM use
    }
    const float* __restrict__ sg = sigma + B.row_base + lo;

    extern __shared__ unsigned s_keys[];            // this CTA's slice of order keys, if it fits
    __shared__ unsigned hist[2][256];
    __shared__ int warp_sums[32];
    __shared__ unsigned s_digit, s_above;
    __shared__ int s_cnt[2];                        // this CTA: #gt, #eq

    const bool cached = len <= cache_cap;
    if (cached) {
        for (int i = tid; i < len; i += kSelThreads) s_keys[i] = order_key(sg[i]);
        __syncthreads();
    }
    auto key_at = [&](int i) -> unsigned { return cached ? s_keys[i] : order_key(sg[i]); };

    constexpr int U = 4;                            // keys per thread per sweep (load ILP)
    unsigned prefix = 0, pmask = 0;
    int krem = K;
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        unsigned* h = hist[pass & 1];
        for (int i = tid; i < 256; i += kSelThreads) h[i] = 0;
        __syncthreads();
        for (int base = 0; base < len; base += kSelThreads * U) {
            unsigned kk[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = base + u * kSelThreads + tid;
                kk[u] = i < len ? key_at(i) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = base + u * kSelThreads + tid;
                const bool match = i < len && (kk[u] & pmask) == prefix;
                const unsigned bin = (kk[u] >> shift) & 255u;
                const unsigned want = __ballot_sync(kFull, match);
                if (match) {
                    const unsigned grp = __match_any_sync(want, bin);
                    if (lane == __ffs(grp) - 1) atomicAdd(&h[bin], static_cast<unsigned>(__popc(grp)));
                }
            }
        }
        cluster.sync();
        if (tid < 32) {
            // lane l owns bins 255-8l .. 248-8l (descending); sum over the cluster
            unsigned cnt[8];
            unsigned mine = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int bin = 255 - 8 * lane - k;
                unsigned c = 0;
#pragma unroll
                for (int cr = 0; cr < kSelCluster; ++cr) c += cluster.map_shared_rank(h, cr)[bin];
                cnt[k] = c;
                mine += c;
            }
            unsigned incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += y;
            }
            const unsigned excl = incl - mine;   // keys in bins above my 8
            const bool here = excl < static_cast<unsigned>(krem) && incl >= static_cast<unsigned>(krem);
            if (here) {
                unsigned above = excl;
                int k = 0;
                while (above + cnt[k] < static_cast<unsigned>(krem)) { above += cnt[k]; ++k; }
                s_digit = 255u - 8u * lane - k;
                s_above = above;
            }
        }
        __syncthreads();
        prefix |= s_digit << shift;
        pmask |= 255u << shift;
        krem -= static_cast<int>(s_above);
        __syncthreads();
    }
    const unsigned T = prefix;       // the K-th largest key
    const int need_eq = krem;        // keys == T to take (>= 1), smallest indices first

    // ---- counts of this slice, shared with the cluster
    int ngt = 0, neq = 0;
    for (int i = tid; i < len; i += kSelThreads) {
        const unsigned key = key_at(i);
        ngt += key > T;
        neq += key == T;
    }
    int tot;
    cta_exclusive_scan(ngt, warp_sums, &tot);
    if (tid == 0) s_cnt[0] = tot;
    cta_exclusive_scan(neq, warp_sums, &tot);
    if (tid == 0) s_cnt[1] = tot;
    cluster.sync();
    int sel_before = 0, eq_before = 0;
    for (int cr = 0; cr < crank; ++cr) {
        const int* rc = cluster.map_shared_rank(s_cnt, cr);
        const int g = rc[0], e = rc[1];
        const int take = max(0, min(e, need_eq - eq_before));
        sel_before += g + take;
        eq_before += e;
    }

    // ---- stable compaction of the slice, kSelItems consecutive keys per thread
    for (int base = 0; base < len; base += kSelThreads * kSelItems) {
        const int i0 = base + tid * kSelItems;
        unsigned keys[kSelItems];
        int my_eq = 0;
#pragma unroll
        for (int e = 0; e < kSelItems; ++e) {
            const int i = i0 + e;
            keys[e] = i < len ? key_at(i) : 0u;
            my_eq += (i < len && keys[e] == T);
        }
        int eq_total;
        int eq_rank = eq_before + cta_exclusive_scan(my_eq, warp_sums, &eq_total);
        bool take[kSelItems];
        int my_sel = 0;
#pragma unroll
        for (int e = 0; e < kSelItems; ++e) {
            bool t = false;
            if (i0 + e < len) {
                if (keys[e] > T) t = true;
                else if (keys[e] == T) { t = eq_rank < need_eq; ++eq_rank; }
            }
            take[e] = t;
            my_sel += t;
        }
        int sel_total;
        int pos = sel_before + cta_exclusive_scan(my_sel, warp_sums, &sel_total);
#pragma unroll
        for (int e = 0; e < kSelItems; ++e)
            if (take[e]) out[pos++] = lo + i0 + e;
        sel_before += sel_total;
        eq_before += eq_total;
    }
    cluster.sync();   // keep shared memory alive until every CTA has read it
}

// =============================================================================
// S4 (+S5, S6 when G == 1): one warp per selected row.
//   (DENSE blocks first apply eq:ef21m-1, since the sketch pass skips them)
//   C_i = h_i - g_i on row I_k; g_i <- g_i + C_i                    eq:ef21m-2 (R12)
//   mode 0: A = C_0 + C_1 + ... (ascending node); val = A / N;
//           gbar <- gbar + val; values[k] = val                     P:242, R13
//   mode 1: wire[k] = local node sum      (NCCL All-Reduce follows)
//   mode 2: wire[i][k] = C_i              (ordered exchange follows)
// =============================================================================
// 4 consecutive floats of a row: one 128-bit access when the quad is whole and
// 16-byte aligned, else element by element (masked by `valid` columns).
struct Quad {
    float v[4];
};
__device__ __forceinline__ Quad load_quad(const float* p, bool vec4, int nvalid) {
    Quad x;
    if (vec4) {
        const float4 t = *reinterpret_cast<const float4*>(p);
        x.v[0] = t.x; x.v[1] = t.y; x.v[2] = t.z; x.v[3] = t.w;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) x.v[k] = k < nvalid ? p[k] : 0.0f;
    }
    return x;
}
__device__ __forceinline__ void store_quad(float* p, const Quad& x, bool vec4, int nvalid) {
    if (vec4) {
        *reinterpret_cast<float4*>(p) = make_float4(x.v[0], x.v[1], x.v[2], x.v[3]);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < nvalid) p[k] = x.v[k];
    }
}

__global__ void __launch_bounds__(256) k_gather_ef(const GatherLaunch a) {
    constexpr int U = 4;                  // quads per lane in flight
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int w = gw; w < a.num_rows; w += nw) {
        const SelRow R = a.rows[w];
        const BlockDev& B = a.blocks[R.b];
        const int p = a.sel[B.sel_base + R.k];
        const int n = B.n;
        const int nv = row_valid_cols(B, p);
        const long long e0 = B.off + static_cast<long long>(p) * n;
        const long long o0 = B.val_base + static_cast<long long>(R.k) * n;
        const bool dense = B.kind == ARC_BLOCK_DENSE;
        // wire / values rows are 16-byte aligned when n % 4 == 0 (val_base is a sum of K n)
        const bool vrow = B.vec && (o0 % 4 == 0);
        const int nq = (n + 3) >> 2;
        for (int f0 = 0; f0 < nq; f0 += 32 * U) {
            int cnt[U];           // valid state columns of each quad
            int ocnt[U];          // columns of each quad inside the row (padding -> +0)
            bool v4[U], ov4[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = 4 * (f0 + 32 * u + lane);
                cnt[u] = max(0, min(4, nv - q));
                ocnt[u] = max(0, min(4, n - q));
                v4[u] = B.vec && cnt[u] == 4;
                ov4[u] = vrow && ocnt[u] == 4;
            }
            Quad A[U];
            for (int i = 0; i < a.nodes_local; ++i) {
                float* __restrict__ ph = a.nodes.h[i];
                float* __restrict__ pg = a.nodes.g[i];
                Quad hq[U], gq[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const long long e = e0 + 4 * (f0 + 32 * u + lane);
                    if (cnt[u] > 0) {
                        gq[u] = load_quad(pg + e, v4[u], cnt[u]);
                        if (dense) {   // DENSE block: eq:ef21m-1 applied here (R11, R20)
                            const Quad hv = load_quad(ph + e, v4[u], cnt[u]);
                            const Quad gr = load_quad(a.nodes.grad[i] + e, v4[u], cnt[u]);
#pragma unroll
                            for (int k = 0; k < 4; ++k) hq[u].v[k] = fadd(fmul(a.ome, hv.v[k]), fmul(a.eta, gr.v[k]));
                            store_quad(ph + e, hq[u], v4[u], cnt[u]);
                        } else {
                            hq[u] = load_quad(ph + e, v4[u], cnt[u]);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (ocnt[u] == 0) continue;
                    const long long e = e0 + 4 * (f0 + 32 * u + lane);
                    Quad c, gn;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        c.v[k] = k < cnt[u] ? fsub(hq[u].v[k], gq[u].v[k]) : 0.0f;   // C_i (+0 padding)
                        gn.v[k] = fadd(gq[u].v[k], c.v[k]);                            // R12
                        A[u].v[k] = (i == 0) ? c.v[k] : fadd(A[u].v[k], c.v[k]);
                    }
                    if (cnt[u] > 0) store_quad(pg + e, gn, v4[u], cnt[u]);
                    if (a.mode == 2)
                        store_quad(a.values + static_cast<long long>(i) * a.sum_Kn + o0 + 4 * (f0 + 32 * u + lane),
                                   c, ov4[u] && (a.sum_Kn % 4 == 0), ocnt[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (ocnt[u] == 0) continue;
                const int q = 4 * (f0 + 32 * u + lane);
                if (a.mode == 0) {
                    const long long e = e0 + q;
                    Quad val, gb;
#pragma unroll
                    for (int k = 0; k < 4; ++k) val.v[k] = k < cnt[u] ? __fdiv_rn(A[u].v[k], a.Nf) : 0.0f;   // R3
                    if (cnt[u] > 0) {
                        gb = load_quad(a.gbar + e, v4[u], cnt[u]);
#pragma unroll
                        for (int k = 0; k < 4; ++k) gb.v[k] = fadd(gb.v[k], val.v[k]);                    // R13
                        store_quad(a.gbar + e, gb, v4[u], cnt[u]);
                    }
                    if (a.values != nullptr) store_quad(a.values + o0 + q, val, ov4[u], ocnt[u]);
                } else if (a.mode == 1) {
                    store_quad(a.values + o0 + q, A[u], ov4[u], ocnt[u]);
                }
            }
        }
    }
}

// =============================================================================
// S6 for G > 1: gbar[I] += A / N after exchange #2.
//   mode 0: wire holds the summed rows (NCCL All-Reduce)
//   mode 1: wire holds [N][sumKn] per-node rows: ordered sum (R9) first
// =============================================================================
__global__ void __launch_bounds__(256) k_scatter(const ScatterLaunch a) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int w = gw; w < a.num_rows; w += nw) {
        const SelRow R = a.rows[w];
        const BlockDev& B = a.blocks[R.b];
        const int p = a.sel[B.sel_base + R.k];
        const int n = B.n;
        const int nv = row_valid_cols(B, p);
        const long long e0 = B.off + static_cast<long long>(p) * n;
        const long long o0 = B.val_base + static_cast<long long>(R.k) * n;
        for (int q = lane; q < n; q += 32) {
            if (q < nv) {
                float A;
                if (a.mode == 0) {
                    A = a.wire[o0 + q];
                } else {
                    A = a.wire[o0 + q];
                    for (int i = 1; i < a.nodes_total; ++i) A = fadd(A, a.wire[static_cast<long long>(i) * a.sum_Kn + o0 + q]);
                }
                const float val = __fdiv_rn(A, a.Nf);
                a.gbar[e0 + q] = fadd(a.gbar[e0 + q], val);
                if (a.values != nullptr) a.values[o0 + q] = val;
            } else if (a.values != nullptr) {
                a.values[o0 + q] = 0.0f;
            }
        }
    }
}

}  // namespace

// ---- launchers ---------------------------------------------------------------

void launch_vgen(const BlockDev* blocks_dev, int num_blocks, int max_nR4, int r, uint64_t seed, int64_t t,
                 float* V, cudaStream_t s) {
    const int threads = 256;
    int gx = (max_nR4 + threads - 1) / threads;
    if (gx < 1) gx = 1;
    if (gx > 64) gx = 64;
    dim3 grid(gx, num_blocks);
    const uint2 key = make_uint2(static_cast<unsigned>(seed), static_cast<unsigned>(seed >> 32));
    k_vgen<<<grid, threads, 0, s>>>(blocks_dev, r, key, static_cast<unsigned>(static_cast<uint64_t>(t)),
                                    static_cast<unsigned>(static_cast<uint64_t>(t) >> 32), V);
}

void launch_sketch_reduce(const float* xrecv, int M, int G, int nodes_local, int r, float Nf, float* sigma,
                          unsigned* status, cudaStream_t s) {
    int grid = (M + 255) / 256;
    if (grid < 1) grid = 1;
    if (grid > 4096) grid = 4096;
    k_sketch_reduce<<<grid, 256, 0, s>>>(xrecv, M, G, nodes_local, r, Nf, sigma, status);
}

constexpr int kSelCacheMaxBytes = 200 * 1024;

void launch_select(const BlockDev* blocks, int num_blocks, const float* sigma, int32_t* sel, int max_slice,
                   cudaStream_t s) {
    static int configured = -1;
    int cap = max_slice;
    if (cap * 4 > kSelCacheMaxBytes) cap = kSelCacheMaxBytes / 4;
    if (cap < 1) cap = 1;
    const int bytes = cap * 4;
    if (bytes > 48 * 1024 && configured < bytes) {
        cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, kSelCacheMaxBytes);
        configured = kSelCacheMaxBytes;
    }
    k_select<<<num_blocks * kSelCluster, kSelThreads, bytes, s>>>(blocks, sigma, sel, cap);
}

int select_max_slice(int max_m) { return (max_m + kSelCluster - 1) / kSelCluster; }

static int rows_grid(int num_rows) {
    int grid = (num_rows + 7) / 8;   // 8 warps per CTA, one warp per row
    if (grid < 1) grid = 1;
    if (grid > 148 * 16) grid = 148 * 16;
    return grid;
}

void launch_gather_ef(const GatherLaunch& a, cudaStream_t s) {
    k_gather_ef<<<rows_grid(a.num_rows), 256, 0, s>>>(a);
}

void launch_scatter(const ScatterLaunch& a, cudaStream_t s) {
    k_scatter<<<rows_grid(a.num_rows), 256, 0, s>>>(a);
}

}  // namespace arc
