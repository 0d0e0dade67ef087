// arc_sketch.cu — S1 (+S2 when the GPU holds every node and there is one):
// the fused streaming pass of the EF21M + ARC-Top-K step, the one kernel that
// moves ~98 % of the step's HBM bytes.
//
// Per element (eq:ef21m-1 P:325; ARC-NUM v1 O1-O3, R11, R4):
//     h' = fma(eta, grad, (1 - eta) h)      (h' stored)      Delta = h' - g
// Per row p and sketch column j (Alg.1 l.4; ARC-NUM v1 O6, R2, R9):
//     P'_i[p][j] = O6 dot product of Delta_p with column j of V: row chunks of
//     1024 columns; in chunk c lane l accumulates a_l <- fma(Delta_q, V_qj, a_l)
//     over q = 1024c + 128s + 4l + e (s = 0..7, e = 0..3, q < nv); a butterfly
//     gives w_c = a_0; P' = ((w_0 + w_1) + ...) left to right.
// With one node on this GPU and no exchange (mode 0): S = P'_0 and
//     Sigma_p = fma(S_p,r-1, S_p,r-1, ... fma(S_p0, S_p0, +0))       (O8, R3)
// plus the digit-1 histogram of Sigma's order key for the selection.
//
// Layout.  The O6 order maps one row to one warp: lane l owns the float4 at
// columns 128s + 4l of every 512-byte row segment, so a warp streams its row
// front to back — every load and store is a fully coalesced 512-byte warp
// access, and consecutive segments of a row are contiguous (DRAM-page
// friendly).  Delta stays in registers and meets V_b^T (stored transposed,
// [r][n], staged in shared memory per block when it fits) in the lane's fma
// chain.  UN segments are loaded per batch (3 UN float4 per lane in flight).
// A CTA walks a host-balanced list of tiles (8 or 32 rows of one block for one
// node); warp w takes rows w, w + 8, ... of each tile, independently of the
// other warps; the CTA meets at a barrier only when the block changes, to
// publish its shared histogram and stage the next block's V.
#include <cuda_runtime.h>

#include <cstdint>

#include "arc_device.cuh"
#include "arc_internal.cuh"
#include "arc_rng.cuh"

namespace arc {
namespace {
using namespace dev;

constexpr int kThreads = kSketchThreads;   // 256 = 8 warps
constexpr int kTileCache = 128;            // tile descriptors cached in shared memory

// valid columns of row p of a block (the last row of a padded flat block is short, R14)
__device__ __forceinline__ int row_cols(long long len, int n, int p) {
    const long long rest = len - static_cast<long long>(p) * n;
    return rest < n ? static_cast<int>(rest) : n;
}

// Cache policy of the streaming pass's loads (build-time knobs for A/B runs):
// ARC_SK_LDG for the gradient (read once), ARC_SK_LDS for the state h, g;
// 0 = streaming (evict-first), 1 = cache global (L2, normal eviction),
// 4 = cache global + 256-byte L2 prefetch.  ARC_SK_ST: the h' store.
// Measured (profiles/r02_cache_policy.txt): the state through L2 with normal
// eviction and the gradient evict-first is within 0.6 % of the best on every
// layout tried (C3 -2.3 % step time against all-streaming); the gradient through
// L2 as well gains 0.5 % on C3 but costs 16 % on C2 (d = 11.7M: h and g then no
// longer stay in the 126 MB L2 between steps).
#ifndef ARC_SK_LDG
#define ARC_SK_LDG 0
#endif
#ifndef ARC_SK_LDS
#define ARC_SK_LDS 1
#endif
#ifndef ARC_SK_ST
#define ARC_SK_ST 0
#endif
template <int POL>
__device__ __forceinline__ float4 sk_ld4p(const float* p) {
    if constexpr (POL == 1) {
        return __ldcg(reinterpret_cast<const float4*>(p));
    } else if constexpr (POL == 4) {
        float4 v;
        asm volatile("ld.global.cg.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
        return v;
    } else {
        return __ldcs(reinterpret_cast<const float4*>(p));
    }
}
__device__ __forceinline__ float4 sk_ld4(const float* p) { return sk_ld4p<ARC_SK_LDS>(p); }    // h, g
__device__ __forceinline__ float4 sk_ld4g(const float* p) { return sk_ld4p<ARC_SK_LDG>(p); }   // grad
// scalar loads (rows that are not 16-byte aligned): streaming, so the 4 loads of a
// quad meet in L1 (cache-global scalar loads measured 23 % slower on n = 5461 rows)
__device__ __forceinline__ float sk_ld1(const float* p) { return __ldcs(p); }
__device__ __forceinline__ void sk_st4(float* p, float4 v) {
#if ARC_SK_ST == 1      // write-back (default policy)
    *reinterpret_cast<float4*>(p) = v;
#elif ARC_SK_ST == 2    // no L1 allocation, default L2 policy
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
#else                   // streaming store, the measured default
    __stcs(reinterpret_cast<float4*>(p), v);
#endif
}

// sum over the 32 lanes, butterfly order of O6 (every lane ends with the same value)
__device__ __forceinline__ float butterfly(float a) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) a = fadd(a, __shfl_xor_sync(kFull, a, o));
    return a;
}

// V_b^T of the CTA's current block is staged in (dynamic) shared memory when it
// fits (a.vs_cap floats), so the lane chains read it with conflict-free 16-byte
// loads next to the streaming traffic instead of through L1/L2.
constexpr int kVsMax = 12288;              // floats of V_b^T staged at most (48 KB)
// The second launch (RANGED instantiation: blocks whose V_b^T exceeds kVsMax,
// and blocks of rows of <= 4 columns) runs one CTA per SM with the warps of
// two main-kernel CTAs, so the whole of V_b^T up to 196 KB is staged once per
// block; only wider V is staged in ranges.
constexpr int kVsBig = 50176;
__host__ __device__ constexpr int wide_threads(int rj) { return rj <= 16 ? 512 : 256; }
__host__ __device__ constexpr int wide_un(int rj) { return rj <= 8 ? 4 : 3; }

// One segment (columns q..q+3 of lane l) of one row: momentum, residual, the
// h' store and the lane's O6 fma chains; at the end of a 1024-column chunk the
// butterfly folds the lane sums into P (left to right over chunks).
template <int RJ, bool NOEF>
__device__ __forceinline__ void segment(const SketchLaunch& a, int k, int nseg, int q, int nv, long long base, bool vec,
                                        int vld, int vc0, const float* Vb, bool V_vec, bool v_smem, bool sketch, float* ph,
                                        const float (&gx)[4], const float (&hx)[4], const float (&dx)[4], float eta,
                                        float ome, int r, float (&acc)[RJ], float (&P)[RJ]) {
    const long long e = base + q;
    float hn[4], dl[4];
    if (NOEF) {
        // compressed MSGD without EF: the sketch sees the gradient itself; the
        // replicated momentum u (kept in gbar) decays, u <- beta u (eta = beta),
        // once per element (node-0 tiles, ph == gbar; others ph == nullptr)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            hn[kk] = fmul(eta, hx[kk]);
            dl[kk] = gx[kk];
        }
    } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            hn[kk] = ffma(eta, gx[kk], fmul(ome, hx[kk]));   // O2, R11
            dl[kk] = fsub(hn[kk], dx[kk]);                   // O3, R4
        }
    }
    if (NOEF && ph == nullptr) {
    } else if (q + 3 < nv && vec) {
        sk_st4(ph + e, make_float4(hn[0], hn[1], hn[2], hn[3]));
    } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
            if (q + kk < nv) ph[e + kk] = hn[kk];
    }
    if (sketch) {
        // V_b^T row j, columns q..q+3: one 16-byte load per lane
#pragma unroll
        for (int j = 0; j < RJ; ++j) {
            if (j >= r) break;
            const float* vj = Vb + static_cast<long long>(j) * vld + (q - vc0);   // V_b^T [r][vld] from column vc0
            float v[4];
            if (q + 3 < nv && V_vec) {
                const float4 t4 = v_smem ? *reinterpret_cast<const float4*>(vj) : __ldg(reinterpret_cast<const float4*>(vj));
                v[0] = t4.x; v[1] = t4.y; v[2] = t4.z; v[3] = t4.w;
            } else {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) v[kk] = q + kk < nv ? vj[kk] : 0.0f;
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                if (q + kk < nv) acc[j] = ffma(dl[kk], v[kk], acc[j]);   // O6 (padding never summed)
        }
    } else if (a.mode == 2) {                                           // Top-K baseline: ||Delta_p||^2
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
            if (q + kk < nv) acc[0] = ffma(dl[kk], dl[kk], acc[0]);
    }
    if (a.mode != 3 && ((k & 7) == 7 || k == nseg - 1)) {               // end of a 1024-column chunk
#pragma unroll
        for (int j = 0; j < RJ; ++j) {
            const float w = butterfly(acc[j]);
            P[j] = (k < 8) ? w : fadd(P[j], w);
            acc[j] = 0.0f;
        }
    }
}

// Per-row epilogue (P[j] is the same in every lane).
// Rand-K key of row p of block b at this step's t (R16; ARC_FLAG_DEVICE_T: t from the device counter)
__device__ __forceinline__ float randk_key_t(const unsigned long long* t_dev, unsigned t_lo, unsigned t_hi, uint2 key, int p,
                                           int b) {
    if (t_dev != nullptr) {
        const unsigned long long t = __ldcg(t_dev);
        t_lo = static_cast<unsigned>(t);
        t_hi = static_cast<unsigned>(t >> 32);
    }
    const uint4 x = rng::philox4x32_10(make_uint4(static_cast<unsigned>(p), static_cast<unsigned>(b) | 0x80000000u, t_lo, t_hi),
                                       key);
    return __uint_as_float(x.x >> 2);
}
__device__ __forceinline__ float randk_key(const SketchLaunch& a, int p, int b) {
    return randk_key_t(a.t_dev, a.t_lo, a.t_hi, a.key, p, b);
}

template <int RJ>
__device__ __forceinline__ void row_epilogue(const SketchLaunch& a, int p, int row_base, int b, int node, int lane, int r,
                                             const float (&P)[RJ], unsigned* s_hist) {
    if (a.mode == 3) {
        // Rand-K: row p's shared key (R16), written once (node-0 tiles)
        if (lane == 0 && node == 0) {
            const float sig = randk_key(a, p, b);
            a.sigma[row_base + p] = sig;
            atomicAdd(&s_hist[order_key_dev(sig) >> kHist1Shift], 1u);
        }
    } else if (a.mode == 2) {
        // Top-K baseline: this node's own ||row||^2 and its selection histogram
        if (lane == 0) {
            const float sig = P[0];
            a.sigma[static_cast<long long>(node) * a.M + row_base + p] = sig;
            atomicAdd(&s_hist[order_key_dev(sig) >> kHist1Shift], 1u);   // slot (node, block)
            if (!isfinite(sig)) atomicOr(a.status, kStatusNonfinite);
        }
    } else {
        if (a.pnodes != nullptr && lane < r) {                           // P'_i for the exchange / node sum
            float v = P[0];
#pragma unroll
            for (int j = 1; j < RJ; ++j)
                if (lane == j) v = P[j];
            a.pnodes[(static_cast<long long>(row_base + p) * a.nodes_local + node) * r + lane] = v;
        }
        if (a.mode == 0 && lane == 0) {                                  // S = P'_0: Sigma (O8)
            float sig = 0.0f;
#pragma unroll
            for (int j = 0; j < RJ; ++j)
                if (j < r) sig = ffma(P[j], P[j], sig);
            a.sigma[row_base + p] = sig;
            atomicAdd(&s_hist[order_key_dev(sig) >> kHist1Shift], 1u);   // digit-1 histogram
            if (!isfinite(sig)) atomicOr(a.status, kStatusNonfinite);
        }
    }
}

// The register path: the same per-segment arithmetic with the batch loaded
// straight into registers (UN segments, 3 UN float4 per lane), warps streaming
// their rows independently; V_b^T staged in shared memory as above.
// RANGED: the launch over the blocks whose V_b^T does not fit the stage; V is
// staged in ranges of whole 1024-column chunks and every row carries its P'
// across ranges in shared memory (the O6 order is unchanged)
template <int RJ, int UN, int MINB, bool NOEF, bool RANGED>
__global__ void __launch_bounds__(RANGED ? wide_threads(RJ) : kThreads, MINB) k_ef_sketch(const SketchLaunch a) {
    constexpr int NT = RANGED ? wide_threads(RJ) : kThreads, NW = NT / 32;
    __shared__ TileDesc s_tile[kTileCache];
    __shared__ unsigned s_hist[kHist1Bins];     // digit-1 histogram of this CTA's Sigma (modes 0, 3)
    __shared__ float s_P[RANGED ? 32 : 1][RJ];  // (RANGED) the tile rows' running P' between ranges
    extern __shared__ __align__(16) float4 dyn[];   // V_b^T
    float* Vs = reinterpret_cast<float*>(dyn);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int list_begin = a.cta_begin[blockIdx.x], list_end = a.cta_begin[blockIdx.x + 1];
    if (list_begin >= list_end) return;
    const int ntile = list_end - list_begin;
    for (int i = tid; i < min(ntile, kTileCache) * 4; i += NT)
        reinterpret_cast<uint4*>(s_tile)[i] = __ldg(reinterpret_cast<const uint4*>(a.tiles + list_begin) + i);
    for (int i = tid; i < kHist1Bins; i += NT) s_hist[i] = 0;
    __syncthreads();
    grid_dependency_wait();   // the previous kernel (g, V, histogram reset) is complete

    const int r = a.r;
    const float eta = a.eta, ome = a.ome;
    const int mode = a.mode;
    const bool sketch = mode <= 1;
    const bool cta_hist = true;                 // every mode histograms its keys in shared memory first
    auto flush_hist = [&](int b) {
        unsigned* gh = a.hist1 + static_cast<long long>(b) * kHist1Bins;
        for (int i = tid; i < kHist1Bins; i += NT) {
            const unsigned v = s_hist[i];
            if (v) { atomicAdd(gh + i, v); s_hist[i] = 0; }
        }
    };
    auto tile = [&](int li) -> const TileDesc* {
        return li - list_begin < kTileCache ? &s_tile[li - list_begin] : a.tiles + li;
    };

    int carry = warp;                           // (RANGED) this warp's first row of the next tile
    int cur_b = -1;                             // histogram slot of the current tile: block (mode 2: node, block)
    bool v_smem = false;
    for (int li = list_begin; li < list_end; ++li) {
        const TileDesc* Tp = tile(li);
        const long long T_off = Tp->off, T_len = Tp->len, T_voff = Tp->v_off;
        const int T_n = Tp->n, T_row0 = Tp->row0, T_rows = Tp->rows, T_row_base = Tp->row_base, T_b = Tp->b;
        const bool T_vec = Tp->vec != 0;
        const int node = Tp->node;
        const int hslot = mode == 2 ? node * a.num_blocks + T_b : T_b;
        if (hslot != cur_b) {
            __syncthreads();
            if (cta_hist && cur_b >= 0) flush_hist(cur_b);
            const int nvf = r * ((T_n + 3) & ~3);
            v_smem = sketch && nvf <= a.vs_cap;
            if (v_smem) {
                const float* __restrict__ src = a.V + T_voff;
                if ((T_voff & 3) == 0 && (nvf & 3) == 0) {
                    for (int i = tid; i < (nvf >> 2); i += NT)
                        reinterpret_cast<float4*>(Vs)[i] = __ldg(reinterpret_cast<const float4*>(src) + i);
                } else {
                    for (int i = tid; i < nvf; i += NT) Vs[i] = __ldg(src + i);
                }
            }
            __syncthreads();
        }
        cur_b = hslot;
        const float* __restrict__ pg = a.nodes.grad[node];
        // (without EF: h is the replicated momentum u = gbar, read and scaled by node 0 only; no g)
        float* __restrict__ ph = NOEF ? (node == 0 ? a.gbar : nullptr) : a.nodes.h[node];
        const float* __restrict__ pgg = NOEF ? nullptr : a.nodes.g[node];
        const float* Vb = v_smem ? Vs : a.V + T_voff;
        const bool V_vec = true;   // V_b^T rows start 16-byte aligned (padded to ldv = round_up(n, 4))

        bool streamed = false;                  // (RANGED) tile done by the per-thread or ranged path
        if constexpr (RANGED) {
          streamed = T_n <= 4 || !v_smem;
          if (T_n <= 4) {
            // rows of at most 4 columns (e.g. n = 1): one row per THREAD (tiles of up
            // to 256 rows).  In O6 terms only lane 0 holds data, so the butterfly
            // yields a_0 (+) (+0): the lane's own fma chain with -0 turned into +0.
            const int rr = tid;
            if (rr < T_rows) {
                const int p = T_row0 + rr;
                const int nv = row_cols(T_len, T_n, p);
                const long long base = T_off + static_cast<long long>(p) * T_n;
                const int ldv = (T_n + 3) & ~3;   // (V_b^T read from global: r x 4 floats)
                float P[RJ];
#pragma unroll
                for (int j = 0; j < RJ; ++j) P[j] = 0.0f;
                for (int e = 0; e < nv; ++e) {
                    const long long x = base + e;
                    const float gv = __ldcs(pg + x);
                    float dl;
                    if (NOEF) {
                        if (ph != nullptr) ph[x] = fmul(eta, ph[x]);          // u <- beta u (node 0)
                        dl = gv;
                    } else {
                        const float hn = ffma(eta, gv, fmul(ome, __ldcs(ph + x)));   // O2, R11
                        __stcs(ph + x, hn);
                        dl = fsub(hn, __ldcs(pgg + x));                       // O3, R4
                    }
                    if (sketch) {
#pragma unroll
                        for (int j = 0; j < RJ; ++j)
                            if (j < r) P[j] = ffma(dl, Vb[static_cast<long long>(j) * ldv + e], P[j]);   // O6 lane 0
                    } else if (mode == 2) {
                        P[0] = ffma(dl, dl, P[0]);
                    }
                }
#pragma unroll
                for (int j = 0; j < RJ; ++j) P[j] = fadd(P[j], 0.0f);    // the butterfly with idle lanes
                if (mode == 3) {
                    if (node == 0) {
                        const float sig = randk_key(a, p, T_b);
                        a.sigma[T_row_base + p] = sig;
                        atomicAdd(&s_hist[order_key_dev(sig) >> kHist1Shift], 1u);
                    }
                } else if (mode == 2) {
                    const float sig = P[0];
                    a.sigma[static_cast<long long>(node) * a.M + T_row_base + p] = sig;
                    atomicAdd(&s_hist[order_key_dev(sig) >> kHist1Shift], 1u);
                    if (!isfinite(sig)) atomicOr(a.status, kStatusNonfinite);
                } else {
                    if (a.pnodes != nullptr)
                        for (int j = 0; j < r; ++j) {
                            float v = P[0];
#pragma unroll
                            for (int jj = 1; jj < RJ; ++jj)
                                if (jj == j) v = P[jj];
                            a.pnodes[(static_cast<long long>(T_row_base + p) * a.nodes_local + node) * r + j] = v;
                        }
                    if (mode == 0) {
                        float sig = 0.0f;
#pragma unroll
                        for (int j = 0; j < RJ; ++j)
                            if (j < r) sig = ffma(P[j], P[j], sig);                   // O8
                        a.sigma[T_row_base + p] = sig;
                        atomicAdd(&s_hist[order_key_dev(sig) >> kHist1Shift], 1u);
                        if (!isfinite(sig)) atomicOr(a.status, kStatusNonfinite);
                    }
                }
            }
          } else if (!v_smem) {
            const int ldv = (T_n + 3) & ~3;
            const int range_w = (a.vs_cap / r) / 1024 * 1024;
            for (int c0 = 0; c0 < T_n; c0 += range_w) {
                __syncthreads();                         // stage V_b^T[:, c0 : c0 + range_w)
                const int w = min(range_w, ldv - c0);
                for (int i = tid; i < r * (w >> 2); i += NT) {
                    const int j = i / (w >> 2), f = i - j * (w >> 2);
                    reinterpret_cast<float4*>(Vs + j * range_w)[f] =
                        __ldg(reinterpret_cast<const float4*>(a.V + T_voff + static_cast<long long>(j) * ldv + c0) + f);
                }
                __syncthreads();
                for (int rr = warp; rr < T_rows; rr += NW) {
                    const int p = T_row0 + rr;
                    const int nv = row_cols(T_len, T_n, p);
                    const long long base = T_off + static_cast<long long>(p) * T_n;
                    const int nseg = (nv + 127) >> 7;
                    const int kb = c0 >> 7, ke = min(nseg, (c0 + range_w) >> 7);
                    if (kb >= ke) continue;              // (a short last row ends in an earlier range)
                    float acc[RJ], P[RJ];
#pragma unroll
                    for (int j = 0; j < RJ; ++j) { acc[j] = 0.0f; P[j] = c0 > 0 ? s_P[rr][j] : 0.0f; }
                    for (int k0 = kb; k0 < ke; k0 += UN) {
                        float4 xg[UN], xh[UN], xd[UN];
#pragma unroll
                        for (int u = 0; u < UN; ++u) {
                            const int q = 128 * (k0 + u) + 4 * lane;
                            const long long e = base + q;
                            float tg[4] = {0.f, 0.f, 0.f, 0.f}, th[4] = {0.f, 0.f, 0.f, 0.f}, td[4] = {0.f, 0.f, 0.f, 0.f};
                            if (k0 + u < ke && q + 3 < nv && T_vec) {
                                const float4 g4 = sk_ld4g(pg + e);
                                tg[0] = g4.x; tg[1] = g4.y; tg[2] = g4.z; tg[3] = g4.w;
                                if (!NOEF || ph != nullptr) {
                                    const float4 h4 = sk_ld4(ph + e);
                                    th[0] = h4.x; th[1] = h4.y; th[2] = h4.z; th[3] = h4.w;
                                }
                                if (!NOEF) {
                                    const float4 d4 = sk_ld4(pgg + e);
                                    td[0] = d4.x; td[1] = d4.y; td[2] = d4.z; td[3] = d4.w;
                                }
                            } else if (k0 + u < ke) {
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    if (q + k < nv) {
                                        tg[k] = sk_ld1(pg + e + k);
                                        if (!NOEF || ph != nullptr) th[k] = sk_ld1(ph + e + k);
                                        if (!NOEF) td[k] = sk_ld1(pgg + e + k);
                                    }
                            }
                            xg[u] = make_float4(tg[0], tg[1], tg[2], tg[3]);
                            xh[u] = make_float4(th[0], th[1], th[2], th[3]);
                            xd[u] = make_float4(td[0], td[1], td[2], td[3]);
                        }
#pragma unroll
                        for (int u = 0; u < UN; ++u) {
                            const int k = k0 + u;
                            if (k >= ke) break;
                            const float gx[4] = {xg[u].x, xg[u].y, xg[u].z, xg[u].w};
                            const float hx[4] = {xh[u].x, xh[u].y, xh[u].z, xh[u].w};
                            const float dx[4] = {xd[u].x, xd[u].y, xd[u].z, xd[u].w};
                            segment<RJ, NOEF>(a, k, nseg, 128 * k + 4 * lane, nv, base, T_vec, range_w, c0, Vs, true, true,
                                              sketch, ph, gx, hx, dx, eta, ome, r, acc, P);
                        }
                    }
                    if (ke < nseg) {                     // the row continues in the next range
                        if (lane == 0)
#pragma unroll
                            for (int j = 0; j < RJ; ++j) s_P[rr][j] = P[j];
                        continue;
                    }
                    row_epilogue<RJ>(a, p, T_row_base, T_b, node, lane, r, P, s_hist);
                }
            }
          }
        }
        if (!streamed) {
        // (RANGED: the CTA's warps take its rows round-robin across tiles, so a
        // tile height that is not a multiple of the warp count idles no warp)
        int rr = RANGED ? carry : warp;
        for (; rr < T_rows; rr += NW) {
            const int p = T_row0 + rr;
            const int nv = row_cols(T_len, T_n, p);
            const long long base = T_off + static_cast<long long>(p) * T_n;
            const int nseg = (nv + 127) >> 7;
            float acc[RJ], P[RJ];
#pragma unroll
            for (int j = 0; j < RJ; ++j) { acc[j] = 0.0f; P[j] = 0.0f; }
            for (int k0 = 0; k0 < nseg; k0 += UN) {
                float4 xg[UN], xh[UN], xd[UN];
#pragma unroll
                for (int u = 0; u < UN; ++u) {
                    const int q = 128 * (k0 + u) + 4 * lane;
                    const long long e = base + q;
                    if (q + 3 < nv && T_vec) {
                        xg[u] = sk_ld4g(pg + e);
                        xh[u] = (!NOEF || ph != nullptr) ? sk_ld4(ph + e) : make_float4(0.f, 0.f, 0.f, 0.f);
                        xd[u] = !NOEF ? sk_ld4(pgg + e) : make_float4(0.f, 0.f, 0.f, 0.f);
                    } else {
                        float tg[4] = {0.f, 0.f, 0.f, 0.f}, th[4] = {0.f, 0.f, 0.f, 0.f}, td[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (q + k < nv) {
                                tg[k] = sk_ld1(pg + e + k);
                                if (!NOEF || ph != nullptr) th[k] = sk_ld1(ph + e + k);
                                if (!NOEF) td[k] = sk_ld1(pgg + e + k);
                            }
                        xg[u] = make_float4(tg[0], tg[1], tg[2], tg[3]);
                        xh[u] = make_float4(th[0], th[1], th[2], th[3]);
                        xd[u] = make_float4(td[0], td[1], td[2], td[3]);
                    }
                }
#pragma unroll
                for (int u = 0; u < UN; ++u) {
                    const int k = k0 + u;
                    if (k >= nseg) break;
                    const float gx[4] = {xg[u].x, xg[u].y, xg[u].z, xg[u].w};
                    const float hx[4] = {xh[u].x, xh[u].y, xh[u].z, xh[u].w};
                    const float dx[4] = {xd[u].x, xd[u].y, xd[u].z, xd[u].w};
                    segment<RJ, NOEF>(a, k, nseg, 128 * k + 4 * lane, nv, base, T_vec, (T_n + 3) & ~3, 0, Vb, V_vec, v_smem, sketch, ph,
                                gx, hx, dx, eta, ome, r, acc, P);
                }
            }
            row_epilogue<RJ>(a, p, T_row_base, T_b, node, lane, r, P, s_hist);
        }
        if constexpr (RANGED) carry = rr - T_rows;
        }
    }
    if (cta_hist) {
        __syncthreads();
        flush_hist(cur_b);
    }
}

template <int RJ, int UN, int MINB, bool NOEF = false, bool RANGED = false>
void launch_reg(const SketchLaunch& a, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(a.grid);
    cfg.blockDim = dim3(RANGED ? wide_threads(RJ) : kThreads);
    cfg.dynamicSmemBytes = sizeof(float) * a.vs_cap;
    cfg.stream = s;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_ef_sketch<RJ, UN, MINB, NOEF, RANGED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(float) * (RANGED ? kVsBig : kVsMax)));
        attr_set = true;
    }
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_ef_sketch<RJ, UN, MINB, NOEF, RANGED>, a);
}
template <int RJ, int UN, int MINB, bool NOEF = false, bool RANGED = false>
int occupancy_reg(int vs_cap) {
    cudaFuncSetAttribute(k_ef_sketch<RJ, UN, MINB, NOEF, RANGED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(float) * (RANGED ? kVsBig : kVsMax)));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ef_sketch<RJ, UN, MINB, NOEF, RANGED>,
                                                  RANGED ? wide_threads(RJ) : kThreads, sizeof(float) * vs_cap);
    return per_sm;
}

// variant (a.shape): UN segments per batch / CTAs per SM: 0 = 3 / 3, 1 = 2 / 4,
// 2 = 4 / 2, 3 = 6 / 2 (r <= 8; wider sketches get fewer CTAs).  0 and 2 are chosen per
// layout (arc_api.cu); 1 and 3 measured no better (C3: 3 / 3 325.7 us, 6 / 2 326.3 us)
template <int RJ>
void launch_rj(const SketchLaunch& a, cudaStream_t s) {
    if (a.ranged) {   // the wide blocks' launch (one variant)
        if (a.noef) launch_reg<RJ, wide_un(RJ), 1, true, true>(a, s);
        else launch_reg<RJ, wide_un(RJ), 1, false, true>(a, s);
        return;
    }
    if (a.noef) {   // (the without-EF baseline: one variant)
        launch_reg<RJ, 3, (RJ <= 8 ? 3 : 2), true>(a, s);
        return;
    }
    switch (a.shape) {
        case 1: launch_reg<RJ, 2, (RJ <= 8 ? 4 : 2)>(a, s); break;
        case 2: launch_reg<RJ, 4, 2>(a, s); break;
        case 3: launch_reg<RJ, (RJ <= 8 ? 6 : 2), 2>(a, s); break;
        default: launch_reg<RJ, 3, (RJ <= 8 ? 3 : 2)>(a, s); break;
    }
}
template <int RJ>
int occupancy_rj(int shape, int vs_cap) {
    switch (shape) {
        case 1: return occupancy_reg<RJ, 2, (RJ <= 8 ? 4 : 2)>(vs_cap);
        case 2: return occupancy_reg<RJ, 4, 2>(vs_cap);
        case 3: return occupancy_reg<RJ, (RJ <= 8 ? 6 : 2), 2>(vs_cap);
        default: return occupancy_reg<RJ, 3, (RJ <= 8 ? 3 : 2)>(vs_cap);
    }
}

}  // namespace

int sketch_tile_rows(int) { return 32; }   // (plan_tiles takes 8 for small single-block layouts)
int sketch_tile_cols(int) { return 128; }
int sketch_shape_ok(int shape, int) { return shape >= 0 && shape <= 3; }

void launch_ef_sketch(const SketchLaunch& a, cudaStream_t s) {
    // Top-K baseline and Rand-K need no sketch columns
    const int r = a.mode >= 2 ? 1 : a.r;
    if (r <= 4) launch_rj<4>(a, s);
    else if (r <= 8) launch_rj<8>(a, s);
    else if (r <= 16) launch_rj<16>(a, s);
    else launch_rj<32>(a, s);
}

int sketch_vs_cap(int r, int max_n) {
    const long long need = static_cast<long long>(r) * ((max_n + 3) / 4 * 4);   // padded V_b^T rows
    return static_cast<int>(need <= kVsMax ? need : 0) & ~3;   // 0: V read from global memory
}

int sketch_ranged_cap(int r) { return kVsBig / (1024 * r) * (1024 * r); }
int sketch_wide_threads(int r) { return wide_threads(r <= 4 ? 4 : r <= 8 ? 8 : r <= 16 ? 16 : 32); }

int ef_sketch_resident_ctas_ranged(int r, int vs_cap) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_sm = r <= 4 ? occupancy_reg<4, wide_un(4), 1, false, true>(vs_cap)
                       : r <= 8 ? occupancy_reg<8, wide_un(8), 1, false, true>(vs_cap)
                       : r <= 16 ? occupancy_reg<16, wide_un(16), 1, false, true>(vs_cap)
                                 : occupancy_reg<32, wide_un(32), 1, false, true>(vs_cap);
    return sms * (per_sm < 1 ? 1 : per_sm);
}

int ef_sketch_resident_ctas(int r, int shape, int vs_cap) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_sm = r <= 4 ? occupancy_rj<4>(shape, vs_cap) : r <= 8 ? occupancy_rj<8>(shape, vs_cap)
                       : r <= 16 ? occupancy_rj<16>(shape, vs_cap) : occupancy_rj<32>(shape, vs_cap);
    return sms * (per_sm < 1 ? 1 : per_sm);
}

}  // namespace arc
