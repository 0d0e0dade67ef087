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
#include <type_traits>

#include "arc_device.cuh"
#include "arc_internal.cuh"
#include "arc_rng.cuh"
#include "arc_select_common.cuh"

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
#ifndef ARC_SK_FAST   // predicate-free loop for full aligned rows in the 4-segment variant (A/B knob)
#define ARC_SK_FAST 1
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

// ---- the fused small-problem tail: S3..S6 in the last CTA ------
// Every CTA, after its tiles, fences its writes and increments the done
// counter once (then draws its share of the next step's V, off the critical
// path).  The CTA that brings the counter to the
// grid size has every other CTA's Sigma rows and digit-1 histogram bins
// visible, and runs the selection of k_select_gather on keys held in shared
// memory: per ARC block, the boundary digit 1 from the complete histogram,
// digits 2 and 3 (key[20:10], key[9:0]) by two shared-memory histogram passes
// over the keys whose higher digits match, so T = the K_b-th largest key and
// need_eq = how many keys equal to T are taken; then ONE ordered pass writes
// I_b ascending (key > T, or key == T among the need_eq smallest rows: ties
// -> smaller row, R5; NaN keys largest, R15).  S4..S6 follow on the selected
// rows with the arithmetic of gather_rows_local (one node on this GPU, N = 1:
// C = h' - g [R25 rounding], g <- g + C, gbar <- gbar + C / N, R3, R12, R13).
// No grid barrier, no second launch: nothing waits on another CTA.
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <int NT>
__device__ __forceinline__ bool tail_arrive(const SketchLaunch& a) {
    __shared__ unsigned s_last;
    const TailArgs& T = a.tail;
    __threadfence();   // this thread's Sigma, histogram and h' writes, before the CTA's increment
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(T.done, 1u) == gridDim.x - 1 ? 1u : 0u;
    __syncthreads();
    if (s_last) __threadfence();
    return s_last != 0;
}

// The CTA's share of the next step's V (S0, speculative: V depends only on (seed, t, b)):
// item i on CTA i mod grid, drawn AFTER the CTA's increment, off the path to the last
// arrival.  The last CTA leaves its items to k_tail_update (it records its index), so
// they do not delay the grid's completion either; the kernels that read V_next wait
// for both grids.
template <int NT>
__device__ __forceinline__ void tail_next_V(const SketchLaunch& a, bool last) {
    const TailArgs& T = a.tail;
    if (T.V_next == nullptr) return;
    if (last) {
        if (threadIdx.x == 0) *T.last_cta = blockIdx.x;
        return;
    }
    for (long long i = threadIdx.x * static_cast<long long>(gridDim.x) + blockIdx.x; i < T.v_items;
         i += static_cast<long long>(gridDim.x) * NT)
        rng::gen_V_item(a.blocks, a.num_blocks, a.r, a.key, T.tn_lo, T.tn_hi, i, T.V_next);
}

template <int NT>
__device__ void tail_select(const SketchLaunch& a, unsigned* sh, unsigned* s_keys) {
    __shared__ int warp_sums[32];
    __shared__ unsigned s_dig;
    __shared__ int s_abv, s_cnt;
    constexpr int kTailCand = 256;   // boundary-bin keys ranked directly, O(E^2) (sh holds keys | rows);
                                     // a more crowded bin takes the two histogram passes
    const int tid = threadIdx.x;
    const TailArgs& T = a.tail;
#define TAIL_STAMP(k) \
    if (T.stamps != nullptr && tid == 0) T.stamps[k] = globaltimer_ns()
    TAIL_STAMP(1);
    // the update kernel behind this launch may become resident now (it waits for this grid)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // ---- S3 per ARC block
    for (int b = 0; b < a.num_blocks; ++b) {
        const BlockDev& B = a.blocks[b];
        if (B.kind != ARC_BLOCK_ARC) continue;
        const int m = B.m, K = B.K, sel_base = B.sel_base;
        __syncthreads();                                     // (sh, s_keys of the previous block)
        // the block's digit-1 histogram and order keys (R15): every load of a
        // batch in flight before the first is used (one L2 round trip per batch)
        unsigned* gh = a.hist1 + static_cast<long long>(b) * kHist1Bins;
        {
            constexpr int HB = kHist1Bins / NT;
            unsigned hv[HB];
#pragma unroll
            for (int k = 0; k < HB; ++k) hv[k] = __ldcg(gh + tid + k * NT);
            // 16-byte loads of the aligned superset [row_base & ~3, row_base + m) (the
            // Sigma buffer is 256-byte aligned and padded), 8 per thread per round trip
            const int a0 = B.row_base & 3;
            const float4* __restrict__ s4 = reinterpret_cast<const float4*>(a.sigma + (B.row_base - a0));
            const int nq = (m + a0 + 3) >> 2;
            for (int i0 = 0; i0 < nq; i0 += 8 * NT) {
                float4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = i0 + u * NT + tid;
                    v[u] = i < nq ? __ldcg(s4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = 4 * (i0 + u * NT + tid) - a0;   // block row of v[u].x
                    const float w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (i + k >= 0 && i + k < m) s_keys[i + k] = order_key_dev(w[k]);   // R15
                }
            }
#pragma unroll
            for (int k = 0; k < HB; ++k) {
                sh[tid + k * NT] = hv[k];
                gh[tid + k * NT] = 0u;                       // (the next step's histogram starts empty)
            }
        }
        __syncthreads();
        TAIL_STAMP(2);
        // T = the K-th largest key; selected: key > T, or key == T and (use_peq)
        // row <= P_eq / (else) among the need_eq smallest rows with key T
        unsigned Tk = 0u;   // K = m: every row (key >= +0, P_eq = m - 1)
        int Peq = m - 1, need_eq = m;
        bool use_peq = true;
        if (K < m) {
            int above;
            const unsigned b1 = selc::top_digit<NT>(sh, kHist1Bins, K, warp_sums, &s_dig, &s_abv, &above);
            int krem = K - above;
            // the keys of the boundary bin b1 (usually a handful) listed in sh, then
            // ranked in the order (key desc, row asc): the krem-th is (T, P_eq)
            unsigned* ck = sh;
            int* ci = reinterpret_cast<int*>(sh + kTailCand);
            if (tid == 0) s_cnt = 0;
            __syncthreads();
            for (int i = tid; i < m; i += NT) {
                const unsigned k = s_keys[i];
                if ((k >> 21) == b1) {
                    const int slot = atomicAdd(&s_cnt, 1);
                    if (slot < kTailCand) { ck[slot] = k; ci[slot] = i; }
                }
            }
            __syncthreads();
            const int E = s_cnt;
            if (E <= kTailCand) {
                for (int c = tid; c < E; c += NT) {
                    const unsigned key = ck[c];
                    const int row = ci[c];
                    int rank = 0;
#pragma unroll 4
                    for (int j = 0; j < E; ++j) rank += ck[j] > key || (ck[j] == key && ci[j] < row);
                    if (rank == krem - 1) { s_dig = key; s_abv = row; }
                }
                __syncthreads();
                Tk = s_dig;
                Peq = s_abv;
                __syncthreads();
            } else {   // a crowded boundary bin (massive ties): digits 2 and 3 by histogram passes
                use_peq = false;
                for (int i = tid; i < 2048; i += NT) sh[i] = 0u;
                __syncthreads();
                for (int i = tid; i < m; i += NT) {
                    const unsigned k = s_keys[i];
                    if ((k >> 21) == b1) atomicAdd(&sh[(k >> 10) & 2047u], 1u);
                }
                __syncthreads();
                const unsigned b2 = selc::top_digit<NT>(sh, 2048, krem, warp_sums, &s_dig, &s_abv, &above);
                krem -= above;
                const unsigned pre = (b1 << 11) | b2;        // key[31:10] of the K-th key
                for (int i = tid; i < 1024; i += NT) sh[i] = 0u;
                __syncthreads();
                for (int i = tid; i < m; i += NT) {
                    const unsigned k = s_keys[i];
                    if ((k >> 10) == pre) atomicAdd(&sh[k & 1023u], 1u);
                }
                __syncthreads();
                const unsigned b3 = selc::top_digit<NT>(sh, 1024, krem, warp_sums, &s_dig, &s_abv, &above);
                krem -= above;
                Tk = (pre << 10) | b3;
                need_eq = krem;                              // >= 1 keys equal to T are taken
            }
        }
        TAIL_STAMP(3);
        // ordered pass: thread tid owns rows [r0, r1); I_b written ascending
        const int R = (m + NT - 1) / NT;
        const int r0 = min(m, tid * R), r1 = min(m, r0 + R);
        int tot, pos;
        if (use_peq) {
            int cnt = 0;
            for (int i = r0; i < r1; ++i) {
                const unsigned k = s_keys[i];
                cnt += k > Tk || (k == Tk && i <= Peq);
            }
            pos = selc::cta_exclusive_scan(cnt, warp_sums, &tot);
            for (int i = r0; i < r1; ++i) {
                const unsigned k = s_keys[i];
                if (k > Tk || (k == Tk && i <= Peq)) {
                    T.sel[sel_base + pos] = i;
                    ++pos;
                }
            }
        } else {
            int gt = 0, eq = 0;
            for (int i = r0; i < r1; ++i) {
                const unsigned k = s_keys[i];
                gt += k > Tk;
                eq += k == Tk;
            }
            int eq_seen = selc::cta_exclusive_scan(eq, warp_sums, &tot);
            const int take_eq = max(0, min(eq, need_eq - eq_seen));
            pos = selc::cta_exclusive_scan(gt + take_eq, warp_sums, &tot);
            for (int i = r0; i < r1; ++i) {
                const unsigned k = s_keys[i];
                bool take = k > Tk;
                if (k == Tk) take = eq_seen++ < need_eq;
                if (take) {
                    T.sel[sel_base + pos] = i;
                    ++pos;
                }
            }
        }
    }
    __syncthreads();
    TAIL_STAMP(4);
    if (tid == 0) {
        if (T.t_advance != nullptr) *T.t_advance += 1ull;   // (every reader of this step's t is done)
        *T.done = 0u;                                       // (the next launch counts from zero)
    }
#undef TAIL_STAMP
}

// S4..S6 on the tail's selected rows (one node on this GPU, N = 1 here): one
// quad (4 columns of one selected row) per thread, the arithmetic of
// gather_rows_local — C = h' - g [R25 rounding], g <- g + C, gbar <- gbar + C / N
// (R3, R12, R13), A / N into the values when requested.  Launched right behind
// the streaming launch: with programmatic dependent launch its CTAs are resident
// while the last CTA selects (that CTA triggers its dependents first) and wait
// here for the streaming grid to complete; the selection is then visible.  (One
// CTA updating the rows itself measured 9-14 us for 10 rows of 1024 columns.)
__global__ void __launch_bounds__(256) k_tail_update(const SketchLaunch a) {
    // the next kernel (the next step's streaming launch) may become resident and run
    // its prologue now; it waits for this grid before touching the state
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    grid_dependency_wait();
    const TailArgs& T = a.tail;
    const bool pow2 = (T.N_int & (T.N_int - 1)) == 0;
    const float invN = 1.0f / a.Nf;
    const bool noef = a.noef != 0;
    const float* __restrict__ ph = noef ? a.nodes.grad[0] : a.nodes.h[0];   // (without EF: C = the gradient rows)
    float* __restrict__ pg = a.nodes.g[0];
    float* __restrict__ gbar = a.gbar;
    if (T.V_next != nullptr) {   // the streaming launch's last CTA's share of V_next (see tail_next_V)
        const long long g = T.sk_grid, last = __ldcg(T.last_cta), nt = gridDim.x * 256ll;
        for (long long i = last + (nt - 1 - (blockIdx.x * 256ll + threadIdx.x)) * g; i < T.v_items; i += nt * g)
            rng::gen_V_item(a.blocks, a.num_blocks, a.r, a.key, T.tn_lo, T.tn_hi, i, T.V_next);
    }
    for (long long item = blockIdx.x * 256ll + threadIdx.x; item < T.quads; item += gridDim.x * 256ll) {
        int b = 0;
        while (b + 1 < T.nblk && item >= T.blk[b + 1].q_begin) ++b;
        const TailBlk& B = T.blk[b];
        const int nq = (B.n + 3) >> 2;
        const long long rel = item - B.q_begin;
        const int j = static_cast<int>(rel / nq), q = 4 * static_cast<int>(rel - static_cast<long long>(j) * nq);
        const int p = __ldcg(T.sel + B.sel_base + j);
        const int cnt = max(0, min(4, row_cols(B.len, B.n, p) - q)), ocnt = min(4, B.n - q);
        const long long e = B.off + static_cast<long long>(p) * B.n + q;
        const long long o = B.val_base + static_cast<long long>(j) * B.n + q;
        const bool v4 = cnt == 4 && B.vec;
        float hq[4] = {0.f, 0.f, 0.f, 0.f}, gq[4] = {0.f, 0.f, 0.f, 0.f}, bq[4] = {0.f, 0.f, 0.f, 0.f};
        if (v4) {
            const float4 h4 = __ldcg(reinterpret_cast<const float4*>(ph + e));
            const float4 b4 = __ldcg(reinterpret_cast<const float4*>(gbar + e));
            const float4 g4 = noef ? make_float4(0.f, 0.f, 0.f, 0.f) : __ldcg(reinterpret_cast<const float4*>(pg + e));
            hq[0] = h4.x; hq[1] = h4.y; hq[2] = h4.z; hq[3] = h4.w;
            bq[0] = b4.x; bq[1] = b4.y; bq[2] = b4.z; bq[3] = b4.w;
            gq[0] = g4.x; gq[1] = g4.y; gq[2] = g4.z; gq[3] = g4.w;
        } else {   // unaligned rows, the short last row
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                if (kk < cnt) {
                    hq[kk] = __ldcg(ph + e + kk);
                    bq[kk] = __ldcg(gbar + e + kk);
                    if (!noef) gq[kk] = __ldcg(pg + e + kk);
                }
        }
        float gn[4], val[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const float c = kk < cnt ? wire_round(noef ? hq[kk] : fsub(hq[kk], gq[kk]), T.bf16) : 0.0f;   // C (R25; +0 padding)
            gn[kk] = fadd(gq[kk], c);                                                          // R12
            val[kk] = kk < cnt ? (pow2 ? fmul(c, invN) : __fdiv_rn(c, a.Nf)) : 0.0f;           // A / N, R3
            bq[kk] = fadd(bq[kk], val[kk]);                                                    // R13
        }
        if (v4) {
            if (!noef) *reinterpret_cast<float4*>(pg + e) = make_float4(gn[0], gn[1], gn[2], gn[3]);
            *reinterpret_cast<float4*>(gbar + e) = make_float4(bq[0], bq[1], bq[2], bq[3]);
        } else {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                if (kk < cnt) {
                    if (!noef) pg[e + kk] = gn[kk];
                    gbar[e + kk] = bq[kk];
                }
        }
        if (T.values != nullptr) {
            if (B.vec && ocnt == 4 && (o & 3) == 0) {
                *reinterpret_cast<float4*>(T.values + o) = make_float4(val[0], val[1], val[2], val[3]);
            } else {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    if (kk < ocnt) T.values[o + kk] = val[kk];
            }
        }
    }
    if (T.stamps != nullptr && blockIdx.x == 0 && threadIdx.x == 0) T.stamps[5] = globaltimer_ns();
}

// The register path: the same per-segment arithmetic with the batch loaded
// straight into registers (UN segments, 3 UN float4 per lane), warps streaming
// their rows independently; V_b^T staged in shared memory as above.
// RANGED: the launch over the blocks whose V_b^T does not fit the stage; V is
// staged in ranges of whole 1024-column chunks and every row carries its P'
// across ranges in shared memory (the O6 order is unchanged)
template <int RJ, int UN, int MINB, bool NOEF, bool RANGED, bool TAIL>
__global__ void __launch_bounds__(RANGED ? wide_threads(RJ) : kThreads, MINB) k_ef_sketch(const SketchLaunch a) {
    constexpr int NT = RANGED ? wide_threads(RJ) : kThreads, NW = NT / 32;
    __shared__ TileDesc s_tile[kTileCache];
    __shared__ unsigned s_hist[kHist1Bins];     // digit-1 histogram of this CTA's Sigma (modes 0, 3)
    __shared__ float s_P[RANGED ? 32 : 1][RJ];  // (RANGED) the tile rows' running P' between ranges
    extern __shared__ __align__(16) float4 dyn[];   // V_b^T
    float* Vs = reinterpret_cast<float*>(dyn);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int list_begin = a.cta_begin[blockIdx.x], list_end = a.cta_begin[blockIdx.x + 1];
    if (list_begin >= list_end) {
        if constexpr (TAIL) {   // (an idle CTA still counts, and draws its share of V)
            grid_dependency_wait();
            const bool last = tail_arrive<NT>(a);
            if (last) tail_select<NT>(a, s_hist, reinterpret_cast<unsigned*>(dyn));
            tail_next_V<NT>(a, last);
        }
        return;
    }
    const int ntile = list_end - list_begin;
    for (int i = tid; i < min(ntile, kTileCache) * 4; i += NT)
        reinterpret_cast<uint4*>(s_tile)[i] = __ldg(reinterpret_cast<const uint4*>(a.tiles + list_begin) + i);
    for (int i = tid; i < kHist1Bins; i += NT) s_hist[i] = 0;
    __syncthreads();
    grid_dependency_wait();   // the previous kernel (g, V, histogram reset) is complete
    if constexpr (TAIL) {
        if (a.tail.stamps != nullptr && blockIdx.x == 0 && tid == 0) a.tail.stamps[0] = globaltimer_ns();
    }

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
            // Full rows of whole 128-column segments, 16-byte aligned, V_b^T staged,
            // r == RJ: the same O6 arithmetic with no per-element predicates.  Only in
            // the 4-segment / 2-CTA variant (128 registers): C2 sketch 36.9 -> 33.4 us,
            // C5 d = 1e8 -1 %; in the 80-register variant (C3) it spilled: +3 % (fast
            // path alone) / +32 % (both paths) (profiles/r02_sketch_fastpath.txt)
            if constexpr (ARC_SK_FAST && !NOEF && !RANGED && !TAIL && RJ == 4 && (UN == 4 || UN == 3) && MINB == 2) {
            if (sketch && v_smem && T_vec && r == RJ && nv == T_n && (T_n & 127) == 0) {
                const int ldv4 = T_n >> 2;
                const float4* __restrict__ V4 = reinterpret_cast<const float4*>(Vs);
                for (int k0 = 0; k0 < nseg; k0 += UN) {
                    float4 xg[UN], xh[UN], xd[UN];
#pragma unroll
                    for (int u = 0; u < UN; ++u) {
                        if (k0 + u < nseg) {
                            const long long e = base + 128 * (k0 + u) + 4 * lane;
                            xg[u] = sk_ld4g(pg + e);
                            xh[u] = sk_ld4(ph + e);
                            xd[u] = sk_ld4(pgg + e);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < UN; ++u) {
                        const int k = k0 + u;
                        if (k >= nseg) break;
                        const int q4 = 32 * k + lane;   // quad index of columns q .. q + 3
                        const float hn0 = ffma(eta, xg[u].x, fmul(ome, xh[u].x)), hn1 = ffma(eta, xg[u].y, fmul(ome, xh[u].y));
                        const float hn2 = ffma(eta, xg[u].z, fmul(ome, xh[u].z)), hn3 = ffma(eta, xg[u].w, fmul(ome, xh[u].w));
                        sk_st4(ph + base + 4 * q4, make_float4(hn0, hn1, hn2, hn3));                  // O2, R11
                        const float d0 = fsub(hn0, xd[u].x), d1 = fsub(hn1, xd[u].y);                // O3, R4
                        const float d2 = fsub(hn2, xd[u].z), d3 = fsub(hn3, xd[u].w);
#pragma unroll
                        for (int j = 0; j < RJ; ++j) {
                            const float4 v = V4[j * ldv4 + q4];
                            acc[j] = ffma(d0, v.x, acc[j]);                                      // O6
                            acc[j] = ffma(d1, v.y, acc[j]);
                            acc[j] = ffma(d2, v.z, acc[j]);
                            acc[j] = ffma(d3, v.w, acc[j]);
                        }
                        if ((k & 7) == 7 || k == nseg - 1) {                                       // end of a 1024-column chunk
#pragma unroll
                            for (int j = 0; j < RJ; ++j) {
                                const float w = butterfly(acc[j]);
                                P[j] = (k < 8) ? w : fadd(P[j], w);
                                acc[j] = 0.0f;
                            }
                        }
                    }
                }
                row_epilogue<RJ>(a, p, T_row_base, T_b, node, lane, r, P, s_hist);
                continue;
            }
            }
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
    if constexpr (TAIL) {
        const bool last = tail_arrive<NT>(a);
        if (last) tail_select<NT>(a, s_hist, reinterpret_cast<unsigned*>(dyn));
        tail_next_V<NT>(a, last);
    }
}

// dynamic shared memory (floats) a variant may request: V_b^T (RANGED: the wide stage), or
// for the fused tail also the keys of one ARC block
template <bool RANGED, bool TAIL>
constexpr int dyn_max() {
    return RANGED ? kVsBig : (TAIL && kTailMaxRows > kVsMax ? kTailMaxRows : kVsMax);
}

template <int RJ, int UN, int MINB, bool NOEF = false, bool RANGED = false, bool TAIL = false>
void launch_reg(const SketchLaunch& a, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(a.grid);
    cfg.blockDim = dim3(RANGED ? wide_threads(RJ) : kThreads);
    cfg.dynamicSmemBytes = sizeof(float) * (TAIL && a.tail.key_cap > a.vs_cap ? a.tail.key_cap : a.vs_cap);
    cfg.stream = s;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_ef_sketch<RJ, UN, MINB, NOEF, RANGED, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(float) * dyn_max<RANGED, TAIL>()));
        attr_set = true;
    }
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_ef_sketch<RJ, UN, MINB, NOEF, RANGED, TAIL>, a);
}
template <int RJ, int UN, int MINB, bool NOEF = false, bool RANGED = false, bool TAIL = false>
int occupancy_reg(int vs_cap) {
    cudaFuncSetAttribute(k_ef_sketch<RJ, UN, MINB, NOEF, RANGED, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(float) * dyn_max<RANGED, TAIL>()));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ef_sketch<RJ, UN, MINB, NOEF, RANGED, TAIL>,
                                                  RANGED ? wide_threads(RJ) : kThreads, sizeof(float) * vs_cap);
    return per_sm;
}

// variant (a.shape): UN segments per batch / CTAs per SM: 0 = 3 / 3, 1 = 2 / 4,
// 2 = 4 / 2, 3 = 6 / 2 (r <= 8; wider sketches get fewer CTAs), 5 = 3 / 2 (with the
// predicate-free loop).  0, 2 and 5 are chosen per layout (arc_api.cu); 1 and 3 measured
// no better (C3: 3 / 3 325.7 us, 6 / 2 326.3 us)
template <int RJ>
void launch_rj(const SketchLaunch& a, cudaStream_t s) {
    if (a.ranged) {   // the wide blocks' launch (one variant)
        if (a.noef) launch_reg<RJ, wide_un(RJ), 1, true, true>(a, s);
        else launch_reg<RJ, wide_un(RJ), 1, false, true>(a, s);
        return;
    }
    if constexpr (RJ <= 8) {   // the fused small-problem tail (r <= 8): shapes 0 and 2 (the chosen ones)
        if (a.tail.done != nullptr) {
            if (a.noef) launch_reg<RJ, 3, 3, true, false, true>(a, s);
            else if (a.shape == 2) launch_reg<RJ, 4, 2, false, false, true>(a, s);
            else launch_reg<RJ, 3, 3, false, false, true>(a, s);
            return;
        }
    }
    if (a.noef) {   // (the without-EF baseline: one variant)
        launch_reg<RJ, 3, (RJ <= 8 ? 3 : 2), true>(a, s);
        return;
    }
    switch (a.shape) {
        case 1: launch_reg<RJ, 2, (RJ <= 8 ? 4 : 2)>(a, s); break;
        case 5: launch_reg<RJ, 3, 2>(a, s); break;
        case 2: launch_reg<RJ, 4, 2>(a, s); break;
        case 3: launch_reg<RJ, (RJ <= 8 ? 6 : 2), 2>(a, s); break;
        default: launch_reg<RJ, 3, (RJ <= 8 ? 3 : 2)>(a, s); break;
    }
}
template <int RJ>
int occupancy_rj(int shape, int vs_cap) {
    switch (shape) {
        case 1: return occupancy_reg<RJ, 2, (RJ <= 8 ? 4 : 2)>(vs_cap);
        case 5: return occupancy_reg<RJ, 3, 2>(vs_cap);
        case 2: return occupancy_reg<RJ, 4, 2>(vs_cap);
        case 3: return occupancy_reg<RJ, (RJ <= 8 ? 6 : 2), 2>(vs_cap);
        default: return occupancy_reg<RJ, 3, (RJ <= 8 ? 3 : 2)>(vs_cap);
    }
}

}  // namespace

void launch_tail_update(const SketchLaunch& a, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    const long long ctas = (a.tail.quads + 255) / 256;
    cfg.gridDim = dim3(static_cast<unsigned>(ctas < 1 ? 1 : ctas > 1184 ? 1184 : ctas));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_tail_update, a);
}

int sketch_tile_rows(int) { return 32; }   // (plan_tiles takes 8 for small single-block layouts)
int sketch_tile_cols(int) { return 128; }
int sketch_shape_ok(int shape, int) { return shape >= 0 && shape <= 3 || shape == 5; }

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

int ef_sketch_resident_ctas_tail(int r, int shape, bool noef, int dyn_floats) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    auto occ = [&](auto rj) {   // the instantiation launch_rj takes for the tail
        constexpr int RJ = decltype(rj)::value;
        if (noef) return occupancy_reg<RJ, 3, 3, true, false, true>(dyn_floats);
        if (shape == 2) return occupancy_reg<RJ, 4, 2, false, false, true>(dyn_floats);
        return occupancy_reg<RJ, 3, 3, false, false, true>(dyn_floats);
    };
    const int per_sm = r <= 4 ? occ(std::integral_constant<int, 4>{}) : occ(std::integral_constant<int, 8>{});
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
