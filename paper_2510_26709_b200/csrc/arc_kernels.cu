// arc_kernels.cu — sm_100a kernels of the EF21M + ARC-Top-K step.
//
// Every floating-point operation on the path is an explicitly rounded IEEE
// binary32 intrinsic (__fadd_rn, __fmul_rn, ...) in the order DESIGN.md §3
// fixes (R9, R11), so results are bit-identical to the plain definition; the
// library is also built with -fmad=false -ftz=false -prec-div=true.
//
// Kernels here (DESIGN.md §5 has the roofline of each; the two big ones,
// k_ef_sketch and k_select_gather, have their own files):
//   k_vgen          S0  V_b = Gaussian(seed, t, b)                     P:229-230, Alg.1 l.3
//   k_sigma_slice   S2 on a row slice: S = sum of the nodes' P_i in    P:232, zn28373 P:236
//                   global node order, P = S / N, Sigma = sum_j P_j^2   (R3, R9, R21)
//   k_dense         S1+S4..S6 of DENSE blocks (identity compressor)    P:510, R11, R20
//   k_scatter       S6 after exchange #2                               eq:ef21m-3 P:327
//   k_dense_scatter S6 of DENSE blocks after exchange #2
//   k_topk_merge    Top-K baseline: merge of the all-gathered payloads  Table I "Top-K"
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "arc_device.cuh"
#include "arc_internal.cuh"
#include "arc_rng.cuh"

namespace cg = cooperative_groups;

namespace arc {
namespace {
using namespace dev;
using namespace rng;

// V_b[q][j]: one thread per (q, jj) of block b = blockIdx.y; counter
// (q*R4 + jj, b, lo32 t, hi32 t), key (lo32 seed, hi32 seed).  V_b is stored
// transposed ([r][n_b], column j contiguous: the streaming pass reads it so).
__global__ void __launch_bounds__(256) k_vgen(const BlockDev* __restrict__ blocks, int r, uint2 key,
                                              unsigned t_lo, unsigned t_hi, float* __restrict__ V,
                                              const unsigned long long* __restrict__ t_dev) {
    const int b = blockIdx.y;
    // (programmatic dependent launch: the streaming pass behind may become resident now;
    // this kernel waits for the previous step's kernels -- they read V, advanced t_dev)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    grid_dependency_wait();
    if (t_dev != nullptr) {   // ARC_FLAG_DEVICE_T: this step's t from the device counter
        const unsigned long long t = __ldcg(t_dev);
        t_lo = static_cast<unsigned>(t);
        t_hi = static_cast<unsigned>(t >> 32);
    }
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
        float* dst = V + v_off + q;
        const int ldv = (n + 3) & ~3;   // rows of V_b^T padded to 16 bytes
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (j0 + k < r) dst[static_cast<long long>(j0 + k) * ldv] = z[k];
    }
}

__device__ __forceinline__ int row_valid_cols(const BlockDev& B, int p) {
    const long long rest = B.len - static_cast<long long>(p) * B.n;
    return rest < B.n ? static_cast<int>(rest) : B.n;
}


// =============================================================================
// S6 for G > 1: gbar[I] += A / N after exchange #2.
//   mode 0: wire holds the summed rows (NCCL All-Reduce)
//   mode 1: wire holds [N][sumKn] per-node rows: ordered sum (R9) first
// CTA b takes a contiguous range of row segments; their descriptors and
// selected rows are staged in shared memory first (one round of independent
// loads), then every thread runs 4 quads per batch with all of the batch's
// loads issued before any result is used (the per-quad chain descriptor ->
// block -> selection -> data of the grid-stride version ran the scatter at
// ~0.4 of its HBM roofline at K n = 1e7).
// =============================================================================
constexpr int kScatterStage = 1024;   // segments staged per round (16 KB)

// payload quad o..o+3 of node row `node` (float or bf16 entries; ocnt valid)
__device__ __forceinline__ float4 wire_quad(const void* w, long long o, int ocnt, int bf16) {
    if (!bf16 && ocnt == 4 && (o & 3) == 0) return __ldcg(reinterpret_cast<const float4*>(static_cast<const float*>(w) + o));
    float t[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (k < ocnt) t[k] = pay_ld(w, o + k, bf16);
    return make_float4(t[0], t[1], t[2], t[3]);
}

__global__ void __launch_bounds__(256) k_scatter(const ScatterLaunch a) {
    __shared__ int4 stage[kScatterStage];
    constexpr int UN = 4;
    const bool pow2 = (a.N_int & (a.N_int - 1)) == 0;
    const float invN = 1.0f / a.Nf;
    const long long S = a.num_rows;
    const int seg_begin = static_cast<int>(S * blockIdx.x / gridDim.x);
    const int seg_end = static_cast<int>(S * (blockIdx.x + 1) / gridDim.x);
    for (int seg0 = seg_begin; seg0 < seg_end; seg0 += kScatterStage) {
        const int seg1 = min(seg_end, seg0 + kScatterStage);
        __syncthreads();
        for (int sg = seg0 + static_cast<int>(threadIdx.x); sg < seg1; sg += blockDim.x) {
            const SelRow R = a.rows[sg];
            stage[sg - seg0] = make_int4(R.b, R.k, R.q0, __ldcg(a.sel + a.blocks[R.b].sel_base + R.k));
        }
        __syncthreads();
        const int items = (seg1 - seg0) * kSegQuads;
        for (int base = 0; base < items; base += static_cast<int>(blockDim.x) * UN) {
            long long e0[UN], o0[UN];
            int cnt[UN], ocnt[UN];
            bool v4[UN];
#pragma unroll
            for (int u = 0; u < UN; ++u) {
                const int item = base + u * static_cast<int>(blockDim.x) + static_cast<int>(threadIdx.x);
                cnt[u] = ocnt[u] = 0;
                e0[u] = o0[u] = 0;
                v4[u] = false;
                if (item < items) {
                    const int4 R = stage[item / kSegQuads];         // (block, k, q0, selected row)
                    const BlockDev& B = a.blocks[R.x];
                    const int q = 4 * (R.z + item % kSegQuads);
                    if (q < B.n) {
                        const int nv = row_valid_cols(B, R.w);
                        cnt[u] = max(0, min(4, nv - q));
                        ocnt[u] = min(4, B.n - q);
                        e0[u] = B.off + static_cast<long long>(R.w) * B.n + q;
                        o0[u] = B.val_base + static_cast<long long>(R.y) * B.n + q;
                        v4[u] = B.vec && cnt[u] == 4;
                    }
                }
            }
            float4 A[UN], gb[UN];
#pragma unroll
            for (int u = 0; u < UN; ++u) {   // the batch's loads first
                gb[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (v4[u]) gb[u] = *reinterpret_cast<const float4*>(a.gbar + e0[u]);
                A[u] = ocnt[u] > 0 ? wire_quad(a.wire, o0[u], ocnt[u], a.bf16) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            if (a.mode == 1)
                for (int i = 1; i < a.nodes_total; ++i)
#pragma unroll
                    for (int u = 0; u < UN; ++u) {
                        if (ocnt[u] <= 0) continue;
                        const float4 c = wire_quad(a.wire, static_cast<long long>(i) * a.sum_Kn + o0[u], ocnt[u], a.bf16);
                        A[u].x = fadd(A[u].x, c.x); A[u].y = fadd(A[u].y, c.y);   // R9 node order
                        A[u].z = fadd(A[u].z, c.z); A[u].w = fadd(A[u].w, c.w);
                    }
#pragma unroll
            for (int u = 0; u < UN; ++u) {
                if (ocnt[u] <= 0) continue;
                const float Av[4] = {A[u].x, A[u].y, A[u].z, A[u].w};
                float val[4];
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    val[k] = k < cnt[u] ? (pow2 ? fmul(Av[k], invN) : __fdiv_rn(Av[k], a.Nf)) : 0.0f;   // R3; +0 padding
                if (v4[u]) {
                    float4 g = gb[u];
                    g.x = fadd(g.x, val[0]); g.y = fadd(g.y, val[1]); g.z = fadd(g.z, val[2]); g.w = fadd(g.w, val[3]);
                    *reinterpret_cast<float4*>(a.gbar + e0[u]) = g;                                   // R13
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (k < cnt[u]) a.gbar[e0[u] + k] = fadd(a.gbar[e0[u] + k], val[k]);
                }
                if (a.values != nullptr)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (k < ocnt[u]) a.values[o0[u] + k] = val[k];
            }
        }
    }
}

// =============================================================================
// Top-K baseline (ARC_METHOD_TOPK_ALLGATHER), S6: node j's gathered rows
// merged into the replicated tracker, gbar[I_j[k]] += C_j[k] / N (one launch per
// node, in node order: the nodes' supports overlap).
// =============================================================================
__global__ void __launch_bounds__(256) k_topk_merge(const MergeLaunch a) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const bool pow2 = (a.N_int & (a.N_int - 1)) == 0;
    const float invN = 1.0f / a.Nf;
    for (int w = gw; w < a.num_rows; w += nw) {
        const SelRow R = a.rows[w];
        const BlockDev& B = a.blocks[R.b];
        const int p = a.idx[B.sel_base + R.k];
        const int n = B.n;
        const int nv = row_valid_cols(B, p);
        const long long e0 = B.off + static_cast<long long>(p) * n;
        const long long o0 = B.val_base + static_cast<long long>(R.k) * n;
        const int qend = min(nv, 4 * (R.q0 + kSegQuads));
        for (int q = 4 * R.q0 + lane; q < qend; q += 32) {
            const float v = a.values[o0 + q];
            const float c = pow2 ? fmul(v, invN) : __fdiv_rn(v, a.Nf);   // R3: c / N
            a.gbar[e0 + q] = fadd(a.gbar[e0 + q], c);
        }
    }
}

// =============================================================================
// DENSE blocks (R20) when every node is on this GPU: the identity compressor
// as one coalesced streaming pass per element e of the block:
//   h_i <- (1-eta) h_i + eta grad_i ; C_i = h_i - g_i ; g_i <- g_i + C_i
//   A = C_0 + C_1 + ... ; gbar <- gbar + A / N ; values[e] = A / N
// (the same operations, in the same order, as the selected-row path).
// =============================================================================
__global__ void __launch_bounds__(256) k_dense(const DenseLaunch a) {
    const bool pow2 = (a.N_int & (a.N_int - 1)) == 0;
    const float invN = 1.0f / a.Nf;
    for (int db = 0; db < a.num_dense; ++db) {
        const BlockDev& B = a.blocks[a.dense_ids[db]];
        const long long len = B.len;
        // identity selection
        for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < B.m; p += (long long)gridDim.x * blockDim.x)
            a.sel[B.sel_base + p] = static_cast<int32_t>(p);
        // payload element (block-relative q) of node i (mode 2) or of the local sum (mode 1)
        auto put = [&](long long q, int i, float v) {
            pay_st(a.payload, (a.mode == 2 ? static_cast<long long>(i) * a.sum_Kn : 0LL) + B.val_base + q, v, a.bf16);
        };
        // element loop: quads when the block is 16-byte aligned, else scalars
        const bool vec = (B.off % 4) == 0;
        const long long nq = vec ? len / 4 : 0;
        for (long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x; f < nq; f += (long long)gridDim.x * blockDim.x) {
            const long long e = B.off + 4 * f;
            float A[4];
            for (int i = 0; i < a.nodes_local; ++i) {
                const float4 gr = __ldcs(reinterpret_cast<const float4*>(a.nodes.grad[i] + e));
                if (a.noef) {   // without EF: C_i = grad_i (identity compressor), no h / g
                    const float r4[4] = {wire_round(gr.x, a.bf16), wire_round(gr.y, a.bf16), wire_round(gr.z, a.bf16),
                                         wire_round(gr.w, a.bf16)};   // (R25)
#pragma unroll
                    for (int k = 0; k < 4; ++k) A[k] = (i == 0) ? r4[k] : fadd(A[k], r4[k]);
                    if (a.mode == 2)
#pragma unroll
                        for (int k = 0; k < 4; ++k) put(4 * f + k, i, r4[k]);
                    continue;
                }
                const float4 hv = *reinterpret_cast<const float4*>(a.nodes.h[i] + e);
                const float4 gv = *reinterpret_cast<const float4*>(a.nodes.g[i] + e);
                const float h4[4] = {hv.x, hv.y, hv.z, hv.w}, r4[4] = {gr.x, gr.y, gr.z, gr.w}, g4[4] = {gv.x, gv.y, gv.z, gv.w};
                float hn[4], gn[4], c4[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    hn[k] = ffma(a.eta, r4[k], fmul(a.ome, h4[k]));   // O2, R11
                    c4[k] = wire_round(fsub(hn[k], g4[k]), a.bf16);          // R4, R25
                    gn[k] = fadd(g4[k], c4[k]);                              // R12
                    A[k] = (i == 0) ? c4[k] : fadd(A[k], c4[k]);             // R9 node order
                }
                *reinterpret_cast<float4*>(a.nodes.h[i] + e) = make_float4(hn[0], hn[1], hn[2], hn[3]);
                *reinterpret_cast<float4*>(a.nodes.g[i] + e) = make_float4(gn[0], gn[1], gn[2], gn[3]);
                if (a.mode == 2)
#pragma unroll
                    for (int k = 0; k < 4; ++k) put(4 * f + k, i, c4[k]);
            }
            if (a.noef && a.mode != 0) {   // u <- eta u here; the scatter adds A / N
                const float4 bv = *reinterpret_cast<const float4*>(a.gbar + e);
                *reinterpret_cast<float4*>(a.gbar + e) =
                    make_float4(fmul(a.eta, bv.x), fmul(a.eta, bv.y), fmul(a.eta, bv.z), fmul(a.eta, bv.w));
            }
            if (a.mode == 1) {
#pragma unroll
                for (int k = 0; k < 4; ++k) put(4 * f + k, 0, A[k]);
                continue;
            }
            if (a.mode == 2) continue;
            const float4 bv = *reinterpret_cast<const float4*>(a.gbar + e);
            float b4[4] = {bv.x, bv.y, bv.z, bv.w};
            if (a.noef)
#pragma unroll
                for (int k = 0; k < 4; ++k) b4[k] = fmul(a.eta, b4[k]);   // u <- eta u
            float v[4], bn[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                v[k] = pow2 ? fmul(A[k], invN) : __fdiv_rn(A[k], a.Nf);    // R3
                bn[k] = fadd(b4[k], v[k]);                                   // R13
            }
            *reinterpret_cast<float4*>(a.gbar + e) = make_float4(bn[0], bn[1], bn[2], bn[3]);
            if (a.values != nullptr)
#pragma unroll
                for (int k = 0; k < 4; ++k) a.values[B.val_base + 4 * f + k] = v[k];
        }
        // scalar remainder (unaligned blocks, tails) and the padded tail of the values
        const long long total = static_cast<long long>(B.m) * B.n;
        for (long long q = 4 * nq + blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
             q += (long long)gridDim.x * blockDim.x) {
            if (q >= len) {
                if (a.mode == 2) {
                    for (int i = 0; i < a.nodes_local; ++i) put(q, i, 0.0f);
                } else if (a.mode == 1) {
                    put(q, 0, 0.0f);
                } else if (a.values != nullptr) {
                    a.values[B.val_base + q] = 0.0f;
                }
                continue;
            }
            const long long e = B.off + q;
            float A = 0.0f;
            if (a.noef) {   // without EF: C_i = grad_i, u <- eta u (+ A / N in mode 0)
                for (int i = 0; i < a.nodes_local; ++i) {
                    const float c = wire_round(a.nodes.grad[i][e], a.bf16);   // (R25)
                    A = (i == 0) ? c : fadd(A, c);
                    if (a.mode == 2) put(q, i, c);
                }
                const float us = fmul(a.eta, a.gbar[e]);
                if (a.mode == 1) put(q, 0, A);
                if (a.mode != 0) { a.gbar[e] = us; continue; }
                const float v = pow2 ? fmul(A, invN) : __fdiv_rn(A, a.Nf);
                a.gbar[e] = fadd(us, v);
                if (a.values != nullptr) a.values[B.val_base + q] = v;
                continue;
            }
            for (int i = 0; i < a.nodes_local; ++i) {
                const float hn = ffma(a.eta, a.nodes.grad[i][e], fmul(a.ome, a.nodes.h[i][e]));   // O2, R11
                a.nodes.h[i][e] = hn;
                const float gv = a.nodes.g[i][e];
                const float c = wire_round(fsub(hn, gv), a.bf16);   // (R25)
                a.nodes.g[i][e] = fadd(gv, c);
                A = (i == 0) ? c : fadd(A, c);
                if (a.mode == 2) put(q, i, c);
            }
            if (a.mode == 1) { put(q, 0, A); continue; }
            if (a.mode == 2) continue;
            const float v = pow2 ? fmul(A, invN) : __fdiv_rn(A, a.Nf);
            a.gbar[e] = fadd(a.gbar[e], v);
            if (a.values != nullptr) a.values[B.val_base + q] = v;
        }
    }
}

__global__ void __launch_bounds__(256) k_dense_scatter(const DenseScatterLaunch a) {
    const bool pow2 = (a.N_int & (a.N_int - 1)) == 0;
    const float invN = 1.0f / a.Nf;
    for (int db = 0; db < a.num_dense; ++db) {
        const BlockDev& B = a.blocks[a.dense_ids[db]];
        const long long total = static_cast<long long>(B.m) * B.n;
        for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
             q += (long long)gridDim.x * blockDim.x) {
            const long long o = B.val_base + q;
            float A = pay_ld(a.wire, o, a.bf16);
            if (a.mode == 1)
                for (int i = 1; i < a.nodes_total; ++i) A = fadd(A, pay_ld(a.wire, static_cast<long long>(i) * a.sum_Kn + o, a.bf16));
            const float v = q < B.len ? (pow2 ? fmul(A, invN) : __fdiv_rn(A, a.Nf)) : 0.0f;
            if (q < B.len) a.gbar[B.off + q] = fadd(a.gbar[B.off + q], v);
            if (a.values != nullptr) a.values[o] = v;
        }
    }
}

// S2 for the rows of one slice: x holds, for every source rank g and local node
// l, the slice's per-node sketches P_{gL+l} ([G][Ms][L][r]); the sum runs in
// ascending global node id g L + l (R9, R21).  One thread per row.
__global__ void __launch_bounds__(256) k_sigma_slice(const SigmaLaunch a) {
    const long long p = blockIdx.x * 256LL + threadIdx.x;
    if (p >= a.rows) return;
    const int L = a.L, r = a.r;
    float sig = 0.0f;
    if (r == 4) {
        float4 S = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int g = 0; g < a.G; ++g)
            for (int l = 0; l < L; ++l) {
                const float4 v = __ldcs(reinterpret_cast<const float4*>(a.x + ((g * a.Ms + p) * L + l) * 4));
                if (g == 0 && l == 0) S = v;
                else { S.x = fadd(S.x, v.x); S.y = fadd(S.y, v.y); S.z = fadd(S.z, v.z); S.w = fadd(S.w, v.w); }
            }
        const float P[4] = {S.x, S.y, S.z, S.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) sig = ffma(P[j], P[j], sig);                             // O8, zn28373
    } else {
        for (int j = 0; j < r; ++j) {
            float S = 0.0f;
            for (int g = 0; g < a.G; ++g)
                for (int l = 0; l < L; ++l) {
                    const float v = __ldcs(a.x + ((g * a.Ms + p) * L + l) * r + j);
                    S = (g == 0 && l == 0) ? v : fadd(S, v);
                }
            sig = ffma(S, S, sig);                                                             // O8
        }
    }
    a.sigma[p] = sig;
    if (!isfinite(sig)) atomicOr(a.status, kStatusNonfinite);
}

// ARC_METHOD_EXACT (test mode, SURVEY 8(b) ARC_SKETCH_EXACT, 8(f) row 3): the
// quantity the sketch estimates, Sigma_p = || sum_i Delta_i[p, :] ||^2
// (z72ena P:254-261, up to the factor N^2).  Runs after the streaming pass has
// stored h'_i, before the select kernel (which reads Sigma and histograms it).
// Per element S_q = ((D_0 + D_1) + ...) + D_{N-1}, D_i = h'_i - g_i (node order,
// R9); the squares summed in the O6 lane / chunk order with fma.  One warp per
// row, lane l owns columns 1024 c + 128 s + 4 l + e.
__global__ void __launch_bounds__(256) k_exact_sigma(const ExactSigmaLaunch a) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * 256LL + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * 256) >> 5;
    for (int b = 0; b < a.num_blocks; ++b) {
        const BlockDev& B = a.blocks[b];
        if (B.kind != ARC_BLOCK_ARC) continue;
        for (long long p = warp; p < B.m; p += nwarps) {
            const long long base = B.off + p * B.n;
            const long long rem = B.len - p * B.n;
            const int nv = static_cast<int>(rem < B.n ? rem : B.n);
            float P = 0.0f;
            for (int c = 0; 1024 * c < nv; ++c) {
                float acc = 0.0f;
                for (int sgm = 0; sgm < 8; ++sgm)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int q = 1024 * c + 128 * sgm + 4 * lane + e;
                        if (q < nv) {
                            float S = fsub(a.nodes.h[0][base + q], a.nodes.g[0][base + q]);
                            for (int i = 1; i < a.L; ++i)
                                S = fadd(S, fsub(a.nodes.h[i][base + q], a.nodes.g[i][base + q]));
                            acc = ffma(S, S, acc);                                  // O6
                        }
                    }
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) acc = fadd(acc, __shfl_xor_sync(kFull, acc, o));
                P = (c == 0) ? acc : fadd(P, acc);
            }
            if (lane == 0) {
                a.sigma[B.row_base + p] = P;
                if (!isfinite(P)) atomicOr(a.status, kStatusNonfinite);
            }
        }
    }
}

}  // namespace

// ---- launchers ---------------------------------------------------------------

void launch_vgen(const BlockDev* blocks_dev, int num_blocks, int max_nR4, int r, uint64_t seed, int64_t t,
                 float* V, cudaStream_t s, const unsigned long long* t_dev, int pdl) {
    const int threads = 256;
    int gx = (max_nR4 + threads - 1) / threads;
    if (gx < 1) gx = 1;
    if (gx > 64) gx = 64;
    const uint2 key = make_uint2(static_cast<unsigned>(seed), static_cast<unsigned>(seed >> 32));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(gx, num_blocks);
    cfg.blockDim = dim3(threads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_vgen, blocks_dev, r, key, static_cast<unsigned>(static_cast<uint64_t>(t)),
                       static_cast<unsigned>(static_cast<uint64_t>(t) >> 32), V, t_dev);
}

__global__ void k_advance_t(unsigned long long* t_dev) { *t_dev += 1ull; }
void launch_advance_t(unsigned long long* t_dev, cudaStream_t s) { k_advance_t<<<1, 1, 0, s>>>(t_dev); }
__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }
void launch_set_u64(unsigned long long* p, unsigned long long v, cudaStream_t s) { k_set_u64<<<1, 1, 0, s>>>(p, v); }

static int rows_grid(int num_rows) {
    int grid = (num_rows + 7) / 8;   // 8 warps per CTA, one warp per row segment
    if (grid < 1) grid = 1;
    if (grid > 148 * 16) grid = 148 * 16;
    return grid;
}

void launch_dense(const DenseLaunch& a, cudaStream_t s) {
    k_dense<<<148 * 8, 256, 0, s>>>(a);
}

void launch_dense_scatter(const DenseScatterLaunch& a, cudaStream_t s) {
    k_dense_scatter<<<148 * 8, 256, 0, s>>>(a);
}

void launch_topk_merge(const MergeLaunch& a, cudaStream_t s) {
    k_topk_merge<<<rows_grid(a.num_rows), 256, 0, s>>>(a);
}

void launch_exact_sigma(const ExactSigmaLaunch& a, cudaStream_t s) {
    k_exact_sigma<<<148 * 8, 256, 0, s>>>(a);
}

void launch_sigma_slice(const SigmaLaunch& a, cudaStream_t s) {
    if (a.rows > 0) k_sigma_slice<<<static_cast<unsigned>((a.rows + 255) / 256), 256, 0, s>>>(a);
}

void launch_scatter(const ScatterLaunch& a, cudaStream_t s) {
    const long long quads = static_cast<long long>(a.num_rows) * kSegQuads;
    long long grid = (quads + 255) / 256;
    if (grid > 148 * 8) grid = 148 * 8;
    if (grid < 1) grid = 1;
    k_scatter<<<static_cast<int>(grid), 256, 0, s>>>(a);
}


// ARC_Q_S (debug): S = P'_0 (+) P'_1 (+) ... of every ARC row, ascending node id
// (R9), from the per-node sketches [M][L][r] of one GPU holding every node.
namespace {
__global__ void __launch_bounds__(256) k_node_sum(const float* __restrict__ pn, long long M, int L, int r,
                                                  float* __restrict__ dst) {
    for (long long e = blockIdx.x * 256LL + threadIdx.x; e < M * r; e += static_cast<long long>(gridDim.x) * 256) {
        const long long p = e / r;
        const int j = static_cast<int>(e - p * r);
        float S = pn[p * L * r + j];
        for (int l = 1; l < L; ++l) S = dev::fadd(S, pn[(p * L + l) * r + j]);
        dst[e] = S;
    }
}
}  // namespace

void launch_node_sum(const float* pnodes, long long M, int L, int r, float* dst, cudaStream_t s) {
    const long long n = M * r;
    if (n <= 0) return;
    const int grid = static_cast<int>(n / 256 + 1 < 148 * 8 ? n / 256 + 1 : 148 * 8);
    k_node_sum<<<grid, 256, 0, s>>>(pnodes, M, L, r, dst);
}

}  // namespace arc
