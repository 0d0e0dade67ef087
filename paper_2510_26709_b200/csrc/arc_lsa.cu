// arc_lsa.cu — exchange #2 fused with S6 over NVLink peer memory
// (value_reduce = ARC_REDUCE_LSA).
//
// Alg. 1 l.8 all-reduces the K dense rows C_i ("index-free
// All-Reduce") and eq:ef21m-3 consumes their mean in the
// replicated tracker: gbar[I_k] <- gbar[I_k] + A_k / N.  Here every rank's
// select kernel writes its per-node payload C_{gL+l} ([L][sum_Kn] floats) into
// an NCCL symmetric window (ncclCommWindowRegister, NCCL_WIN_COLL_SYMMETRIC);
// one kernel per block kind then
//   1. meets the other ranks at an LSA barrier (CTA b of every rank; acq_rel:
//      every rank's payload kernel has finished and its stores are visible),
//   2. reads each payload element of every node straight from the owning
//      peer's window over NVLink (ncclGetLsaPointer), sums it in ascending
//      global node id (the ORDERED mode's order, R9 / R21 — so gbar is
//      bit-identical to the oracle on any number of GPUs), and adds A / N into
//      gbar (and values_out),
//   3. meets the peers again so no rank overwrites its window (next step's
//      payload) while a peer is still reading it.
// This replaces the all-gather into a staging buffer and the separate scatter
// launch of the ORDERED mode: the payload crosses NVLink once and lands in
// registers, not in HBM.  k_lsa_sigma does the same for exchange #1 (below).
#include <cuda_runtime.h>

#include <cstdint>

#include "nccl.h"
#include "nccl_device.h"

#include "arc_device.cuh"
#include "arc_internal.cuh"

namespace arc {
namespace {
using namespace dev;

constexpr int kLsaMaxPeers = 72;   // one NVLink domain (NVL72); checked at create

struct PeerBase {
    const float* p[kLsaMaxPeers];
};

__device__ __forceinline__ void load_peers(const LsaScatter& x, PeerBase& pb) {
    for (int g = threadIdx.x; g < x.G; g += blockDim.x)
        pb.p[g] = static_cast<const float*>(ncclGetLsaPointer(x.win, 0, g));
    __syncthreads();
}

// payload element o of node i = g L + l at peer g (float or bf16 entries, R25)
__device__ __forceinline__ float peer_ld(const PeerBase& pb, const LsaScatter& x, int i, long long o) {
    const int g = i / x.L, l = i - g * x.L;
    return pay_ld(pb.p[g], static_cast<long long>(l) * x.sum_Kn + o, x.bf16);
}

// A = C_0 ⊕ C_1 ⊕ ... ⊕ C_{N-1} of payload element o, node i = g L + l at
// peer g, offset l * sum_Kn + o (R9: the order of the ORDERED mode).
__device__ __forceinline__ float node_sum(const PeerBase& pb, const LsaScatter& x, long long o) {
    float A = peer_ld(pb, x, 0, o);
    for (int i = 1; i < x.N; ++i) A = fadd(A, peer_ld(pb, x, i, o));
    return A;
}

__global__ void __launch_bounds__(256) k_lsa_scatter(const ScatterLaunch a, const LsaScatter x) {
    __shared__ PeerBase pb;
    load_peers(x, pb);
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), *x.dev_comm, ncclTeamTagLsa(), blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    const bool pow2 = (a.N_int & (a.N_int - 1)) == 0;
    const float invN = 1.0f / a.Nf;
    const long long items = static_cast<long long>(a.num_rows) * kSegQuads;
    for (long long it = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; it < items;
         it += static_cast<long long>(gridDim.x) * blockDim.x) {
        const SelRow R = a.rows[it / kSegQuads];
        const BlockDev& B = a.blocks[R.b];
        const int q = 4 * (R.q0 + static_cast<int>(it % kSegQuads));
        if (q >= B.n) continue;
        const int p = a.sel[B.sel_base + R.k];
        const long long rest = B.len - static_cast<long long>(p) * B.n;
        const int nv = rest < B.n ? static_cast<int>(rest) : B.n;
        const long long e0 = B.off + static_cast<long long>(p) * B.n;
        const long long o0 = B.val_base + static_cast<long long>(R.k) * B.n;
        const int cnt = max(0, min(4, nv - q)), ocnt = min(4, B.n - q);
        if (!x.bf16 && ocnt == 4 && (((o0 + q) | x.sum_Kn) & 3) == 0) {   // 16-byte payload loads
            float4 A = __ldcg(reinterpret_cast<const float4*>(pb.p[0] + o0 + q));
            for (int i = 1; i < x.N; ++i) {
                const int g = i / x.L, l = i - g * x.L;
                const float4 c = __ldcg(reinterpret_cast<const float4*>(pb.p[g] + static_cast<long long>(l) * x.sum_Kn + o0 + q));
                A.x = fadd(A.x, c.x); A.y = fadd(A.y, c.y); A.z = fadd(A.z, c.z); A.w = fadd(A.w, c.w);
            }
            const float Av[4] = {A.x, A.y, A.z, A.w};
            float val[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) val[k] = k < cnt ? (pow2 ? fmul(Av[k], invN) : __fdiv_rn(Av[k], a.Nf)) : 0.0f;
            if (B.vec && cnt == 4) {
                float4* gp = reinterpret_cast<float4*>(a.gbar + e0 + q);
                float4 gb = *gp;
                gb.x = fadd(gb.x, val[0]); gb.y = fadd(gb.y, val[1]); gb.z = fadd(gb.z, val[2]); gb.w = fadd(gb.w, val[3]);
                *gp = gb;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (k < cnt) a.gbar[e0 + q + k] = fadd(a.gbar[e0 + q + k], val[k]);
            }
            if (a.values != nullptr)
                *reinterpret_cast<float4*>(a.values + o0 + q) = make_float4(val[0], val[1], val[2], val[3]);
            continue;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k >= ocnt) continue;
            const float A = node_sum(pb, x, o0 + q + k);
            const float v = k < cnt ? (pow2 ? fmul(A, invN) : __fdiv_rn(A, a.Nf)) : 0.0f;   // R3; +0 padding
            if (k < cnt) a.gbar[e0 + q + k] = fadd(a.gbar[e0 + q + k], v);                   // R13
            if (a.values != nullptr) a.values[o0 + q + k] = v;
        }
    }
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

__global__ void __launch_bounds__(256) k_lsa_dense_scatter(const DenseScatterLaunch a, const LsaScatter x) {
    __shared__ PeerBase pb;
    load_peers(x, pb);
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), *x.dev_comm, ncclTeamTagLsa(), blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    const bool pow2 = (a.N_int & (a.N_int - 1)) == 0;
    const float invN = 1.0f / a.Nf;
    for (int db = 0; db < a.num_dense; ++db) {
        const BlockDev& B = a.blocks[a.dense_ids[db]];
        const long long total = static_cast<long long>(B.m) * B.n;
        for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
             q += (long long)gridDim.x * blockDim.x) {
            const long long o = B.val_base + q;
            const float A = node_sum(pb, x, o);
            const float v = q < B.len ? (pow2 ? fmul(A, invN) : __fdiv_rn(A, a.Nf)) : 0.0f;
            if (q < B.len) a.gbar[B.off + q] = fadd(a.gbar[B.off + q], v);
            if (a.values != nullptr) a.values[o] = v;
        }
    }
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

// Exchange #1 + S2 over peer memory (replaces the all-to-all of P' slices,
// k_sigma_slice and the all-gather of Sigma): after barrier 1 (every rank's
// sketch pass has completed) CTA b forms Sigma of sub-range b of this rank's
// slice from every node's P' rows read in the owners' windows, summed in
// ascending global node id and squared-summed with the O8 fma chain (R9, R21;
// the k_sigma_slice order); after barrier 2 it copies sub-range b of every
// other rank's Sigma slice from that rank's window (CTA b of that rank wrote
// it); barrier 3 keeps every rank's P' and Sigma unchanged until all peers have
// read them.
__global__ void __launch_bounds__(256) k_lsa_sigma(const LsaSigma a) {
    __shared__ const float* pk[kLsaMaxPeers];   // peers' P' (window offset 0)
    __shared__ const float* ps[kLsaMaxPeers];   // peers' Sigma
    for (int g = threadIdx.x; g < a.G; g += blockDim.x) {
        pk[g] = static_cast<const float*>(ncclGetLsaPointer(a.win, 0, g));
        ps[g] = static_cast<const float*>(ncclGetLsaPointer(a.win, a.sigma_off, g));
    }
    __syncthreads();
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), *a.dev_comm, ncclTeamTagLsa(), blockIdx.x);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    const long long chunk = (a.Ms + gridDim.x - 1) / gridDim.x;
    const long long lo = blockIdx.x * chunk, hi = min(a.Ms, lo + chunk);
    const int L = a.L, r = a.r;
    const long long base = a.me * a.Ms;
    for (long long p = lo + threadIdx.x; p < hi; p += blockDim.x) {
        const long long row = base + p;
        if (row >= a.M) break;
        float sig = 0.0f;
        if (r == 4) {   // one 16-byte load per node (P' rows are 16-byte aligned: r = 4)
            float4 S = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int g = 0; g < a.G; ++g)
                for (int l = 0; l < L; ++l) {
                    const float4 v = __ldcg(reinterpret_cast<const float4*>(pk[g] + (row * L + l) * 4));
                    if (g == 0 && l == 0) S = v;
                    else { S.x = fadd(S.x, v.x); S.y = fadd(S.y, v.y); S.z = fadd(S.z, v.z); S.w = fadd(S.w, v.w); }
                }
            const float P[4] = {S.x, S.y, S.z, S.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) sig = ffma(P[j], P[j], sig);                         // O8
            a.sigma[row] = sig;
            if (!isfinite(sig)) atomicOr(a.status, kStatusNonfinite);
            continue;
        }
        for (int j = 0; j < r; ++j) {
            float S = 0.0f;
            for (int g = 0; g < a.G; ++g)
                for (int l = 0; l < L; ++l) {
                    const float v = __ldcg(pk[g] + (row * L + l) * r + j);
                    S = (g == 0 && l == 0) ? v : fadd(S, v);
                }
            sig = ffma(S, S, sig);                                                             // O8
        }
        a.sigma[row] = sig;
        if (!isfinite(sig)) atomicOr(a.status, kStatusNonfinite);
    }
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    for (int g = 0; g < a.G; ++g) {
        if (g == a.me) continue;
        const long long gb = g * a.Ms;
        for (long long p = lo + threadIdx.x; p < hi; p += blockDim.x) {
            if (gb + p >= a.M) break;
            a.sigma[gb + p] = __ldcg(ps[g] + gb + p);
        }
    }
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

}  // namespace

void launch_lsa_sigma(const LsaSigma& a, cudaStream_t s) {
    long long grid = (a.Ms + 255) / 256;
    if (grid > kLsaCtas) grid = kLsaCtas;
    if (grid < 1) grid = 1;
    k_lsa_sigma<<<static_cast<int>(grid), 256, 0, s>>>(a);
}

void launch_lsa_scatter(const ScatterLaunch& a, const LsaScatter& x, cudaStream_t s) {
    const long long quads = static_cast<long long>(a.num_rows) * kSegQuads;
    long long grid = (quads + 255) / 256;
    if (grid > kLsaCtas) grid = kLsaCtas;
    if (grid < 1) grid = 1;
    k_lsa_scatter<<<static_cast<int>(grid), 256, 0, s>>>(a, x);
}

void launch_lsa_dense_scatter(const DenseScatterLaunch& a, const LsaScatter& x, cudaStream_t s) {
    k_lsa_dense_scatter<<<kLsaCtas, 256, 0, s>>>(a, x);
}

}  // namespace arc
