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
// registers, not in HBM.
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

// A = C_0 ⊕ C_1 ⊕ ... ⊕ C_{N-1} of payload element o, node i = g L + l at
// peer g, offset l * sum_Kn + o (R9: the order of the ORDERED mode).
__device__ __forceinline__ float node_sum(const PeerBase& pb, const LsaScatter& x, long long o) {
    float A = __ldcg(pb.p[0] + o);
    for (int i = 1; i < x.N; ++i) {
        const int g = i / x.L, l = i - g * x.L;
        A = fadd(A, __ldcg(pb.p[g] + static_cast<long long>(l) * x.sum_Kn + o));
    }
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

}  // namespace

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
