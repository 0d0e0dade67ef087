// arc_loopback.cu — an in-process communicator that emulates G ranks inside ONE
// process on ONE GPU, so the library's G > 1 step (exchange #1's all-to-all of
// row slices + the Sigma all-gather, exchange #2's all-reduce / all-gather, the
// params-hash check at create) runs on hardware with one GPU.
//
// Each emulated rank is a host thread with its own context and CUDA stream.
// A collective is three host-side steps per rank:
//   1. record `ready[j]` on the rank's stream (everything the rank enqueued before
//      the collective), post the buffers, meet the other ranks at a host barrier;
//   2. make the stream wait for every rank's `ready` event, then enqueue this
//      rank's share of the data movement (device-to-device copies, or a kernel that
//      sums every rank's send buffer into a scratch buffer), record `done[j]`;
//      host barrier;
//   3. make the stream wait for every rank's `done` event (no rank may overwrite a
//      buffer a peer still reads), then (all-reduce) copy the scratch sum into the
//      receive buffer.
// Dependencies between the ranks' streams are stream-event waits only: no kernel
// spins on another rank's progress, so nothing relies on two kernels being
// co-scheduled (B200_PROFILING.md: ranks that wait on one another must not run
// as separate launches on one GPU).
//
// The all-reduce sums the ranks in DESCENDING rank order — a different order
// from the oracle's ascending node order, standing in for NCCL's unspecified
// one, so the ARC_REDUCE_NCCL tolerance contract is exercised.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "arc_internal.cuh"
#include "arc_loopback.h"

namespace arc {

constexpr int kLoopbackMaxRanks = 64;

struct LoopbackGroup {
    int G = 0;
    int device = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    bool broken = false;                         // a barrier timed out: every later call fails
    struct Post {
        const void* send = nullptr;
        void* recv = nullptr;
        size_t bytes = 0;                        // all-gather: bytes per rank; all-reduce: floats
        const size_t* scount = nullptr;          // all-to-all (floats), host arrays [G]
        const size_t* sdispl = nullptr;
        int kind = -1;
    };
    std::vector<Post> posts;
    std::vector<cudaEvent_t> ready, done;
    std::vector<void*> scratch;                  // all-reduce sums, one per rank (bytes: scratch_n)
    std::vector<size_t> scratch_n;
    std::vector<LoopbackComm> handles;
};

struct LoopbackComm {
    LoopbackGroup* grp = nullptr;
    int rank = 0;
};

namespace {

// host barrier with a timeout (a rank that failed before a collective must not
// hang the others forever)
bool barrier(LoopbackGroup* g) {
    std::unique_lock<std::mutex> lk(g->mu);
    if (g->broken) return false;
    const uint64_t gen = g->generation;
    if (++g->arrived == g->G) {
        g->arrived = 0;
        ++g->generation;
        g->cv.notify_all();
        return true;
    }
    const bool ok = g->cv.wait_for(lk, std::chrono::seconds(120), [&] { return g->generation != gen || g->broken; });
    if (!ok || g->broken) {
        g->broken = true;
        g->cv.notify_all();
        return false;
    }
    return true;
}

struct SumArgs {
    const void* src[kLoopbackMaxRanks];
    int G;
    long long n;
    void* dst;
};

// dst[e] = src[G-1][e] + src[G-2][e] + ... + src[0][e], left to right, in
// binary32; bfloat16 buffers (the R25 wire): the binary32 sum rounded once
template <class T>
__global__ void k_loopback_sum(const SumArgs a) {
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < a.n;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        float s = static_cast<float>(static_cast<const T*>(a.src[a.G - 1])[e]);
        for (int k = a.G - 2; k >= 0; --k) s = __fadd_rn(s, static_cast<float>(static_cast<const T*>(a.src[k])[e]));
        static_cast<T*>(a.dst)[e] = static_cast<T>(s);
    }
}

enum { kAllGather = 0, kAllReduce = 1, kAllToAll = 2, kAllReduceBf16 = 3 };

arc_status collective(LoopbackComm* c, int kind, const void* send, void* recv, size_t bytes, const size_t* scount,
                      const size_t* sdispl, const size_t* rcount, const size_t* rdispl, cudaStream_t s) {
    LoopbackGroup* g = c->grp;
    const int me = c->rank;
    if (cudaEventRecord(g->ready[me], s) != cudaSuccess) return ARC_ERR_CUDA;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        LoopbackGroup::Post& p = g->posts[me];
        p.send = send;
        p.recv = recv;
        p.bytes = bytes;
        p.scount = scount;
        p.sdispl = sdispl;
        p.kind = kind;
    }
    if (!barrier(g)) return ARC_ERR_NCCL;
    arc_status st = ARC_OK;
    for (int k = 0; k < g->G; ++k)
        if (k != me && cudaStreamWaitEvent(s, g->ready[k], 0) != cudaSuccess) st = ARC_ERR_CUDA;
    for (int k = 0; k < g->G && st == ARC_OK; ++k)
        if (g->posts[k].kind != kind) st = ARC_ERR_NCCL;   // ranks issued different collectives
    if (st == ARC_OK) {
        if (kind == kAllGather) {
            for (int k = 0; k < g->G; ++k) {
                unsigned char* dst = static_cast<unsigned char*>(recv) + static_cast<size_t>(k) * bytes;
                const void* src = g->posts[k].send;
                if (bytes == 0 || src == dst) continue;
                if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess) st = ARC_ERR_CUDA;
            }
        } else if (kind == kAllToAll) {
            for (int k = 0; k < g->G; ++k) {
                const LoopbackGroup::Post& p = g->posts[k];
                const size_t n = p.scount[me];   // floats rank k sends to me
                if (n != rcount[k]) { st = ARC_ERR_NCCL; break; }
                if (n == 0) continue;
                const float* src = static_cast<const float*>(p.send) + p.sdispl[me];
                float* dst = static_cast<float*>(recv) + rdispl[k];
                if (cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToDevice, s) != cudaSuccess)
                    st = ARC_ERR_CUDA;
            }
        } else {   // all-reduce (sum): every rank's send buffer summed into this rank's scratch
            const size_t n = bytes;
            const size_t esz = kind == kAllReduceBf16 ? 2 : sizeof(float);
            for (int k = 0; k < g->G; ++k)
                if (g->posts[k].bytes != n) st = ARC_ERR_NCCL;
            if (st == ARC_OK && n > 0) {
                if (g->scratch_n[me] < n * esz) {
                    if (g->scratch[me]) cudaFree(g->scratch[me]);
                    g->scratch[me] = nullptr;
                    g->scratch_n[me] = 0;
                    if (cudaMalloc(&g->scratch[me], n * esz) != cudaSuccess) st = ARC_ERR_CUDA;
                    else g->scratch_n[me] = n * esz;
                }
                if (st == ARC_OK) {
                    SumArgs a{};
                    for (int k = 0; k < g->G; ++k) a.src[k] = g->posts[k].send;
                    a.G = g->G;
                    a.n = static_cast<long long>(n);
                    a.dst = g->scratch[me];
                    const int grid = static_cast<int>(std::min<long long>((a.n + 255) / 256, 148 * 8));
                    if (kind == kAllReduceBf16) k_loopback_sum<__nv_bfloat16><<<grid, 256, 0, s>>>(a);
                    else k_loopback_sum<float><<<grid, 256, 0, s>>>(a);
                    if (cudaPeekAtLastError() != cudaSuccess) { (void)cudaGetLastError(); st = ARC_ERR_CUDA; }
                }
            }
        }
    }
    if (cudaEventRecord(g->done[me], s) != cudaSuccess) st = ARC_ERR_CUDA;
    if (!barrier(g)) return ARC_ERR_NCCL;
    for (int k = 0; k < g->G; ++k)
        if (k != me && cudaStreamWaitEvent(s, g->done[k], 0) != cudaSuccess) st = ARC_ERR_CUDA;
    if (st == ARC_OK && (kind == kAllReduce || kind == kAllReduceBf16) && bytes > 0 &&
        cudaMemcpyAsync(recv, g->scratch[me], bytes * (kind == kAllReduceBf16 ? 2 : sizeof(float)),
                        cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        st = ARC_ERR_CUDA;
    return st;
}

}  // namespace

int loopback_nranks(const LoopbackComm* c) { return c->grp->G; }
int loopback_rank(const LoopbackComm* c) { return c->rank; }

arc_status loopback_all_gather(LoopbackComm* c, const void* send, void* recv, size_t bytes, cudaStream_t s) {
    return collective(c, kAllGather, send, recv, bytes, nullptr, nullptr, nullptr, nullptr, s);
}
arc_status loopback_all_reduce_f32(LoopbackComm* c, const float* send, float* recv, size_t count, cudaStream_t s) {
    return collective(c, kAllReduce, send, recv, count, nullptr, nullptr, nullptr, nullptr, s);
}
arc_status loopback_all_reduce_bf16(LoopbackComm* c, const void* send, void* recv, size_t count, cudaStream_t s) {
    return collective(c, kAllReduceBf16, send, recv, count, nullptr, nullptr, nullptr, nullptr, s);
}
arc_status loopback_all_to_all_f32(LoopbackComm* c, const float* send, const size_t* scount, const size_t* sdispl,
                                   float* recv, const size_t* rcount, const size_t* rdispl, cudaStream_t s) {
    return collective(c, kAllToAll, send, recv, 0, scount, sdispl, rcount, rdispl, s);
}

}  // namespace arc

using namespace arc;

extern "C" {

arc_status arc_topk_loopback_create(int32_t G, void** group) {
    if (group == nullptr) return ARC_ERR_INVALID_ARG;
    *group = nullptr;
    if (G < 1 || G > kLoopbackMaxRanks) return ARC_ERR_INVALID_ARG;
    LoopbackGroup* g = new (std::nothrow) LoopbackGroup();
    if (g == nullptr) return ARC_ERR_INVALID_ARG;
    g->G = G;
    if (cudaGetDevice(&g->device) != cudaSuccess) { delete g; return ARC_ERR_CUDA; }
    g->posts.resize(G);
    g->ready.assign(G, nullptr);
    g->done.assign(G, nullptr);
    g->scratch.assign(G, nullptr);
    g->scratch_n.assign(G, 0);
    g->handles.resize(G);
    for (int k = 0; k < G; ++k) {
        g->handles[k].grp = g;
        g->handles[k].rank = k;
        if (cudaEventCreateWithFlags(&g->ready[k], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&g->done[k], cudaEventDisableTiming) != cudaSuccess) {
            arc_topk_loopback_destroy(g);
            return ARC_ERR_CUDA;
        }
    }
    *group = g;
    return ARC_OK;
}

arc_status arc_topk_loopback_comm(void* group, int32_t rank, void** comm) {
    LoopbackGroup* g = static_cast<LoopbackGroup*>(group);
    if (g == nullptr || comm == nullptr || rank < 0 || rank >= g->G) return ARC_ERR_INVALID_ARG;
    *comm = &g->handles[rank];
    return ARC_OK;
}

arc_status arc_topk_loopback_destroy(void* group) {
    LoopbackGroup* g = static_cast<LoopbackGroup*>(group);
    if (g == nullptr) return ARC_ERR_INVALID_ARG;
    cudaDeviceSynchronize();
    for (cudaEvent_t e : g->ready) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : g->done) if (e) cudaEventDestroy(e);
    for (void* p : g->scratch) if (p) cudaFree(p);
    delete g;
    return ARC_OK;
}

}  // extern "C"
