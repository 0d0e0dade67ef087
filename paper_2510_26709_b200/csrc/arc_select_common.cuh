// arc_select_common.cuh — CTA-wide scan and radix-digit helpers shared by the
// selection kernel (arc_select.cu) and the fused small-problem tail of the
// streaming pass (arc_sketch.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>

#include "arc_device.cuh"

namespace arc {
namespace selc {
using dev::kFull;

// exclusive scan of one int per thread over the CTA; *total = CTA sum.
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
        if (lane < nw) warp_sums[lane] = w;   // inclusive
    }
    __syncthreads();
    const int excl = x - v + (warp > 0 ? warp_sums[warp - 1] : 0);
    *total = warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
    return excl;
}

// The bin of a histogram (largest bin first) where the running count reaches
// `krem`; *above = count in higher bins.  All threads call; h in shared memory.
template <int NT = 256>
__device__ __forceinline__ unsigned top_digit(const unsigned* h, int nbins, int krem, int* warp_sums,
                                              unsigned* s_dig, int* s_abv, int* above) {
    const int per = nbins / NT;   // 8 or 4
    const int hi_bin = nbins - 1 - per * static_cast<int>(threadIdx.x);
    int mine = 0;
    for (int k = 0; k < per; ++k) mine += static_cast<int>(h[hi_bin - k]);
    int tot;
    const int ex = cta_exclusive_scan(mine, warp_sums, &tot);
    if (ex < krem && ex + mine >= krem) {
        int acc = ex, k = 0;
        while (acc + static_cast<int>(h[hi_bin - k]) < krem) { acc += static_cast<int>(h[hi_bin - k]); ++k; }
        *s_dig = static_cast<unsigned>(hi_bin - k);
        *s_abv = acc;
    }
    __syncthreads();
    *above = *s_abv;
    const unsigned d = *s_dig;
    __syncthreads();
    return d;
}

}  // namespace selc
}  // namespace arc
