// Floor of the EF gather pattern: K random rows of n floats in three d-float
// arrays (read h, g, gbar; write g, gbar), one node.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_gather tools/microbench_gather.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

template <int UN>
__global__ void k_gather(const int* __restrict__ rows, int K, int n, const float* __restrict__ h, float* g, float* gbar) {
    const int nq = n / 4;
    const long long items = (long long)K * nq;
    for (long long base = (long long)blockIdx.x * blockDim.x * UN; base < items; base += (long long)gridDim.x * blockDim.x * UN) {
        float4 hv[UN], gv[UN], bv[UN];
        long long e[UN];
        bool ok[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) {
            long long it = base + u * blockDim.x + threadIdx.x;
            ok[u] = it < items;
            int j = ok[u] ? (int)(it / nq) : 0, f = ok[u] ? (int)(it % nq) : 0;
            e[u] = (long long)rows[j] * n + 4 * f;
            if (ok[u]) {
                hv[u] = *reinterpret_cast<const float4*>(h + e[u]);
                gv[u] = *reinterpret_cast<const float4*>(g + e[u]);
                bv[u] = *reinterpret_cast<const float4*>(gbar + e[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < UN; ++u) {
            if (!ok[u]) continue;
            float4 c = make_float4(hv[u].x - gv[u].x, hv[u].y - gv[u].y, hv[u].z - gv[u].z, hv[u].w - gv[u].w);
            *reinterpret_cast<float4*>(g + e[u]) = make_float4(gv[u].x + c.x, gv[u].y + c.y, gv[u].z + c.z, gv[u].w + c.w);
            *reinterpret_cast<float4*>(gbar + e[u]) = make_float4(bv[u].x + c.x, bv[u].y + c.y, bv[u].z + c.z, bv[u].w + c.w);
        }
    }
}

int main() {
    const long long d = 124439808LL;
    const int n = 768, m = (int)(d / n), K = 1621;
    float *h, *g, *gb, *flush;
    int* rows;
    cudaMalloc(&h, d * 4); cudaMalloc(&g, d * 4); cudaMalloc(&gb, d * 4); cudaMalloc(&flush, 512 << 20);
    cudaMemset(h, 0, d * 4); cudaMemset(g, 0, d * 4); cudaMemset(gb, 0, d * 4);
    std::vector<int> r(m);
    for (int i = 0; i < m; ++i) r[i] = i;
    srand(1);
    std::random_shuffle(r.begin(), r.end());
    std::sort(r.begin(), r.begin() + K);
    cudaMalloc(&rows, K * 4);
    cudaMemcpy(rows, r.data(), K * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int grid : {148, 296, 592, 1184}) {
        for (int un : {1, 4}) {
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                cudaMemset(flush, rep, 512 << 20);   // evict L2
                cudaEventRecord(a);
                if (un == 1) k_gather<1><<<grid, 256>>>(rows, K, n, h, g, gb);
                else k_gather<4><<<grid, 256>>>(rows, K, n, h, g, gb);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                best = std::min(best, ms);
            }
            double bytes = (double)K * n * 4 * 5;
            printf("grid %5d UN %d: %.2f us  (%.2f TB/s of 20 B/elem)\n", grid, un, best * 1e3, bytes / (best * 1e-3) / 1e12);
        }
    }
    // empty-kernel reference
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        k_gather<1><<<148, 256>>>(rows, 0, n, h, g, gb);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        best = std::min(best, ms);
    }
    printf("empty launch: %.2f us\n", best * 1e3);
    return 0;
}
