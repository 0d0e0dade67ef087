// Micro-benchmark: launch and grid-barrier costs on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_coop.cu && /tmp/mb
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int SYNCS, int SMEM>
__global__ void __launch_bounds__(256, 3) k_coop(int* out) {
    __shared__ int buf[SMEM / 4];
    cg::grid_group g = cg::this_grid();
    buf[threadIdx.x] = threadIdx.x;
    for (int i = 0; i < SYNCS; ++i) g.sync();
    if (threadIdx.x == 0 && buf[5] == 12345) out[blockIdx.x] = 1;
}
template <int SMEM>
__global__ void __launch_bounds__(256) k_plain(int* out) {
    __shared__ int buf[SMEM / 4];
    buf[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && buf[5] == 12345) out[blockIdx.x] = 1;
}

template <class F>
float time_it(F f, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 10; ++i) f();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1000.f / reps;
}

template <int SYNCS, int SMEM>
void coop(int grid, int* out) {
    void* args[] = {&out};
    float us = time_it([&] { cudaLaunchCooperativeKernel((void*)k_coop<SYNCS, SMEM>, grid, 256, args, 0, 0); }, 200);
    printf("coop grid=%d smem=%d syncs=%d: %.2f us/launch (%s)\n", grid, SMEM, SYNCS, us,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int* out;
    cudaMalloc(&out, 1 << 20);
    for (int grid : {148, 317, 444}) {
        float us = time_it([&] { k_plain<1024><<<grid, 256>>>(out); }, 200);
        printf("plain grid=%d: %.2f us/launch\n", grid, us);
        coop<0, 1024>(grid, out);
        coop<1, 1024>(grid, out);
        coop<3, 1024>(grid, out);
        coop<0, 40960>(grid, out);
        coop<3, 40960>(grid, out);
    }
    return 0;
}
