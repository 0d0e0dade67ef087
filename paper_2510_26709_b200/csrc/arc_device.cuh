// arc_device.cuh — device helpers shared by the kernel files of libarctopk.so:
// explicitly rounded binary32 operations (no contraction, R9) and streaming loads.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace arc {
namespace dev {

constexpr unsigned kFull = 0xFFFFFFFFu;

static __device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
static __device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
static __device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
static __device__ __forceinline__ float ffma(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// ---- streaming loads (read-once data: no L1 allocation) ----------------------
static __device__ __forceinline__ float ld_nc(const float* p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
static __device__ __forceinline__ float4 ld_nc4(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
// h is read and then rewritten by the same thread: coherent load, no L1 allocation
static __device__ __forceinline__ float ld_na(const float* p) {
    float v;
    asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
static __device__ __forceinline__ float4 ld_na4(const float* p) {
    float4 v;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

// ---- the value wire (R25): binary32, or bfloat16 rounded at the source --------
// what a node sends: c itself, or bf16(c) (round to nearest even), as binary32
static __device__ __forceinline__ float wire_round(float c, int bf16) {
    return bf16 ? __bfloat162float(__float2bfloat16_rn(c)) : c;
}
// element i of a payload buffer of binary32 or bfloat16 entries
static __device__ __forceinline__ float pay_ld(const void* base, long long i, int bf16) {
    return bf16 ? __bfloat162float(__ldcg(static_cast<const __nv_bfloat16*>(base) + i))
                : __ldcg(static_cast<const float*>(base) + i);
}
static __device__ __forceinline__ void pay_st(void* base, long long i, float v, int bf16) {
    if (bf16) static_cast<__nv_bfloat16*>(base)[i] = __float2bfloat16_rn(v);
    else static_cast<float*>(base)[i] = v;
}

// Order key of a Sigma value (R15): its binary32 bit pattern (Sigma >= +0, so
// unsigned order is numeric order); every NaN maps to the largest key.
static __device__ __forceinline__ unsigned order_key_dev(float s) {
    return isnan(s) ? 0xFFFFFFFFu : __float_as_uint(s);
}

// Programmatic dependent launch: wait until the preceding kernel's writes are
// visible (a no-op when the kernel was launched without the PDL attribute).
static __device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

}  // namespace dev
}  // namespace arc
