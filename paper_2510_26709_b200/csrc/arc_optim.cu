// arc_optim.cu — the model update that consumes gbar:
//   SGD  x <- x - gamma gbar                                 eq:ef21m-3, P:327 (R23)
//   Adam on gbar, no weight decay (Kingma & Ba Alg. 1)      P:572, P:578     (R24)
// One HBM-streaming pass: 12 B per element (SGD: read x, gbar; write x) or
// 28 B (Adam: read x, gbar, m, v; write x, m, v).  Grid-stride over 16-byte
// quads with two quads in flight per thread, 148 x 8 CTAs of 256 threads (one
// full-occupancy wave), a scalar tail for d % 4.  Every operation explicitly
// rounded in the order the header states (R9).
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

#include "arc_device.cuh"
#include "arc_topk.h"

namespace arc {
namespace {

using dev::fadd;
using dev::ffma;
using dev::fmul;
using dev::fsub;

struct AdamCoef {
    float gamma, b1, b2, om1, om2, bc1, bc2, eps;
};

static __device__ __forceinline__ float sgd1(float x, float gb, float gamma) {
    return fsub(x, fmul(gamma, gb));
}

static __device__ __forceinline__ void adam1(float& x, float& m, float& v, float gb, const AdamCoef& c) {
    m = ffma(c.om1, gb, fmul(c.b1, m));
    v = ffma(c.om2, fmul(gb, gb), fmul(c.b2, v));
    const float mhat = __fdiv_rn(m, c.bc1);
    const float vhat = __fdiv_rn(v, c.bc2);
    x = fsub(x, fmul(c.gamma, __fdiv_rn(mhat, fadd(__fsqrt_rn(vhat), c.eps))));
}

constexpr int kThreads = 256;
constexpr int kGrid = 148 * 8;

__global__ void __launch_bounds__(kThreads) k_apply_sgd(float* __restrict__ x, const float* __restrict__ gbar,
                                                        long long d, float gamma) {
    const long long nq = d / 4;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    long long f = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    float4* x4 = reinterpret_cast<float4*>(x);
    const float4* g4 = reinterpret_cast<const float4*>(gbar);
    for (; f + stride < nq; f += 2 * stride) {
        const float4 xa = x4[f], xb = x4[f + stride];
        const float4 ga = __ldcs(g4 + f), gb = __ldcs(g4 + f + stride);
        x4[f] = make_float4(sgd1(xa.x, ga.x, gamma), sgd1(xa.y, ga.y, gamma), sgd1(xa.z, ga.z, gamma),
                            sgd1(xa.w, ga.w, gamma));
        x4[f + stride] = make_float4(sgd1(xb.x, gb.x, gamma), sgd1(xb.y, gb.y, gamma), sgd1(xb.z, gb.z, gamma),
                                     sgd1(xb.w, gb.w, gamma));
    }
    if (f < nq) {
        const float4 xa = x4[f];
        const float4 ga = __ldcs(g4 + f);
        x4[f] = make_float4(sgd1(xa.x, ga.x, gamma), sgd1(xa.y, ga.y, gamma), sgd1(xa.z, ga.z, gamma),
                            sgd1(xa.w, ga.w, gamma));
    }
    const long long e = 4 * nq + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e < d) x[e] = sgd1(x[e], gbar[e], gamma);
}

__global__ void __launch_bounds__(kThreads) k_apply_adam(float* __restrict__ x, float* __restrict__ m,
                                                         float* __restrict__ v, const float* __restrict__ gbar,
                                                         long long d, const AdamCoef c) {
    const long long nq = d / 4;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    long long f = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    float4* x4 = reinterpret_cast<float4*>(x);
    float4* m4 = reinterpret_cast<float4*>(m);
    float4* v4 = reinterpret_cast<float4*>(v);
    const float4* g4 = reinterpret_cast<const float4*>(gbar);
    auto quad = [&](float4 xq, float4 mq, float4 vq, const float4 gq, long long at) {
        adam1(xq.x, mq.x, vq.x, gq.x, c);
        adam1(xq.y, mq.y, vq.y, gq.y, c);
        adam1(xq.z, mq.z, vq.z, gq.z, c);
        adam1(xq.w, mq.w, vq.w, gq.w, c);
        x4[at] = xq;
        m4[at] = mq;
        v4[at] = vq;
    };
    for (; f + stride < nq; f += 2 * stride) {
        const float4 xa = x4[f], xb = x4[f + stride];
        const float4 ma = m4[f], mb = m4[f + stride];
        const float4 va = v4[f], vb = v4[f + stride];
        const float4 ga = __ldcs(g4 + f), gb = __ldcs(g4 + f + stride);
        quad(xa, ma, va, ga, f);
        quad(xb, mb, vb, gb, f + stride);
    }
    if (f < nq) quad(x4[f], m4[f], v4[f], __ldcs(g4 + f), f);
    const long long e = 4 * nq + static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e < d) {
        float xe = x[e], me = m[e], ve = v[e];
        adam1(xe, me, ve, gbar[e], c);
        x[e] = xe;
        m[e] = me;
        v[e] = ve;
    }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace
}  // namespace arc

extern "C" arc_status arc_topk_apply_update(const arc_opt_params* p, int64_t t, float* x, const float* gbar,
                                            float* m, float* v, int64_t d, void* stream) {
    using namespace arc;
    if (p == nullptr || d < 0 || !std::isfinite(p->gamma)) return ARC_ERR_INVALID_ARG;
    if (p->kind != ARC_OPT_SGD && p->kind != ARC_OPT_ADAM) return ARC_ERR_UNSUPPORTED;
    const bool adam = p->kind == ARC_OPT_ADAM;
    if (adam && (t < 1 || !(p->beta1 >= 0.0f && p->beta1 < 1.0f) || !(p->beta2 >= 0.0f && p->beta2 < 1.0f) ||
                 !(p->eps >= 0.0f) || !std::isfinite(p->eps)))
        return ARC_ERR_INVALID_ARG;
    if (d == 0) return ARC_OK;
    if (x == nullptr || gbar == nullptr || !aligned16(x) || !aligned16(gbar)) return ARC_ERR_INVALID_ARG;
    if (adam && (m == nullptr || v == nullptr || !aligned16(m) || !aligned16(v))) return ARC_ERR_INVALID_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // one full-occupancy wave, fewer CTAs when d is small
    const long long quads = d / 4 + 1;
    long long grid = (quads + kThreads - 1) / kThreads;
    if (grid > kGrid) grid = kGrid;
    if (!adam) {
        k_apply_sgd<<<static_cast<unsigned>(grid), kThreads, 0, s>>>(x, gbar, d, p->gamma);
    } else {
        AdamCoef c;
        c.gamma = p->gamma;
        c.b1 = p->beta1;
        c.b2 = p->beta2;
        c.om1 = 1.0f - p->beta1;   // host fp32, SSE, no contraction
        c.om2 = 1.0f - p->beta2;
        c.bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(p->beta1), static_cast<double>(t)));
        c.bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(p->beta2), static_cast<double>(t)));
        c.eps = p->eps;
        k_apply_adam<<<static_cast<unsigned>(grid), kThreads, 0, s>>>(x, m, v, gbar, d, c);
    }
    return cudaGetLastError() == cudaSuccess ? ARC_OK : ARC_ERR_CUDA;
}
