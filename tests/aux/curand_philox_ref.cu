// Test-only: cuRAND's own Philox4x32-10 (curand_philox4x32_x.h, host-capable
// through NV_IF_ELSE_TARGET) exported for the oracle's pin against a library
// routine.  Not part of the product.
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>

extern "C" void curand_ref_philox(const unsigned* ctr, const unsigned* key, unsigned* out, long long n) {
    for (long long i = 0; i < n; ++i) {
        uint4 c = make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]);
        uint2 k = make_uint2(key[2 * i], key[2 * i + 1]);
        const uint4 o = curand_Philox4x32_10(c, k);
        out[4 * i] = o.x; out[4 * i + 1] = o.y; out[4 * i + 2] = o.z; out[4 * i + 3] = o.w;
    }
}
