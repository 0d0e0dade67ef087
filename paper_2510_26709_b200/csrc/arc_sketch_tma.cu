// arc_sketch_tma.cu — S1 (+S2 with one node per GPU) for the blocks the main
// streaming launch handles worst: rows that are not 16-byte aligned (n % 4 != 0,
// e.g. the LLaMA down projections, n = 5461), which the register path reads with
// scalar loads (4x the L1 sectors and load instructions).  Same arithmetic and the same O6 order as
// k_ef_sketch (arc_sketch.cu; eq:ef21m-1 P:325, Alg.1 l.4, R2, R9,
// R11, R4); only the way the data reaches the lanes differs.
//
// Feed (warp-specialised).  Consumer warp c streams its own rows (rows c, c + NW,
// ... of the CTA's tiles) out of a private ring of D stages in shared memory; a
// stage holds one batch (UN row segments = 128 UN columns) of grad, h and g,
// brought in by three 1-D bulk copies (cp.async.bulk, the TMA unit) of the
// 16-byte-aligned superset window of the batch.  One producer warp issues every
// copy of the CTA: its lane c walks consumer c's batches in the same order and
// refills a stage as soon as the consumer releases it (full / empty mbarriers
// per stage, expect_tx byte counts).  The misaligned row start costs nothing:
// the batch's column c sits at shared index c + a (a = row start mod 4).
//
// Lanes.  Lane l owns columns 128s + 4l + e of each segment (the O6 lane map).
// Reading them as 4 scalar words would hit each bank 4 times (lanes l, l + 8,
// l + 16, l + 24 share banks); lane group G = l / 8 reads its 4 words rotated by
// G (word (e + G) mod 4 in read e), which is conflict-free, computes h' and Delta
// elementwise in that order, and un-rotates Delta (two conditional register
// rotations) before the O6 fma chain against V_b^T (staged whole per block).
//
// Store.  h' goes into a per-warp output buffer at its window index (two batch
// halves, so the words past a window — the next window's head — land where the
// next batch stores them); the aligned interior leaves as 16-byte stores, the
// quads shared with the neighbour rows word by word.  Nothing written by the
// threads is read by the copy engine, so no proxy fence is needed.
//
// Geometry (measured on B200, profiles/r02_sketch_tma.txt): the per-batch cost
// (barrier round trips, the producer's three copies) dominates, so batches are
// 512 columns (UN = 4) with D = 2 stages for 8 consumer warps; deeper rings
// with smaller batches, more warps or one producer lane per consumer warp's own
// lane 0 all measured slower.
//
// Reads past the end.  The last window of a row may extend up to 12 bytes past
// the last element of the vector when d % 4 != 0; it never leaves the 16-byte
// granule that holds that element (the vectors' bases are 16-byte aligned,
// checked by arc_topk_step), hence never the page.  Those bytes are loaded into
// shared memory and never used.
#include <cuda_runtime.h>

#include <cstdint>

#include "arc_device.cuh"
#include "arc_internal.cuh"

namespace arc {
namespace {
using namespace dev;

constexpr int kTmaTileCache = 32;     // tile descriptors cached in shared memory
constexpr int kTmaSmemMax = 232448;   // opt-in shared memory per CTA (227 KB)

#ifndef ARC_TMA_BACKOFF_NS
#define ARC_TMA_BACKOFF_NS 100
#endif

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, unsigned parity) {   // non-blocking
    unsigned ok;
    asm volatile(
        "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    while (!mbar_try(b, parity)) {
    }
}
// global -> shared, completing on an mbarrier; an L2 eviction hint per array
__device__ __forceinline__ void bulk_load(float* dst, const float* src, unsigned bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ float butterfly(float a) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) a = fadd(a, __shfl_xor_sync(kFull, a, o));
    return a;
}
__device__ __forceinline__ int row_cols(long long len, int n, int p) {
    const long long rest = len - static_cast<long long>(p) * n;
    return rest < n ? static_cast<int>(rest) : n;
}

// the warp's position in its stream of batches: tile li, its row rr of that tile, segment k0
struct BatchIt {
    int li, rr, k0;
};

template <int RJ, int UN, int D, int NW>
__global__ void __launch_bounds__((NW + 1) * 32, 1) k_ef_sketch_tma(const SketchLaunch a) {
    static_assert(D >= 2 && NW <= 32, "at least two stages; one producer lane per consumer warp");
    constexpr int NT = NW * 32;      // consumer threads (warp NW is the producer)
    constexpr int BF = 128 * UN;     // columns per batch
    constexpr int SLOT = BF + 4;     // floats per array per stage (the window starts up to 3 floats early)
    constexpr int STAGE = 3 * SLOT;  // grad | h | g
    __shared__ TileDesc s_tile[kTmaTileCache];
    __shared__ unsigned s_hist[kHist1Bins];
    __shared__ __align__(8) uint64_t s_full[NW][D];    // stage loaded (producer's expect_tx + the copies)
    __shared__ __align__(8) uint64_t s_empty[NW][D];   // stage consumed (consumer lane 0)
    extern __shared__ __align__(16) float4 dyn[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float* const ring_base = reinterpret_cast<float*>(dyn);
    float* const ring = ring_base + warp * (D * STAGE);                       // (consumer warps)
    float* const obuf = ring_base + NW * D * STAGE + warp * (2 * BF + 4);    // h' of two batches (+ a carry)
    float* const Vs = ring_base + NW * (D * STAGE + 2 * BF + 4);

    const int grp = (lane >> 3) & 3;   // read rotation of this lane's words
    const int rot[4] = {grp, (grp + 1) & 3, (grp + 2) & 3, (grp + 3) & 3};
    const int list_begin = a.cta_begin[blockIdx.x], list_end = a.cta_begin[blockIdx.x + 1];
    if (list_begin >= list_end) return;
    const int ntile = list_end - list_begin;
    for (int i = tid; i < min(ntile, kTmaTileCache) * 4; i += NT + 32)
        reinterpret_cast<uint4*>(s_tile)[i] = __ldg(reinterpret_cast<const uint4*>(a.tiles + list_begin) + i);
    for (int i = tid; i < kHist1Bins; i += NT + 32) s_hist[i] = 0;
    if (warp == NW && lane < NW)
        for (int s = 0; s < D; ++s) {
            mbar_init(&s_full[lane][s], 1);
            mbar_init(&s_empty[lane][s], 1);
        }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    grid_dependency_wait();   // the previous kernel (g, V, histogram reset) is complete

    auto tile = [&](int li) -> const TileDesc* {
        return li - list_begin < kTmaTileCache ? &s_tile[li - list_begin] : a.tiles + li;
    };
    // skip tiles in which a warp has no rows left (rows are dealt round-robin across tiles)
    auto settle = [&](BatchIt& x) {
        while (x.li < list_end) {
            const int rows = tile(x.li)->rows;
            if (x.rr < rows) break;
            x.rr -= rows;
            ++x.li;
        }
    };

    if (warp == NW) {
        // ---- producer: lane c keeps consumer warp c's ring full, in that warp's batch order
        const uint64_t pol_once = policy_evict_first();    // grad: read once
        const uint64_t pol_state = policy_evict_normal();  // h, g (may stay in L2 between steps)
        BatchIt it{list_begin, lane, 0};
        bool done = lane >= NW;
        if (!done) {
            settle(it);
            done = it.li >= list_end;
        }
        // the producer's copy of the current row (recomputed when the row changes)
        long long row_start = 0;
        int row_nv = 0, row_node = 0, cached_li = -1, cached_rr = -1;
        int issued = 0;
        while (__any_sync(kFull, !done)) {
            const int s = issued % D;
            const bool go = !done && (issued < D || mbar_test(&s_empty[lane][s], static_cast<unsigned>(issued / D - 1) & 1u));
            if (!__any_sync(kFull, go)) {   // every ring is full: back off instead of spinning on issue slots
                __nanosleep(ARC_TMA_BACKOFF_NS);
                continue;
            }
            if (!go) continue;
            if (it.li != cached_li || it.rr != cached_rr) {
                const TileDesc* T = tile(it.li);
                const int p = T->row0 + it.rr;
                row_nv = row_cols(T->len, T->n, p);
                row_start = T->off + static_cast<long long>(p) * T->n;
                row_node = T->node;
                cached_li = it.li;
                cached_rr = it.rr;
            }
            const long long start = row_start + 128 * it.k0;
            const int nb = min(BF, row_nv - 128 * it.k0);
            const int al = static_cast<int>(start & 3);
            const long long W0 = start - al;
            const unsigned bytes = static_cast<unsigned>(((al + nb + 3) & ~3) * 4);
            float* st = ring_base + (lane * D + s) * STAGE;
            uint64_t* bar = &s_full[lane][s];
            mbar_expect_tx(bar, 3 * bytes);
            bulk_load(st, a.nodes.grad[row_node] + W0, bytes, bar, pol_once);
            bulk_load(st + SLOT, a.nodes.h[row_node] + W0, bytes, bar, pol_state);
            bulk_load(st + 2 * SLOT, a.nodes.g[row_node] + W0, bytes, bar, pol_state);
            ++issued;
            it.k0 += UN;
            if (128 * it.k0 >= row_nv) {
                it.k0 = 0;
                it.rr += NW;
                settle(it);
                done = it.li >= list_end;
            }
        }
        return;
    }

    // ---- consumers
    const int r = a.r;
    const float eta = a.eta, ome = a.ome;
    auto consumers_sync = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory"); };
    int kk = 0;   // batches consumed (batch kk lives in stage kk % D)

    int carry = warp;   // this warp's first row of the next tile
    int cur_b = -1;
    for (int li = list_begin; li < list_end; ++li) {
        const TileDesc* Tp = tile(li);
        const long long T_off = Tp->off, T_len = Tp->len, T_voff = Tp->v_off;
        const int T_n = Tp->n, T_row0 = Tp->row0, T_rows = Tp->rows, T_row_base = Tp->row_base, T_b = Tp->b;
        const int node = Tp->node;
        const int ldv = (T_n + 3) & ~3;
        if (T_b != cur_b) {
            consumers_sync();
            if (cur_b >= 0) {
                unsigned* gh = a.hist1 + static_cast<long long>(cur_b) * kHist1Bins;
                for (int i = tid; i < kHist1Bins; i += NT) {
                    const unsigned v = s_hist[i];
                    if (v) { atomicAdd(gh + i, v); s_hist[i] = 0; }
                }
            }
            const int nvf4 = (r * ldv) >> 2;
            for (int i = tid; i < nvf4; i += NT)
                reinterpret_cast<float4*>(Vs)[i] = __ldg(reinterpret_cast<const float4*>(a.V + T_voff) + i);
            consumers_sync();
        }
        cur_b = T_b;
        float* __restrict__ ph = a.nodes.h[node];

        int rr = carry;
        for (; rr < T_rows; rr += NW) {
            const int p = T_row0 + rr;
            const int nv = row_cols(T_len, T_n, p);
            const long long base = T_off + static_cast<long long>(p) * T_n;
            const int al = static_cast<int>(base & 3);
            const int nseg = (nv + 127) >> 7;
            float acc[RJ], P[RJ];
#pragma unroll
            for (int j = 0; j < RJ; ++j) { acc[j] = 0.0f; P[j] = 0.0f; }
            for (int k0 = 0; k0 < nseg; k0 += UN) {
                const int s = kk % D;
                mbar_wait(&s_full[warp][s], static_cast<unsigned>(kk / D) & 1u);
                const float* const sg = ring + s * STAGE;   // grad | h | g of the batch window
                float* const ob = obuf + (kk & 1) * BF;     // h' of the window (index as in the stage)
                const bool first = k0 == 0, last = k0 + UN >= nseg;
                const bool full = 128 * (k0 + UN) <= nv;    // every column of every segment valid
                const int nb = min(BF, nv - 128 * k0);
                // (1) every word of the batch from the stage (rotated reads), all in flight
                // together; word e of lane l at index 128u + 4l + al + ((e + grp) mod 4)
                const int wofs = 4 * lane + al;
                float xg[UN][4], xh[UN][4], xd[UN][4];
#pragma unroll
                for (int u = 0; u < UN; ++u)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float* w = sg + wofs + rot[e] + 128 * u;   // (in the slot even past the row end)
                        xg[u][e] = w[0];
                        xh[u][e] = w[SLOT];
                        xd[u][e] = w[2 * SLOT];
                    }
                // (2) h' and Delta elementwise (rotated word order); h' into the output buffer
                // at its window index (a word past the window, i >= BF, is the next window's head)
#pragma unroll
                for (int u = 0; u < UN; ++u)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float hn = ffma(eta, xg[u][e], fmul(ome, xh[u][e]));   // O2, R11
                        xd[u][e] = fsub(hn, xd[u][e]);                               // Delta (O3, R4)
                        if (full || 128 * (k0 + u) + 4 * lane + rot[e] < nv) ob[wofs + rot[e] + 128 * u] = hn;
                    }
                // every lane has consumed its words of the stage: hand it back to the producer
                __syncwarp();
                if (lane == 0) mbar_arrive(&s_empty[warp][s]);
                // (3) h' to global memory: window indices [first ? al : 0, last ? nb + al : BF),
                // the aligned interior [lo, hi) as 16-byte stores, the rest (quads shared with
                // the neighbour rows) word by word
                {
                    const int lo = (first && al) ? 4 : 0;
                    const int hi = last ? ((nb + al) & ~3) : BF;
                    const int w_end = last ? nb + al : BF;
                    float* const gdst = ph + (base + 128 * k0 - al);
                    for (int j = lo + 4 * lane; j < hi; j += 128)
                        __stcs(reinterpret_cast<float4*>(gdst + j), *reinterpret_cast<const float4*>(ob + j));
                    if (first && al && al + lane < min(lo, w_end)) __stcs(gdst + al + lane, ob[al + lane]);
                    for (int j = max(hi, lo) + lane; j < w_end; j += 32) __stcs(gdst + j, ob[j]);
                }
                __syncwarp();
                if ((kk & 1) && al && !last && lane < al) obuf[lane] = obuf[2 * BF + lane];   // head of the next window
                // (4) the O6 chains: Delta un-rotated (xd[u][e] held word (e + grp) mod 4)
#pragma unroll
                for (int u = 0; u < UN; ++u) {
                    const int k = k0 + u;
                    if (k >= nseg) break;
                    const int q = 128 * k + 4 * lane;
                    float dl[4] = {xd[u][0], xd[u][1], xd[u][2], xd[u][3]};
                    if (grp & 1) {
                        const float t = dl[3];
                        dl[3] = dl[2]; dl[2] = dl[1]; dl[1] = dl[0]; dl[0] = t;
                    }
                    if (grp & 2) {
                        float t = dl[0]; dl[0] = dl[2]; dl[2] = t;
                        t = dl[1]; dl[1] = dl[3]; dl[3] = t;
                    }
                    if (r == RJ && 128 * (k + 1) <= nv) {   // a full segment, every sketch column
                        float4 v4[RJ];
#pragma unroll
                        for (int j = 0; j < RJ; ++j) v4[j] = *reinterpret_cast<const float4*>(Vs + j * ldv + q);
#pragma unroll
                        for (int j = 0; j < RJ; ++j) {
                            acc[j] = ffma(dl[0], v4[j].x, acc[j]);   // O6
                            acc[j] = ffma(dl[1], v4[j].y, acc[j]);
                            acc[j] = ffma(dl[2], v4[j].z, acc[j]);
                            acc[j] = ffma(dl[3], v4[j].w, acc[j]);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < RJ; ++j) {
                            if (j >= r) break;
                            // (a lane past the row end reads nothing: V_b^T has ldv >= q + 4 columns only for q < nv)
                            const float4 v4 = q < nv ? *reinterpret_cast<const float4*>(Vs + j * ldv + q)
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
                            const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e)
                                if (q + e < nv) acc[j] = ffma(dl[e], v[e], acc[j]);   // O6 (padding never summed)
                        }
                    }
                    if ((k & 7) == 7 || k == nseg - 1) {   // end of a 1024-column chunk
#pragma unroll
                        for (int j = 0; j < RJ; ++j) {
                            const float w = butterfly(acc[j]);
                            P[j] = (k < 8) ? w : fadd(P[j], w);
                            acc[j] = 0.0f;
                        }
                    }
                }
                ++kk;
            }
            // row epilogue (P[j] is the same in every lane)
            if (a.pnodes != nullptr && lane < r) {
                float v = P[0];
#pragma unroll
                for (int j = 1; j < RJ; ++j)
                    if (lane == j) v = P[j];
                a.pnodes[(static_cast<long long>(T_row_base + p) * a.nodes_local + node) * r + lane] = v;
            }
            if (a.mode == 0 && lane == 0) {   // S = P'_0: Sigma (O8) and its digit-1 histogram
                float sig = 0.0f;
#pragma unroll
                for (int j = 0; j < RJ; ++j)
                    if (j < r) sig = ffma(P[j], P[j], sig);
                a.sigma[T_row_base + p] = sig;
                atomicAdd(&s_hist[order_key_dev(sig) >> kHist1Shift], 1u);
                if (!isfinite(sig)) atomicOr(a.status, kStatusNonfinite);
            }
        }
        carry = rr - T_rows;
    }
    consumers_sync();
    if (cur_b >= 0) {
        unsigned* gh = a.hist1 + static_cast<long long>(cur_b) * kHist1Bins;
        for (int i = tid; i < kHist1Bins; i += NT) {
            const unsigned v = s_hist[i];
            if (v) atomicAdd(gh + i, v);
        }
    }
}

// ring geometry (UN segments per batch, D stages, NW consumer warps; build-time knobs for A/B runs)
#ifndef ARC_TMA_UN
#define ARC_TMA_UN 4
#endif
#ifndef ARC_TMA_D
#define ARC_TMA_D 2
#endif
#ifndef ARC_TMA_NW
#define ARC_TMA_NW 8
#endif
constexpr int kUN = ARC_TMA_UN, kD = ARC_TMA_D, kNW = ARC_TMA_NW;
constexpr int ring_bytes() { return kNW * (kD * 3 * (128 * kUN + 4) + 2 * 128 * kUN + 4) * static_cast<int>(sizeof(float)); }

template <int RJ>
int tma_static_smem() {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_ef_sketch_tma<RJ, kUN, kD, kNW>);
    return static_cast<int>(fa.sharedSizeBytes);
}
int static_smem(int r) {
    return r <= 4 ? tma_static_smem<4>() : r <= 8 ? tma_static_smem<8>() : r <= 16 ? tma_static_smem<16>() : tma_static_smem<32>();
}

template <int RJ>
void launch_tma_rj(const SketchLaunch& a, cudaStream_t s) {
    const int dyn = ring_bytes() + static_cast<int>(sizeof(float)) * a.vs_cap;
    static int attr_set = 0;
    if (attr_set < dyn) {
        cudaFuncSetAttribute(k_ef_sketch_tma<RJ, kUN, kD, kNW>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        attr_set = dyn;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(a.grid);
    cfg.blockDim = dim3((kNW + 1) * 32);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_ef_sketch_tma<RJ, kUN, kD, kNW>, a);
}

}  // namespace

// floats of V_b^T the TMA launch can stage next to its rings (0: none)
int sketch_tma_vs_cap(int r) {
    const int free_bytes = kTmaSmemMax - static_smem(r) - ring_bytes();
    return free_bytes > 0 ? (free_bytes / 4) & ~3 : 0;
}

int sketch_tma_threads() { return (kNW + 1) * 32; }

void launch_ef_sketch_tma(const SketchLaunch& a, cudaStream_t s) {
    if (a.r <= 4) launch_tma_rj<4>(a, s);
    else if (a.r <= 8) launch_tma_rj<8>(a, s);
    else if (a.r <= 16) launch_tma_rj<16>(a, s);
    else launch_tma_rj<32>(a, s);
}

}  // namespace arc
