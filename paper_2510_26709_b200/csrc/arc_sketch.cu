// arc_sketch.cu — S1 (+S2 when every node is local): the fused streaming pass
// of the EF21M + ARC-Top-K step, the one kernel that moves ~98 % of the step's
// HBM bytes.
//
// Per element (eq:ef21m-1 P:325, R11, R4):   h' = ((1-eta) h) + (eta grad)
//                                             Delta = h' - g          (h' stored)
// Per row p and sketch column j (Alg.1 l.4, R2, R9):
//   P'_i[p][j] = (((0 + Delta_p0 V_0j) + Delta_p1 V_1j) + ...)   left to right
//   P_i = (1/sqrt r) P'_i ; (G == 1) S = P_0 + P_1 + ... ; P = S / N ;
//   Sigma_p = ((0 + P_p0^2) + P_p1^2) + ...                        (zn28373 P:236)
//
// Layout: a CTA walks a host-balanced list of tiles; a tile is <= R rows of
// one ARC block, consumed in chunks of W columns:
//   load  : all 256 threads stream grad, h, g of the R x W chunk (128-bit when
//           the block's rows are 16-byte aligned, else 32-bit), compute h' and
//           Delta, store h' and put Delta in shared memory;
//   chain : 4 lanes per row (lane jl owns j = jl + 4s) walk the chunk's W
//           columns in order — the plain sequential sum, one rounding per op.
// The next chunk's loads are issued before the current chunk's chains, and the
// Delta tile is double buffered, so each CTA keeps a chunk in flight while it
// computes.  Tile/block descriptors are read once per tile through the
// read-only path, never re-read per chunk.
#include <cuda_runtime.h>

#include <cstdint>

#include "arc_device.cuh"
#include "arc_internal.cuh"
#include "arc_rng.cuh"

namespace arc {
namespace {
using namespace dev;

constexpr int kThreads = kSketchThreads;   // 256

// Per-tile scalars kept in registers.
struct TileRegs {
    long long off, len;      // block
    int n, m_rows, row0;     // block row length; rows in this tile; first row
    int vec;                 // 16-byte aligned rows
    int nchunks;
    long long v_off;
    int row_base;
    int b;
    int node;
};

template <int W>
__device__ __forceinline__ TileRegs tile_regs(const TileDesc& T) {
    TileRegs t;
    t.b = T.b;
    t.off = T.off;
    t.len = T.len;
    t.n = T.n;
    t.vec = T.vec;
    t.v_off = T.v_off;
    t.row_base = T.row_base;
    t.row0 = T.row0;
    t.m_rows = T.rows;
    t.node = T.node;
    t.nchunks = (t.n + W - 1) / W;
    return t;
}

// the descriptor of tile li into shared memory, asynchronously (threads 0..3,
// one 16-byte word each; they wait for it before a later __syncthreads)
__device__ __forceinline__ void fetch_tile(const TileDesc* tiles, int li, TileDesc* dst) {
    if (threadIdx.x < 4) {
        const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(reinterpret_cast<char*>(dst) + 16 * threadIdx.x));
        const char* src = reinterpret_cast<const char*>(tiles + li) + 16 * threadIdx.x;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n\tcp.async.commit_group;" ::"r"(d), "l"(src) : "memory");
    }
}
template <int kPending>
__device__ __forceinline__ void fetch_wait() {
    if (threadIdx.x < 4) asm volatile("cp.async.wait_group %0;" ::"n"(kPending) : "memory");
}

// valid columns of tile row `row` (0 for rows beyond the tile): the last row of
// a padded flat block is short (R14)
__device__ __forceinline__ int row_cols(const TileRegs& t, int row) {
    if (row >= t.m_rows) return 0;
    const long long rest = t.len - static_cast<long long>(t.row0 + row) * t.n;
    return rest < t.n ? static_cast<int>(rest) : t.n;
}

template <int R, int W, int RPT, int NR>
__global__ void __launch_bounds__(kThreads, 4) k_ef_sketch(const SketchLaunch a) {
    static_assert(R * W == 2048 * NR, "one load round = 2048 elements = 8 per thread");
    static_assert(W % 32 == 0 && W <= 256, "W in {32, 64, 128, 256}");
    constexpr int RR = R / NR;                  // rows per load round
    constexpr int NB = NR == 1 ? 2 : 1;         // Delta / V buffers
    constexpr int NE = RR * W / kThreads;       // elements per thread per stream = 8
    constexpr int LPR = W / 4;                  // vec: threads per row segment (one float4 each)
    constexpr int DS = W + 4;                   // Delta row stride (floats): 16-byte rows,
                                                // rows t..t+7 on distinct banks
    constexpr int VS = 4 * RPT;                 // V row stride in smem (padded r)
    __shared__ __align__(16) float Ds[NB][R][DS];
    __shared__ __align__(16) float Vs[NB][W * VS];
    __shared__ unsigned hist[kHist1Bins];       // digit-1 histogram of this CTA's Sigma (mode 0)
    __shared__ TileDesc s_tile[3];              // tile descriptors, list position mod 3

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int crow = tid >> 2, jl = tid & 3;    // chain role (threads < 4R)
    const int list_begin = a.cta_begin[blockIdx.x], list_end = a.cta_begin[blockIdx.x + 1];
    if (list_begin >= list_end) return;
    const int r = a.r;
    for (int i = tid; i < kHist1Bins; i += kThreads) hist[i] = 0;
    for (int k = 0; k < 3 && list_begin + k < list_end; ++k) fetch_tile(a.tiles, list_begin + k, &s_tile[k]);
    fetch_wait<0>();
    __syncthreads();
    grid_dependency_wait();   // the previous kernel (g, V, histogram reset) is complete
    // (the first __syncthreads of the main loop orders this before any use)
    auto flush_hist = [&](int b) {               // all threads; after a __syncthreads
        unsigned* gh = a.hist1 + static_cast<long long>(b) * kHist1Bins;
        for (int i = tid; i < kHist1Bins; i += kThreads) {
            const unsigned v = hist[i];
            if (v) { atomicAdd(gh + i, v); hist[i] = 0; }
        }
    };

    // element e of this thread in a chunk -> (row, column within chunk)
    // (vec: float4 number q = tid + 256 (e / 4) of the chunk, row-major)
    auto vrow = [&](int e) { return (tid + kThreads * (e >> 2)) / LPR; };
    auto vcol = [&](int e) { return 4 * ((tid + kThreads * (e >> 2)) % LPR) + (e & 3); };
    auto srow = [&](int e) { return warp + 8 * (e / (W / 32)); };
    auto scol = [&](int e) { return lane + 32 * (e % (W / 32)); };

    float xg[NE], xh[NE], xd[NE];
    constexpr int NV = (W * VS + kThreads - 1) / kThreads;
    float xv[NV];                                // this thread's V entries of the chunk


    // A load round is NP parts of 4 elements per thread per stream; part 0 also
    // carries the thread's V entries of the chunk (round 0).  Staging part p of
    // the current round frees its registers, which immediately take part p of
    // the next round: one round stays in flight without a gap at the barrier.
    constexpr int NP = NE / 4;
    auto load_part = [&](const TileRegs& t, int chunk, int rnd, int part) {
        const float* __restrict__ pg = a.nodes.grad[t.node];
        const float* __restrict__ ph = a.nodes.h[t.node];
        const float* __restrict__ pgg = a.nodes.g[t.node];
        const int c0 = chunk * W;
        if (rnd == 0 && part == 0) {   // V rows [c0, c0 + W) of the block, r values each -> stride VS (zero padded)
            const float* __restrict__ Vb = a.V + t.v_off;
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                const int i = tid + k * kThreads, q = i / VS, j = i % VS;
                xv[k] = (i < W * VS && c0 + q < t.n && j < r) ? __ldg(Vb + static_cast<long long>(c0 + q) * r + j) : 0.0f;
            }
        }
        if (t.vec) {
            const int e4 = 4 * part;
            const int row = rnd * RR + vrow(e4), col = c0 + vcol(e4);
            const int nv = row_cols(t, row);
            const long long e = t.off + static_cast<long long>(t.row0 + row) * t.n + col;
            if (col + 3 < nv) {
                const float4 vg = __ldcs(reinterpret_cast<const float4*>(pg + e));
                const float4 vh = __ldcs(reinterpret_cast<const float4*>(ph + e));
                const float4 vd = __ldcs(reinterpret_cast<const float4*>(pgg + e));
                xg[e4] = vg.x; xg[e4 + 1] = vg.y; xg[e4 + 2] = vg.z; xg[e4 + 3] = vg.w;
                xh[e4] = vh.x; xh[e4 + 1] = vh.y; xh[e4 + 2] = vh.z; xh[e4 + 3] = vh.w;
                xd[e4] = vd.x; xd[e4 + 1] = vd.y; xd[e4 + 2] = vd.z; xd[e4 + 3] = vd.w;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (col + k < nv) {
                        xg[e4 + k] = __ldcs(pg + e + k);
                        xh[e4 + k] = __ldcs(ph + e + k);
                        xd[e4 + k] = __ldcs(pgg + e + k);
                    }
                }
            }
        } else {
#pragma unroll
            for (int e1 = 4 * part; e1 < 4 * part + 4; ++e1) {
                const int row = rnd * RR + srow(e1), col = c0 + scol(e1);
                const long long e = t.off + static_cast<long long>(t.row0 + row) * t.n + col;
                if (col < row_cols(t, row)) {
                    xg[e1] = __ldcs(pg + e);
                    xh[e1] = __ldcs(ph + e);
                    xd[e1] = __ldcs(pgg + e);
                }
            }
        }
    };

    auto stage_part = [&](const TileRegs& t, int chunk, int rnd, int part, int buf) {
        float* __restrict__ ph = a.nodes.h[t.node];
        const int c0 = chunk * W;
        if (t.vec) {
            const int e4 = 4 * part;
            const int row = rnd * RR + vrow(e4), cl = vcol(e4), col = c0 + cl;
            const int nv = row_cols(t, row);
            const long long e = t.off + static_cast<long long>(t.row0 + row) * t.n + col;
            float hn[4], dl[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                hn[k] = fadd(fmul(a.ome, xh[e4 + k]), fmul(a.eta, xg[e4 + k]));   // R11
                dl[k] = fsub(hn[k], xd[e4 + k]);                                   // R4
            }
            if (col + 3 < nv) {
                __stcs(reinterpret_cast<float4*>(ph + e), make_float4(hn[0], hn[1], hn[2], hn[3]));
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (col + k < nv) ph[e + k] = hn[k];
            }
            *reinterpret_cast<float4*>(&Ds[buf][row][cl]) = make_float4(dl[0], dl[1], dl[2], dl[3]);
        } else {
#pragma unroll
            for (int e1 = 4 * part; e1 < 4 * part + 4; ++e1) {
                const int row = rnd * RR + srow(e1), cl = scol(e1), col = c0 + cl;
                const long long e = t.off + static_cast<long long>(t.row0 + row) * t.n + col;
                const float hn = fadd(fmul(a.ome, xh[e1]), fmul(a.eta, xg[e1]));
                if (col < row_cols(t, row)) ph[e] = hn;
                Ds[buf][row][cl] = fsub(hn, xd[e1]);
            }
        }
        if (rnd == 0 && part == 0) {   // V, loaded with the chunk
#pragma unroll
            for (int k = 0; k < NV; ++k)
                if (tid + k * kThreads < W * VS) Vs[buf][tid + k * kThreads] = xv[k];
        }
    };

    float acc[RPT], S[RPT];
#pragma unroll
    for (int s = 0; s < RPT; ++s) { acc[s] = 0.0f; S[s] = 0.0f; }

    // the unit = one load round (tile li, chunk, round); cursor on the unit being
    // staged, its successor's loads issued part by part while it is staged
    int li = list_begin, chunk = 0, rnd = 0;
    TileRegs tc = tile_regs<W>(s_tile[0]); // tile of the unit being staged / chained
#pragma unroll
    for (int p = 0; p < NP; ++p) load_part(tc, 0, 0, p);
    int buf = 0;
    bool first = true;
    while (true) {
        int nli = li, nchunk = chunk, nrnd = rnd + 1;
        if (nrnd == NR || nrnd * RR >= tc.m_rows) {   // (rounds past the tile's rows are skipped)
            nrnd = 0;
            if (++nchunk == tc.nchunks) {
                nchunk = 0;
                ++nli;
            }
        }
        const bool more = nli < list_end;
        TileRegs tl = tc;                  // tile of the successor unit
        if (more && nli != li) {
            tl = tile_regs<W>(s_tile[(nli - list_begin) % 3]);
            if (nli + 2 < list_end) fetch_tile(a.tiles, nli + 2, &s_tile[(nli + 2 - list_begin) % 3]);
        }
        if (NB == 1 && rnd == 0 && !first) __syncthreads();   // the single Delta buffer is free again
        first = false;
        // Several rounds per chunk: the successor's loads go out part by part as
        // this round is staged.  One round per chunk: after the barrier, all at
        // once (measured faster for 32 x 64 on C3 / C4 / C5).
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            stage_part(tc, chunk, rnd, p, buf);
            if (NR > 1 && more) load_part(tl, nchunk, nrnd, p);
        }
        if (more && nrnd != 0) {           // the chunk has more rounds
            rnd = nrnd;
            continue;
        }
        fetch_wait<1>();                   // (descriptors go two tiles ahead: the latest may fly on)
        __syncthreads();
        if (NR == 1 && more) {
#pragma unroll
            for (int p = 0; p < NP; ++p) load_part(tl, nchunk, nrnd, p);
        }
        const int node = tc.node;

        // ------------------------------------------------------------ chains
        const bool live = crow < tc.m_rows;
        const int c0 = chunk * W;
        if (a.mode == 3) {
            // Rand-K: no sketch, the selection does not look at the data
        } else if (a.mode == 2) {
            // Top-K baseline: lane 0 of the row sums Delta_q^2 in column order
            if (crow < R && jl == 0) {
                const int qmax = live ? min(W, row_cols(tc, crow) - c0) : 0;
                const float* __restrict__ drow = &Ds[buf][crow][0];
                for (int q = 0; q < qmax; ++q) acc[0] = fadd(acc[0], fmul(drow[q], drow[q]));
            }
        } else if (crow < R) {
            const int qmax = live ? min(W, row_cols(tc, crow) - c0) : 0;
            const float* __restrict__ drow = &Ds[buf][crow][0];
            const float* __restrict__ vb = &Vs[buf][jl];
            if (qmax == W) {
#pragma unroll 16
                for (int q = 0; q < W; ++q) {
                    const float dq = drow[q];
#pragma unroll
                    for (int s = 0; s < RPT; ++s) acc[s] = fadd(acc[s], fmul(dq, vb[q * VS + 4 * s]));   // R9
                }
            } else {
                for (int q = 0; q < qmax; ++q) {
                    const float dq = drow[q];
#pragma unroll
                    for (int s = 0; s < RPT; ++s) acc[s] = fadd(acc[s], fmul(dq, vb[q * VS + 4 * s]));
                }
            }
        }

        // ------------------------------------------------ per-(tile, node) epilogue
        if (chunk == tc.nchunks - 1 && a.mode == 3) {
            // Rand-K: row p's shared key (R16), written once (node-0 tiles)
            const int p = tc.row0 + crow;
            if (jl == 0 && live && node == 0) {
                const uint4 x = rng::philox4x32_10(
                    make_uint4(static_cast<unsigned>(p), static_cast<unsigned>(tc.b) | 0x80000000u, a.t_lo, a.t_hi), a.key);
                const float sig = __uint_as_float(x.x >> 2);
                a.sigma[tc.row_base + p] = sig;
                atomicAdd(&hist[order_key_dev(sig) >> kHist1Shift], 1u);
            }
        } else if (chunk == tc.nchunks - 1 && a.mode == 2) {
            // Top-K baseline: this node's own ||row||^2 and its selection histogram
            const int p = tc.row0 + crow;
            if (jl == 0 && live) {
                const float sig = acc[0];
                a.sigma[static_cast<long long>(node) * a.M + tc.row_base + p] = sig;
                atomicAdd(&a.hist1[(static_cast<long long>(node) * a.num_blocks + tc.b) * kHist1Bins +
                                   (order_key_dev(sig) >> kHist1Shift)], 1u);
                if (!isfinite(sig)) atomicOr(a.status, kStatusNonfinite);
            }
#pragma unroll
            for (int s2 = 0; s2 < RPT; ++s2) acc[s2] = 0.0f;
        } else if (chunk == tc.nchunks - 1) {
            const int p = tc.row0 + crow;
#pragma unroll
            for (int s = 0; s < RPT; ++s) {
                const int j = jl + 4 * s;
                const float Pi = fmul(a.c_r, acc[s]);                                    // R2
                if (a.pnodes != nullptr && live && j < r)
                    a.pnodes[(static_cast<long long>(tc.row_base + p) * a.nodes_local + node) * r + j] = Pi;
                S[s] = Pi;        // mode 0 has one local node: S = P_0 (more nodes: ordered sum pass)
                acc[s] = 0.0f;
            }
            if (a.mode == 0) {
                float sig = 0.0f;
#pragma unroll
                for (int s = 0; s < RPT; ++s) {
                    const float pv = __fdiv_rn(S[s], a.Nf);                               // R3
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const float v = __shfl_sync(kFull, pv, (lane & ~3) | jj);
                        if (4 * s + jj < r) sig = fadd(sig, fmul(v, v));                 // zn28373
                    }
                }
                if (jl == 0 && live) {
                    a.sigma[tc.row_base + p] = sig;
                    atomicAdd(&hist[order_key_dev(sig) >> kHist1Shift], 1u);   // digit-1 histogram
                    if (!isfinite(sig)) atomicOr(a.status, kStatusNonfinite);
                }
            }
        }
        if (!more || tl.b != tc.b) {             // block boundary: publish the histogram
            __syncthreads();
            if (a.mode == 0 || a.mode == 3) flush_hist(tc.b);
            __syncthreads();
        }
        if (!more) break;
        if (nli != li) tc = tl;
        li = nli;
        chunk = nchunk;
        rnd = 0;
        buf ^= NB - 1;
    }
}

// RPT (sums per lane) = ceil(r / 4); the widest shape stops at r <= 16 (shared memory)
template <class K>
void launch_pdl(K kernel, const SketchLaunch& a, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(a.grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kernel, a);
}

template <int R, int W, int NR = 1>
void launch_rw(const SketchLaunch& a, cudaStream_t s) {
    if (a.r <= 4) launch_pdl(k_ef_sketch<R, W, 1, NR>, a, s);
    else if constexpr (W <= 128) {
        if (a.r <= 8) launch_pdl(k_ef_sketch<R, W, 2, NR>, a, s);
    }
    if constexpr (W <= 128 && NR == 1) {
        if (a.r > 8 && a.r <= 16) launch_pdl(k_ef_sketch<R, W, 4, NR>, a, s);
        else if constexpr (W < 128) { if (a.r > 16) launch_pdl(k_ef_sketch<R, W, 8, NR>, a, s); }
    }
}

template <int R, int W, int NR = 1>
int occupancy_rw(int r) {
    int per_sm = 0;
    if (r <= 4) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ef_sketch<R, W, 1, NR>, kThreads, 0);
    else if constexpr (W <= 128) {
        if (r <= 8) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ef_sketch<R, W, 2, NR>, kThreads, 0);
    }
    if constexpr (W <= 128 && NR == 1) {
        if (r > 8 && r <= 16) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ef_sketch<R, W, 4, NR>, kThreads, 0);
        else if constexpr (W < 128) { if (r > 16) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ef_sketch<R, W, 8, NR>, kThreads, 0); }
    }
    return per_sm;
}

}  // namespace

// tile shapes R x W (load rounds): 0 = 64 x 32, 1 = 32 x 64, 2 = 16 x 128 (r <= 16),
// 3 = 32 x 256 in 4 rounds of 8 rows (r <= 4), 4 = 32 x 128 in 2 rounds of 16 rows (r <= 8)
int sketch_tile_rows(int shape) { return shape == 0 ? 64 : shape == 2 ? 16 : 32; }
int sketch_tile_cols(int shape) { return shape == 0 ? 32 : shape == 1 ? 64 : shape == 3 ? 256 : 128; }
int sketch_shape_ok(int shape, int r) {
    return shape <= 1 || (shape == 2 && r <= 16) || (shape == 3 && r <= 4) || (shape == 4 && r <= 8);
}

void launch_ef_sketch(const SketchLaunch& a, cudaStream_t s) {
    switch (a.shape) {
        case 0: launch_rw<64, 32>(a, s); break;
        case 1: launch_rw<32, 64>(a, s); break;
        case 2: launch_rw<16, 128>(a, s); break;
        case 3: launch_rw<32, 256, 4>(a, s); break;
        default: launch_rw<32, 128, 2>(a, s); break;
    }
}

int ef_sketch_resident_ctas(int r, int shape) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = shape == 0 ? occupancy_rw<64, 32>(r)
                 : shape == 1 ? occupancy_rw<32, 64>(r)
                 : shape == 2 ? occupancy_rw<16, 128>(r)
                 : shape == 3 ? occupancy_rw<32, 256, 4>(r)
                              : occupancy_rw<32, 128, 2>(r);
    if (per_sm < 1) per_sm = 1;
    return sms * per_sm;
}

}  // namespace arc
