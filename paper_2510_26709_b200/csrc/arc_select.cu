// arc_select.cu — S3 (+S4, and S5/S6 when every node is local) in ONE
// cooperative kernel: the shared Top-K selection and the compaction / EF update
// of the selected rows.
//
// S3  I_b = argtop_{K_b}(Sigma_b)  (zn28373 P:236-237; ties -> smaller row,
//     R5; NaN above +Inf, R15): an MSB-first radix select on the 32-bit order
//     keys, digits key[31:21] | key[20:10] | key[9:0].  A slice is <= 4096
//     consecutive rows of one block; the kernel is persistent (CTA b takes slices
//     b, b + grid, ...), and a CTA with one slice keeps its keys in shared memory.
//     Digit 1 was histogrammed by the pass that produced Sigma (phase 0 here
//     when Sigma came from the exchange or several local nodes), so each slice
//     knows the boundary bin b1 at once: it counts its keys above b1 and appends
//     its keys in b1 (the candidates) to a per-block list.  After ONE grid
//     barrier every CTA resolves the K-th key T and the tie cutoff P_eq from the
//     candidate list in shared memory (digit 2, then a rank count); a block
//     whose boundary bin overflows the list takes the digit-by-digit path
//     (digits 2 and 3 through global histograms, two more barriers).  Nothing
//     is serial in the number of tied keys.
// S4  each slice writes its selected rows in ascending order at its prefix
//     offset and applies, for every selected row k (row p) and node i,
//       C_i = h_i - g_i ; g_i <- g_i + C_i                      eq:ef21m-2 (R12)
//     and, when every node is on this GPU (mode 0),
//       A = C_0 + C_1 + ... ; val = A / N ; gbar <- gbar + val  P:242, R3, R13
//     or writes the exchange payload (modes 1, 2; mode 3: the Top-K baseline).
//     Early mode (mode 0, no values requested): the rows above b1 are updated
//     between the arrive and the wait of barrier 1, the selected boundary rows
//     after the resolution — no second barrier.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "arc_device.cuh"
#include "arc_internal.cuh"
#include "arc_rng.cuh"
#include "arc_select_common.cuh"

namespace cg = cooperative_groups;

namespace arc {
namespace {
using namespace dev;
using selc::cta_exclusive_scan;
using selc::top_digit;

constexpr int kThreads = 256;

__device__ __forceinline__ unsigned order_key(float s) { return order_key_dev(s); }

// load a block's global histogram into shared memory
__device__ __forceinline__ void load_hist(unsigned* h, const unsigned* g, int nbins) {
    unsigned v[8];   // nbins / kThreads <= 8 loads in flight per thread
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int i = threadIdx.x + k * kThreads;
        v[k] = i < nbins ? __ldcg(g + i) : 0u;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int i = threadIdx.x + k * kThreads;
        if (i < nbins) h[i] = v[k];
    }
    __syncthreads();
}
// add this CTA's nonzero bins to the block's global histogram, then clear
__device__ __forceinline__ void flush_hist(unsigned* h, unsigned* g, int nbins) {
    __syncthreads();
    for (int i = threadIdx.x; i < nbins; i += kThreads) {
        const unsigned v = h[i];
        if (v) atomicAdd(g + i, v);
    }
}

// ---- compaction / EF update of one selected row --------------------------------
struct Quad {
    float v[4];
};
__device__ __forceinline__ Quad load_quad(const float* p, bool vec4, int nvalid) {
    Quad x;
    if (vec4) {
        const float4 t = *reinterpret_cast<const float4*>(p);
        x.v[0] = t.x; x.v[1] = t.y; x.v[2] = t.z; x.v[3] = t.w;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) x.v[k] = k < nvalid ? p[k] : 0.0f;
    }
    return x;
}
// Two-step loads for the segment gather's batch of quads: issue_quad issues the
// 16-byte load unconditionally (from a zero quad when the quad is not 16-byte
// loadable), so the batch's loads are all in flight before the first result is
// used; patch_quad then fills the quads that are not (unaligned rows, the short
// last row) with scalar loads.  (With the load inside a vector/scalar branch the
// compiler merged each result right after its LDG, serialising the batch: ncu
// source page; C5 d = 1e9 at 10 %: 772 -> 564 us.  The early-gather path keeps
// load_quad: this form measured no faster there and slower on unaligned rows.)
__device__ const float4 k_zero_quad = {0.f, 0.f, 0.f, 0.f};
__device__ __forceinline__ Quad issue_quad(const float* p, bool vec4) {
    const float4 t = *(vec4 ? reinterpret_cast<const float4*>(p) : &k_zero_quad);
    Quad x;
    x.v[0] = t.x; x.v[1] = t.y; x.v[2] = t.z; x.v[3] = t.w;
    return x;
}
__device__ __forceinline__ void patch_quad(Quad& x, const float* p, bool vec4, int nvalid) {
    if (!vec4)
#pragma unroll
        for (int k = 0; k < 4; ++k) x.v[k] = k < nvalid ? p[k] : 0.0f;
}
__device__ __forceinline__ void store_quad(float* p, const Quad& x, bool vec4, int nvalid) {
    if (vec4) {
        *reinterpret_cast<float4*>(p) = make_float4(x.v[0], x.v[1], x.v[2], x.v[3]);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < nvalid) p[k] = x.v[k];
    }
}

__device__ __forceinline__ int row_valid_cols(const BlockDev& B, int p) {
    const long long rest = B.len - static_cast<long long>(p) * B.n;
    return rest < B.n ? static_cast<int>(rest) : B.n;
}

// Balanced S4 (+S5, S6): the selected rows of every block cut into segments of
// kSegQuads quads (host table), CTA b processes segments [seg0, seg1); every
// (segment, quad) pair is one item, kThreads * UN items in flight per pass.
// The segments' descriptors and selected rows are staged in shared memory first
// (`cap` at a time: one round of independent loads), so an item's data loads do
// not wait on a chain of descriptor -> block -> selection loads (that chain cost
// the unstaged version ~2.5 x its bandwidth at K n = 1e8, C5 d = 1e9, 10 %).
// A / N: for N a power of two the product with the exact reciprocal is the
// same correctly rounded value as the quotient (R3), and much cheaper.
__device__ __forceinline__ float div_N(float A, float Nf, float invN, bool pow2) {
    return pow2 ? fmul(A, invN) : __fdiv_rn(A, Nf);
}

template <int UN>
__device__ void gather_segments(const GatherLaunch& a, int seg_begin, int seg_end, int4* stage, int cap) {
    const bool pow2 = (a.N_int & (a.N_int - 1)) == 0;
    const float invN = 1.0f / a.Nf;
    for (int seg0 = seg_begin; seg0 < seg_end; seg0 += cap) {
    const int seg1 = min(seg_end, seg0 + cap);
    __syncthreads();                                 // (the previous round's stage is consumed)
    for (int sg = seg0 + static_cast<int>(threadIdx.x); sg < seg1; sg += kThreads) {
        const SelRow R = a.rows[sg];
        stage[sg - seg0] = make_int4(R.b, R.k, R.q0, __ldcg(a.sel + a.blocks[R.b].sel_base + R.k));
    }
    __syncthreads();
    const int items = (seg1 - seg0) * kSegQuads;
    for (int base = 0; base < items; base += kThreads * UN) {
        int cnt[UN], ocnt[UN], nd[UN];
        long long e[UN], o[UN];
        bool v4[UN], ov4[UN], dense[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) {
            const int item = base + u * kThreads + static_cast<int>(threadIdx.x);
            cnt[u] = ocnt[u] = 0;
            nd[u] = -1;
            e[u] = o[u] = 0;
            v4[u] = ov4[u] = dense[u] = false;
            if (item < items) {
                const int4 R = stage[item / kSegQuads];      // (block, k, q0, selected row)
                const BlockDev& B = a.blocks[R.x];
                const int f = R.z + item % kSegQuads;
                const int q = 4 * f;
                if (q < B.n) {
                    const int p = R.w;
                    const int nv = row_valid_cols(B, p);
                    cnt[u] = max(0, min(4, nv - q));
                    ocnt[u] = min(4, B.n - q);
                    e[u] = B.off + static_cast<long long>(p) * B.n + q;
                    o[u] = B.val_base + static_cast<long long>(R.y) * B.n + q;
                    v4[u] = B.vec && cnt[u] == 4;
                    ov4[u] = B.vec && (o[u] % 4 == 0) && ocnt[u] == 4;
                    dense[u] = B.kind == ARC_BLOCK_DENSE;
                    nd[u] = B.node;
                }
            }
        }
        Quad A[UN], gb[UN];
        // Top-K baseline (mode 3): a selection block belongs to one node (nd)
        const bool per_node = a.mode == 3;
        for (int i = 0; i < a.nodes_local; ++i) {
            // (without EF the compressed rows are the gradient's: C_i = grad_i, no g)
            float* __restrict__ ph = a.noef ? const_cast<float*>(a.nodes.grad[i]) : a.nodes.h[i];
            float* __restrict__ pg = a.nodes.g[i];
            Quad hq[UN], gq[UN];
            bool act[UN];
#pragma unroll
            for (int u = 0; u < UN; ++u) {   // issue every load of the batch ...
                act[u] = cnt[u] > 0 && (!per_node || nd[u] == i);
                const bool gbl = i == 0 && a.mode == 0 && cnt[u] > 0;
                if (i == 0) gb[u] = issue_quad(a.gbar + e[u], v4[u] && gbl);
                gq[u] = issue_quad(pg + e[u], v4[u] && act[u] && !a.noef);
                hq[u] = issue_quad(ph + e[u], v4[u] && act[u]);
            }
#pragma unroll
            for (int u = 0; u < UN; ++u) {   // ... then the scalar quads and DENSE rows
                if (i == 0 && a.mode == 0 && cnt[u] > 0) patch_quad(gb[u], a.gbar + e[u], v4[u], cnt[u]);
                if (!act[u]) continue;
                if (!a.noef) patch_quad(gq[u], pg + e[u], v4[u], cnt[u]);
                patch_quad(hq[u], ph + e[u], v4[u], cnt[u]);
                if (dense[u]) {   // DENSE block: eq:ef21m-1 here (R11, R20); hq held h
                    Quad gr = issue_quad(a.nodes.grad[i] + e[u], v4[u]);
                    patch_quad(gr, a.nodes.grad[i] + e[u], v4[u], cnt[u]);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) hq[u].v[kk] = ffma(a.eta, gr.v[kk], fmul(a.ome, hq[u].v[kk]));   // O2
                    store_quad(ph + e[u], hq[u], v4[u], cnt[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < UN; ++u) {
                if (ocnt[u] <= 0 || (per_node && nd[u] != i)) continue;
                Quad c, gn;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    c.v[kk] = kk < cnt[u] ? wire_round(a.noef ? hq[u].v[kk] : fsub(hq[u].v[kk], gq[u].v[kk]), a.bf16)
                                          : 0.0f;   // C_i, what node i sends (R25; +0 padding)
                    gn.v[kk] = a.noef ? 0.0f : fadd(gq[u].v[kk], c.v[kk]);                             // R12
                    A[u].v[kk] = (i == 0 || per_node) ? c.v[kk] : fadd(A[u].v[kk], c.v[kk]);   // R9 node order
                }
                if (cnt[u] > 0 && !a.noef) store_quad(pg + e[u], gn, v4[u], cnt[u]);
                if (a.mode == 2) {
                    if (a.bf16) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            if (kk < ocnt[u]) pay_st(a.values, static_cast<long long>(i) * a.sum_Kn + o[u] + kk, c.v[kk], 1);
                    } else {
                        store_quad(a.values + static_cast<long long>(i) * a.sum_Kn + o[u], c,
                                   ov4[u] && (a.sum_Kn % 4 == 0), ocnt[u]);
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < UN; ++u) {
            if (ocnt[u] <= 0) continue;
            if (a.mode == 0) {
                Quad val;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) val.v[kk] = kk < cnt[u] ? div_N(A[u].v[kk], a.Nf, invN, pow2) : 0.0f;   // R3
                if (cnt[u] > 0) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) gb[u].v[kk] = fadd(gb[u].v[kk], val.v[kk]);              // R13
                    store_quad(a.gbar + e[u], gb[u], v4[u], cnt[u]);
                }
                if (a.values != nullptr) store_quad(a.values + o[u], val, ov4[u], ocnt[u]);
            } else if (a.mode == 1 && a.bf16) {   // the local node sum, rounded for the bf16 all-reduce
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    if (kk < ocnt[u]) pay_st(a.values, o[u] + kk, A[u].v[kk], 1);
            } else if (a.mode == 1 || a.mode == 3) {
                store_quad(a.values + o[u], A[u], ov4[u] && a.mode == 1, ocnt[u]);
            }
        }
    }
    }
}

// S4 + S5 + S6 of a list of selected rows of one block, every node local (mode 0,
// no values output): the same arithmetic as gather_segments mode 0.  Row j of
// the list is lo + list[j] (list == nullptr: lo + j).  The row's position in
// the selection is not needed, so a CTA can run this before the selection of
// the other slices is known.
template <int UN>
__device__ void gather_rows_local(const GatherLaunch& a, const BlockDev& B, int lo, const int* list, int cnt) {
    const int nq = (B.n + 3) >> 2;
    const int items = cnt * nq;
    const bool pow2 = (a.N_int & (a.N_int - 1)) == 0;
    const float invN = 1.0f / a.Nf;
    for (int base = 0; base < items; base += kThreads * UN) {
        int nv[UN];
        long long e[UN];
        bool v4[UN];
#pragma unroll
        for (int u = 0; u < UN; ++u) {
            const int item = base + u * kThreads + static_cast<int>(threadIdx.x);
            nv[u] = 0;
            e[u] = 0;
            if (item < items) {
                const int j = item / nq, q = 4 * (item - j * nq);
                const int p = lo + (list != nullptr ? list[j] : j);
                nv[u] = max(0, min(4, row_valid_cols(B, p) - q));
                e[u] = B.off + static_cast<long long>(p) * B.n + q;
            }
            v4[u] = B.vec && nv[u] == 4;
        }
        Quad A[UN], gb[UN];
        for (int i = 0; i < a.nodes_local; ++i) {
            // (without EF the compressed rows are the gradient's: C_i = grad_i, no g)
            float* __restrict__ ph = a.noef ? const_cast<float*>(a.nodes.grad[i]) : a.nodes.h[i];
            float* __restrict__ pg = a.nodes.g[i];
            Quad hq[UN], gq[UN];
#pragma unroll
            for (int u = 0; u < UN; ++u) {
                if (nv[u] == 0) continue;
                if (i == 0) gb[u] = load_quad(a.gbar + e[u], v4[u], nv[u]);
                if (!a.noef) gq[u] = load_quad(pg + e[u], v4[u], nv[u]);
                hq[u] = load_quad(ph + e[u], v4[u], nv[u]);
            }
#pragma unroll
            for (int u = 0; u < UN; ++u) {
                if (nv[u] == 0) continue;
                Quad gn;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const float c = wire_round(a.noef ? hq[u].v[kk] : fsub(hq[u].v[kk], gq[u].v[kk]), a.bf16);   // C_i (R25)
                    gn.v[kk] = a.noef ? 0.0f : fadd(gq[u].v[kk], c);                       // R12
                    A[u].v[kk] = i == 0 ? c : fadd(A[u].v[kk], c);                 // R9 node order
                }
                if (!a.noef) store_quad(pg + e[u], gn, v4[u], nv[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < UN; ++u) {
            if (nv[u] == 0) continue;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) gb[u].v[kk] = fadd(gb[u].v[kk], div_N(A[u].v[kk], a.Nf, invN, pow2));   // R3, R13
            store_quad(a.gbar + e[u], gb[u], v4[u], nv[u]);
        }
    }
}

// S4 + S5 + S6 of one selected row (mode 0, no values output) by one warp: lane
// l takes columns 4l, 4l + 128, ...; the same arithmetic as gather_rows_local.
__device__ __forceinline__ void gather_row_warp(const GatherLaunch& a, const BlockDev& B, int p, int lane) {
    const int nvr = row_valid_cols(B, p);
    const bool pow2 = (a.N_int & (a.N_int - 1)) == 0;
    const float invN = 1.0f / a.Nf;
    for (int q = 4 * lane; q < nvr; q += 128) {
        const int nv = min(4, nvr - q);
        const long long e = B.off + static_cast<long long>(p) * B.n + q;
        const bool v4 = B.vec && nv == 4;
        Quad A, gb = load_quad(a.gbar + e, v4, nv);
        for (int i = 0; i < a.nodes_local; ++i) {
            float* __restrict__ ph = a.noef ? const_cast<float*>(a.nodes.grad[i]) : a.nodes.h[i];
            float* __restrict__ pg = a.nodes.g[i];
            const Quad hq = load_quad(ph + e, v4, nv);
            Quad gq, gn;
            if (!a.noef) gq = load_quad(pg + e, v4, nv);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const float c = wire_round(a.noef ? hq.v[kk] : fsub(hq.v[kk], gq.v[kk]), a.bf16);   // C_i (R25)
                gn.v[kk] = a.noef ? 0.0f : fadd(gq.v[kk], c);                 // R12
                A.v[kk] = i == 0 ? c : fadd(A.v[kk], c);                      // R9 node order
            }
            if (!a.noef) store_quad(pg + e, gn, v4, nv);
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) gb.v[kk] = fadd(gb.v[kk], div_N(A.v[kk], a.Nf, invN, pow2));   // R3, R13
        store_quad(a.gbar + e, gb, v4, nv);
    }
}

constexpr int kMaxSliceRows = 4096;
constexpr int kMaxSlicesPerCta = 32;   // slices one CTA of the persistent selection kernel takes at most

// Candidate resolution on a small list in shared memory (every CTA of the block
// computes the same result): T = the krem-th largest key among the candidates
// (digits key[20:10], key[9:0] below the common digit 1), and the row cutoff
// P_eq among the candidates equal to T (the need_eq smallest rows are taken).
__device__ void resolve_candidates(const unsigned* ck, const int* ci, int C, unsigned b1, int krem, unsigned* sh,
                                   int* warp_sums, unsigned* s_dig, int* s_abv, unsigned* T_out, int* Peq_out) {
    const int tid = threadIdx.x;
    // digit 2 (key[20:10]) of the candidates
    for (int i = tid; i < 2048; i += kThreads) sh[i] = 0;
    __syncthreads();
    for (int i = tid; i < C; i += kThreads) atomicAdd(&sh[(ck[i] >> 10) & 2047u], 1u);
    __syncthreads();
    int above;
    const unsigned b2 = top_digit(sh, 2048, krem, warp_sums, s_dig, s_abv, &above);
    krem -= above;
    const unsigned pre = (b1 << 11) | b2;            // key[31:10] of the K-th key
    // the candidates of bin (b1, b2) — usually a handful — compacted into a
    // short list (sh is free again), then ranked in the order (key desc, row asc):
    // the krem-th one is (T, P_eq)
    constexpr int kList = 1024;
    unsigned* lk = sh;
    int* li = reinterpret_cast<int*>(sh + kList);
    int mine = 0;
    for (int i = tid; i < C; i += kThreads) mine += (ck[i] >> 10) == pre;
    int E;
    int pos = cta_exclusive_scan(mine, warp_sums, &E);
    if (E <= kList) {
        for (int i = tid; i < C; i += kThreads)
            if ((ck[i] >> 10) == pre) { lk[pos] = ck[i]; li[pos] = ci[i]; ++pos; }
        __syncthreads();
        for (int i = tid; i < E; i += kThreads) {
            const unsigned key = lk[i];
            const int row = li[i];
            int rank = 0;
#pragma unroll 8
            for (int j = 0; j < E; ++j) rank += lk[j] > key || (lk[j] == key && li[j] < row);
            if (rank == krem - 1) { *s_dig = key; *s_abv = row; }
        }
    } else {   // massive ties inside one sub-bin: rank against the whole list
        for (int i = tid; i < C; i += kThreads) {
            if ((ck[i] >> 10) != pre) continue;
            int rank = 0;
#pragma unroll 8
            for (int j = 0; j < C; ++j)
                rank += ((ck[j] >> 10) == pre) && (ck[j] > ck[i] || (ck[j] == ck[i] && ci[j] < ci[i]));
            if (rank == krem - 1) { *s_dig = ck[i]; *s_abv = ci[i]; }
        }
    }
    __syncthreads();
    *T_out = *s_dig;
    *Peq_out = *s_abv;
    __syncthreads();
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// One selection slice: rows [lo, hi) of one selection block.
struct Slice {
    BlockDev B;
    long long bb;   // selection block index
    int c;          // slice index in the block
    int lo, hi, nk;
    int sidx;       // global slice index (slice_gt / slice_eq)
    bool arc;       // a real selection (ARC block with K < m); otherwise identity
};
__device__ __forceinline__ Slice slice_of(const SelectGatherLaunch& s, int item) {
    Slice x;
    const SliceItem it = s.items[item];
    x.B = s.blocks[it.b];
    x.bb = it.b;
    x.c = it.c;
    x.lo = it.c * s.slice_rows;
    x.hi = min(x.B.m, x.lo + s.slice_rows);
    x.nk = x.hi - x.lo;
    x.sidx = x.B.slice_base + it.c;
    x.arc = x.B.kind == ARC_BLOCK_ARC && x.B.K < x.B.m;
    return x;
}

// the slice's order keys (R15) from Sigma in global memory into shared memory
__device__ __forceinline__ void load_keys(const float* __restrict__ sigma, const Slice& x, unsigned* s_keys) {
    const float* __restrict__ sg = sigma + x.B.row_base + x.lo;
    for (int i0 = 0; i0 < x.nk; i0 += 4 * kThreads) {
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = i0 + k * kThreads + static_cast<int>(threadIdx.x);
            v[k] = i < x.nk ? __ldcg(sg + i) : 0.0f;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = i0 + k * kThreads + static_cast<int>(threadIdx.x);
            if (i < x.nk) s_keys[i] = order_key(v[k]);
        }
    }
}

// Grid-wide barriers.  The kernel normally runs as a cooperative grid (cg grid
// barriers through global memory).  A small selection (at most 16 slices) runs
// as ONE thread-block cluster instead: the cluster's hardware barrier
// (barrier.cluster arrive.release / wait.acquire, memory-ordered at cluster
// scope, which here is every thread of the grid) replaces the grid barrier, and
// the launch is an ordinary one — no cooperative launch.
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire;" ::: "memory"); }

// The selection kernel is PERSISTENT: CTA b handles slices b, b + grid, b + 2 grid,
// ... (at most kMaxSlicesPerCta), so any block table is accepted whatever the
// number of co-resident CTAs.  With one slice per CTA (the common case) the
// slice's keys stay in shared memory across the grid barriers; with several
// they are re-read from Sigma (L2) for each slice.
template <bool kPhase0, bool kMulti, bool kCluster>
__global__ void __launch_bounds__(kThreads, 2) k_select_gather(const SelectGatherLaunch s, const GatherLaunch ga) {
    cg::grid_group grid = cg::this_grid();
    auto grid_sync = [&]() {
        if constexpr (kCluster) {
            cluster_arrive();
            cluster_wait();
        } else {
            grid.sync();
        }
    };
#define STAMP(k) \
    if (s.stamps != nullptr && threadIdx.x == 0) s.stamps[blockIdx.x * 8 + (k)] = globaltimer()
    STAMP(0);
    __shared__ unsigned sh[2048];                   // histogram
    __shared__ __align__(16) unsigned s_keys[kMaxSliceRows];   // the current slice's order keys
    __shared__ int s_rows[kMaxSliceRows];           // boundary-bin candidates (keys | rows) / row lists
    __shared__ int warp_sums[32];
    __shared__ unsigned s_dig;
    __shared__ int s_abv;
    __shared__ int s_nb;                            // early mode: selected boundary-bin rows
    __shared__ unsigned s_b1[kMaxSlicesPerCta];     // per slice of this CTA: digit-1 boundary bin
    __shared__ int s_krem[kMaxSlicesPerCta];        //   and the rank still to find inside it

    const int tid = threadIdx.x;
    // (kMulti: grid < num_items, some CTAs take several slices; else one slice per CTA)
    const int nmine = kMulti ? (s.num_items - static_cast<int>(blockIdx.x) + static_cast<int>(gridDim.x) - 1) /
                                   static_cast<int>(gridDim.x)
                             : 1;
    const bool cached = !kMulti;                    // keys survive in s_keys across the barriers
    auto item_of = [&](int k) { return static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x); };
    grid_dependency_wait();   // Sigma and the digit-1 histogram are complete
    const int par = static_cast<int>(__ldcg(s.parity) & 1u);   // read by every CTA before barrier 1
    unsigned* ccount = s.cand_count + par * s.num_blocks;                 // this step's counters

    // ------------------------------------------------ phase 0
    // Sigma was not formed by the streaming pass: either the kernel forms it here
    // from this GPU's per-node sketches ([M][L][r], several local nodes, no
    // exchange: S2 summed in node order, R9, R21), or k_sigma_slice + the Sigma
    // all-gather left it in s.sigma (exchange path).  Then the slices' keys, the
    // blocks' digit-1 histograms, and a grid barrier so they are complete.
    if constexpr (kPhase0) {
        for (int k = 0; k < nmine; ++k) {
            const Slice x = slice_of(s, item_of(k));
            const BlockDev& B = x.B;
            const int lo = x.lo, nk = x.nk;
            if (B.kind == ARC_BLOCK_ARC && (x.arc || s.xsk != nullptr)) {   // every ARC block gets its Sigma
                __syncthreads();                                            // (s_keys / sh of the previous slice)
                for (int i = tid; i < kHist1Bins; i += kThreads) sh[i] = 0;
                __syncthreads();
                auto finish = [&](int i, float sig) {
                    const unsigned key = order_key(sig);
                    s_keys[i] = key;
                    atomicAdd(&sh[key >> kHist1Shift], 1u);
                };
                if (s.xsk == nullptr) {
                    const float* __restrict__ sg = s.sigma + B.row_base + lo;
                    for (int i0 = 0; i0 < nk; i0 += 4 * kThreads) {
                        float v[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int i = i0 + q * kThreads + tid;
                            v[q] = i < nk ? __ldcg(sg + i) : 0.0f;
                        }
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int i = i0 + q * kThreads + tid;
                            if (i < nk) finish(i, v[q]);
                        }
                    }
                } else {
                    const int L = s.L;
                    auto sigma_of = [&](int i, const float* S) {
                        float sig = 0.0f;
                        for (int j = 0; j < s.r; ++j) {
                            sig = ffma(S[j], S[j], sig);                           // O8, zn28373
                        }
                        s.sigma_w[B.row_base + lo + i] = sig;
                        if (!isfinite(sig)) atomicOr(s.status, kStatusNonfinite);
                        finish(i, sig);
                    };
                    if (s.r == 4) {
                        // 4 rows per thread, 4 nodes per round: 16 float4 loads in flight
                        for (int i0 = 0; i0 < nk; i0 += 4 * kThreads) {
                            float S[4][4];
                            for (int n0 = 0; n0 < L; n0 += 4) {
                                float4 v[4][4];
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    const int i = i0 + u * kThreads + tid;
                                    const long long p = B.row_base + lo + i;
#pragma unroll
                                    for (int q = 0; q < 4; ++q)
                                        if (i < nk && n0 + q < L)
                                            v[u][q] = __ldcg(reinterpret_cast<const float4*>(s.xsk + (p * L + n0 + q) * 4));
                                }
#pragma unroll
                                for (int u = 0; u < 4; ++u)
#pragma unroll
                                    for (int q = 0; q < 4; ++q) {
                                        if (n0 + q >= L) continue;
                                        const float4 w = v[u][q];
                                        if (n0 + q == 0) { S[u][0] = w.x; S[u][1] = w.y; S[u][2] = w.z; S[u][3] = w.w; }
                                        else {                                               // R9 node order
                                            S[u][0] = fadd(S[u][0], w.x); S[u][1] = fadd(S[u][1], w.y);
                                            S[u][2] = fadd(S[u][2], w.z); S[u][3] = fadd(S[u][3], w.w);
                                        }
                                    }
                            }
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int i = i0 + u * kThreads + tid;
                                if (i < nk) sigma_of(i, S[u]);
                            }
                        }
                    } else {
                        for (int i = tid; i < nk; i += kThreads) {
                            const long long p = B.row_base + lo + i;
                            float S[32];
                            for (int j = 0; j < s.r; ++j) {
                                float a = 0.0f;
                                for (int l = 0; l < L; ++l) {
                                    const float v = __ldcg(s.xsk + (p * L + l) * s.r + j);
                                    a = l == 0 ? v : fadd(a, v);
                                }
                                S[j] = a;
                            }
                            sigma_of(i, S);
                        }
                    }
                }
                if (x.arc) flush_hist(sh, s.hist1 + x.bb * kHist1Bins, kHist1Bins);
            }
        }
        grid_sync();                                 // ---------------- barrier 0
    }
    // ------------------------------------------------ phase A (per slice)
    // the digit-1 boundary bin b1 of the slice's block, the slice's count of keys
    // above it, and its keys in b1 appended to the block's candidate list
    int gt_pos = 0, gt_tot = 0;                      // (one slice per CTA: this thread's / the slice's rows above b1)
    for (int k = 0; k < nmine; ++k) {
        const Slice x = slice_of(s, item_of(k));
        if (!x.arc) continue;
        const BlockDev& B = x.B;
        __syncthreads();                             // (s_keys, sh of the previous slice)
        unsigned hv[8];                              // digit-1 histogram, loaded alongside the keys
#pragma unroll
        for (int q = 0; q < 8; ++q) hv[q] = __ldcg(s.hist1 + x.bb * kHist1Bins + tid + q * kThreads);
        if (!(kPhase0 && cached)) load_keys(s.sigma, x, s_keys);
#pragma unroll
        for (int q = 0; q < 8; ++q) sh[tid + q * kThreads] = hv[q];
        __syncthreads();
        int above;
        const unsigned b1 = top_digit(sh, kHist1Bins, B.K, warp_sums, &s_dig, &s_abv, &above);
        const int krem = B.K - above;
        // keys above bin b1 and the candidates (keys in bin b1) of this slice;
        // both counts in one packed scan (each <= 4096)
        int gt1 = 0, nc = 0;
        for (int i = tid; i < x.nk; i += kThreads) {
            const unsigned d1 = s_keys[i] >> 21;
            gt1 += d1 > b1;
            nc += d1 == b1;
        }
        int packed_tot;
        const int packed = cta_exclusive_scan((gt1 << 16) | nc, warp_sums, &packed_tot);
        const int ctot = packed_tot & 0xFFFF;
        gt_pos = packed >> 16;
        gt_tot = packed_tot >> 16;
        if (tid == 0) {
            s.slice_gt[x.sidx] = packed_tot >> 16;
            s_abv = ctot > 0 ? static_cast<int>(atomicAdd(ccount + x.bb, static_cast<unsigned>(ctot))) : 0;
            s_b1[k] = b1;
            s_krem[k] = krem;
        }
        __syncthreads();
        unsigned* cand = s.cand + (static_cast<long long>(par) * s.num_blocks + x.bb) * (2 * kCandCap);
        int cpos = s_abv + (packed & 0xFFFF);
        for (int i = tid; i < x.nk && nc > 0; i += kThreads) {
            const unsigned key = s_keys[i];
            if ((key >> 21) == b1) {
                if (cpos < kCandCap) { cand[cpos] = key; cand[kCandCap + cpos] = static_cast<unsigned>(x.lo + i); }
                ++cpos;
            }
        }
    }
    // S0 of the next step, generated here speculatively (V depends only on
    // (seed, t, b)); the host uses it only if the next step's t matches
    // (the blocks' first items staged in shared memory — s_rows is free here — so
    // the per-item block search makes no dependent global loads: with C4's 171
    // blocks the global search cost ~20 us of this phase)
    if (s.V_next != nullptr) {
        const int R4 = (s.r + 3) >> 2;
        long long* first = reinterpret_cast<long long*>(s_rows);
        const bool tab = s.num_vblocks <= kMaxSliceRows / 2;
        __syncthreads();
        if (tab)
            for (int b = tid; b < s.num_vblocks; b += kThreads) first[b] = (s.vblocks[b].v_off / s.r) * R4;
        __syncthreads();
        for (long long i = blockIdx.x * static_cast<long long>(kThreads) + tid; i < s.v_items;
             i += static_cast<long long>(gridDim.x) * kThreads) {
            if (tab) rng::gen_V_item_tab(s.vblocks, first, s.num_vblocks, s.r, s.key, s.t_lo, s.t_hi, i, s.V_next);
            else rng::gen_V_item(s.vblocks, s.num_vblocks, s.r, s.key, s.t_lo, s.t_hi, i, s.V_next);
        }
        __syncthreads();   // (s_rows is reused below)
    }
    STAMP(1);
    for (int k = 0; k < nmine; ++k) {                // next step's candidate counter of each block
        const SliceItem it = s.items[item_of(k)];
        if (it.c == 0 && tid == 0) s.cand_count[(par ^ 1) * s.num_blocks + it.b] = 0;
    }
    if (s.early) {
        // split barrier 1: the rows of a slice above the boundary bin b1 are
        // selected whatever the candidates resolve to (fewer than K keys lie above
        // b1), so their S4..S6 runs while the other CTAs reach the barrier
        auto early_gather = [&]() {
            for (int k = 0; k < nmine; ++k) {
                const Slice x = slice_of(s, item_of(k));
                if (x.arc) {
                    __syncthreads();                     // (s_rows / s_keys of the previous slice)
                    if (!cached) {
                        load_keys(s.sigma, x, s_keys);
                        __syncthreads();
                        int g1 = 0;
                        for (int i = tid; i < x.nk; i += kThreads) g1 += (s_keys[i] >> 21) > s_b1[k];
                        gt_pos = cta_exclusive_scan(g1, warp_sums, &gt_tot);
                    }
                    const unsigned b1 = s_b1[k];
                    int pos = gt_pos;
                    for (int i = tid; i < x.nk; i += kThreads)
                        if ((s_keys[i] >> 21) > b1) s_rows[pos++] = i;
                    __syncthreads();
                    gather_rows_local<4>(ga, x.B, x.lo, s_rows, gt_tot);
                } else {
                    gather_rows_local<4>(ga, x.B, x.lo, nullptr, x.nk);   // K = m: every row
                }
            }
            __syncthreads();                             // s_rows is reused below
        };
        if constexpr (kCluster) {
            cluster_arrive();
            early_gather();
            cluster_wait();
        } else {
            auto token = grid.barrier_arrive();
            early_gather();
            grid.barrier_wait(std::move(token));
        }
    } else {
        grid_sync();                                 // ---------------- barrier 1
    }
    STAMP(2);
    // every CTA has read this step's parity (before barrier 1): the next step uses the other one
    if (blockIdx.x == 0 && tid == 0) *s.parity = static_cast<unsigned>(par ^ 1);
    // ARC_FLAG_DEVICE_T: the step's kernels that read t (V, Rand-K keys) ran before this one
    if (s.t_advance != nullptr && blockIdx.x == 0 && tid == 0) *s.t_advance += 1ull;
    // any block with more candidates than fit takes the digit-by-digit path
    // (uniform across the grid, so every CTA meets the same barriers)
    bool overflow = false;
    for (int b = tid; b < s.num_blocks; b += kThreads) overflow |= __ldcg(ccount + b) > static_cast<unsigned>(kCandCap);
    overflow = __syncthreads_or(overflow);
    for (int k = 0; k < nmine; ++k) {                // hist1 was read by every slice before barrier 1: reset
        const Slice x = slice_of(s, item_of(k));
        if (x.B.kind == ARC_BLOCK_ARC && x.c == 0)
            for (int i = tid; i < kHist1Bins; i += kThreads) s.hist1[x.bb * kHist1Bins + i] = 0;
    }
    STAMP(3);
    int32_t* __restrict__ sel_all = s.sel;
    // one slice's compaction: its selected rows (key > T, or key == T and
    // [use_peq] row <= P_eq / [else] within the slice's quota of equal keys) in
    // ascending order at sel_before; early mode: its selected boundary-bin rows
    // (still to update) listed in s_rows[0 .. s_nb)
    auto compact = [&](const Slice& x, unsigned b1, unsigned T, int P_eq, int need_eq, int sel_before, bool use_peq) {
        int32_t* __restrict__ out = sel_all + x.B.sel_base;
        const int per = (s.slice_rows + kThreads - 1) / kThreads;   // consecutive rows per thread
        int my_eq = 0;
        if (!use_peq)
            for (int q = 0; q < per; ++q) {
                const int i = tid * per + q;
                my_eq += (i < x.nk && s_keys[i] == T);
            }
        int eq_tot;
        int eq_rank = use_peq ? 0 : cta_exclusive_scan(my_eq, warp_sums, &eq_tot);
        int my_sel = 0;
        unsigned take_mask = 0;                      // per <= 16
        for (int q = 0; q < per; ++q) {
            const int i = tid * per + q;
            bool t = false;
            if (i < x.nk) {
                const unsigned key = s_keys[i];
                if (key > T) t = true;
                else if (key == T) {
                    if (use_peq) t = x.lo + i <= P_eq;
                    else { t = eq_rank < need_eq; ++eq_rank; }
                }
            }
            if (t) { take_mask |= 1u << q; ++my_sel; }
        }
        if (tid == 0) s_nb = 0;
        int nsel;
        int pos = cta_exclusive_scan(my_sel, warp_sums, &nsel);
        for (int q = 0; q < per; ++q) {
            if (take_mask & (1u << q)) {
                const int i = tid * per + q;
                out[sel_before + pos] = x.lo + i;
                ++pos;
                // early mode: the selected rows of the boundary bin are still to do
                if (s.early && (s_keys[i] >> 21) == b1) s_rows[atomicAdd(&s_nb, 1)] = i;
            }
        }
        __syncthreads();
    };
    auto identity = [&](const Slice& x) {            // DENSE blocks and K = m
        int32_t* __restrict__ out = sel_all + x.B.sel_base;
        for (int p = x.lo + tid; p < x.hi; p += kThreads) out[p] = p;
    };
    // early mode after an overflow: this CTA's selected boundary rows, appended to one list
    auto append_boundary = [&](const Slice& x) {
        if (tid == 0) s_abv = s_nb > 0 ? static_cast<int>(atomicAdd(ga.bnd_count + par, static_cast<unsigned>(s_nb))) : 0;
        __syncthreads();
        for (int i = tid; i < s_nb; i += kThreads) ga.bnd[s_abv + i] = make_int2(static_cast<int>(x.bb), x.lo + s_rows[i]);
        __syncthreads();
    };
    if (!overflow) {
        for (int k = 0; k < nmine; ++k) {
            const Slice x = slice_of(s, item_of(k));
            if (!x.arc) { identity(x); continue; }
            __syncthreads();                         // (s_rows / s_keys of the previous slice)
            const unsigned* cand = s.cand + (static_cast<long long>(par) * s.num_blocks + x.bb) * (2 * kCandCap);
            // this block's candidate slots (all of them: one round, no wait for the count)
            // and the preceding slices' counts, loaded together
            const int C = static_cast<int>(min(__ldcg(ccount + x.bb), static_cast<unsigned>(kCandCap)));
            int before = 0;
            for (int c = tid; c < x.c; c += kThreads) before += __ldcg(s.slice_gt + x.B.slice_base + c);
            unsigned* ck = reinterpret_cast<unsigned*>(s_rows);
            int* ci = s_rows + kCandCap;
#pragma unroll
            for (int q = 0; q < kCandCap / kThreads; ++q) {
                const int i = tid + q * kThreads;
                ck[i] = __ldcg(cand + i);
                ci[i] = static_cast<int>(__ldcg(cand + kCandCap + i));
            }
            if (!cached) load_keys(s.sigma, x, s_keys);
            __syncthreads();
            unsigned T;
            int P_eq;
            const unsigned b1 = s_b1[k];
            resolve_candidates(ck, ci, C, b1, s_krem[k], sh, warp_sums, &s_dig, &s_abv, &T, &P_eq);
            // rows selected before this slice: keys above bin b1 in earlier slices,
            // plus the selected candidates at earlier rows
            for (int i = tid; i < C; i += kThreads)
                before += (ci[i] < x.lo && (ck[i] > T || (ck[i] == T && ci[i] <= P_eq)));
            int sel_before;
            cta_exclusive_scan(before, warp_sums, &sel_before);
            STAMP(4);
            compact(x, b1, T, P_eq, 0, sel_before, true);
            STAMP(5);
            if (s.early) gather_rows_local<4>(ga, x.B, x.lo, s_rows, s_nb);
        }
        if (s.early) {
            STAMP(6);
            STAMP(7);
            return;
        }
    } else {
        // ---- digit by digit (some block's boundary bin overflowed the candidate
        // list): digit-2 histogram of bin b1, then digit 3, one barrier each
        for (int k = 0; k < nmine; ++k) {
            const Slice x = slice_of(s, item_of(k));
            if (!x.arc) continue;
            __syncthreads();
            if (!cached) load_keys(s.sigma, x, s_keys);
            for (int i = tid; i < 2048; i += kThreads) sh[i] = 0;
            __syncthreads();
            const unsigned b1 = s_b1[k];
            for (int i = tid; i < x.nk; i += kThreads)
                if ((s_keys[i] >> 21) == b1) atomicAdd(&sh[(s_keys[i] >> 10) & 2047u], 1u);
            flush_hist(sh, s.hist2 + x.bb * 2048, 2048);
        }
        grid_sync();                                 // ---------------- barrier 1b
        for (int k = 0; k < nmine; ++k) {
            const Slice x = slice_of(s, item_of(k));
            if (!x.arc) continue;
            __syncthreads();
            const unsigned b1 = s_b1[k];
            const int kr = s_krem[k];
            if (!cached) load_keys(s.sigma, x, s_keys);
            load_hist(sh, s.hist2 + x.bb * 2048, 2048);   // (ends with a barrier: b1, kr read by all)
            int above;
            const unsigned b2 = top_digit(sh, 2048, kr, warp_sums, &s_dig, &s_abv, &above);
            const unsigned pre = (b1 << 11) | b2;
            if (tid == 0) { s_b1[k] = pre; s_krem[k] = kr - above; }   // from here on: key[31:10] of the K-th key
            for (int i = tid; i < 1024; i += kThreads) sh[i] = 0;
            __syncthreads();
            for (int i = tid; i < x.nk; i += kThreads)
                if ((s_keys[i] >> 10) == pre) atomicAdd(&sh[s_keys[i] & 1023u], 1u);
            flush_hist(sh, s.hist3 + x.bb * 1024, 1024);
        }
        grid_sync();                                 // ---------------- barrier 2
        for (int k = 0; k < nmine; ++k) {
            const Slice x = slice_of(s, item_of(k));
            if (!x.arc) continue;
            __syncthreads();
            if (x.c == 0)
                for (int i = tid; i < 2048; i += kThreads) s.hist2[x.bb * 2048 + i] = 0;
            const unsigned pre = s_b1[k];
            const int kr = s_krem[k];
            if (!cached) load_keys(s.sigma, x, s_keys);
            load_hist(sh, s.hist3 + x.bb * 1024, 1024);   // (ends with a barrier: pre, kr read by all)
            int above;
            const unsigned b3 = top_digit(sh, 1024, kr, warp_sums, &s_dig, &s_abv, &above);
            const unsigned T = (pre << 10) | b3;
            if (tid == 0) { s_b1[k] = T; s_krem[k] = kr - above; }   // (T, need_eq) of the block
            int gt = 0, eq = 0;
            for (int i = tid; i < x.nk; i += kThreads) {
                gt += s_keys[i] > T;
                eq += s_keys[i] == T;
            }
            int tg, te;
            cta_exclusive_scan(gt, warp_sums, &tg);
            cta_exclusive_scan(eq, warp_sums, &te);
            if (tid == 0) { s.slice_gt[x.sidx] = tg; s.slice_eq[x.sidx] = te; }
        }
        grid_sync();                                 // ---------------- barrier 3
        if (s.early && blockIdx.x == 0 && tid == 0) ga.bnd_count[par ^ 1] = 0;   // the next step's counter
        for (int k = 0; k < nmine; ++k) {
            const Slice x = slice_of(s, item_of(k));
            if (!x.arc) { identity(x); continue; }
            __syncthreads();
            if (x.c == 0)
                for (int i = tid; i < 1024; i += kThreads) s.hist3[x.bb * 1024 + i] = 0;
            if (!cached) load_keys(s.sigma, x, s_keys);
            int gb = 0, eb = 0;
            for (int c = tid; c < x.c; c += kThreads) {
                gb += __ldcg(s.slice_gt + x.B.slice_base + c);
                eb += __ldcg(s.slice_eq + x.B.slice_base + c);
            }
            int gtot, etot;
            cta_exclusive_scan(gb, warp_sums, &gtot);
            cta_exclusive_scan(eb, warp_sums, &etot);
            const int need_eq = s_krem[k];
            const unsigned T = s_b1[k];
            const int sel_before = gtot + min(etot, need_eq);
            // b1 of the block = T's top 11 bits (the boundary rows of early mode)
            compact(x, T >> 21, T, 0x7FFFFFFF, max(0, need_eq - etot), sel_before, false);
            if (s.early) append_boundary(x);
        }
        if (s.early) {
            // a candidate overflow (massive ties): the selected boundary rows may crowd
            // a few slices, so every slice appended them to one list and, after a
            // barrier, the grid's warps take them row by row
            __threadfence();
            grid_sync();                             // ---------------- the boundary list is complete
            const int total = static_cast<int>(__ldcg(ga.bnd_count + par));
            const int lane = tid & 31, warps = kThreads / 32;
            for (int j = blockIdx.x * warps + (tid >> 5); j < total; j += gridDim.x * warps) {
                const int2 br = __ldcg(ga.bnd + j);
                gather_row_warp(ga, ga.blocks[br.x], br.y, lane);
            }
            STAMP(6);
            STAMP(7);
            return;
        }
    }
    // S4 (+S5, S6): all selected-row segments spread evenly over the grid
    constexpr int UN = 4;
    const long long S = ga.num_rows;
    const int seg0 = static_cast<int>(S * blockIdx.x / gridDim.x);
    const int seg1 = static_cast<int>(S * (blockIdx.x + 1) / gridDim.x);
    __threadfence();
    grid_sync();                                     // ---------------- the selection is complete
    STAMP(6);
    // (s_keys, 16 KB, is free now: the segment stage)
    gather_segments<UN>(ga, seg0, seg1, reinterpret_cast<int4*>(s_keys), kMaxSliceRows / 4);
    __syncthreads();
    STAMP(7);

#undef STAMP
}

}  // namespace

int select_gather_resident_ctas() {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_select_gather<false, false, false>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_select_gather<true, false, false>, kThreads, 0);
    if (per_sm2 < per_sm) per_sm = per_sm2;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_select_gather<false, true, false>, kThreads, 0);
    if (per_sm2 < per_sm) per_sm = per_sm2;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_select_gather<true, true, false>, kThreads, 0);
    if (per_sm2 < per_sm) per_sm = per_sm2;
    return sms * (per_sm < 1 ? 1 : per_sm);
}

int select_max_slice_rows() { return kMaxSliceRows; }
int select_max_slices_per_cta() { return kMaxSlicesPerCta; }

cudaError_t launch_select_gather(const SelectGatherLaunch& s, const GatherLaunch& ga, cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(s.grid);   // persistent: CTA b takes slices b, b + grid, ...
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    if (s.cluster) {   // the whole grid is one cluster (its hardware barrier is the grid barrier)
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(s.grid);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
    }
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = s.pdl ? 2 : 1;
    if (s.cluster)
        return s.build_hist ? cudaLaunchKernelEx(&cfg, k_select_gather<true, false, true>, s, ga)
                            : cudaLaunchKernelEx(&cfg, k_select_gather<false, false, true>, s, ga);
    const bool multi = s.grid < s.num_items;
    if (s.build_hist)
        return multi ? cudaLaunchKernelEx(&cfg, k_select_gather<true, true, false>, s, ga)
                     : cudaLaunchKernelEx(&cfg, k_select_gather<true, false, false>, s, ga);
    return multi ? cudaLaunchKernelEx(&cfg, k_select_gather<false, true, false>, s, ga)
                 : cudaLaunchKernelEx(&cfg, k_select_gather<false, false, false>, s, ga);
}

// the largest grid (<= want) the selection kernel can run as one thread-block cluster (0: none)
int select_cluster_max(int want) {
    const void* fns[2] = {reinterpret_cast<const void*>(k_select_gather<false, false, true>),
                          reinterpret_cast<const void*>(k_select_gather<true, false, true>)};
    int best = want;
    for (const void* f : fns) {
        cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        int c = best;
        for (; c >= 1; --c) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(c);
            cfg.blockDim = dim3(kThreads);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = static_cast<unsigned>(c);
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, f, &cfg) == cudaSuccess && n >= 1) break;
            cudaGetLastError();
        }
        best = c;
    }
    return best;
}

}  // namespace arc
