// arc_api.cu — the C ABI of libarctopk.so (include/arc_topk.h): validation,
// workspace layout, the tile scheduler for the streaming pass, NCCL plumbing
// and the per-step launch sequence.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <new>
#include <queue>
#include <vector>

#include "arc_internal.cuh"
#include "arc_loopback.h"
#include "nccl.h"   // types only (torch wheel's NCCL 2.28); functions are resolved with dlsym
#include "nccl_device.h"   // ncclDevComm / requirements types (ARC_REDUCE_LSA)

using namespace arc;

namespace {

constexpr size_t kAlign = 256;
constexpr int kMinTileRows = 8;
constexpr int kMaxGrid = 8192;

size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

// ---- NCCL, resolved at run time from the libnccl.so.2 torch already loaded ----
struct Nccl {
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*commUserRank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    // symmetric windows + device communicator (ARC_REDUCE_LSA; NCCL >= 2.28)
    ncclResult_t (*memAlloc)(void**, size_t) = nullptr;
    ncclResult_t (*memFree)(void*) = nullptr;
    ncclResult_t (*winRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
    ncclResult_t (*winDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
    ncclResult_t (*devCommCreate)(ncclComm_t, const ncclDevCommRequirements_t*, ncclDevComm_t*) = nullptr;
    ncclResult_t (*devCommDestroy)(ncclComm_t, const ncclDevComm_t*) = nullptr;
    ncclTeam_t (*teamLsa)(ncclComm_t) = nullptr;
    bool ok = false;
};

bool load_nccl(Nccl& n) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) return false;
    n.allGather = reinterpret_cast<decltype(n.allGather)>(dlsym(h, "ncclAllGather"));
    n.allReduce = reinterpret_cast<decltype(n.allReduce)>(dlsym(h, "ncclAllReduce"));
    n.commCount = reinterpret_cast<decltype(n.commCount)>(dlsym(h, "ncclCommCount"));
    n.commUserRank = reinterpret_cast<decltype(n.commUserRank)>(dlsym(h, "ncclCommUserRank"));
    n.commGetAsyncError = reinterpret_cast<decltype(n.commGetAsyncError)>(dlsym(h, "ncclCommGetAsyncError"));
    n.send = reinterpret_cast<decltype(n.send)>(dlsym(h, "ncclSend"));
    n.recv = reinterpret_cast<decltype(n.recv)>(dlsym(h, "ncclRecv"));
    n.groupStart = reinterpret_cast<decltype(n.groupStart)>(dlsym(h, "ncclGroupStart"));
    n.groupEnd = reinterpret_cast<decltype(n.groupEnd)>(dlsym(h, "ncclGroupEnd"));
    n.memAlloc = reinterpret_cast<decltype(n.memAlloc)>(dlsym(h, "ncclMemAlloc"));
    n.memFree = reinterpret_cast<decltype(n.memFree)>(dlsym(h, "ncclMemFree"));
    n.winRegister = reinterpret_cast<decltype(n.winRegister)>(dlsym(h, "ncclCommWindowRegister"));
    n.winDeregister = reinterpret_cast<decltype(n.winDeregister)>(dlsym(h, "ncclCommWindowDeregister"));
    n.devCommCreate = reinterpret_cast<decltype(n.devCommCreate)>(dlsym(h, "ncclDevCommCreate"));
    n.devCommDestroy = reinterpret_cast<decltype(n.devCommDestroy)>(dlsym(h, "ncclDevCommDestroy"));
    n.teamLsa = reinterpret_cast<decltype(n.teamLsa)>(dlsym(h, "ncclTeamLsa"));
    n.ok = n.allGather && n.allReduce && n.commCount && n.commUserRank && n.commGetAsyncError && n.send && n.recv &&
           n.groupStart && n.groupEnd;
    return n.ok;
}

// ---- the step's collectives: NCCL, or the in-process loopback group ------------
// (arc_loopback.cu: G emulated ranks on one GPU, for tests without G GPUs).
// Every call also tallies the floats this rank hands to the collective, for the
// Table I ledger audit (arc_topk_comm_tally).
struct Comm {
    const Nccl* nccl = nullptr;
    ncclComm_t nc = nullptr;
    LoopbackComm* lb = nullptr;
    bool any() const { return nc != nullptr || lb != nullptr; }
    arc_status all_gather_bytes(const void* send, void* recv, size_t bytes, cudaStream_t s) const {
        if (lb) return loopback_all_gather(lb, send, recv, bytes, s);
        return nccl->allGather(send, recv, bytes, ncclUint8, nc, s) == ncclSuccess ? ARC_OK : ARC_ERR_NCCL;
    }
    arc_status all_gather_f32(const float* send, float* recv, size_t count, cudaStream_t s) const {
        if (lb) return loopback_all_gather(lb, send, recv, count * sizeof(float), s);
        return nccl->allGather(send, recv, count, ncclFloat32, nc, s) == ncclSuccess ? ARC_OK : ARC_ERR_NCCL;
    }
    arc_status all_reduce_f32(const float* send, float* recv, size_t count, cudaStream_t s) const {
        if (lb) return loopback_all_reduce_f32(lb, send, recv, count, s);
        return nccl->allReduce(send, recv, count, ncclFloat32, ncclSum, nc, s) == ncclSuccess ? ARC_OK : ARC_ERR_NCCL;
    }
    // the bfloat16 value wire (R25): NCCL sums in bfloat16 (rounded partial sums)
    arc_status all_reduce_bf16(const void* send, void* recv, size_t count, cudaStream_t s) const {
        if (lb) return loopback_all_reduce_bf16(lb, send, recv, count, s);
        return nccl->allReduce(send, recv, count, ncclBfloat16, ncclSum, nc, s) == ncclSuccess ? ARC_OK : ARC_ERR_NCCL;
    }
    // grouped point-to-point all-to-all (counts / displacements in floats, host arrays [G])
    arc_status all_to_all_f32(const float* send, const size_t* scount, const size_t* sdispl, float* recv,
                              const size_t* rcount, const size_t* rdispl, int G, cudaStream_t s) const {
        if (lb) return loopback_all_to_all_f32(lb, send, scount, sdispl, recv, rcount, rdispl, s);
        if (nccl->groupStart() != ncclSuccess) return ARC_ERR_NCCL;
        for (int j = 0; j < G; ++j) {
            if (scount[j] > 0 && nccl->send(send + sdispl[j], scount[j], ncclFloat32, j, nc, s) != ncclSuccess) {
                nccl->groupEnd();
                return ARC_ERR_NCCL;
            }
            if (rcount[j] > 0 && nccl->recv(recv + rdispl[j], rcount[j], ncclFloat32, j, nc, s) != ncclSuccess) {
                nccl->groupEnd();
                return ARC_ERR_NCCL;
            }
        }
        return nccl->groupEnd() == ncclSuccess ? ARC_OK : ARC_ERR_NCCL;
    }
};

// ledger tally slots (floats this rank handed to each collective, summed over steps)
enum { kTallySketch = 0, kTallySigma = 1, kTallyValues = 2, kTallyCalls = 3, kTallySteps = 4, kTallyN = 8 };

// ---- derived layout -----------------------------------------------------------
struct Plan {
    int G = 1, L = 1;
    bool exchange = false;       // run the G>1 sequence
    bool keep_pnodes = false;
    int M = 0;                   // sum of ARC m_b (global ARC rows)
    int64_t Ms = 0;              // exchange #1: rows per rank slice, ceil(M / G)
    int64_t sumK = 0, sumKn = 0, sum_nr = 0;
    int64_t num_segs = 0;        // gather / scatter row segments
    int num_slices = 0;          // selection slices (all blocks)
    int slice_rows = kSliceMin;
    std::vector<SliceItem> items;
    int max_nR4 = 0;
    int max_tiles = 0;
    std::vector<BlockDev> bdev;      // the caller's blocks
    bool topk = false;               // ARC_METHOD_TOPK_ALLGATHER baseline
    bool randk = false;              // ARC_METHOD_RANDK: data-independent shared selection
    bool exact = false;              // ARC_METHOD_EXACT: Sigma = exact row norms of the node sum
    bool noef = false;               // ARC_METHOD_NOEF_MSGD: sketch the gradient, u = gbar (no h, g)
    int64_t W = 0;                   // Top-K: payload words per node (sum K n values + sum K indices)
    std::vector<BlockDev> sbdev;     // selection blocks: bdev, or (Top-K) one copy per local node
    std::vector<SelRow> segs;        // gather segments over sbdev
    std::vector<SelRow> segs_real;   // segments over bdev (scatter, Top-K merge)
    bool dense_fast = false;         // DENSE blocks handled by the streaming k_dense (not Top-K)
    std::vector<int> dense_ids;
    // workspace offsets (bytes)
    size_t o_cta_w = 0, o_cta_t = 0, o_tdev = 0;
    size_t o_blocks = 0, o_tiles = 0, o_cta = 0, o_selrows = 0, o_V = 0, o_sigma = 0, o_sel = 0,
           o_status = 0, o_pnodes = 0, o_xrecv = 0, o_wire = 0, o_wire_all = 0, o_staging = 0,
           o_vals = 0, o_hash = 0, o_hist1 = 0, o_hist2 = 0, o_hist3 = 0, o_slice_gt = 0, o_slice_eq = 0,
           o_items = 0, o_cand = 0, o_cand_count = 0, o_sblocks = 0, o_segs_real = 0, o_dense_ids = 0, total = 0,
           o_bnd = 0, o_bnd_count = 0;
};

arc_status validate(const arc_topk_params* p) {
    if (p == nullptr) return ARC_ERR_INVALID_ARG;
    if (p->abi_version != ARC_TOPK_ABI_VERSION) return ARC_ERR_INVALID_ARG;
    if (p->N < 1 || p->nodes_local < 1 || p->nodes_local > ARC_MAX_NODES_LOCAL) return ARC_ERR_INVALID_ARG;
    if (p->N % p->nodes_local != 0) return ARC_ERR_INVALID_ARG;
    const int G = p->N / p->nodes_local;
    if (p->rank < 0 || p->rank >= G) return ARC_ERR_INVALID_ARG;
    if (p->d < 1 || p->r < 1 || p->r > 32) return ARC_ERR_INVALID_ARG;
    // eta: the EF21M momentum, 0 < eta <= 1; without EF it is the heavy-ball beta, 0 <= beta < 1
    if (p->method == ARC_METHOD_NOEF_MSGD ? !(p->eta >= 0.0f && p->eta < 1.0f) : !(p->eta > 0.0f && p->eta <= 1.0f))
        return ARC_ERR_INVALID_ARG;
    if (p->value_reduce != ARC_REDUCE_NCCL && p->value_reduce != ARC_REDUCE_ORDERED && p->value_reduce != ARC_REDUCE_LSA)
        return ARC_ERR_INVALID_ARG;
    if (p->wire != ARC_WIRE_F32 && p->wire != ARC_WIRE_BF16) return ARC_ERR_INVALID_ARG;
    if (p->reserved != 0) return ARC_ERR_INVALID_ARG;
    if (p->wire == ARC_WIRE_BF16 && p->method == ARC_METHOD_TOPK_ALLGATHER) return ARC_ERR_UNSUPPORTED;
    if (p->num_blocks < 1 || p->blocks == nullptr) return ARC_ERR_INVALID_ARG;
    if (p->flags & ~(ARC_FLAG_HOST_STAGING | ARC_FLAG_DEBUG_SKETCH | ARC_FLAG_FORCE_EXCHANGE | ARC_FLAG_LOOPBACK_COMM |
                     ARC_FLAG_DEVICE_T))
        return ARC_ERR_INVALID_ARG;
    if (p->method != ARC_METHOD_ARC && p->method != ARC_METHOD_TOPK_ALLGATHER && p->method != ARC_METHOD_RANDK &&
        p->method != ARC_METHOD_NOEF_MSGD && p->method != ARC_METHOD_EXACT)
        return ARC_ERR_INVALID_ARG;
    if (p->method == ARC_METHOD_EXACT && (p->nodes_local != p->N || (p->flags & ARC_FLAG_FORCE_EXCHANGE)))
        return ARC_ERR_UNSUPPORTED;
    int64_t pos = 0, M = 0, sumK = 0;
    for (int b = 0; b < p->num_blocks; ++b) {
        const arc_block& B = p->blocks[b];
        if (B.offset != pos) return ARC_ERR_INVALID_ARG;                  // tile [0, d) in order
        if (B.m < 1 || B.n < 1 || B.len < 1) return ARC_ERR_INVALID_ARG;
        if (B.m > INT32_MAX || B.n > INT32_MAX) return ARC_ERR_INVALID_ARG;
        if (B.len > B.m * B.n || B.len <= (B.m - 1) * B.n) return ARC_ERR_INVALID_ARG;
        if (B.K < 1 || B.K > B.m) return ARC_ERR_INVALID_ARG;
        if (B.kind != ARC_BLOCK_ARC && B.kind != ARC_BLOCK_DENSE) return ARC_ERR_INVALID_ARG;
        if (B.kind == ARC_BLOCK_DENSE && B.K != B.m) return ARC_ERR_INVALID_ARG;
        if (B.reserved != 0) return ARC_ERR_INVALID_ARG;
        pos += B.len;
        if (B.kind == ARC_BLOCK_ARC) M += B.m;
        sumK += B.K;
    }
    if (pos != p->d) return ARC_ERR_INVALID_ARG;
    if (M > INT32_MAX || sumK > INT32_MAX / 64) return ARC_ERR_INVALID_ARG;
    return ARC_OK;
}

// The single-block shorthand (num_blocks == 0, blocks == NULL): one ARC block
// of rows of n floats over [0, d), m = ceil(d / n), K rows kept (
// Alg. 1's K).  `out` is the params with the block table filled in (`one`).
arc_status normalize(const arc_topk_params* in, arc_topk_params& out, arc_block& one) {
    if (in == nullptr) return ARC_ERR_INVALID_ARG;
    out = *in;
    if (in->num_blocks == 0 && in->blocks == nullptr) {
        if (in->n < 1 || in->d < 1) return ARC_ERR_INVALID_ARG;
        one = arc_block{0, in->d, (in->d + in->n - 1) / in->n, in->n, in->K, ARC_BLOCK_ARC, 0};
        out.num_blocks = 1;
        out.blocks = &one;
    }
    return validate(&out);
}

void make_plan(const arc_topk_params* p, Plan& pl, int slice_rows = kSliceMin) {
    pl.slice_rows = slice_rows;
    pl.L = p->nodes_local;
    pl.G = p->N / p->nodes_local;
    pl.exchange = pl.G > 1 || (p->flags & ARC_FLAG_FORCE_EXCHANGE);
    pl.randk = p->method == ARC_METHOD_RANDK;
    pl.noef = p->method == ARC_METHOD_NOEF_MSGD;
    pl.exact = p->method == ARC_METHOD_EXACT;
    pl.keep_pnodes = !pl.randk && (pl.exchange || pl.L > 1 || pl.exact || (p->flags & ARC_FLAG_DEBUG_SKETCH));
    pl.bdev.resize(p->num_blocks);
    int64_t M = 0, sumK = 0, sumKn = 0, sum_nr = 0;
    int max_tiles = 0;
    const int R4 = (p->r + 3) / 4;
    for (int b = 0; b < p->num_blocks; ++b) {
        const arc_block& B = p->blocks[b];
        BlockDev& D = pl.bdev[b];
        D.off = B.offset;
        D.len = B.len;
        D.m = static_cast<int>(B.m);
        D.n = static_cast<int>(B.n);
        D.K = static_cast<int>(B.K);
        D.kind = B.kind;
        D.v_off = sum_nr;
        D.row_base = static_cast<int>(M);
        D.sel_base = static_cast<int>(sumK);
        D.val_base = sumKn;
        D.vec = (B.offset % 4 == 0) && (B.n % 4 == 0);
        D.slice_base = 0;
        D.node = 0;
        D.pad_ = 0;
        if (B.kind == ARC_BLOCK_ARC) {
            M += B.m;
            sum_nr += (B.n + 3) / 4 * 4 * p->r;   // V_b^T rows padded to 16 bytes
            pl.max_nR4 = std::max<int64_t>(pl.max_nR4, B.n * R4);
            max_tiles += static_cast<int>((B.m + kMinTileRows - 1) / kMinTileRows) *
                         (p->method == ARC_METHOD_TOPK_ALLGATHER || p->nodes_local > 1 ? p->nodes_local : 1);
        }
        sumK += B.K;
        sumKn += B.K * B.n;
        if (!(B.kind == ARC_BLOCK_DENSE && p->method != ARC_METHOD_TOPK_ALLGATHER)) {   // DENSE: streaming kernels
            const int nq = static_cast<int>((B.n + 3) / 4);
            for (int64_t k = 0; k < B.K; ++k)
                for (int q0 = 0; q0 < nq; q0 += kSegQuads) pl.segs_real.push_back(SelRow{b, static_cast<int>(k), q0});
        }
    }
    pl.M = static_cast<int>(M);
    pl.sumK = sumK;
    pl.sumKn = sumKn;
    pl.sum_nr = sum_nr;
    pl.max_tiles = max_tiles + 2 * kMaxGrid;   // (+ plan_tiles' balancing of a single block, per launch)
    // selection blocks: one per (local node, block) for the Top-K baseline, whose
    // nodes rank their own rows; the node's payload is [values | indices]
    pl.topk = p->method == ARC_METHOD_TOPK_ALLGATHER;
    pl.W = sumKn + sumK;
    // every node local and ARC: DENSE blocks take the streaming kernel, not the selection
    pl.dense_fast = !pl.topk;
    for (int b = 0; b < p->num_blocks; ++b)
        if (pl.dense_fast && pl.bdev[b].kind == ARC_BLOCK_DENSE) pl.dense_ids.push_back(b);
    const int nl = pl.topk ? pl.L : 1;
    for (int l = 0; l < nl; ++l) {
        for (int b = 0; b < p->num_blocks; ++b) {
            BlockDev S = pl.bdev[b];
            if (pl.dense_fast && S.kind == ARC_BLOCK_DENSE) {   // keep indices aligned with bdev
                S.slice_base = pl.num_slices;
                pl.sbdev.push_back(S);
                continue;
            }
            S.node = l;
            if (pl.topk) {
                S.row_base = l * pl.M + S.row_base;
                S.sel_base = static_cast<int>(l * pl.W + sumKn + S.sel_base);
                S.val_base = l * pl.W + S.val_base;
            }
            S.slice_base = pl.num_slices;
            const int nsl = (S.m + pl.slice_rows - 1) / pl.slice_rows;
            const int vb = static_cast<int>(pl.sbdev.size());
            for (int c = 0; c < nsl; ++c) pl.items.push_back(SliceItem{vb, c});
            pl.num_slices += nsl;
            const int nq = (S.n + 3) / 4;
            for (int k = 0; k < S.K; ++k)
                for (int q0 = 0; q0 < nq; q0 += kSegQuads) pl.segs.push_back(SelRow{vb, k, q0});
            pl.sbdev.push_back(S);
        }
    }
    pl.num_segs = static_cast<int64_t>(pl.segs.size());
    const int nsb = static_cast<int>(pl.sbdev.size());

    size_t off = 0;
    auto take = [&](size_t bytes) { const size_t o = off; off = align_up(off + std::max<size_t>(bytes, 1)); return o; };
    pl.o_blocks = take(sizeof(BlockDev) * p->num_blocks);
    pl.o_sblocks = take(sizeof(BlockDev) * nsb);
    pl.o_segs_real = take(sizeof(SelRow) * pl.segs_real.size());
    pl.o_dense_ids = take(sizeof(int) * pl.dense_ids.size());
    pl.o_tiles = take(sizeof(TileDesc) * pl.max_tiles);
    pl.o_cta = take(sizeof(int) * (kMaxGrid + 1));
    pl.o_cta_w = take(sizeof(int) * (kMaxGrid + 1));
    pl.o_cta_t = take(sizeof(int) * (kMaxGrid + 1));
    pl.o_selrows = take(sizeof(SelRow) * pl.num_segs);
    pl.o_V = take(sizeof(float) * sum_nr * 2);   // double-buffered by t parity
    pl.Ms = (M + pl.G - 1) / pl.G;
    pl.o_sigma = take(sizeof(float) * std::max<int64_t>(std::max<int64_t>(M * nl, pl.G * pl.Ms), 1));
    pl.o_sel = take(sizeof(int32_t) * sumK);
    pl.o_status = take(16);
    pl.o_tdev = take(16);
    pl.o_hist1 = take(sizeof(unsigned) * kHist1Bins * nsb);
    pl.o_hist2 = take(sizeof(unsigned) * 2048 * nsb);
    pl.o_hist3 = take(sizeof(unsigned) * 1024 * nsb);
    pl.o_slice_gt = take(sizeof(int) * pl.num_slices);
    pl.o_slice_eq = take(sizeof(int) * pl.num_slices);
    pl.o_items = take(sizeof(SliceItem) * pl.items.size());
    pl.o_cand = take(sizeof(unsigned) * 2 * 2 * kCandCap * nsb);
    pl.o_cand_count = take(sizeof(unsigned) * 2 * nsb);
    pl.o_bnd = take(sizeof(int) * 2 * std::max<int64_t>(sumK, 1));
    pl.o_bnd_count = take(sizeof(unsigned) * 2);
    pl.o_hash = take(sizeof(uint64_t) * (pl.G + 1));
    const size_t pn = sizeof(float) * static_cast<size_t>(M) * pl.L * p->r;
    pl.o_pnodes = pl.keep_pnodes ? take(pn) : 0;
    if (pl.topk) {
        pl.exchange = false;   // the baseline has its own exchange (all-gather of the payloads)
        pl.o_wire = take(sizeof(float) * pl.W * pl.L);
        pl.o_wire_all = pl.G > 1 ? take(sizeof(float) * pl.W * pl.L * pl.G) : 0;
    } else if (pl.exchange) {
        pl.o_xrecv = pl.randk ? 0 : take(sizeof(float) * static_cast<size_t>(pl.Ms) * pl.L * p->r * pl.G);
        // ORDERED and LSA carry per-node payloads; LSA's live in the library's
        // symmetric window instead of the workspace
        const bool ordered = p->value_reduce == ARC_REDUCE_ORDERED;
        const bool lsa = p->value_reduce == ARC_REDUCE_LSA;
        const size_t we = p->wire == ARC_WIRE_BF16 ? 2 : sizeof(float);   // payload entry bytes (R25)
        pl.o_wire = lsa ? 0 : take(we * sumKn * (ordered ? pl.L : 1));
        pl.o_wire_all = ordered ? take(we * sumKn * pl.L * pl.G) : 0;
    }
    if (p->flags & ARC_FLAG_HOST_STAGING) {
        // each node's staged gradient starts 256-byte aligned (the kernels' 16-byte loads)
        pl.o_staging = take(sizeof(float) * static_cast<size_t>((p->d + 63) / 64 * 64) * pl.L);
        pl.o_vals = take(sizeof(float) * sumKn);
    }
    pl.total = off;
}

// ---- the tile scheduler: balance the streaming pass over the resident CTAs ----
// A tile is <= R_shape rows of one ARC block for one local node (a row's sums
// are sequential, R9, so a row never spans two CTAs; different nodes are
// independent).  A chunk costs about the same whether or not all R_shape rows
// are live (masked rows still run the load and staging code), so a tile of r
// rows is charged nchunks * max(r, 0.6 R_shape); tiles go longest-first to the
// least-loaded CTA (LPT).
void plan_tiles(const Plan& pl, const std::vector<char>& use, int resident, int tile_rows_max, int W,
                std::vector<Tile>& tiles, std::vector<int>& cta_begin, int& grid, int tiny_rows = 0) {
    struct Cand { int64_t makespan = INT64_MAX; std::vector<Tile> tiles; std::vector<int> begin; int grid = 0; };
    Cand best;
    resident = std::max(1, std::min(resident, kMaxGrid));
    const int nodes = pl.topk || pl.L > 1 ? pl.L : 1;
    // Tile height: 8 rows (one per warp, the finest balance of the last round:
    // -1 % on C3, -1.7 % on C5 d = 1e8, -6 % on C2 against 32 rows) when the
    // layout has few blocks and the CTAs' tile lists stay in the kernel's shared
    // descriptor cache; 32 rows otherwise (many blocks: fewer block changes per
    // CTA, each restaging V; C4 +5 % and C5 d = 1e9 +0.4 % with 8-row tiles).
    {
        int arc_blocks = 0;
        int64_t tiles8 = 0;
        for (size_t b = 0; b < pl.bdev.size(); ++b)
            if (pl.bdev[b].kind == ARC_BLOCK_ARC && use[b]) { ++arc_blocks; tiles8 += (pl.bdev[b].m + 7) / 8 * nodes; }
        if (tiny_rows == 0 && arc_blocks <= 8 && tiles8 <= static_cast<int64_t>(resident) * 96)
            tile_rows_max = std::min(tile_rows_max, 8);
    }
    const int64_t floor_rows = (tile_rows_max * 6 + 9) / 10;
    const int R_pick = tile_rows_max;
    int R_lo = R_pick, R_hi = R_pick;
    if (const char* e = getenv("ARC_TILE_ROWS")) {   // debug knob: one tile height
        const int v = atoi(e);
        if (v >= 1 && v <= 32) R_lo = R_hi = v;
    }
    int used_blocks = 0;
    for (size_t b = 0; b < pl.bdev.size(); ++b) used_blocks += pl.bdev[b].kind == ARC_BLOCK_ARC && use[b];
    // variant 1 (one block in the second launch): raise the tile count to a multiple of the resident
    // CTAs, so every CTA streams the same number of rows (e.g. m = 18,315 rows
    // of 8 over 444 CTAs is 5.16 tiles per CTA: the last wave would be 16 % idle)
    for (int variant = 0; variant < (used_blocks == 1 && tiny_rows > 0 ? 2 : 1); ++variant)
    for (int R = R_hi; R >= R_lo; --R) {
        std::vector<Tile> ts;
        std::vector<int64_t> cost;
        for (size_t b = 0; b < pl.bdev.size(); ++b) {
            const BlockDev& B = pl.bdev[b];
            if (B.kind != ARC_BLOCK_ARC || !use[b]) continue;
            const int Rb = std::min(B.n <= 4 && tiny_rows > 0 ? tiny_rows : R, B.m);   // (<= 4 columns: a row per thread)
            int nt = (B.m + Rb - 1) / Rb;
            if (variant == 1) {
                const int64_t want = (static_cast<int64_t>(nt) * nodes + resident - 1) / resident * resident;
                nt = static_cast<int>(std::min<int64_t>(B.m, (want + nodes - 1) / nodes));
            }
            const int64_t nch = (B.n + W - 1) / W;
            for (int l = 0; l < nodes; ++l)
                for (int i = 0; i < nt; ++i) {   // rows spread evenly over the block's tiles
                    const int r0 = static_cast<int>(static_cast<int64_t>(B.m) * i / nt);
                    const int r1 = static_cast<int>(static_cast<int64_t>(B.m) * (i + 1) / nt);
                    ts.push_back(Tile{static_cast<int>(b), r0, r1 - r0, l});
                    cost.push_back(nch * std::max<int64_t>(r1 - r0, floor_rows) + 4);
                }
        }
        if (static_cast<int>(ts.size()) > pl.max_tiles) continue;
        const int g = std::min<int>(resident, static_cast<int>(ts.size()));
        std::vector<int> order(ts.size());
        for (size_t i = 0; i < ts.size(); ++i) order[i] = static_cast<int>(i);
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return cost[x] > cost[y]; });
        using Slot = std::pair<int64_t, int>;
        std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> heap;
        for (int c = 0; c < g; ++c) heap.push({0, c});
        std::vector<std::vector<int>> lists(g);
        int64_t makespan = 0;
        for (int idx : order) {
            Slot sl = heap.top();
            heap.pop();
            sl.first += cost[idx];
            makespan = std::max(makespan, sl.first);
            lists[sl.second].push_back(idx);
            heap.push(sl);
        }
        if (makespan < best.makespan) {
            Cand c;
            c.makespan = makespan;
            c.grid = g;
            c.begin.push_back(0);
            for (int k = 0; k < g; ++k) {
                std::sort(lists[k].begin(), lists[k].end());
                for (int idx : lists[k]) c.tiles.push_back(ts[idx]);
                c.begin.push_back(static_cast<int>(c.tiles.size()));
            }
            best = std::move(c);
        }
    }
    tiles = std::move(best.tiles);
    cta_begin = std::move(best.begin);
    grid = best.grid;
}

uint64_t fnv1a(uint64_t h, const void* data, size_t n) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) { h ^= p[i]; h *= 1099511628211ull; }
    return h;
}

uint64_t params_hash(const arc_topk_params* p) {
    uint64_t h = 1469598103934665603ull;
    h = fnv1a(h, &p->abi_version, sizeof p->abi_version);
    h = fnv1a(h, &p->N, sizeof p->N);
    h = fnv1a(h, &p->nodes_local, sizeof p->nodes_local);
    h = fnv1a(h, &p->d, sizeof p->d);
    h = fnv1a(h, &p->r, sizeof p->r);
    h = fnv1a(h, &p->num_blocks, sizeof p->num_blocks);
    h = fnv1a(h, p->blocks, sizeof(arc_block) * p->num_blocks);
    h = fnv1a(h, &p->eta, sizeof p->eta);
    h = fnv1a(h, &p->value_reduce, sizeof p->value_reduce);
    h = fnv1a(h, &p->seed, sizeof p->seed);
    h = fnv1a(h, &p->method, sizeof p->method);
    h = fnv1a(h, &p->wire, sizeof p->wire);
    const uint32_t f = p->flags & ~(ARC_FLAG_HOST_STAGING | ARC_FLAG_LOOPBACK_COMM);
    h = fnv1a(h, &f, sizeof f);
    return h;
}

}  // namespace

struct arc_topk_ctx {
    arc_topk_params p{};
    std::vector<arc_block> blocks;
    Plan pl;
    Nccl nccl;
    ncclComm_t comm = nullptr;       // NCCL communicator (borrowed), or
    LoopbackComm* lb = nullptr;      // the loopback group's rank handle (ARC_FLAG_LOOPBACK_COMM)
    Comm xc;                         // the step's collectives over either
    int64_t tally[kTallyN] = {};
    unsigned char* ws = nullptr;
    int grid = 0, num_tiles = 0, shape = 0, vs_cap = 0;
    int sel_grid = 0;                             // CTAs of the (persistent) selection kernel
    bool sel_cluster = false;                     // ... launched as one thread-block cluster
    int grid_w = 0, vs_cap_w = 0, tiles_w0 = 0;   // the wide blocks' ranged launch (grid_w == 0: none)
    int grid_t = 0, vs_cap_t = 0;                 // the bulk-copy fed launch (grid_t == 0: none)
    float ome = 0.f, Nf = 0.f;
    cudaStream_t last = nullptr;
    // per-phase timing
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;   // (ARC_TIMING_PHASES + 1) per timed step
    int timed_steps = 0;
    unsigned long long* stamps = nullptr;   // debug (ARC_DEBUG_STAMPS=1): library-owned device buffer
    int64_t v_ready = -1;        // t whose V the previous step generated speculatively
    bool pdl = true;             // programmatic dependent launch between the step's kernels (ARC_PDL=0: off)
    bool early = true;           // early gather of the certain rows in the select kernel (ARC_EARLY=0: off)
    bool tail = false;           // S3..S6 in the streaming launch's last CTA (small single-node selections)
    int tail_keys = 0;           // the largest ARC block's rows (keys staged in shared memory by the tail)
    int64_t last_t = 0;
    int64_t v_items = 0;
    // ARC_REDUCE_LSA: library-owned symmetric window and device communicator
    bool lsa = false;
    void* win_buf = nullptr;
    ncclWindow_t win = nullptr;
    bool dev_comm_ok = false;
    ncclDevComm dev_comm{};
    ncclDevComm* dev_comm_d = nullptr;
    // exchange #1 over peer memory: P' ([M][L][r]) and Sigma in one more window
    bool lsa1 = false;
    void* sk_buf = nullptr;
    ncclWindow_t sk_win = nullptr;
    size_t sk_sigma_off = 0;
    float* pnodes_ptr() const { return lsa1 ? static_cast<float*>(sk_buf) : at<float>(pl.o_pnodes); }
    float* sigma_ptr() const {
        return lsa1 ? reinterpret_cast<float*>(static_cast<unsigned char*>(sk_buf) + sk_sigma_off) : at<float>(pl.o_sigma);
    }

    template <class T> T* at(size_t off) const { return reinterpret_cast<T*>(ws + off); }
};

#define ARC_CUDA(call)                                     \
    do {                                                   \
        if ((call) != cudaSuccess) return ARC_ERR_CUDA;    \
    } while (0)
#define ARC_LAUNCHED()                                               \
    do {                                                             \
        if (cudaPeekAtLastError() != cudaSuccess) {                  \
            (void)cudaGetLastError();                                \
            return ARC_ERR_CUDA;                                     \
        }                                                            \
    } while (0)

// ARC_REDUCE_LSA (collective: every rank calls it at create, after the params
// check).  The payload window [L][sum_Kn] floats comes from ncclMemAlloc and is
// registered as a symmetric window; the device communicator carries one LSA
// barrier per CTA of the fused scatter kernels (arc_lsa.cu).
static void lsa_release(arc_topk_ctx* c) {
    if (c->dev_comm_ok && c->nccl.devCommDestroy) c->nccl.devCommDestroy(c->comm, &c->dev_comm);
    if (c->sk_win && c->nccl.winDeregister) c->nccl.winDeregister(c->comm, c->sk_win);
    if (c->sk_buf && c->nccl.memFree) c->nccl.memFree(c->sk_buf);
    c->sk_win = nullptr;
    c->sk_buf = nullptr;
    c->lsa1 = false;
    if (c->win && c->nccl.winDeregister) c->nccl.winDeregister(c->comm, c->win);
    if (c->win_buf && c->nccl.memFree) c->nccl.memFree(c->win_buf);
    if (c->dev_comm_d) cudaFree(c->dev_comm_d);
    c->dev_comm_ok = false;
    c->win = nullptr;
    c->win_buf = nullptr;
    c->dev_comm_d = nullptr;
    c->lsa = false;
}

static arc_status lsa_setup(arc_topk_ctx* c, cudaStream_t s) {
    const Plan& pl = c->pl;
    if (pl.topk || c->comm == nullptr) return pl.topk ? ARC_ERR_UNSUPPORTED : ARC_ERR_INVALID_ARG;
    Nccl& n = c->nccl;
    if (!n.memAlloc || !n.memFree || !n.winRegister || !n.winDeregister || !n.devCommCreate || !n.devCommDestroy ||
        !n.teamLsa)
        return ARC_ERR_UNSUPPORTED;   // NCCL older than 2.28
    const ncclTeam_t team = n.teamLsa(c->comm);
    if (team.nRanks != pl.G || pl.G > 72) return ARC_ERR_UNSUPPORTED;   // every rank in one NVLink domain
    if (cudaStreamSynchronize(s) != cudaSuccess) return ARC_ERR_CUDA;
    size_t bytes = (c->p.wire == ARC_WIRE_BF16 ? 2 : sizeof(float)) * static_cast<size_t>(std::max<int64_t>(pl.sumKn, 1)) * pl.L;
    bytes = (bytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
    if (n.memAlloc(&c->win_buf, bytes) != ncclSuccess) return ARC_ERR_NCCL;
    if (n.winRegister(c->comm, c->win_buf, bytes, &c->win, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess) return ARC_ERR_NCCL;
    if (pl.exchange && pl.keep_pnodes && !pl.randk && pl.M > 0) {   // exchange #1 window: [P' | Sigma]
        const size_t pn = sizeof(float) * static_cast<size_t>(pl.M) * pl.L * c->p.r;
        c->sk_sigma_off = (pn + 255) / 256 * 256;
        size_t sb = c->sk_sigma_off + sizeof(float) * static_cast<size_t>(std::max<int64_t>(pl.M, pl.G * pl.Ms));
        sb = (sb + NCCL_WIN_REQUIRED_ALIGNMENT - 1) / NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
        if (n.memAlloc(&c->sk_buf, sb) != ncclSuccess) return ARC_ERR_NCCL;
        if (n.winRegister(c->comm, c->sk_buf, sb, &c->sk_win, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess) return ARC_ERR_NCCL;
        c->lsa1 = true;
    }
    ncclDevCommRequirements_t reqs;
    std::memset(&reqs, 0, sizeof(reqs));
    reqs.lsaBarrierCount = arc::kLsaCtas;
    if (n.devCommCreate(c->comm, &reqs, &c->dev_comm) != ncclSuccess) return ARC_ERR_NCCL;
    c->dev_comm_ok = true;
    if (cudaMalloc(&c->dev_comm_d, sizeof(ncclDevComm)) != cudaSuccess ||
        cudaMemcpy(c->dev_comm_d, &c->dev_comm, sizeof(ncclDevComm), cudaMemcpyHostToDevice) != cudaSuccess)
        return ARC_ERR_CUDA;
    c->lsa = true;
    return ARC_OK;
}

extern "C" {

const char* arc_topk_status_string(arc_status s) {
    switch (s) {
        case ARC_OK: return "ok";
        case ARC_ERR_INVALID_ARG: return "invalid argument";
        case ARC_ERR_UNSUPPORTED: return "unsupported";
        case ARC_ERR_PARAM_MISMATCH: return "parameters differ across ranks";
        case ARC_ERR_CUDA: return "CUDA error";
        case ARC_ERR_NCCL: return "NCCL error";
        case ARC_ERR_NONFINITE: return "non-finite row importance";
    }
    return "unknown status";
}

arc_status arc_topk_workspace_bytes(const arc_topk_params* params_in, size_t* bytes) {
    if (bytes == nullptr) return ARC_ERR_INVALID_ARG;
    arc_topk_params np;
    arc_block one;
    const arc_status v = normalize(params_in, np, one);
    if (v != ARC_OK) return v;
    const arc_topk_params* params = &np;
    Plan pl;
    make_plan(params, pl);
    *bytes = pl.total;
    return ARC_OK;
}

arc_status arc_topk_create(const arc_topk_params* params_in, void* nccl_comm, void* workspace, size_t workspace_bytes,
                           void* stream, arc_topk_ctx** out) {
    if (out == nullptr) return ARC_ERR_INVALID_ARG;
    *out = nullptr;
    arc_topk_params np;
    arc_block one;
    const arc_status v = normalize(params_in, np, one);
    if (v != ARC_OK) return v;
    const arc_topk_params* params = &np;
    if (workspace == nullptr || (reinterpret_cast<uintptr_t>(workspace) % kAlign) != 0) return ARC_ERR_INVALID_ARG;
    arc_topk_ctx* c = new (std::nothrow) arc_topk_ctx();
    if (c == nullptr) return ARC_ERR_INVALID_ARG;
    c->p = *params;
    c->blocks.assign(params->blocks, params->blocks + params->num_blocks);
    c->p.blocks = c->blocks.data();
    make_plan(&c->p, c->pl);
    if (workspace_bytes < c->pl.total) { delete c; return ARC_ERR_INVALID_ARG; }
    {   // the select/gather kernel is cooperative: one CTA per slice, all co-resident
        // the smallest slice (multiple of 32 rows) whose slices all fit, so the
        // grid fills the GPU; ARC_SLICE_ROWS forces a size (experiments)
        const int resident = select_gather_resident_ctas();
        auto slices = [&](int rows) {
            int64_t n = 0;
            for (const BlockDev& B : c->pl.sbdev)
                if (!(c->pl.dense_fast && B.kind == ARC_BLOCK_DENSE)) n += (B.m + rows - 1) / rows;
            return n;
        };
        // (more slices than co-resident CTAs: the kernel is persistent, every CTA
        // takes ceil(slices / resident) of them, at most select_max_slices_per_cta())
        int rows = kSliceMin;
        while (rows < select_max_slice_rows() && slices(rows) > resident) rows += 32;
        // a small selection (<= 16 slices of the smallest height, one per CTA) runs
        // as one thread-block cluster: hardware barriers instead of grid barriers
        // through global memory and no cooperative launch (C5 d = 1e6: step 25.0 ->
        // 21.1 us).  Taller slices to fit a cluster measured slower (C1: 16 CTAs of
        // 4096 rows instead of 256 of 256: 20.9 -> 22.2 us), so only selections that
        // are small anyway take it (ARC_SELECT_CLUSTER: the largest cluster, 0 = off)
        c->sel_cluster = false;
        {
            int cl = 16;
            if (const char* e = std::getenv("ARC_SELECT_CLUSTER")) cl = std::atoi(e);
            const int64_t ns = slices(rows);
            if (cl > 0 && ns >= 1 && ns <= cl && select_cluster_max(static_cast<int>(ns)) == ns) c->sel_cluster = true;
        }
        if (const char* e = std::getenv("ARC_SLICE_ROWS")) {
            const int f = std::atoi(e);
            if (f >= kSliceMin && f <= select_max_slice_rows()) {
                rows = f;
                c->sel_cluster = false;
            }
        }
        int grid = static_cast<int>(std::min<int64_t>(slices(rows), resident));
        if (const char* e = std::getenv("ARC_SELECT_GRID")) {   // debug knob: fewer CTAs (several slices each)
            const int f = std::atoi(e);
            if (f >= 1 && f < grid) {
                grid = f;
                c->sel_cluster = false;
            }
        }
        if (grid > 0 && (slices(rows) + grid - 1) / grid > select_max_slices_per_cta()) {
            delete c;
            return ARC_ERR_UNSUPPORTED;
        }
        c->sel_grid = grid;
        const size_t total = c->pl.total;
        if (rows != kSliceMin) {
            c->pl = Plan();
            make_plan(&c->p, c->pl, rows);
            c->pl.total = total;   // fewer slices: the workspace laid out for 1024-row slices is larger
        }
    }
    c->ws = static_cast<unsigned char*>(workspace);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    c->last = s;

    const int G = c->pl.G;
    if ((params->flags & ARC_FLAG_LOOPBACK_COMM) != 0) {
        // the in-process loopback group (tests: G emulated ranks on one GPU)
        if (nccl_comm == nullptr) { delete c; return ARC_ERR_INVALID_ARG; }
        if (params->value_reduce == ARC_REDUCE_LSA) { delete c; return ARC_ERR_UNSUPPORTED; }
        c->lb = static_cast<LoopbackComm*>(nccl_comm);
        if (loopback_nranks(c->lb) != G || loopback_rank(c->lb) != (G > 1 ? params->rank : 0)) {
            delete c;
            return ARC_ERR_INVALID_ARG;
        }
        c->xc.lb = c->lb;
    } else if (G > 1) {
        if (nccl_comm == nullptr) { delete c; return ARC_ERR_INVALID_ARG; }
        if (!load_nccl(c->nccl)) { delete c; return ARC_ERR_NCCL; }
        c->comm = static_cast<ncclComm_t>(nccl_comm);
        int cnt = 0, rk = -1;
        if (c->nccl.commCount(c->comm, &cnt) != ncclSuccess || c->nccl.commUserRank(c->comm, &rk) != ncclSuccess) {
            delete c;
            return ARC_ERR_NCCL;
        }
        if (cnt != G || rk != params->rank) { delete c; return ARC_ERR_INVALID_ARG; }
    } else if (nccl_comm != nullptr) {
        if (!load_nccl(c->nccl)) { delete c; return ARC_ERR_NCCL; }
        c->comm = static_cast<ncclComm_t>(nccl_comm);
    }
    if (c->comm != nullptr) {
        c->xc.nccl = &c->nccl;
        c->xc.nc = c->comm;
    }

    // static tables
    std::vector<Tile> tiles;
    std::vector<int> cta_begin, cta_begin_w, cta_begin_t;
    {   // streaming-pass variant: 0 = 4 row segments per batch (>= 3 CTAs/SM),
        // 1 = 2 segments per batch at 4 CTAs/SM, 2 = 4 segments at 2 CTAs/SM
        // (ARC_SKETCH_SHAPE, experiments).  A row of n columns is ceil(n/128)
        // segments; the batch size that leaves fewer padded slots (weighted by
        // the blocks' bytes) wins: 3 for n = 768 (C3), 4 for n = 512, 1024,
        // 2048 (C2 -6 %, C5 -3 %, LLaMA layout -1 %, measured).
        double waste3 = 0.0, waste4 = 0.0;
        for (const BlockDev& B : c->pl.bdev) {
            if (B.kind != ARC_BLOCK_ARC) continue;
            const double nseg = static_cast<double>((B.n + 127) / 128);
            waste3 += static_cast<double>(B.len) * (1.0 - nseg / (std::ceil(nseg / 3.0) * 3.0));
            waste4 += static_cast<double>(B.len) * (1.0 - nseg / (std::ceil(nseg / 4.0) * 4.0));
        }
        c->shape = waste4 <= waste3 ? 2 : 0;
        {   // one node on this GPU, r <= 4, a few ARC blocks of full 16-byte-aligned rows of
            // whole 128-column segments: 3 segments per batch at 2 CTAs/SM (128 registers)
            // with the predicate-free loop (profiles/r02_sketch_shape5.txt: C3 step -1.6 %,
            // sketch at the measured HBM peak; C5 d = 1e9 -1.8 %; C2 one node equal; C4's
            // 171 blocks +1.4 % and several local nodes +7 % keep the rule above)
            // (layouts small enough for the fused tail keep its measured variant)
            int nb = 0, max_m = 0;
            bool full = c->pl.L == 1 && c->p.r <= 4 && !c->pl.topk && !c->pl.randk && !c->pl.noef;
            for (const BlockDev& B : c->pl.bdev) {
                if (B.kind != ARC_BLOCK_ARC) continue;
                ++nb;
                max_m = std::max(max_m, B.m);
                full = full && B.vec && B.n % 128 == 0;
            }
            if (full && nb >= 1 && nb <= 8 && max_m > kTailMaxRows) c->shape = 5;
        }
        if (const char* e = getenv("ARC_SKETCH_SHAPE")) {
            const int v = atoi(e);
            if (sketch_shape_ok(v, c->p.r)) c->shape = v;
        }
    }
    {
        // blocks whose V_b^T fits the shared-memory stage stream in one launch; the
        // wider ones (methods with a sketch) and blocks of rows of <= 4 columns (one
        // row per thread) in a second launch, so the main kernel carries neither path
        //
        // Blocks of the sketch methods (EF21M) whose rows are not 16-byte aligned
        // (n >= 256) go to a third launch fed by bulk copies (arc_sketch_tma.cu)
        // when their V_b^T fits next to its rings: the main launch would read them
        // with scalar loads (ARC_SKETCH_TMA: 0 = off, 2 = every ARC block of more
        // than 4 columns, for A/B runs)
        const bool sketches = !c->pl.topk && !c->pl.randk;
        int tma_mode = 1;
        if (const char* e = getenv("ARC_SKETCH_TMA")) tma_mode = atoi(e);
        const int tma_cap = sketches && !c->pl.noef && tma_mode > 0 ? sketch_tma_vs_cap(c->p.r) : 0;
        std::vector<char> narrow(c->pl.bdev.size(), 1), wide(c->pl.bdev.size(), 0), viatma(c->pl.bdev.size(), 0);
        c->vs_cap = 0;
        c->vs_cap_t = 0;
        bool any_wide = false, any_tma = false;
        for (size_t b = 0; b < c->pl.bdev.size(); ++b) {
            const BlockDev& B = c->pl.bdev[b];
            if (B.kind != ARC_BLOCK_ARC) continue;
            const int cap = sketch_vs_cap(c->p.r, B.n);
            const int64_t need = static_cast<int64_t>(c->p.r) * ((B.n + 3) / 4 * 4);
            if (B.n > 4 && need <= tma_cap && (tma_mode >= 2 || (!B.vec && B.n >= 256))) {
                narrow[b] = 0;
                viatma[b] = 1;
                any_tma = true;
                c->vs_cap_t = std::max<int>(c->vs_cap_t, static_cast<int>(need));
            } else if (((cap == 0 && sketches) || B.n <= 4) && sketch_ranged_cap(c->p.r) > 0) {
                narrow[b] = 0;
                wide[b] = 1;
                any_wide = true;
            } else {
                c->vs_cap = std::max(c->vs_cap, cap);
            }
        }
        {   // the fused small-problem tail (arc_sketch.cu): S3 in the streaming launch's
            // last CTA (+ S4..S6 in a small update kernel) when the GPU holds the one node,
            // there is no exchange and every ARC block's keys fit that CTA's shared memory
            // (ARC_TAIL=0: off, the selection kernel instead)
            const Plan& P = c->pl;
            int arc_blocks = 0, max_m = 0;
            for (const BlockDev& B : P.bdev)
                if (B.kind == ARC_BLOCK_ARC) {
                    ++arc_blocks;
                    max_m = std::max(max_m, B.m);
                }
            bool on = true;
            if (const char* e = getenv("ARC_TAIL")) on = e[0] != '0';
            const int r_eff = P.randk ? 1 : c->p.r;
            c->tail = on && !P.exchange && P.L == 1 && c->p.N == 1 && !P.topk && !P.exact && !any_wide && !any_tma &&
                      r_eff <= 8 && arc_blocks >= 1 && arc_blocks <= kTailMaxBlocks && max_m <= kTailMaxRows;
            c->tail_keys = max_m;
        }
        // (the tail's launch may stage more shared memory than V_b^T: its keys)
        const int resident = c->tail ? ef_sketch_resident_ctas_tail(c->p.r, c->shape, c->pl.noef,
                                                                    std::max(c->vs_cap, c->tail_keys))
                                     : ef_sketch_resident_ctas(c->p.r, c->shape, c->vs_cap);
        plan_tiles(c->pl, narrow, resident, sketch_tile_rows(c->shape), sketch_tile_cols(c->shape), tiles, cta_begin,
                   c->grid);
        if (c->grid <= 0) c->tail = false;

        c->grid_w = 0;
        if (any_wide) {
            // shared memory: the widest fully staged V_b^T, or the range stage
            // (rows of <= 4 columns read V from global memory)
            const int cap_w = sketch_ranged_cap(c->p.r);
            c->vs_cap_w = 0;
            for (size_t b = 0; b < c->pl.bdev.size(); ++b) {
                const BlockDev& B = c->pl.bdev[b];
                if (wide[b] && B.n > 4)
                    c->vs_cap_w = std::max<int>(c->vs_cap_w, std::min<int64_t>(cap_w, c->p.r * ((B.n + 3) / 4 * 4)));
            }
            std::vector<Tile> tw;
            std::vector<int> cbw;
            plan_tiles(c->pl, wide, ef_sketch_resident_ctas_ranged(c->p.r, c->vs_cap_w), 32, sketch_tile_cols(c->shape),
                       tw, cbw, c->grid_w, sketch_wide_threads(c->p.r));
            c->tiles_w0 = static_cast<int>(tiles.size());
            for (int& x : cbw) x += c->tiles_w0;
            tiles.insert(tiles.end(), tw.begin(), tw.end());
            cta_begin_w = std::move(cbw);
        }
        c->grid_t = 0;
        if (any_tma) {
            std::vector<Tile> tt;
            std::vector<int> cbt;
            int sms = 0, dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            plan_tiles(c->pl, viatma, std::max(sms, 1), 32, sketch_tile_cols(c->shape), tt, cbt, c->grid_t);
            const int t0 = static_cast<int>(tiles.size());
            for (int& x : cbt) x += t0;
            tiles.insert(tiles.end(), tt.begin(), tt.end());
            cta_begin_t = std::move(cbt);
        }
    }
    c->num_tiles = static_cast<int>(tiles.size());
    std::vector<TileDesc> tdesc(tiles.size());
    for (size_t i = 0; i < tiles.size(); ++i) {
        const BlockDev& B = c->pl.bdev[tiles[i].b];
        TileDesc& D = tdesc[i];
        D = TileDesc{};
        D.off = B.off;
        D.len = B.len;
        D.v_off = B.v_off;
        D.n = B.n;
        D.row0 = tiles[i].row0;
        D.rows = tiles[i].rows;
        D.vec = B.vec;
        D.row_base = B.row_base;
        D.b = tiles[i].b;
        D.node = tiles[i].node;
    }
    const std::vector<SelRow>& rows = c->pl.segs;

#define UPLOAD(off, vec) \
    if (!(vec).empty()) ARC_CUDA(cudaMemcpyAsync(c->ws + (off), (vec).data(), sizeof((vec)[0]) * (vec).size(), cudaMemcpyHostToDevice, s))
    do {
        arc_status st = ARC_OK;
        auto up = [&]() -> arc_status {
            UPLOAD(c->pl.o_blocks, c->pl.bdev);
            UPLOAD(c->pl.o_sblocks, c->pl.sbdev);
            UPLOAD(c->pl.o_segs_real, c->pl.segs_real);
            UPLOAD(c->pl.o_dense_ids, c->pl.dense_ids);
            UPLOAD(c->pl.o_tiles, tdesc);
            UPLOAD(c->pl.o_cta, cta_begin);
            UPLOAD(c->pl.o_cta_w, cta_begin_w);
            UPLOAD(c->pl.o_cta_t, cta_begin_t);
            UPLOAD(c->pl.o_selrows, rows);
            UPLOAD(c->pl.o_items, c->pl.items);
            ARC_CUDA(cudaMemsetAsync(c->ws + c->pl.o_cand_count, 0, sizeof(unsigned) * 2 * c->pl.sbdev.size(), s));
            ARC_CUDA(cudaMemsetAsync(c->ws + c->pl.o_bnd_count, 0, sizeof(unsigned) * 2, s));
            ARC_CUDA(cudaMemsetAsync(c->ws + c->pl.o_hist2, 0, sizeof(unsigned) * 2048 * c->pl.sbdev.size(), s));
            ARC_CUDA(cudaMemsetAsync(c->ws + c->pl.o_hist3, 0, sizeof(unsigned) * 1024 * c->pl.sbdev.size(), s));
            ARC_CUDA(cudaMemsetAsync(c->ws + c->pl.o_status, 0, 16, s));
            ARC_CUDA(cudaMemsetAsync(c->ws + c->pl.o_tdev, 0, 16, s));   // ARC_FLAG_DEVICE_T: t = 0
            ARC_CUDA(cudaMemsetAsync(c->ws + c->pl.o_hist1, 0, sizeof(unsigned) * kHist1Bins * c->pl.sbdev.size(), s));
            ARC_CUDA(cudaStreamSynchronize(s));
            return ARC_OK;
        };
        st = up();
        if (st != ARC_OK) { delete c; return st; }
    } while (0);
#undef UPLOAD

    for (const BlockDev& B : c->pl.bdev)
        if (B.kind == ARC_BLOCK_ARC) c->v_items += static_cast<int64_t>((B.n + 3) / 4 * 4) * ((c->p.r + 3) / 4);
    if (const char* e = getenv("ARC_PDL")) c->pdl = e[0] != '0';
    if (const char* e = getenv("ARC_EARLY")) c->early = e[0] != '0';
    c->ome = 1.0f - c->p.eta;                       // R11, fp32
    c->Nf = static_cast<float>(c->p.N);             // R3

    if (G > 1) {   // every rank checks that all ranks passed identical params
        const uint64_t mine = params_hash(&c->p);
        uint64_t* dh = c->at<uint64_t>(c->pl.o_hash);
        std::vector<uint64_t> all(G, 0);
        if (cudaMemcpyAsync(dh + G, &mine, 8, cudaMemcpyHostToDevice, s) != cudaSuccess ||
            c->xc.all_gather_bytes(dh + G, dh, 8, s) != ARC_OK ||
            cudaMemcpyAsync(all.data(), dh, 8 * G, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) {
            delete c;
            return ARC_ERR_NCCL;
        }
        for (uint64_t x : all)
            if (x != mine) { delete c; return ARC_ERR_PARAM_MISMATCH; }
    }
    if (c->p.value_reduce == ARC_REDUCE_LSA && (c->pl.exchange || c->pl.topk)) {
        const arc_status ls = lsa_setup(c, s);
        if (ls != ARC_OK) { lsa_release(c); delete c; return ls; }
    }
    if (const char* e = getenv("ARC_DEBUG_STAMPS")) {
        if (e[0] == '1' && cudaMalloc(&c->stamps, sizeof(unsigned long long) * 8 * c->pl.items.size()) != cudaSuccess)
            c->stamps = nullptr;
    }
    *out = c;
    return ARC_OK;
}

static arc_status mark(arc_topk_ctx* c, int phase_edge, cudaStream_t s) {
    if (!c->timing) return ARC_OK;
    const size_t idx = static_cast<size_t>(c->timed_steps) * (ARC_TIMING_PHASES + 1) + phase_edge;
    while (c->ev_pool.size() <= idx) {
        cudaEvent_t e;
        ARC_CUDA(cudaEventCreate(&e));
        c->ev_pool.push_back(e);
    }
    ARC_CUDA(cudaEventRecord(c->ev_pool[idx], s));
    return ARC_OK;
}
#define ARC_MARK(edge)                                          \
    do {                                                        \
        const arc_status ms_ = mark(c, (edge), s);              \
        if (ms_ != ARC_OK) return ms_;                          \
    } while (0)

static arc_status run_step(arc_topk_ctx* c, int64_t t, const float* const* grad, float* const* h, float* const* g,
                           float* gbar, int32_t* sel_out, float* values_out, cudaStream_t s) {
    const Plan& pl = c->pl;
    const int L = pl.L;
    NodePtrs np{};
    // base pointers must be 16-byte aligned (the kernels' vector accesses; the ABI)
    auto misaligned = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15u) != 0; };
    for (int i = 0; i < L; ++i) {
        if (grad[i] == nullptr || misaligned(grad[i])) return ARC_ERR_INVALID_ARG;
        np.grad[i] = grad[i];
        if (pl.noef) continue;   // without EF there is no (h, g) state: h, g may be NULL
        if (h == nullptr || g == nullptr || h[i] == nullptr || g[i] == nullptr) return ARC_ERR_INVALID_ARG;
        if (misaligned(h[i]) || misaligned(g[i])) return ARC_ERR_INVALID_ARG;
        np.h[i] = h[i];
        np.g[i] = g[i];
    }
    if (gbar == nullptr || misaligned(gbar)) return ARC_ERR_INVALID_ARG;
    if ((sel_out != nullptr && (reinterpret_cast<uintptr_t>(sel_out) & 3u)) || (values_out != nullptr && misaligned(values_out)))
        return ARC_ERR_INVALID_ARG;
    c->last = s;
    const BlockDev* blocks = c->at<BlockDev>(pl.o_blocks);
    float* V = c->at<float>(pl.o_V);
    float* sigma = c->sigma_ptr();
    int32_t* sel = c->at<int32_t>(pl.o_sel);
    unsigned* status = c->at<unsigned>(pl.o_status);
    unsigned* hist1 = c->at<unsigned>(pl.o_hist1);
    const SelRow* rows = c->at<SelRow>(pl.o_selrows);
    const BlockDev* sblocks = c->at<BlockDev>(pl.o_sblocks);
    if (pl.topk && (sel_out != nullptr || values_out != nullptr)) return ARC_ERR_INVALID_ARG;

    ARC_MARK(0);
    // ARC_FLAG_DEVICE_T: t is the device counter (read by the kernels, advanced by
    // the selection kernel); V single-buffered and drawn by every step
    const bool dev_t = (c->p.flags & ARC_FLAG_DEVICE_T) != 0;
    unsigned long long* t_dev = dev_t ? c->at<unsigned long long>(pl.o_tdev) : nullptr;
    if (dev_t) t = 0;
    // S0 (skipped when the previous step already generated V for this t)
    float* V_t = V + static_cast<size_t>(dev_t ? 0 : (t & 1)) * pl.sum_nr;
    // (a captured step always draws its own V: a replay must not depend on what
    // eager steps between capture and replay left in the double buffer)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) return ARC_ERR_CUDA;
    if (pl.M > 0 && !pl.topk && !pl.randk && (dev_t || c->v_ready != t || cap != cudaStreamCaptureStatusNone)) {
        launch_vgen(blocks, c->p.num_blocks, pl.max_nR4, c->p.r, c->p.seed, t, V_t, s, t_dev, c->pdl && !c->timing ? 1 : 0);
        ARC_LAUNCHED();
    }
    c->last_t = t;
    // S1 (+S2)
    if (pl.M > 0) {
        SketchLaunch a{};
        a.blocks = blocks;
        a.tiles = c->at<TileDesc>(pl.o_tiles);
        a.cta_begin = c->at<int>(pl.o_cta);
        a.num_tiles = c->num_tiles;
        a.grid = c->grid;
        a.nodes = np;
        a.nodes_local = L;
        a.N = c->p.N;
        a.r = c->p.r;
        a.eta = c->p.eta;
        a.ome = c->ome;
        a.Nf = c->Nf;
        a.V = V_t;
        a.t_dev = t_dev;
        a.sigma = sigma;
        a.hist1 = hist1;
        a.pnodes = pl.keep_pnodes ? c->pnodes_ptr() : nullptr;
        a.mode = pl.topk ? 2 : pl.randk ? 3 : ((pl.exchange || L > 1 || pl.exact) ? 1 : 0);
        a.key = make_uint2(static_cast<unsigned>(c->p.seed), static_cast<unsigned>(c->p.seed >> 32));
        a.t_lo = static_cast<unsigned>(static_cast<uint64_t>(t));
        a.t_hi = static_cast<unsigned>(static_cast<uint64_t>(t) >> 32);
        a.M = pl.M;
        a.num_blocks = c->p.num_blocks;
        a.shape = c->shape;
        a.vs_cap = c->vs_cap;
        a.pdl = c->pdl && !c->timing ? 1 : 0;
        a.status = status;
        ARC_MARK(1);
        a.noef = pl.noef ? 1 : 0;
        a.gbar = gbar;
        if (c->tail) {   // S3..S6 in the last CTA (no selection kernel this step)
            TailArgs& ta = a.tail;
            ta.done = status + 2;
            ta.sel = sel;
            ta.values = values_out;
            ta.bf16 = c->p.wire == ARC_WIRE_BF16 ? 1 : 0;
            ta.N_int = c->p.N;
            ta.t_advance = t_dev;
            ta.key_cap = c->tail_keys;
            ta.stamps = c->stamps;
            ta.nblk = 0;
            ta.quads = 0;
            for (const BlockDev& B : pl.bdev) {
                if (B.kind != ARC_BLOCK_ARC) continue;
                TailBlk& tb = ta.blk[ta.nblk++];
                tb.off = B.off;
                tb.len = B.len;
                tb.val_base = B.val_base;
                tb.q_begin = ta.quads;
                tb.n = B.n;
                tb.K = B.K;
                tb.sel_base = B.sel_base;
                tb.vec = B.vec;
                ta.quads += static_cast<long long>(B.K) * ((B.n + 3) / 4);
            }
            const bool spec = !pl.randk && t < INT64_MAX && !dev_t;
            if (spec) {
                const uint64_t tn = static_cast<uint64_t>(t + 1);
                ta.V_next = V + static_cast<size_t>((t + 1) & 1) * pl.sum_nr;
                ta.v_items = c->v_items;
                ta.tn_lo = static_cast<unsigned>(tn);
                ta.tn_hi = static_cast<unsigned>(tn >> 32);
            }
            ta.last_cta = status + 3;
            ta.sk_grid = c->grid;
        }
        if (c->grid > 0) {
            launch_ef_sketch(a, s);
            ARC_LAUNCHED();
            if (c->tail) {   // S4..S6 of the tail's selection
                launch_tail_update(a, s);
                ARC_LAUNCHED();
            }
        }
        if (c->grid_w > 0) {   // blocks with V_b^T wider than the stage
            a.cta_begin = c->at<int>(pl.o_cta_w);
            a.grid = c->grid_w;
            a.vs_cap = c->vs_cap_w;
            a.ranged = 1;
            launch_ef_sketch(a, s);
            ARC_LAUNCHED();
        }
        if (c->grid_t > 0) {   // unaligned rows / wide V through the bulk-copy rings
            a.cta_begin = c->at<int>(pl.o_cta_t);
            a.grid = c->grid_t;
            a.vs_cap = c->vs_cap_t;
            a.ranged = 0;
            launch_ef_sketch_tma(a, s);
            ARC_LAUNCHED();
        }
    } else {
        ARC_MARK(1);
    }
    ARC_MARK(2);
    // (DENSE blocks skip the sketch pass: the select/gather kernel applies their momentum.)
    // Exchange #1 + S2 (Rand-K needs none: every rank draws the same keys).  Rank j
    // owns rows [j Ms, (j+1) Ms) of the M ARC rows: an all-to-all brings it those
    // rows' per-node sketches from every rank, k_sigma_slice sums them in global
    // node order and forms Sigma, and an all-gather of the Sigma slices gives
    // every rank all of Sigma.  (Several local nodes and no exchange: the select
    // kernel forms Sigma from the per-node sketches itself, phase 0.)
    const bool sigma_pass = (pl.exchange || L > 1 || pl.exact) && !pl.randk && !pl.topk && pl.M > 0;
    if (sigma_pass && pl.exchange && c->lsa1) {   // exchange #1 + S2 over peer memory
        LsaSigma ls{};
        ls.dev_comm = c->dev_comm_d;
        ls.win = c->sk_win;
        ls.sigma_off = c->sk_sigma_off;
        ls.sigma = sigma;
        ls.Ms = pl.Ms;
        ls.M = pl.M;
        ls.G = pl.G;
        ls.me = pl.G > 1 ? c->p.rank : 0;
        ls.L = L;
        ls.r = c->p.r;
        ls.status = status;
        launch_lsa_sigma(ls, s);
        ARC_LAUNCHED();
    } else if (sigma_pass && pl.exchange) {
        const int G = pl.G;
        const int me = G > 1 ? c->p.rank : 0;
        const int64_t Ms = pl.Ms;
        const size_t row_floats = static_cast<size_t>(L) * c->p.r;
        auto slice_rows = [&](int j) { return std::max<int64_t>(0, std::min<int64_t>(pl.M, (j + 1) * Ms) - j * Ms); };
        float* xs = c->at<float>(pl.o_pnodes);
        const float* x = xs;
        if (pl.exchange && c->xc.any()) {
            // rank j owns rows [j Ms, (j+1) Ms): send it those rows' sketches of
            // this GPU's nodes, receive this rank's rows from every rank
            float* xr = c->at<float>(pl.o_xrecv);
            std::vector<size_t> sc(G), sd(G), rc(G), rd(G);
            for (int j = 0; j < G; ++j) {
                sc[j] = static_cast<size_t>(slice_rows(j)) * row_floats;
                sd[j] = static_cast<size_t>(j) * Ms * row_floats;
                rc[j] = static_cast<size_t>(slice_rows(me)) * row_floats;
                rd[j] = static_cast<size_t>(j) * Ms * row_floats;
                if (j != me) c->tally[kTallySketch] += static_cast<int64_t>(sc[j]);
            }
            const arc_status xs_st = c->xc.all_to_all_f32(xs, sc.data(), sd.data(), xr, rc.data(), rd.data(), G, s);
            if (xs_st != ARC_OK) return xs_st;
            ++c->tally[kTallyCalls];
            x = xr;
        }
        SigmaLaunch sl{};
        sl.x = x;
        sl.Ms = Ms;
        sl.rows = slice_rows(me);
        sl.G = G;
        sl.L = L;
        sl.r = c->p.r;
        sl.Nf = c->Nf;
        sl.sigma = sigma + me * Ms;
        sl.status = status;
        launch_sigma_slice(sl, s);
        ARC_LAUNCHED();
        if (pl.exchange && c->xc.any()) {
            const arc_status ag = c->xc.all_gather_f32(sigma + me * Ms, sigma, static_cast<size_t>(Ms), s);
            if (ag != ARC_OK) return ag;
            c->tally[kTallySigma] += Ms;
            ++c->tally[kTallyCalls];
        }
    }
    if (sigma_pass && pl.exact) {   // test mode: Sigma from the exact row norms of the node sum
        ExactSigmaLaunch ex{};
        ex.blocks = blocks;
        ex.num_blocks = c->p.num_blocks;
        ex.L = L;
        ex.nodes = np;
        ex.sigma = sigma;
        ex.status = status;
        launch_exact_sigma(ex, s);
        ARC_LAUNCHED();
    }
    ARC_MARK(3);
    // S3 + S4 (+ S5, S6 when every node is local): one cooperative kernel
    GatherLaunch ga{};
    ga.blocks = blocks;
    ga.rows = rows;
    ga.num_rows = static_cast<int>(pl.num_segs);
    ga.sel = sel;
    ga.nodes = np;
    ga.nodes_local = L;
    ga.eta = c->p.eta;
    ga.ome = c->ome;
    ga.Nf = c->Nf;
    ga.N_int = c->p.N;
    ga.sum_Kn = pl.sumKn;
    ga.noef = pl.noef ? 1 : 0;
    ga.bnd = c->at<int2>(pl.o_bnd);
    ga.bnd_count = c->at<unsigned>(pl.o_bnd_count);
    const int bf16 = c->p.wire == ARC_WIRE_BF16 ? 1 : 0;   // R25
    const size_t we = bf16 ? 2 : sizeof(float);           // payload entry bytes
    ga.bf16 = bf16;
    const bool ordered = c->p.value_reduce != ARC_REDUCE_NCCL;   // ORDERED and LSA: per-node payloads
    float* wire = c->lsa ? static_cast<float*>(c->win_buf)
                         : ((pl.exchange || pl.topk) ? c->at<float>(pl.o_wire) : nullptr);
    ga.blocks = sblocks;
    if (pl.topk) {   // baseline: each node's payload [values | indices] in the wire
        ga.mode = 3;
        ga.values = wire;
        ga.sel = reinterpret_cast<const int32_t*>(wire);
    } else if (!pl.exchange) {
        ga.mode = 0;
        ga.gbar = gbar;
        ga.values = values_out;
    } else {
        ga.mode = ordered ? 2 : 1;
        ga.values = wire;
    }
    {
        SelectGatherLaunch sg{};
        sg.blocks = sblocks;
        sg.items = c->at<SliceItem>(pl.o_items);
        sg.num_items = static_cast<int>(pl.items.size());
        sg.grid = std::min(c->sel_grid, sg.num_items);
        sg.slice_rows = pl.slice_rows;
        sg.sigma = sigma;
        sg.hist1 = hist1;
        sg.hist2 = c->at<unsigned>(pl.o_hist2);
        sg.hist3 = c->at<unsigned>(pl.o_hist3);
        sg.slice_gt = c->at<int>(pl.o_slice_gt);
        sg.slice_eq = c->at<int>(pl.o_slice_eq);
        sg.cand = c->at<unsigned>(pl.o_cand);
        sg.cand_count = c->at<unsigned>(pl.o_cand_count);
        sg.num_blocks = static_cast<int>(pl.sbdev.size());
        sg.parity = status + 1;   // device-side parity word (status[1])
        sg.sel = pl.topk ? reinterpret_cast<int32_t*>(wire) : sel;
        sg.stamps = c->stamps;
        sg.pdl = c->pdl && !c->timing && !(pl.exchange && pl.M > 0) ? 1 : 0;
        sg.early = c->early && ga.mode == 0 && ga.values == nullptr ? 1 : 0;
        sg.cluster = c->sel_cluster && sg.grid == sg.num_items ? 1 : 0;
        sg.build_hist = sigma_pass ? 1 : 0;
        if (sigma_pass && !pl.exchange && !pl.exact) {
            sg.xsk = c->pnodes_ptr();
            sg.sigma_w = sigma;
            sg.L = L;
            sg.Nf = c->Nf;
            sg.status = status;
        }
        const bool spec = pl.M > 0 && !pl.topk && !pl.randk && t < INT64_MAX && !dev_t;
        sg.t_advance = t_dev;
        sg.r = c->p.r;   // (phase 0 forms Sigma over r sketch columns)
        if (spec) {
            const uint64_t tn = static_cast<uint64_t>(t + 1);
            sg.vblocks = blocks;
            sg.num_vblocks = c->p.num_blocks;
            sg.V_next = V + static_cast<size_t>((t + 1) & 1) * pl.sum_nr;
            sg.v_items = c->v_items;
            sg.r = c->p.r;
            sg.key = make_uint2(static_cast<unsigned>(c->p.seed), static_cast<unsigned>(c->p.seed >> 32));
            sg.t_lo = static_cast<unsigned>(tn);
            sg.t_hi = static_cast<unsigned>(tn >> 32);
        }
        if (c->tail && pl.M > 0) {   // (S3..S6, the next V and the t advance ran in the streaming launch)
            c->v_ready = (!pl.randk && t < INT64_MAX && !dev_t) ? t + 1 : -1;
            t_dev = nullptr;
        } else {
            c->v_ready = (spec && sg.num_items > 0) ? t + 1 : -1;
            if (sg.num_items > 0 && launch_select_gather(sg, ga, s) != cudaSuccess) {
                (void)cudaGetLastError();
                return ARC_ERR_CUDA;
            }
            if (sg.num_items > 0) t_dev = nullptr;   // (advanced by the selection kernel)
        }
    }
    if (!pl.dense_ids.empty()) {   // DENSE blocks: identity compressor, streaming
        DenseLaunch dl{};
        dl.blocks = blocks;
        dl.dense_ids = c->at<int>(pl.o_dense_ids);
        dl.num_dense = static_cast<int>(pl.dense_ids.size());
        dl.nodes = np;
        dl.nodes_local = L;
        dl.eta = c->p.eta;
        dl.ome = c->ome;
        dl.Nf = c->Nf;
        dl.N_int = c->p.N;
        dl.gbar = gbar;
        dl.sel = sel;
        dl.mode = !pl.exchange ? 0 : (ordered ? 2 : 1);
        dl.noef = pl.noef ? 1 : 0;
        dl.values = !pl.exchange ? values_out : nullptr;
        dl.payload = pl.exchange ? static_cast<void*>(wire) : nullptr;
        dl.bf16 = bf16;
        dl.sum_Kn = pl.sumKn;
        launch_dense(dl, s);
        ARC_LAUNCHED();
    }
    ARC_MARK(4);
    if (pl.topk) {   // baseline: all-gather the payloads, merge them in node order
        const float* all = wire;
        if (pl.G > 1) {
            float* dst = c->at<float>(pl.o_wire_all);
            const arc_status ag = c->xc.all_gather_f32(wire, dst, static_cast<size_t>(pl.W) * L, s);
            if (ag != ARC_OK) return ag;
            c->tally[kTallyValues] += pl.W * L;
            ++c->tally[kTallyCalls];
            all = dst;
        }
        for (int j = 0; j < c->p.N; ++j) {
            MergeLaunch ml{};
            ml.blocks = blocks;
            ml.rows = c->at<SelRow>(pl.o_segs_real);
            ml.num_rows = static_cast<int>(pl.segs_real.size());
            ml.values = all + static_cast<size_t>(j) * pl.W;
            ml.idx = reinterpret_cast<const int32_t*>(all + static_cast<size_t>(j) * pl.W + pl.sumKn);
            ml.Nf = c->Nf;
            ml.N_int = c->p.N;
            ml.gbar = gbar;
            launch_topk_merge(ml, s);
            ARC_LAUNCHED();
        }
    } else if (pl.exchange && c->lsa) {   // exchange #2 fused with S6 over peer memory
        LsaScatter x{};
        x.dev_comm = c->dev_comm_d;
        x.win = c->win;
        x.G = pl.G;
        x.L = L;
        x.N = c->p.N;
        x.sum_Kn = pl.sumKn;
        x.bf16 = bf16;
        if (!pl.segs_real.empty()) {
            ScatterLaunch sa{};
            sa.blocks = blocks;
            sa.rows = c->at<SelRow>(pl.o_segs_real);
            sa.num_rows = static_cast<int>(pl.segs_real.size());
            sa.sel = sel;
            sa.sum_Kn = pl.sumKn;
            sa.Nf = c->Nf;
            sa.N_int = c->p.N;
            sa.gbar = gbar;
            sa.values = values_out;
            launch_lsa_scatter(sa, x, s);
            ARC_LAUNCHED();
        }
        if (!pl.dense_ids.empty()) {
            DenseScatterLaunch ds{};
            ds.blocks = blocks;
            ds.dense_ids = c->at<int>(pl.o_dense_ids);
            ds.num_dense = static_cast<int>(pl.dense_ids.size());
            ds.sum_Kn = pl.sumKn;
            ds.Nf = c->Nf;
            ds.N_int = c->p.N;
            ds.gbar = gbar;
            ds.values = values_out;
            launch_lsa_dense_scatter(ds, x, s);
            ARC_LAUNCHED();
        }
    } else if (pl.exchange) {   // exchange #2 + S6
        const void* reduced = wire;
        if (!ordered) {
            if (c->xc.any() && pl.G > 1) {
                const arc_status ar = bf16 ? c->xc.all_reduce_bf16(wire, wire, static_cast<size_t>(pl.sumKn), s)
                                           : c->xc.all_reduce_f32(wire, wire, static_cast<size_t>(pl.sumKn), s);
                if (ar != ARC_OK) return ar;
                c->tally[kTallyValues] += pl.sumKn;
                ++c->tally[kTallyCalls];
            }
        } else {
            void* all = c->ws + pl.o_wire_all;
            const size_t cnt = static_cast<size_t>(pl.sumKn) * L;
            if (c->xc.any()) {
                const arc_status ag = c->xc.all_gather_bytes(wire, all, cnt * we, s);
                if (ag != ARC_OK) return ag;
                c->tally[kTallyValues] += static_cast<int64_t>(cnt);
                ++c->tally[kTallyCalls];
            } else {
                ARC_CUDA(cudaMemcpyAsync(all, wire, cnt * we, cudaMemcpyDeviceToDevice, s));
            }
            reduced = all;
        }
        ScatterLaunch sa{};
        sa.blocks = blocks;
        sa.rows = c->at<SelRow>(pl.o_segs_real);
        sa.num_rows = static_cast<int>(pl.segs_real.size());
        sa.sel = sel;
        sa.wire = reduced;
        sa.bf16 = bf16;
        sa.mode = ordered ? 1 : 0;
        sa.nodes_total = c->p.N;
        sa.sum_Kn = pl.sumKn;
        sa.Nf = c->Nf;
        sa.N_int = c->p.N;
        sa.gbar = gbar;
        sa.values = values_out;
        if (sa.num_rows > 0) {
            launch_scatter(sa, s);
            ARC_LAUNCHED();
        }
        if (!pl.dense_ids.empty()) {
            DenseScatterLaunch ds{};
            ds.blocks = blocks;
            ds.dense_ids = c->at<int>(pl.o_dense_ids);
            ds.num_dense = static_cast<int>(pl.dense_ids.size());
            ds.wire = reduced;
            ds.bf16 = bf16;
            ds.mode = ordered ? 1 : 0;
            ds.nodes_total = c->p.N;
            ds.sum_Kn = pl.sumKn;
            ds.Nf = c->Nf;
            ds.N_int = c->p.N;
            ds.gbar = gbar;
            ds.values = values_out;
            launch_dense_scatter(ds, s);
            ARC_LAUNCHED();
        }
    }
    ARC_MARK(5);
    if (sel_out != nullptr)
        ARC_CUDA(cudaMemcpyAsync(sel_out, sel, sizeof(int32_t) * pl.sumK, cudaMemcpyDeviceToDevice, s));
    if (t_dev != nullptr) {   // ARC_FLAG_DEVICE_T and no selection kernel ran: advance t here
        launch_advance_t(t_dev, s);
        ARC_LAUNCHED();
    }
    ARC_MARK(6);
    if (c->timing) ++c->timed_steps;
    ++c->tally[kTallySteps];
    return ARC_OK;
}

arc_status arc_topk_step(arc_topk_ctx* c, int64_t t, const float* const* grad, float* const* h, float* const* g,
                         float* gbar, int32_t* sel_out, float* values_out, void* stream) {
    if (c == nullptr || grad == nullptr || gbar == nullptr) return ARC_ERR_INVALID_ARG;   // (h, g: checked per method)
    return run_step(c, t, grad, h, g, gbar, sel_out, values_out, static_cast<cudaStream_t>(stream));
}

arc_status arc_topk_set_iteration(arc_topk_ctx* c, int64_t t, void* stream) {
    if (c == nullptr || t < 0 || !(c->p.flags & ARC_FLAG_DEVICE_T)) return ARC_ERR_INVALID_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const unsigned long long v = static_cast<unsigned long long>(t);
    // (a kernel, not a host copy: the value travels as an argument, so the call is
    // also legal inside a stream capture)
    launch_set_u64(c->at<unsigned long long>(c->pl.o_tdev), v, s);
    if (cudaGetLastError() != cudaSuccess) return ARC_ERR_CUDA;
    c->last = s;
    return ARC_OK;
}

arc_status arc_topk_step_host(arc_topk_ctx* c, int64_t t, const float* const* grad_host, float* const* h,
                              float* const* g, float* gbar, int32_t* sel_host, float* values_host, void* stream) {
    if (c == nullptr || grad_host == nullptr || gbar == nullptr) return ARC_ERR_INVALID_ARG;
    if (!(c->p.flags & ARC_FLAG_HOST_STAGING)) return ARC_ERR_INVALID_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int L = c->pl.L;
    const float* dgrad[ARC_MAX_NODES_LOCAL];
    float* stage = c->at<float>(c->pl.o_staging);
    for (int i = 0; i < L; ++i) {
        if (grad_host[i] == nullptr) return ARC_ERR_INVALID_ARG;
        float* dst = stage + static_cast<size_t>(i) * ((c->p.d + 63) / 64 * 64);
        ARC_CUDA(cudaMemcpyAsync(dst, grad_host[i], sizeof(float) * c->p.d, cudaMemcpyHostToDevice, s));
        dgrad[i] = dst;
    }
    float* vals = c->at<float>(c->pl.o_vals);
    if (c->pl.topk && (sel_host != nullptr || values_host != nullptr)) return ARC_ERR_INVALID_ARG;
    const arc_status st = run_step(c, t, dgrad, h, g, gbar, nullptr, values_host ? vals : nullptr, s);
    if (st != ARC_OK) return st;
    if (sel_host != nullptr)
        ARC_CUDA(cudaMemcpyAsync(sel_host, c->at<int32_t>(c->pl.o_sel), sizeof(int32_t) * c->pl.sumK,
                                 cudaMemcpyDeviceToHost, s));
    if (values_host != nullptr)
        ARC_CUDA(cudaMemcpyAsync(values_host, vals, sizeof(float) * c->pl.sumKn, cudaMemcpyDeviceToHost, s));
    return ARC_OK;
}

arc_status arc_topk_query(arc_topk_ctx* c, int32_t what, void* dst, size_t bytes, void* stream) {
    if (c == nullptr || dst == nullptr) return ARC_ERR_INVALID_ARG;
    const Plan& pl = c->pl;
    size_t off = 0, need = 0;
    switch (what) {
        case ARC_Q_V: off = pl.o_V + sizeof(float) * pl.sum_nr * (c->last_t & 1); need = sizeof(float) * pl.sum_nr; break;
        case ARC_Q_SIGMA: off = pl.o_sigma; need = sizeof(float) * pl.M; break;
        case ARC_Q_SEL: off = pl.o_sel; need = sizeof(int32_t) * pl.sumK; break;
        case ARC_Q_P_NODES:
            if (!pl.keep_pnodes) return ARC_ERR_INVALID_ARG;
            off = pl.o_pnodes;
            need = sizeof(float) * static_cast<size_t>(pl.M) * pl.L * c->p.r;
            break;
        case ARC_Q_S: {   // S = sum_i P'_i (node order), every node on this GPU
            if (!pl.keep_pnodes || pl.G > 1 || pl.randk || pl.topk) return ARC_ERR_UNSUPPORTED;
            need = sizeof(float) * static_cast<size_t>(pl.M) * c->p.r;
            if (bytes < need) return ARC_ERR_INVALID_ARG;
            if (need == 0) return ARC_OK;
            launch_node_sum(c->pnodes_ptr(), pl.M, pl.L, c->p.r, static_cast<float*>(dst), static_cast<cudaStream_t>(stream));
            ARC_LAUNCHED();
            return ARC_OK;
        }
        case ARC_Q_CANDIDATES: {   // counters of the last step's parity (device word status[1], toggled per step)
            unsigned par = 0;
            ARC_CUDA(cudaStreamSynchronize(c->last));
            ARC_CUDA(cudaMemcpy(&par, c->ws + pl.o_status + sizeof(unsigned), sizeof par, cudaMemcpyDeviceToHost));
            off = pl.o_cand_count + sizeof(unsigned) * pl.sbdev.size() * ((par & 1u) ^ 1u);
            need = sizeof(unsigned) * pl.sbdev.size();
            break;
        }
        case ARC_Q_PLAN: {   // host-side facts, copied synchronously
            const int32_t plan[4] = {pl.items.empty() ? 3 : c->tail ? 2 : c->sel_cluster ? 1 : 0,
                                     pl.items.empty() ? 0 : c->tail ? 1 : c->sel_grid,
                                     pl.M > 0 ? (c->grid > 0) + (c->grid_w > 0) + (c->grid_t > 0) : 0,
                                     arc_topk_kernels_per_step(c)};
            if (bytes < sizeof plan) return ARC_ERR_INVALID_ARG;
            ARC_CUDA(cudaMemcpy(dst, plan, sizeof plan, cudaMemcpyDefault));
            return ARC_OK;
        }
        default: return ARC_ERR_INVALID_ARG;
    }
    if (bytes < need) return ARC_ERR_INVALID_ARG;
    if (need == 0) return ARC_OK;
    const void* src = c->ws + off;
    if (what == ARC_Q_SIGMA) src = c->sigma_ptr();
    if (what == ARC_Q_P_NODES) src = c->pnodes_ptr();
    ARC_CUDA(cudaMemcpyAsync(dst, src, need, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
    return ARC_OK;
}

arc_status arc_topk_sizes(const arc_topk_ctx* c, int64_t* sum_K, int64_t* sum_Kn, int64_t* sum_m_arc,
                          int64_t* sum_nr_arc) {
    if (c == nullptr) return ARC_ERR_INVALID_ARG;
    if (sum_K) *sum_K = c->pl.sumK;
    if (sum_Kn) *sum_Kn = c->pl.sumKn;
    if (sum_m_arc) *sum_m_arc = c->pl.M;
    if (sum_nr_arc) *sum_nr_arc = c->pl.sum_nr;
    return ARC_OK;
}

int32_t arc_topk_kernels_per_step(const arc_topk_ctx* c) {
    if (c == nullptr) return -1;
    // steady state with consecutive t: V comes from the previous step's select
    // kernel (k_vgen only when there is none)
    const Plan& pl = c->pl;
    const int sketch = pl.M > 0 ? (c->grid > 0 ? 1 : 0) + (c->grid_w > 0 ? 1 : 0) + (c->grid_t > 0 ? 1 : 0) : 0;
    const int sel = pl.items.empty() ? 0 : 1;   // (the fused tail: S3 in the sketch launch + the update kernel)
    if (pl.topk) return sketch + sel + c->p.N;   // + N ordered merges
    const int vgen = (pl.M > 0 && !pl.topk && !pl.randk && (pl.items.empty() || (c->p.flags & ARC_FLAG_DEVICE_T))) ? 1 : 0;
    const int sigma = (pl.exchange || pl.exact) && !pl.randk && pl.M > 0 ? 1 : 0;
    const int dense = pl.dense_ids.empty() ? 0 : 1;
    const int scatter = pl.exchange ? (pl.segs_real.empty() ? 0 : 1) + dense : 0;
    return vgen + sketch + sigma + sel + dense + scatter;
}

arc_status arc_topk_set_timing(arc_topk_ctx* c, int32_t enable) {
    if (c == nullptr) return ARC_ERR_INVALID_ARG;
    c->timing = enable != 0;
    return ARC_OK;
}

arc_status arc_topk_read_timing(arc_topk_ctx* c, float* ms, int32_t n_phases, int32_t* steps) {
    if (c == nullptr || ms == nullptr || n_phases < 1 || n_phases > ARC_TIMING_PHASES) return ARC_ERR_INVALID_ARG;
    for (int k = 0; k < n_phases; ++k) ms[k] = 0.0f;
    if (c->timed_steps > 0) ARC_CUDA(cudaEventSynchronize(c->ev_pool[static_cast<size_t>(c->timed_steps) * (ARC_TIMING_PHASES + 1) - 1]));
    for (int st = 0; st < c->timed_steps; ++st) {
        const size_t b = static_cast<size_t>(st) * (ARC_TIMING_PHASES + 1);
        for (int k = 0; k < n_phases; ++k) {
            float x = 0.0f;
            ARC_CUDA(cudaEventElapsedTime(&x, c->ev_pool[b + k], c->ev_pool[b + k + 1]));
            ms[k] += x;
        }
    }
    if (steps) *steps = c->timed_steps;
    c->timed_steps = 0;
    return ARC_OK;
}

arc_status arc_topk_comm_tally(const arc_topk_ctx* c, int64_t* out, int32_t n) {
    if (c == nullptr || out == nullptr || n < 1 || n > kTallyN) return ARC_ERR_INVALID_ARG;
    for (int k = 0; k < n; ++k) out[k] = c->tally[k];
    return ARC_OK;
}

arc_status arc_topk_get_status(arc_topk_ctx* c, uint32_t* flags) {
    if (c == nullptr) return ARC_ERR_INVALID_ARG;
    ARC_CUDA(cudaStreamSynchronize(c->last));
    uint32_t st = 0;
    ARC_CUDA(cudaMemcpy(&st, c->ws + c->pl.o_status, 4, cudaMemcpyDeviceToHost));
    ARC_CUDA(cudaMemset(c->ws + c->pl.o_status, 0, 4));
    if (flags) *flags = st;
    if (c->comm != nullptr && c->nccl.ok) {
        ncclResult_t r = ncclSuccess;
        if (c->nccl.commGetAsyncError(c->comm, &r) != ncclSuccess || r != ncclSuccess) return ARC_ERR_NCCL;
    }
    return (st & kStatusNonfinite) ? ARC_ERR_NONFINITE : ARC_OK;
}

arc_status arc_topk_debug_stamps(arc_topk_ctx* c, uint64_t* stamps_host, int64_t n, int32_t* grid) {
    if (c == nullptr || c->stamps == nullptr || stamps_host == nullptr) return ARC_ERR_INVALID_ARG;
    const int64_t all = static_cast<int64_t>(c->tail ? 1 : c->sel_grid) * 8;   // (the fused tail: one row)
    ARC_CUDA(cudaStreamSynchronize(c->last));
    ARC_CUDA(cudaMemcpy(stamps_host, c->stamps, sizeof(uint64_t) * (n < all ? n : all), cudaMemcpyDeviceToHost));
    if (grid) *grid = static_cast<int32_t>(c->tail ? 1 : c->sel_grid);
    return ARC_OK;
}

arc_status arc_topk_destroy(arc_topk_ctx* c) {
    if (c == nullptr) return ARC_ERR_INVALID_ARG;
    cudaStreamSynchronize(c->last);
    if (c->stamps) cudaFree(c->stamps);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    lsa_release(c);
    delete c;
    return ARC_OK;
}

}  // extern "C"
