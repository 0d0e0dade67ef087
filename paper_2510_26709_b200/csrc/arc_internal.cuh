// arc_internal.cuh — device-side layout shared by the kernels and the host
// orchestration of libarctopk.so.  Not part of the public ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "arc_topk.h"

struct ncclDevComm;
struct ncclWindow_vidmem;

namespace arc {

// Per-block descriptor in device memory (built once at create).
struct BlockDev {
    long long off;      // first flat element
    long long len;      // flat elements
    int m, n, K, kind;  // view and rows kept
    long long v_off;    // offset of V_b (floats) in the V buffer      (ARC blocks)
    int row_base;       // first global ARC row (sigma / exchange rows) (ARC blocks)
    int sel_base;       // offset of I_b in the selection array
    long long val_base; // offset of the compact rows in values / wire
    int vec;            // rows 16-byte aligned: off % 4 == 0 && n % 4 == 0
    int slice_base;     // first selection slice of the block
    int node;           // Top-K baseline: the local node whose own rows this selection block ranks
    int pad_;
};

// A sketch tile: rows [row0, row0 + rows) of one ARC block for one local node
// (the nodes' sketches are independent; their ordered sum is a separate pass).
struct Tile {
    int b;
    int row0;
    int rows;
    int node;
};

// A tile with its block's fields, as the streaming kernel reads it (64 B; the
// next tile's descriptor is fetched into shared memory while a tile runs).
struct alignas(16) TileDesc {
    long long off, len, v_off;   // block
    int n, row0, rows, vec, row_base, b, node;
    int pad_[3];
};
static_assert(sizeof(TileDesc) == 64, "TileDesc is four 16-byte words");

// Gather / scatter work item: columns [4*q0, 4*q0 + kSegQuads*4) of the k-th
// selected row of block b.
constexpr int kSegQuads = 64;      // 32 lanes x 2 quads = 256 columns
struct SelRow {
    int b;
    int k;
    int q0;
};

constexpr int kSketchThreads = 256;

constexpr uint32_t kStatusNonfinite = 1u;

// Selection: digit 1 of the order key (bits [31:21]) is histogrammed per block
// by the pass that produces Sigma; k_select resolves the rest on candidates.
constexpr int kHist1Bins = 2048;
constexpr int kHist1Shift = 21;
constexpr unsigned kHist1Mask = 0xFFE00000u;
constexpr int kSliceMin = 256;     // rows per selection slice (one CTA), at least
constexpr int kCandCap = 2048;     // boundary-bin candidates per block resolved in every CTA

struct SliceItem {
    int b;   // block
    int c;   // slice in the block
};


struct SelectGatherLaunch {
    const BlockDev* blocks;
    const SliceItem* items;        // every slice of every block (one CTA each)
    int num_items;
    int grid;                      // CTAs (<= num_items, all co-resident); CTA b takes slices b, b + grid, ...
    int slice_rows;                // rows per slice (<= 4096)
    const float* sigma;
    unsigned* hist1;               // [num_blocks][2048] digit key[31:21] (filled by the Sigma pass)
    unsigned* hist2;               // [num_blocks][2048] digit key[20:10]
    unsigned* hist3;               // [num_blocks][1024] digit key[9:0]
    int* slice_gt;                 // [num_slices] keys > T (or above digit-1 bin)
    int* slice_eq;                 // [num_slices] keys == T
    unsigned* cand;                // [2][num_blocks][2 * kCandCap] boundary-bin candidates (key | row)
    unsigned* cand_count;          // [2][num_blocks]
    int num_blocks;
    unsigned* parity;              // device word: bit 0 selects this step's candidate / boundary
                                   // counters; toggled by the kernel once every CTA has read it, so
                                   // a CUDA-graph replay of a captured step stays consistent
    int32_t* sel;
    unsigned long long* stamps;    // debug: [grid][8] %globaltimer at phase boundaries, or nullptr
    // speculative S0 of the next step: V for t_next (nullptr: none)
    const BlockDev* vblocks;       // the caller's blocks (V offsets)
    int num_vblocks;
    float* V_next;
    long long v_items;             // sum over ARC blocks of n_b * ceil(r / 4)
    int r;
    uint2 key;
    unsigned t_lo, t_hi;
    int pdl;                       // launch with programmatic stream serialization
    int cluster;                   // the grid is one thread-block cluster (<= 16 CTAs, one slice each)
    unsigned long long* t_advance; // ARC_FLAG_DEVICE_T: the device iteration counter, += 1 at the end
    int early;                     // mode 0 without values: gather the certainly selected rows
                                   // (digit 1 above the boundary bin) before barrier 1 completes
    // Sigma not formed by the streaming pass: the kernel builds the digit-1
    // histogram itself, behind one more grid barrier (phase 0) -- from s.sigma
    // (k_sigma_slice + all-gather, exchange path) or, when xsk != nullptr, after
    // forming Sigma from this GPU's per-node sketches (several local nodes)
    int build_hist;
    const float* xsk;              // [M][L][r] per-node sketches, or nullptr
    float* sigma_w;                // Sigma written for queries
    int L;
    float Nf;
    unsigned* status;
};

struct NodePtrs {
    const float* grad[ARC_MAX_NODES_LOCAL];
    float* h[ARC_MAX_NODES_LOCAL];
    float* g[ARC_MAX_NODES_LOCAL];
};

// ---- launchers (arc_kernels.cu) ---------------------------------------------
void launch_vgen(const BlockDev* blocks_dev, int num_blocks, int max_nR4, int r, uint64_t seed,
                 int64_t t, float* V, cudaStream_t s, const unsigned long long* t_dev = nullptr, int pdl = 0);
void launch_advance_t(unsigned long long* t_dev, cudaStream_t s);   // t_dev += 1 (one thread)
void launch_set_u64(unsigned long long* p, unsigned long long v, cudaStream_t s);   // *p = v (one thread)

// The fused small-problem tail of the streaming pass (arc_sketch.cu): with one
// node on the GPU, no exchange and a small selection, the LAST CTA of the
// streaming launch to finish (a done counter) runs S3..S6 itself — no second
// launch, no grid barrier ("fused tail").
constexpr int kTailMaxRows = 8192;      // the largest ARC block's rows: its keys in shared memory (32 KB)
                                        // (C2 with one node, 22,831 rows, measured slower through the tail:
                                        // 59.8 against 46.7 us per step, profiles/r02_tail.txt)
constexpr int kTailMaxBlocks = 8;       // ARC blocks
struct TailBlk {                    // an ARC block as the tail's update kernel reads it (kernel parameter)
    long long off, len, val_base;
    long long q_begin;              // first quad of the block's selected rows in the update's item space
    int n, K, sel_base, vec;
};
struct TailArgs {
    unsigned* done;                 // CTAs finished (workspace word, zero between steps); nullptr: no tail
    int32_t* sel;                   // the selection (sum K_b entries, block sel_base offsets)
    float* values;                  // optional A / N (val_base offsets)
    int bf16;                       // R25: C rounded at the source
    int N_int;
    unsigned long long* t_advance;  // ARC_FLAG_DEVICE_T: += 1 once the step's t readers are done
    float* V_next;                  // speculative S0 of the next step (nullptr: none), drawn by every CTA
    long long v_items;
    unsigned tn_lo, tn_hi;
    unsigned* last_cta;             // the last CTA's index (its V_next items are drawn by k_tail_update)
    int sk_grid;                    // the streaming launch's grid
    int key_cap;                    // floats of dynamic shared memory (keys of one block, m_b <= key_cap)
    unsigned long long* stamps;     // debug (ARC_DEBUG_STAMPS=1): %globaltimer at the tail's phases, or nullptr
    int nblk;                       // ARC blocks (<= kTailMaxBlocks) and their update table
    long long quads;                // sum over them of K_b ceil(n_b / 4): the update's items
    TailBlk blk[kTailMaxBlocks];
};


struct SketchLaunch {
    const BlockDev* blocks;
    const TileDesc* tiles;  // all tiles, grouped by CTA
    const int* cta_begin;   // [grid + 1]: CTA c runs tiles [cta_begin[c], cta_begin[c+1])
    int num_tiles;
    int grid;
    NodePtrs nodes;
    int nodes_local, N, r;
    float eta, ome, Nf;
    const float* V;
    float* sigma;      // mode 0: written
    unsigned* hist1;   // [num_blocks][kHist1Bins] digit-1 histogram of Sigma (mode 0)
    float* pnodes;     // [M][nodes_local][r] P_i, or nullptr (mode 0 without debug)
    int mode;          // 0 = reduce locally -> sigma ; 1 = exchange (write pnodes only) ;
                       // 2 = Top-K baseline: per-node exact ||row||^2 -> sigma[node][M]
                       // 3 = Rand-K: the row's shared random key -> sigma (node-0 tiles)
    int M;
    uint2 key;         // Rand-K: Philox key (seed)
    unsigned t_lo, t_hi;             // ARC rows (stride of the per-node sigma in mode 2)
    int num_blocks;
    int shape;         // variant (arc_sketch.cu)
    int vs_cap;        // floats of dynamic shared memory for V_b^T (0: V from global memory)
    int noef;          // compressed MSGD without EF: sketch the gradient, u = gbar <- eta u
    int ranged;        // the launch over blocks whose V_b^T exceeds the stage (ranges of vs_cap / r columns)
    float* gbar;       // (noef) the replicated momentum u
    const unsigned long long* t_dev;   // ARC_FLAG_DEVICE_T: t in device memory (Rand-K keys), else nullptr
    int pdl;           // launch with programmatic stream serialization (overlap the launch)
    unsigned* status;
    TailArgs tail;     // (mode 0 / 3, one node, no exchange) the fused S3..S6 tail, or tail.done == nullptr
};
void launch_ef_sketch(const SketchLaunch& a, cudaStream_t s);
// S4..S6 of the tail's selection: a small grid launched right behind the streaming
// launch (programmatic dependent launch when a.pdl), waiting for it to complete.
void launch_tail_update(const SketchLaunch& a, cudaStream_t s);
int ef_sketch_resident_ctas(int r, int shape, int vs_cap);   // SMs x occupancy
int ef_sketch_resident_ctas_tail(int r, int shape, bool noef, int dyn_floats);   // (the fused-tail variant)
int sketch_vs_cap(int r, int max_n);   // floats of V_b^T the streaming pass stages in shared memory (0: too wide)
int sketch_ranged_cap(int r);          // floats staged per range by the wide blocks' launch
int ef_sketch_resident_ctas_ranged(int r, int vs_cap);
int sketch_wide_threads(int r);        // threads per CTA of that launch (tiles of <= 4-column rows: one row per thread)
// the bulk-copy (TMA) fed launch for unaligned rows and wide V (arc_sketch_tma.cu): one CTA per SM
void launch_ef_sketch_tma(const SketchLaunch& a, cudaStream_t s);
int sketch_tma_vs_cap(int r);          // floats of V_b^T it stages next to its rings
int sketch_tma_threads();
int sketch_tile_rows(int shape);
int sketch_tile_cols(int shape);
int sketch_shape_ok(int shape, int r);



struct GatherLaunch;
cudaError_t launch_select_gather(const SelectGatherLaunch& s, const GatherLaunch& ga, cudaStream_t st);
int select_gather_resident_ctas();
int select_max_slice_rows();
int select_max_slices_per_cta();
int select_cluster_max(int want);      // largest one-cluster grid <= want the selection kernel can launch

struct GatherLaunch {
    const BlockDev* blocks;
    const SelRow* rows;
    int num_rows;       // number of row segments
    const int32_t* sel;
    NodePtrs nodes;
    int nodes_local;
    float eta, ome;     // DENSE blocks: the momentum update happens here (no sketch pass)
    float Nf;
    int N_int;          // N as an integer (power-of-two test for A / N)
    float* gbar;        // mode 0: updated ; mode 1: nullptr
    float* values;      // mode 0: optional A/N ; mode 1: the wire (local pre-sum or per-node)
    int mode;           // 0 = fused local (G==1); 1 = wire pre-sum; 2 = wire per node [nodes_local][sumKn];
                        // 3 = Top-K baseline: node B.node only, wire values at B.val_base
    long long sum_Kn;
    int noef;           // without EF: C_i = grad_i rows, no h / g (u = gbar, scaled by the sketch pass)
    int bf16;           // bfloat16 value wire (R25): C_i rounded at the source; modes 1, 2 payloads in bf16
    int2* bnd;          // early mode after an overflow: selected boundary rows (block, row)
    unsigned* bnd_count;   // [2] by step parity
};

struct ScatterLaunch {
    const BlockDev* blocks;
    const SelRow* rows;
    int num_rows;
    const int32_t* sel;
    const void* wire;       // reduced sums (mode 0) or gathered per-node wires (mode 1); float or bf16 entries
    int mode;               // 0 = already summed; 1 = [G*nodes_local][sumKn], ordered sum
    int bf16;               // payload entries are bfloat16 (R25)
    int nodes_total;        // N (mode 1)
    long long sum_Kn;
    float Nf;
    int N_int;
    float* gbar;
    float* values;          // optional A/N
};
void launch_scatter(const ScatterLaunch& a, cudaStream_t s);

// S2 on this rank's row slice (after the all-to-all of exchange #1, or on the
// per-node sketches of one GPU with several local nodes).
struct SigmaLaunch {
    const float* x;      // [G][Ms][L][r] per-node sketches of the slice's rows, by source rank
    long long Ms;        // rows per slice (the source-rank stride)
    long long rows;      // rows of this slice
    int G, L, r;
    float Nf;
    float* sigma;        // Sigma of the slice's rows
    unsigned* status;
};
void launch_sigma_slice(const SigmaLaunch& a, cudaStream_t s);

// ARC_METHOD_EXACT: Sigma_p = || sum_i (h'_i - g_i)[p, :] ||^2 for every ARC row.
struct ExactSigmaLaunch {
    const BlockDev* blocks;
    int num_blocks;
    int L;               // local nodes (== N)
    NodePtrs nodes;      // h (already h'), g
    float* sigma;        // [M], indexed by B.row_base + p
    unsigned* status;
};
void launch_exact_sigma(const ExactSigmaLaunch& a, cudaStream_t s);

// ARC_Q_S: the node sum S [M][r] of the per-node sketches [M][L][r] (node order)
void launch_node_sum(const float* pnodes, long long M, int L, int r, float* dst, cudaStream_t s);

// DENSE blocks with every node on this GPU: one streaming pass (identity compressor).
struct DenseLaunch {
    const BlockDev* blocks;
    const int* dense_ids;       // indices of the DENSE blocks
    int num_dense;
    NodePtrs nodes;
    int nodes_local;
    float eta, ome, Nf;
    int N_int;
    float* gbar;
    float* values;              // mode 0: optional A/N (float)
    void* payload;              // modes 1, 2: the exchange payload (float or bf16 entries)
    int bf16;                   // bfloat16 value wire (R25)
    int32_t* sel;               // identity selection written here
    int mode;                   // 0 = fused local; 1 = payload = local node sum; 2 = payload per node
    long long sum_Kn;           // mode 2: per-node payload stride
    int noef;                   // without EF: C_i = grad_i, u = gbar <- eta u (+ A / N in mode 0)
};
void launch_dense(const DenseLaunch& a, cudaStream_t s);

// DENSE blocks after exchange #2: gbar += A / N (A all-reduced, or the ordered
// sum over the all-gathered per-node payloads).
struct DenseScatterLaunch {
    const BlockDev* blocks;
    const int* dense_ids;
    int num_dense;
    const void* wire;           // float or bf16 entries
    int mode;                   // 0 = summed; 1 = [N][sum_Kn] per node, ordered sum
    int bf16;
    int nodes_total;
    long long sum_Kn;
    float Nf;
    int N_int;
    float* gbar;
    float* values;              // optional A/N
};
void launch_dense_scatter(const DenseScatterLaunch& a, cudaStream_t s);

// Exchange #2 fused with S6 over peer memory (ARC_REDUCE_LSA, arc_lsa.cu):
// the per-node payloads live in an NCCL symmetric window on every rank.
constexpr int kLsaCtas = 592;   // grid cap = LSA barriers requested at create (4 per SM)
struct LsaScatter {
    const ncclDevComm* dev_comm;   // device copy of the ncclDevComm (library-owned)
    ncclWindow_vidmem* win;        // window of [L][sum_Kn] floats per rank
    int G, L, N;                   // ranks (= LSA team), local nodes, global nodes
    long long sum_Kn;
    int bf16;                      // window entries are bfloat16 (R25)
};
void launch_lsa_scatter(const ScatterLaunch& a, const LsaScatter& x, cudaStream_t s);
// Exchange #1 over peer memory: every rank's per-node sketches P' ([M][L][r])
// and Sigma ([G * Ms]) live in one symmetric window (P' at byte 0, Sigma at
// sigma_off).  CTA b of every rank owns sub-range b of every rank's row slice.
struct LsaSigma {
    const ncclDevComm* dev_comm;
    ncclWindow_vidmem* win;
    size_t sigma_off;      // bytes
    float* sigma;          // this rank's Sigma (the window's local address + sigma_off)
    long long Ms, M;       // rows per slice, rows in total
    int G, me, L, r;
    unsigned* status;
};
void launch_lsa_sigma(const LsaSigma& a, cudaStream_t s);
void launch_lsa_dense_scatter(const DenseScatterLaunch& a, const LsaScatter& x, cudaStream_t s);

// Top-K baseline merge of one node's gathered payload: gbar[I_j] += C_j / N.
struct MergeLaunch {
    const BlockDev* blocks;     // real blocks
    const SelRow* rows;         // segments over the real blocks
    int num_rows;
    const float* values;        // this node's values (block val_base offsets)
    const int32_t* idx;         // this node's indices (block sel_base offsets)
    float Nf;
    int N_int;
    float* gbar;
};
void launch_topk_merge(const MergeLaunch& a, cudaStream_t s);

}  // namespace arc
