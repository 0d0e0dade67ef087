// arc_internal.cuh — device-side layout shared by the kernels and the host
// orchestration of libarctopk.so.  Not part of the public ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "arc_topk.h"

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
    int pad_;
};

// A sketch tile: rows [row0, row0 + rows) of one ARC block, rows <= kTileRows.
struct Tile {
    int b;
    int row0;
    int rows;
};

// Selected-row work item for gather / scatter: (block, k).
struct SelRow {
    int b;
    int k;
};

constexpr int kSketchThreads = 256;

constexpr uint32_t kStatusNonfinite = 1u;

struct NodePtrs {
    const float* grad[ARC_MAX_NODES_LOCAL];
    float* h[ARC_MAX_NODES_LOCAL];
    float* g[ARC_MAX_NODES_LOCAL];
};

// ---- launchers (arc_kernels.cu) ---------------------------------------------
void launch_vgen(const BlockDev* blocks_dev, int num_blocks, int max_nR4, int r, uint64_t seed,
                 int64_t t, float* V, cudaStream_t s);

struct SketchLaunch {
    const BlockDev* blocks;
    const Tile* tiles;      // all tiles, grouped by CTA
    const int* cta_begin;   // [grid + 1]: CTA c runs tiles [cta_begin[c], cta_begin[c+1])
    int num_tiles;
    int grid;
    NodePtrs nodes;
    int nodes_local, N, r;
    float eta, ome, c_r, Nf;
    const float* V;
    float* sigma;      // mode 0: written
    float* pnodes;     // [M][nodes_local][r] P_i, or nullptr (mode 0 without debug)
    int mode;          // 0 = reduce locally -> sigma ; 1 = exchange (write pnodes only)
    int shape;         // tile shape R x W: 0 = 64 x 32, 1 = 32 x 64, 2 = 16 x 128
    unsigned* status;
};
void launch_ef_sketch(const SketchLaunch& a, cudaStream_t s);
int ef_sketch_resident_ctas(int r, int shape);   // SMs x occupancy
int sketch_tile_rows(int shape);
int sketch_shape_ok(int shape, int r);

void launch_sketch_reduce(const float* xrecv, int M, int G, int nodes_local, int r, float Nf,
                          float* sigma, unsigned* status, cudaStream_t s);

void launch_select(const BlockDev* blocks, int num_blocks, const float* sigma, int32_t* sel, int max_slice,
                   cudaStream_t s);
int select_max_slice(int max_m);   // keys per CTA of the largest selected block

struct GatherLaunch {
    const BlockDev* blocks;
    const SelRow* rows;
    int num_rows;       // sum_b K_b
    const int32_t* sel;
    NodePtrs nodes;
    int nodes_local;
    float eta, ome;     // DENSE blocks: the momentum update happens here (no sketch pass)
    float Nf;
    float* gbar;        // mode 0: updated ; mode 1: nullptr
    float* values;      // mode 0: optional A/N ; mode 1: the wire (local pre-sum or per-node)
    int mode;           // 0 = fused local (G==1); 1 = wire pre-sum; 2 = wire per node [nodes_local][sumKn]
    long long sum_Kn;
};
void launch_gather_ef(const GatherLaunch& a, cudaStream_t s);

struct ScatterLaunch {
    const BlockDev* blocks;
    const SelRow* rows;
    int num_rows;
    const int32_t* sel;
    const float* wire;      // reduced sums (mode 0) or gathered per-node wires (mode 1)
    int mode;               // 0 = already summed; 1 = [G*nodes_local][sumKn], ordered sum
    int nodes_total;        // N (mode 1)
    long long sum_Kn;
    float Nf;
    float* gbar;
    float* values;          // optional A/N
};
void launch_scatter(const ScatterLaunch& a, cudaStream_t s);

}  // namespace arc
