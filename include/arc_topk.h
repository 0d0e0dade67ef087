/*
 * arc_topk.h — C ABI of libarctopk.so: the EF21M + ARC-Top-K compression step
 * on B200 (sm_100a).
 *
 * What one arc_topk_step computes (PAPER.md = arXiv 2510.26709 LaTeX, "P:n" =
 * line n; readings R1..R22 are in DESIGN.md §3, the arithmetic is SURVEY.md
 * §8(c)'s ARC-NUM v1):
 *   for every node i held by this GPU, every block b (an m_b x n_b row-major
 *   view of the flat vector, R1):
 *     h_i   <- fma(eta, grad_i, (1-eta) h_i)                 eq:ef21m-1, P:325 (R11)
 *     Delta_i = h_i - g_i                                     R4
 *     V_b   ~ N(0, I), n_b x r, from (seed, t, b)             P:229-230, Alg.1 l.3 (R7, R8)
 *     P'_i  = G_i V_b  (the O6 lane/chunk order, fma)         P:231-233, Alg.1 l.4 (R2, R9)
 *     S     = sum_i P'_i   (exchange #1, node order)          P:232, Alg.1 l.5 (R3, R9, R21)
 *     Sigma = diag(S S^T); I_b = argtop_{K_b}(Sigma)          zn28373 P:236-237, Alg.1 l.6 (R5, R15)
 *     (the paper's 1/sqrt(r) and 1/N scale every Sigma alike: not applied, R2/R3)
 *     C_i   = [Delta_i]_{I_b,:}                               2zn20 P:241-243, Alg.1 l.7
 *     g_i[I_b] <- g_i[I_b] + C_i                              eq:ef21m-2, P:326 (R12)
 *     C     = (1/N) sum_i C_i        (exchange #2)            P:242, P:278 (index-free All-Reduce)
 *     gbar[I_b] <- gbar[I_b] + C                              eq:ef21m-3 consumes gbar, P:327 (R13)
 *   DENSE blocks (R20) skip the sketch: I_b = all rows.
 *
 * Conventions
 *   - Device pointers unless a name ends in _host.  All base pointers 16-byte
 *     aligned (torch's allocator gives 512; step returns ARC_ERR_INVALID_ARG
 *     otherwise, before enqueueing anything); rows inside a block may be
 *     unaligned (n % 4 != 0) and are handled.
 *   - Every GPU call enqueues on `stream` (a cudaStream_t; NULL = legacy
 *     default stream) and returns without blocking the host, except create
 *     (when a comm is given), get_status and destroy, which synchronise.
 *   - Ownership: the caller owns grad, h, g, gbar, the workspace, sel_out,
 *     values_out, the stream and the NCCL communicator (borrowed; it must
 *     outlive the context).  The library owns only the host context.
 *   - Errors: validation failures return before anything is enqueued and leave
 *     all state untouched.  ARC_ERR_CUDA / ARC_ERR_NCCL leave the state
 *     undefined: destroy the context.  No call aborts or throws.
 *   - SPMD: with G > 1 GPUs every rank calls create/step/destroy in the same
 *     order with identical params (except rank) and t.
 */
#ifndef ARC_TOPK_H
#define ARC_TOPK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ARC_TOPK_ABI_VERSION 2u
#define ARC_MAX_NODES_LOCAL 16

typedef struct arc_topk_ctx arc_topk_ctx;   /* opaque, library-owned */

typedef enum {
    ARC_OK = 0,
    ARC_ERR_INVALID_ARG = 1,     /* bad pointer, size, layout or parameter   */
    ARC_ERR_UNSUPPORTED = 2,     /* valid but not implemented on this build  */
    ARC_ERR_PARAM_MISMATCH = 3,  /* ranks passed different params to create  */
    ARC_ERR_CUDA = 4,            /* a CUDA runtime call failed               */
    ARC_ERR_NCCL = 5,            /* an NCCL call failed / NCCL not loadable  */
    ARC_ERR_NONFINITE = 6        /* get_status: a non-finite Sigma was seen  */
} arc_status;

typedef enum { ARC_BLOCK_ARC = 0, ARC_BLOCK_DENSE = 1 } arc_block_kind;

typedef enum {
    ARC_REDUCE_NCCL = 0,     /* exchange #2 = ncclAllReduce(sum): gbar within tolerance (G > 1) */
    ARC_REDUCE_ORDERED = 1,  /* exchange #2 = all-gather + ascending node-id sum: bit-exact gbar */
    ARC_REDUCE_LSA = 2       /* exchange #2 fused with S6: each rank's per-node
                                payload sits in an NCCL symmetric window (ncclMemAlloc +
                                ncclCommWindowRegister, library-owned, made at create — a collective);
                                one kernel per block kind meets the peers at an LSA barrier, reads
                                every node's payload from its owner over NVLink (ncclGetLsaPointer),
                                sums in ascending node id (bit-exact gbar, like ORDERED) and adds
                                A/N into gbar.  Needs the exchange path (G > 1 or
                                ARC_FLAG_FORCE_EXCHANGE with a comm), every rank in one LSA team
                                (one NVLink domain, <= 72 ranks) and NCCL >= 2.28; otherwise create
                                returns ARC_ERR_UNSUPPORTED (ARC_ERR_INVALID_ARG without a comm).
                                Not for ARC_METHOD_TOPK_ALLGATHER (UNSUPPORTED). */
} arc_reduce_mode;

/* Compressor.  ARC_METHOD_TOPK_ALLGATHER is the baseline of Table I row "Top-K"
 * (P:91): vanilla EF21M where every node keeps the K_b
 * rows of ITS OWN residual with the largest exact ||row||^2 (ties -> smaller
 * row), g_i <- g_i + C_i on those rows, the nodes all-gather K_b n_b values +
 * K_b indices each, and gbar <- gbar + C_j / N for j = 0 .. N-1 in node order.
 * For it sel_out / values_out must be NULL (the payload is per node). */
/* ARC_METHOD_RANDK is Table I row "Rand-K" with a shared seed
 * (R16): each block keeps K_b uniformly random rows, the same on every node
 * (row p's key is Philox(seed; p, b | 2^31, t) >> 2, the K_b largest keys win),
 * with the same EF21M update and index-free value All-Reduce as ARC-Top-K. */
/* ARC_METHOD_NOEF_MSGD is Table II's "(without EF)" baseline (SPEC
 * compressed_msgd_step): compressed momentum SGD with the shared ARC-Top-K
 * selection applied to the gradients themselves, c_i = C_local(grad_i), and the
 * replicated heavy-ball momentum u_t = beta u_{t-1} + (1/N) sum_i c_i kept in
 * `gbar` (beta = params.eta, 0 <= beta < 1): u <- beta (x) u everywhere, then
 * u[I] <- u[I] (+) A (/) N.  There is no (h, g) state: h and g may be NULL. */
typedef enum {
    ARC_METHOD_ARC = 0,
    ARC_METHOD_TOPK_ALLGATHER = 1,
    ARC_METHOD_RANDK = 2,
    ARC_METHOD_NOEF_MSGD = 3,
    ARC_METHOD_EXACT = 4      /* test mode (SURVEY 8(b) ARC_SKETCH_EXACT): the selection uses the
                                 quantity the sketch estimates, Sigma_p = ||sum_i Delta_i[p,:]||^2
                                 (z72ena P:254-261), the squares in the O6 order; every node on this
                                 GPU (nodes_local == N, no FORCE_EXCHANGE), else ARC_ERR_UNSUPPORTED */
} arc_method;

/* flags */
#define ARC_FLAG_HOST_STAGING   0x1u  /* reserve device staging for arc_topk_step_host          */
#define ARC_FLAG_DEBUG_SKETCH   0x2u  /* keep P_i for arc_topk_query(ARC_Q_P_NODES)              */
#define ARC_FLAG_FORCE_EXCHANGE 0x4u  /* G == 1: run the G > 1 kernel sequence (tests)           */
#define ARC_FLAG_LOOPBACK_COMM  0x8u  /* nccl_comm is an arc_topk_loopback_comm() handle: G ranks   */
                                      /* emulated in one process on one GPU (tests; not with LSA)  */
#define ARC_FLAG_DEVICE_T       0x10u /* the iteration t lives in device memory (the workspace):    */
                                      /* arc_topk_step ignores its t argument, its kernels read the */
                                      /* counter and the step advances it by one, so a CUDA graph   */
                                      /* of one captured step replays iterations t, t + 1, ...      */
                                      /* (R7: V and the Rand-K keys depend on t).  Every step draws */
                                      /* its own V (no speculative V for t + 1).  The counter starts */
                                      /* at 0; arc_topk_set_iteration sets it.                      */

/* The value wire (exchange #2's payload, R25):
 * ARC_WIRE_F32 sends the compact rows C_i in binary32; ARC_WIRE_BF16 rounds each
 * entry to bfloat16 at the source (round to nearest, ties to even), halving the
 * payload.  The EF update adds what was sent, g_i <- g_i + bf16(C_i), so the
 * rounding error stays in the residual h_i - g_i (error feedback); every sum
 * (A = sum_i C_i, gbar += A / N) stays binary32.  The rounding is applied on
 * every placement (also with every node on one GPU), so I, h, g and, with
 * ORDERED / LSA, gbar do not depend on G.  With ARC_REDUCE_NCCL the all-reduce
 * runs in bfloat16 (the rank's local pre-sum and NCCL's partial sums are rounded
 * to bf16, u = 2^-8 each): gbar within (G + 1) u M (R25).  The sketch exchange (P'_i, Sigma) stays binary32.  Not for
 * ARC_METHOD_TOPK_ALLGATHER (its payload carries indices): ARC_ERR_UNSUPPORTED. */
typedef enum { ARC_WIRE_F32 = 0, ARC_WIRE_BF16 = 1 } arc_wire;

/* One block: the m x n row-major view of flat elements [offset, offset+len),
 * (m-1) n < len <= m n (only the last row may be short, R14).  K rows kept,
 * 1 <= K <= m; DENSE blocks require K == m.  Blocks must tile [0, d) in order. */
typedef struct {
    int64_t offset, len, m, n, K;
    int32_t kind;        /* arc_block_kind */
    int32_t reserved;    /* 0 */
} arc_block;

typedef struct {
    uint32_t abi_version;   /* ARC_TOPK_ABI_VERSION                                   */
    int32_t  N;             /* paper nodes in the job (all GPUs)                      */
    int32_t  nodes_local;   /* nodes held by this GPU, 1..ARC_MAX_NODES_LOCAL;        */
                            /* G = N / nodes_local GPUs; global node ids of this GPU  */
                            /* are rank*nodes_local + [0, nodes_local)                */
    int32_t  rank;          /* this GPU's rank in the communicator (0 when G == 1)    */
    int64_t  d;             /* per-node vector length in floats                       */
    int32_t  r;             /* sketch width, 1..32 (paper: 4)                         */
    int32_t  num_blocks;    /* >= 1; or 0 with blocks == NULL: the single-block       */
                            /* shorthand below (one ARC block over [0, d))            */
    const arc_block* blocks;/* host array, copied at create                           */
    float    eta;           /* EF21M momentum, 0 < eta <= 1 (NOEF_MSGD: beta, [0, 1)) */
    int32_t  value_reduce;  /* arc_reduce_mode                                        */
    uint64_t seed;          /* shared base seed (R7), identical on every rank         */
    uint32_t flags;         /* ARC_FLAG_*                                             */
    uint32_t method;        /* arc_method: ARC_METHOD_ARC (0) or the baseline below   */
    int64_t  n, K;          /* num_blocks == 0: rows of n floats, m = ceil(d / n)     */
                            /* (the last row short, R14), K rows kept, 1 <= K <= m    */
                            /* (P:226-228 reshape; Alg. 1 input K); else ignored      */
    int32_t  wire;          /* arc_wire: exchange #2's payload precision (R25)        */
    int32_t  reserved;      /* 0                                                      */
} arc_topk_params;

/* Bytes of device workspace `create` needs for these params (host-only call). */
arc_status arc_topk_workspace_bytes(const arc_topk_params* params, size_t* bytes);

/* Create a context.  workspace: >= arc_topk_workspace_bytes() device bytes,
 * 256-byte aligned, owned by the caller, untouched by anyone else while the
 * context lives.  nccl_comm: an ncclComm_t of G ranks (G = N/nodes_local) when
 * G > 1 (borrowed, e.g. from torch's ProcessGroupNCCL); may be NULL when
 * G == 1.  With G > 1, create all-gathers a hash of the params and returns
 * ARC_ERR_PARAM_MISMATCH on every rank if any rank differs (synchronises). */
arc_status arc_topk_create(const arc_topk_params* params, void* nccl_comm,
                           void* workspace, size_t workspace_bytes,
                           void* stream, arc_topk_ctx** out);

/* One EF21M + ARC-Top-K step at iteration t (t keys the shared V, R7).
 *   grad  : host array [nodes_local] of device pointers to d floats (read-only)
 *   h, g  : host arrays [nodes_local] of device pointers to d floats (in/out)
 *   gbar  : device, d floats (in/out), replicated on every rank
 *   sel_out    : optional device int32[sum_b K_b]: I_b per block, ascending
 *   values_out : optional device float[sum_b K_b n_b]: C = (1/N) sum_i C_i,
 *                the compressed global rows in I order (+0 in padding)      */
arc_status arc_topk_step(arc_topk_ctx* ctx, int64_t t,
                         const float* const* grad, float* const* h, float* const* g,
                         float* gbar, int32_t* sel_out, float* values_out, void* stream);

/* ARC_FLAG_DEVICE_T contexts: enqueue (on `stream`, async) the write of t into
 * the context's device iteration counter, which the next step uses (and
 * advances).  ARC_ERR_INVALID_ARG for a context without the flag or t < 0. */
arc_status arc_topk_set_iteration(arc_topk_ctx* ctx, int64_t t, void* stream);

/* Same step with the gradients in HOST memory (pinned for async copies): the
 * call enqueues host->device copies of grad_host[i] (d floats each) into the
 * workspace staging area (needs ARC_FLAG_HOST_STAGING), the step, and
 * device->host copies of the selection and values into sel_host /
 * values_host (each optional).  Returns after enqueueing. */
arc_status arc_topk_step_host(arc_topk_ctx* ctx, int64_t t,
                              const float* const* grad_host, float* const* h, float* const* g,
                              float* gbar, int32_t* sel_host, float* values_host, void* stream);

/* Debug read-back of the last step's intermediates (device dst, async). */
typedef enum {
    ARC_Q_V = 0,        /* float [sum_ARC ldv_b * r]     V_b transposed, [r][ldv_b] with
                           ldv_b = round_up(n_b, 4) (column j of V_b contiguous and 16-byte
                           aligned, the layout the sketch reads; padding undefined), blocks
                           in order                                                        */
    ARC_Q_SIGMA = 1,    /* float [sum_ARC m_b]           Sigma per ARC block row (unscaled, R2) */
    ARC_Q_SEL = 2,      /* int32 [sum_b K_b]             I_b                                   */
    ARC_Q_P_NODES = 3,  /* float [sum_ARC m_b][nodes_local][r]  P'_i = G_i V, unscaled (needs
                           DEBUG_SKETCH, or G > 1, or nodes_local > 1)                         */
    ARC_Q_S = 5,        /* float [sum_ARC m_b][r]  S = sum_i P'_i, the node sum in ascending node id
                           (R9): Alg. 1 l.5 before the 1/(N sqrt r) scaling (R2, R3); every node on
                           this GPU (G == 1) and P' kept (as ARC_Q_P_NODES), else
                           ARC_ERR_UNSUPPORTED (with G > 1 each rank holds only its own nodes')  */
    ARC_Q_CANDIDATES = 4, /* uint32 [num_blocks] rows sharing the boundary bin of the last selection
                            ([nodes_local][num_blocks] for ARC_METHOD_TOPK_ALLGATHER, whose
                            nodes select separately); synchronises the step's stream first;
                            not maintained by the fused tail (ARC_Q_PLAN[0] == 2)             */
    ARC_Q_PLAN = 6      /* int32 [4] how the context runs a step (fixed at create): [0] selection
                           form: 0 cooperative grid, 1 one thread-block cluster, 2 the fused tail
                           (S3 in the streaming launch's last CTA + a small update kernel: one node
                           on this GPU, no exchange, a small selection), 3 none; [1] selection
                           CTAs (1 for the tail); [2] streaming (S1) launches; [3] kernels per
                           step (arc_topk_kernels_per_step)                                     */
} arc_query;
arc_status arc_topk_query(arc_topk_ctx* ctx, int32_t what, void* dst, size_t bytes, void* stream);

/* Sizes of the step's outputs. */
arc_status arc_topk_sizes(const arc_topk_ctx* ctx, int64_t* sum_K, int64_t* sum_Kn,
                          int64_t* sum_m_arc, int64_t* sum_nr_arc);

/* Synchronises the context's last stream; reports ARC_ERR_NONFINITE if a
 * non-finite Sigma was produced since the last call (flag cleared), or an
 * asynchronous NCCL error.  flags (optional) receives the raw status word. */
arc_status arc_topk_get_status(arc_topk_ctx* ctx, uint32_t* flags);

/* Number of kernels one arc_topk_step launches (for bench accounting). */
int32_t arc_topk_kernels_per_step(const arc_topk_ctx* ctx);

/* Per-phase device timing (CUDA events recorded on the step's stream between
 * the step's phases; off by default, and must stay off during graph capture).
 * Phases: 0 S0 vgen, 1 S1 ef_sketch, 2 exchange #1 + S2 reduce,
 * 3 S3 select + S4 gather/EF (+S5/S6 at G == 1), 4 exchange #2 + S6 scatter,
 * 5 output copies.  read_timing synchronises and returns the summed
 * milliseconds of each phase over the timed steps since the last read
 * (n_phases <= 6), then resets. */
#define ARC_TIMING_PHASES 6
arc_status arc_topk_set_timing(arc_topk_ctx* ctx, int32_t enable);
arc_status arc_topk_read_timing(arc_topk_ctx* ctx, float* ms, int32_t n_phases, int32_t* steps);

/* Debug: per-CTA %globaltimer stamps (ns) at the phase boundaries of the last
 * step's select/gather kernel, when the context was created with the
 * environment variable ARC_DEBUG_STAMPS=1 (else ARC_ERR_INVALID_ARG).  Copies
 * min(n, grid * 8) uint64 values into host memory (synchronises).  When the
 * step ran the fused small-problem tail (S3..S6 in the streaming launch's last
 * CTA; no selection kernel) *grid = 1 and the row holds: [0] streaming launch
 * start (CTA 0), [1] tail start (the last CTA's arrival), [2] keys and
 * histogram loaded, [3] digits resolved (last ARC block), [4] selection
 * written, [5] S4..S6 done. */
arc_status arc_topk_debug_stamps(arc_topk_ctx* ctx, uint64_t* stamps_host, int64_t n, int32_t* grid);

/* The model update that consumes gbar (R23,
 * R24).  Context-free: one HBM-streaming kernel over d elements, enqueued on
 * `stream` (call it after arc_topk_step on the same stream, so it reads the
 * step's gbar).
 *   ARC_OPT_SGD  : x <- x - gamma * gbar                  eq:ef21m-3, P:327 (R23)
 *   ARC_OPT_ADAM : "standard Adam" on gbar, no weight decay (R24):
 *                  m <- fma(1-b1, gbar, b1 m);  v <- fma(1-b2, gbar^2, b2 v)
 *                  x <- x - gamma ((m / bc1) / (sqrt(v / bc2) + eps)),
 *                  bc_k = (float)(1 - b_k^t) evaluated in double on the host
 * Arguments: x (in/out), gbar (read-only), m and v (in/out, ADAM only; may be
 * NULL for SGD): device float[d], base pointers 16-byte aligned, caller-owned.
 * t is Adam's step count (>= 1; ignored by SGD).  d == 0 is a no-op.
 * Errors (returned before anything is enqueued): ARC_ERR_INVALID_ARG for a
 * NULL params, d < 0, NULL or unaligned pointers, t < 1 (ADAM), betas outside
 * [0, 1), eps < 0 or a non-finite gamma; ARC_ERR_UNSUPPORTED for an unknown
 * kind; ARC_ERR_CUDA if the launch fails.  Non-finite inputs propagate (IEEE). */
typedef enum { ARC_OPT_SGD = 0, ARC_OPT_ADAM = 1 } arc_opt_kind;
typedef struct {
    uint32_t kind;      /* arc_opt_kind */
    float    gamma;     /* step size                          */
    float    beta1;     /* ADAM first-moment decay, [0, 1)    */
    float    beta2;     /* ADAM second-moment decay, [0, 1)   */
    float    eps;       /* ADAM denominator offset, >= 0      */
} arc_opt_params;
arc_status arc_topk_apply_update(const arc_opt_params* params, int64_t t, float* x, const float* gbar,
                                 float* m, float* v, int64_t d, void* stream);

/* Ledger audit (Table I): the floats this rank handed to the
 * step's collectives since create, summed over steps.  out[0] = sketch entries
 * sent to other ranks in exchange #1 (all-to-all of row slices of P'_i),
 * out[1] = Sigma entries contributed to the Sigma all-gather, out[2] = value
 * entries handed to exchange #2 (all-reduce: sum_b K_b n_b per step; ORDERED:
 * nodes_local x that; Top-K baseline: its all-gathered payload), out[3] =
 * collective calls, out[4] = steps.  n <= 8 slots are copied (the rest are 0).
 * Host-only; ARC_ERR_INVALID_ARG for a NULL ctx / out or n outside [1, 8]. */
arc_status arc_topk_comm_tally(const arc_topk_ctx* ctx, int64_t* out, int32_t n);

/* In-process loopback communicator (tests without G GPUs): G ranks emulated in
 * ONE process on the current GPU.  Each rank is a host thread with its own
 * context (created with ARC_FLAG_LOOPBACK_COMM and the handle of
 * arc_topk_loopback_comm as nccl_comm) and its own stream; the collectives meet
 * at host barriers and order the ranks' streams with CUDA events only (no
 * kernel waits on another rank).  The all-reduce sums the ranks in descending
 * rank order (not the oracle's order: it stands in for NCCL's).  A barrier that
 * waits more than 120 s fails the call with ARC_ERR_NCCL (and every later one).
 *   create : G in [1, 64]; *group receives the group (library-owned)
 *   comm   : *comm receives rank's handle (valid until destroy)
 *   destroy: synchronises the device, frees the group (every context using it
 *            must be destroyed first)                                         */
arc_status arc_topk_loopback_create(int32_t G, void** group);
arc_status arc_topk_loopback_comm(void* group, int32_t rank, void** comm);
arc_status arc_topk_loopback_destroy(void* group);

/* Frees the host context (synchronises first).  Never frees caller memory. */
arc_status arc_topk_destroy(arc_topk_ctx* ctx);

const char* arc_topk_status_string(arc_status s);

#ifdef __cplusplus
}
#endif
#endif /* ARC_TOPK_H */
