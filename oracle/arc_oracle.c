/*
 * arc_oracle.c — the CPU ORACLE for the EF21M + ARC-Top-K compression step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2510_26709_b200/) never imports, links or calls it,
 * and this file includes nothing from the product (no shared headers, tables
 * or helpers).  Its only shared source is the text of the paper plus the
 * readings written down in DESIGN.md §3 ("Readings"), which take SURVEY.md
 * §8(c)'s ARC-NUM v1 / ARC-RNG v1 wherever the paper is silent.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, "P:n" = line n):
 *   EF21M, eq:ef21m-1..3, with the compressor C_local / C realised
 *   by ARC-Top-K, Algorithm 1 alg:ar_topk:
 *     reshape g -> G (m x n)                 z72habsd00111, Alg.1 l.2
 *     V in R^{n x r}, vec(V) ~ N(0, I)       P:229-230,     Alg.1 l.3
 *     P'_i = G_i V                           P:231-233,     Alg.1 l.4
 *     S    = sum_i P'_i        (All-Reduce)  P:232,         Alg.1 l.5
 *     Sigma = diag(S S^T), I = argtop_K      zn28373 P:236-237, Alg.1 l.6
 *     C_local(G_i) = [G_i]_{I,:}             2zn20 P:241-243, Alg.1 l.7
 *     C = (1/N) sum_i C_local (All-Reduce)   P:242, Alg.1 l.8
 *   The factors 1/sqrt(r) and 1/N of P scale every row's Sigma by the
 *   same 1/(r N^2), which leaves argtop_K unchanged in exact arithmetic, so
 *   the selection is computed unscaled [R2, R3].
 *
 * Precision.  The selection I is an argtop (an integer decided by floating
 * point), and h, g feed the next step's Sigma, so every value on that chain is
 * computed in IEEE binary32 — the kernel's precision — each + and * rounded
 * once (built with -ffp-contract=off) and fused multiply-adds only where
 * ARC-NUM v1 writes fmaf: the momentum (O2), the sketch dot products (O6) and
 * Sigma (O8).  The sketch's order over q is ARC-NUM v1's O6 (1024-column
 * chunks, 32 lanes, a butterfly, chunks left to right — o6_dot below,
 * simulated lane by lane); every other sum runs left to right in the order it
 * is written.  The places where the paper is silent (summation order,
 * tie-break, generator, NaN) follow DESIGN.md §3; each is cited as "[Rn]".
 *
 * The definitions are written out with plain loops; nothing is blocked, fused
 * or reordered beyond what ARC-NUM v1 fixes.  It is deliberately slow.
 *
 * Threads.  Loops over independent rows (or elements) may be split across
 * OpenMP threads (orc_set_threads; 1 thread unless asked): every row's or
 * element's arithmetic is the same sequence of operations whichever thread
 * runs it, so the results are bit-identical to one thread (pinned in
 * tests/test_oracle.py).  No sum crosses rows, so nothing is reordered.
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdlib.h>
#include <string.h>

/* Threads for the row-parallel loops (see the header); 1 = the plain oracle. */
void orc_set_threads(int32_t n)
{
#ifdef _OPENMP
    omp_set_num_threads(n > 0 ? n : 1);
#else
    (void)n;
#endif
}

int32_t orc_get_threads(void)
{
#ifdef _OPENMP
    return (int32_t)omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------- */
/* Counter-based generator [R8]: Philox4x32-10 (Salmon et al., SC'11).        */
/* ------------------------------------------------------------------------- */

void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; round++) {
        if (round > 0) {               /* key schedule: bump before rounds 2..10 */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t prod0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
        uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static float bits_to_float(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t float_to_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/*
 * bfloat16 wire [R25] (not in the paper, whose precision is
 * unstated, A10): the binary32 value rounded to the nearest bfloat16 (8
 * significand bits, binary32's exponent range), ties to even, returned as the
 * binary32 number it represents.  Written from the definition: the 16 low bits
 * are dropped, rounding up when they exceed the halfway point 0x8000, or equal
 * it and the kept part is odd.  Infinities stay; any NaN becomes a NaN.
 */
float orc_bf16(float x)
{
    uint32_t u = float_to_bits(x);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu) != 0)
        return bits_to_float((u | 0x00400000u) & 0xFFFF0000u);     /* quiet NaN, sign kept */
    uint32_t low = u & 0xFFFFu, keep = u >> 16;
    if (low > 0x8000u || (low == 0x8000u && (keep & 1u))) keep += 1u;   /* carries into the exponent */
    return bits_to_float(keep << 16);
}

/* the value node i puts on the value wire [R25]: x itself, or bf16(x) */
static float wire_value(float x, int32_t wire) { return wire ? orc_bf16(x) : x; }

/* word -> uniform in (0,1): (x >> 9) * 2^-23 + 2^-24, both operations exact [R8]. */
float orc_uniform(uint32_t x)
{
    float i = (float)(x >> 9);
    return i * 0x1p-23f + 0x1p-24f;
}

/* Natural log of a positive normal float, built only from exactly specified
 * operations (bit split, exact subtraction, explicit fmaf) [R8].  Coefficients:
 * the classic Cephes logf set. */
float orc_ln(float u)
{
    uint32_t b = float_to_bits(u);
    int e = (int)(b >> 23) - 126;                       /* u = f * 2^e, f in [0.5,1) */
    float f = bits_to_float((b & 0x007FFFFFu) | 0x3F000000u);
    float x;
    if (f < 0.707106781186547524f) {                    /* SQRTHF */
        e = e - 1;
        x = (f + f) - 1.0f;                              /* exact */
    } else {
        x = f - 1.0f;                                    /* exact (Sterbenz) */
    }
    float z = x * x;
    float p = 7.0376836292e-2f;
    p = fmaf(p, x, -1.1514610310e-1f);
    p = fmaf(p, x, 1.1676998740e-1f);
    p = fmaf(p, x, -1.2420140846e-1f);
    p = fmaf(p, x, 1.4249322787e-1f);
    p = fmaf(p, x, -1.6668057665e-1f);
    p = fmaf(p, x, 2.0000714765e-1f);
    p = fmaf(p, x, -2.4999993993e-1f);
    p = fmaf(p, x, 3.3333331174e-1f);
    float y = (p * x) * z;
    float fe = (float)e;
    y = fmaf(fe, -2.12194440e-4f, y);
    y = fmaf(-0.5f, z, y);
    float res = x + y;
    res = fmaf(fe, 0.693359375f, res);
    return res;
}

/* sin(pi/2 * f) and cos(pi/2 * f) for |f| <= 1/2: Taylor series of sin/cos at
 * argument (pi/2) f, coefficients (pi/2)^k / k! rounded to float [R8]. */
static float sin_quarter(float f)
{
    float f2 = f * f;
    float p = 1.6044118478735982e-4f;
    p = fmaf(p, f2, -4.6817541353186881e-3f);
    p = fmaf(p, f2, 7.9692626246167046e-2f);
    p = fmaf(p, f2, -6.4596409750624625e-1f);
    p = fmaf(p, f2, 1.5707963267948966f);
    return p * f;
}
static float cos_quarter(float f)
{
    float f2 = f * f;
    float p = -2.5202042373060605e-5f;
    p = fmaf(p, f2, 9.1926027483942659e-4f);
    p = fmaf(p, f2, -2.0863480763352961e-2f);
    p = fmaf(p, f2, 2.5366950790104802e-1f);
    p = fmaf(p, f2, -1.2337005501361697f);
    p = fmaf(p, f2, 1.0f);
    return p;
}

/* sin(2 pi u), cos(2 pi u) for u in (0,1): 2 pi u = (pi/2)(k + f) with
 * k = rint(4u), f = 4u - k, both exact; then a quadrant rotation [R8]. */
void orc_sincos2pi(float u, float* s_out, float* c_out)
{
    float w = 4.0f * u;                 /* exact */
    float kf = rintf(w);                /* exact; never a tie for u = (2i+1) 2^-24 */
    float f = w - kf;                   /* exact */
    float s = sin_quarter(f), c = cos_quarter(f);
    int k = ((int)kf) & 3;
    if (k == 0)      { *s_out = s;  *c_out = c;  }
    else if (k == 1) { *s_out = c;  *c_out = -s; }
    else if (k == 2) { *s_out = -s; *c_out = -c; }
    else             { *s_out = -c; *c_out = s;  }
}

/* V_b in R^{n x r}, row-major (V[q*r + j]), vec(V) ~ N(0, I) — P:229-230, Alg.1
 * l.3.  Entry (q, j) is drawn from Philox with key (lo32 seed, hi32 seed) and
 * counter (q*R4 + j/4, b, lo32 t, hi32 t), R4 = ceil(r/4); the four words give
 * two Box–Muller pairs (u0,u1) -> (z0,z1), (u2,u3) -> (z2,z3) [R8]. */
void orc_gaussian_V(uint64_t seed, int64_t t, int32_t b, int64_t n, int32_t r, float* V)
{
    int64_t R4 = (r + 3) / 4;
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    for (int64_t q = 0; q < n; q++) {
        for (int64_t jj = 0; jj < R4; jj++) {
            uint32_t ctr[4] = { (uint32_t)(q * R4 + jj), (uint32_t)b,
                                (uint32_t)(uint64_t)t, (uint32_t)((uint64_t)t >> 32) };
            uint32_t x[4];
            orc_philox4x32_10(ctr, key, x);
            float z[4];
            for (int pair = 0; pair < 2; pair++) {
                float ua = orc_uniform(x[2 * pair]);
                float ub = orc_uniform(x[2 * pair + 1]);
                float rho = sqrtf(-2.0f * orc_ln(ua));
                float sn, cs;
                orc_sincos2pi(ub, &sn, &cs);
                z[2 * pair] = rho * cs;
                z[2 * pair + 1] = rho * sn;
            }
            for (int k = 0; k < 4; k++) {
                int64_t j = 4 * jj + k;
                if (j < r) V[q * r + j] = z[k];
            }
        }
    }
}

/* ------------------------------------------------------------------------- */
/* Selection: I = argtop_K(Sigma), P:134 + P:237 [R5].                        */
/* ------------------------------------------------------------------------- */

/* Order key of a Sigma value: its binary32 bit pattern (Sigma >= +0, where
 * unsigned bit order is numeric order); every NaN maps to the largest key [R15]. */
uint32_t orc_sigma_key(float s)
{
    if (isnan(s)) return 0xFFFFFFFFu;
    return float_to_bits(s);
}

typedef struct { uint32_t key; int64_t idx; } orc_keyed;

static int cmp_desc_key_asc_idx(const void* a, const void* b)
{
    const orc_keyed* x = (const orc_keyed*)a;
    const orc_keyed* y = (const orc_keyed*)b;
    if (x->key != y->key) return (x->key > y->key) ? -1 : 1;
    if (x->idx != y->idx) return (x->idx < y->idx) ? -1 : 1;
    return 0;
}
static int cmp_i32(const void* a, const void* b)
{
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* The K rows with the largest Sigma (ties -> smaller index), returned in
 * ascending row order. */
void orc_argtop_k(const float* sigma, int64_t m, int64_t K, int32_t* sel)
{
    orc_keyed* a = (orc_keyed*)malloc((size_t)m * sizeof(orc_keyed));
    for (int64_t p = 0; p < m; p++) { a[p].key = orc_sigma_key(sigma[p]); a[p].idx = p; }
    qsort(a, (size_t)m, sizeof(orc_keyed), cmp_desc_key_asc_idx);
    for (int64_t k = 0; k < K; k++) sel[k] = (int32_t)a[k].idx;
    qsort(sel, (size_t)K, sizeof(int32_t), cmp_i32);
    free(a);
}

/* ------------------------------------------------------------------------- */
/* Algorithm 1 (ARC-Top-K) on one m x n block, for all N nodes.               */
/* ------------------------------------------------------------------------- */

typedef struct {
    int64_t offset;   /* first flat element of the block                          */
    int64_t len;      /* flat elements in the block, (m-1) n < len <= m n [R14]   */
    int64_t m, n;     /* the m x n view, row-major [R1]                           */
    int64_t K;        /* rows kept, 1 <= K <= m (K = m for DENSE)                 */
    int32_t kind;     /* 0 = ARC, 1 = DENSE (identity compressor) [R20]           */
    int32_t pad_;
} orc_block;

/* Number of real columns in row p: rows are full except a short last row. */
static int64_t row_len(int64_t len, int64_t n, int64_t p)
{
    int64_t rest = len - p * n;
    return rest < n ? rest : n;
}

/*
 * ARC-NUM v1 O6 [R9]: the dot product sum_{q < nv} x[q] * y[q * ys] in the
 * canonical order.  Row chunk c holds columns [1024 c, 1024 c + 1024); in it,
 * lane l (0..31) starts from a_l = +0 and, for s = 0..7 then e = 0..3, with
 * q = 1024 c + 128 s + 4 l + e < nv, sets a_l <- fma(x[q], y[q ys], a_l).  A
 * butterfly (o = 16, 8, 4, 2, 1: every lane a_l <- a_l + a_{l xor o}, all
 * lanes from the previous values) leaves the chunk value w_c = a_0, and the
 * result is (((w_0 + w_1) + w_2) + ...), left to right.  The 32 lanes are
 * simulated literally.
 */
static float o6_dot(const float* x, const float* y, int64_t ys, int64_t nv)
{
    float P = 0.0f;
    for (int64_t c = 0; c * 1024 < nv; c++) {
        float a[32], b[32];
        for (int l = 0; l < 32; l++) {
            a[l] = 0.0f;
            for (int s = 0; s < 8; s++)
                for (int e = 0; e < 4; e++) {
                    int64_t q = 1024 * c + 128 * s + 4 * l + e;
                    if (q < nv) a[l] = fmaf(x[q], y[q * ys], a[l]);
                }
        }
        for (int o = 16; o >= 1; o >>= 1) {
            for (int l = 0; l < 32; l++) b[l] = a[l] + a[l ^ o];
            memcpy(a, b, sizeof a);
        }
        P = (c == 0) ? a[0] : P + a[0];
    }
    return P;
}

/*
 * orc_arc_round — Algorithm 1 on N node-local m x n matrices.
 *   G[i]      : node i's block as flat floats (len of them), read-only
 *   V         : n x r projection (row-major)
 *   exact     : 0 = Gaussian sketch (the paper); 1 = test mode, Sigma_p =
 *               O6 sum of fma(S_q, S_q, .) with S_q = sum_i G_i[p][q] in node
 *               order: || sum_i G_i[p,:] ||^2, the quantity the sketch
 *               estimates up to the factor N^2 (z72ena P:254-261)
 * Outputs (each optional except sel):
 *   P_nodes [N][m][r] : P'_i = G_i V, each entry an O6 dot product
 *   S_out   [m][r]    : S = ((P'_0 + P'_1) + ...) + P'_{N-1}, node order [R9]
 *   sigma   [m]       : Sigma_p: s = +0; s <- fma(S_pj, S_pj, s), j = 0..r-1 (O8)
 *   sel     [K]       : I, ascending
 *   C_local [N][K][n] : [G_i]_{I,:}, compact rows in I order, +0 in padding
 *                       (wire = 1: each entry rounded to bfloat16 [R25])
 *   C_glob  [K][n]    : (1/N) sum_i C_local_i = A / N, A summed in node order
 */
void orc_arc_round(int32_t N, int64_t len, int64_t m, int64_t n, int64_t K, int32_t r,
                   const float* const* G, const float* V, int32_t exact, int32_t wire,
                   float* P_nodes, float* S_out, float* sigma, int32_t* sel,
                   float* C_local, float* C_glob)
{
    float* Pn = (float*)malloc((size_t)N * (size_t)m * (size_t)r * sizeof(float));
    float* Sa = (float*)malloc((size_t)m * (size_t)r * sizeof(float));
    float* Sg = (float*)calloc((size_t)m, sizeof(float));
    const float Nf = (float)N;

    if (!exact) {
        /* Alg.1 l.4: P'_i = G_i V, entry (p, j) the O6 dot product of row p
         * with column j of V [R2, R9]. */
        for (int32_t i = 0; i < N; i++)
#pragma omp parallel for schedule(static)
            for (int64_t p = 0; p < m; p++) {
                int64_t nv = row_len(len, n, p);
                for (int32_t j = 0; j < r; j++)
                    Pn[((size_t)i * m + p) * r + j] = o6_dot(G[i] + p * n, V + j, r, nv);
            }
        /* Alg.1 l.5: S = sum_i P'_i, the node sum in ascending node id [R9]. */
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < m; p++)
            for (int32_t j = 0; j < r; j++) {
                float s = Pn[(size_t)p * r + j];
                for (int32_t i = 1; i < N; i++) s = s + Pn[((size_t)i * m + p) * r + j];
                Sa[(size_t)p * r + j] = s;
            }
        /* Alg.1 l.6: Sigma = diag(S S^T) (O8) [R3]. */
#pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < m; p++) {
            float s = 0.0f;
            for (int32_t j = 0; j < r; j++) s = fmaf(Sa[(size_t)p * r + j], Sa[(size_t)p * r + j], s);
            Sg[p] = s;
        }
    } else {
        float* row = (float*)malloc((size_t)(n > 0 ? n : 1) * sizeof(float));
        for (int64_t p = 0; p < m; p++) {
            int64_t nv = row_len(len, n, p);
            for (int64_t q = 0; q < nv; q++) {
                float a = G[0][p * n + q];
                for (int32_t i = 1; i < N; i++) a = a + G[i][p * n + q];
                row[q] = a;
            }
            Sg[p] = o6_dot(row, row, 1, nv);
        }
        free(row);
    }
    /* Alg.1 l.6: I = argtop_K(Sigma) */
    orc_argtop_k(Sg, m, K, sel);

    /* Alg.1 l.7-8: C_local(G_i) = [G_i]_{I,:};  C = (1/N) sum_i C_local(G_i). */
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < K; k++) {
        int64_t p = sel[k];
        int64_t nv = row_len(len, n, p);
        for (int64_t q = 0; q < n; q++) {
            float a = 0.0f;
            for (int32_t i = 0; i < N; i++) {
                float c = wire_value((q < nv) ? G[i][p * n + q] : 0.0f, wire);   /* [R25] */
                if (C_local) C_local[((size_t)i * K + k) * n + q] = c;
                a = (i == 0) ? c : a + c;
            }
            if (C_glob) C_glob[(size_t)k * n + q] = a / Nf;
        }
    }

    if (P_nodes && !exact) memcpy(P_nodes, Pn, (size_t)N * m * r * sizeof(float));
    if (S_out && !exact) memcpy(S_out, Sa, (size_t)m * r * sizeof(float));
    if (sigma) memcpy(sigma, Sg, (size_t)m * sizeof(float));
    free(Pn); free(Sa); free(Sg);
}

/* ------------------------------------------------------------------------- */
/* One EF21M step (eq:ef21m-1, eq:ef21m-2) with ARC-Top-K,         */
/* plus the replicated global tracker gbar = (1/N) sum_i g_i that             */
/* eq:ef21m-3 consumes [R13].                                          */
/* ------------------------------------------------------------------------- */

/* ------------------------------------------------------------------------- */
/* Rand-K with a shared seed (Table I row "Rand-K"): K rows   */
/* of each block drawn uniformly without replacement, the same on every node   */
/* [R16].  Row p of block b draws a 30-bit key from Philox (counter            */
/* (p, b | 2^31, lo32 t, hi32 t), first word >> 2) and the K largest keys are  */
/* kept (ties -> smaller row): a uniformly random K-subset.                    */
/* ------------------------------------------------------------------------- */
void orc_randk_keys(uint64_t seed, int64_t t, int32_t b, int64_t m, float* keys)
{
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    for (int64_t p = 0; p < m; p++) {
        uint32_t ctr[4] = { (uint32_t)p, (uint32_t)b | 0x80000000u,
                            (uint32_t)(uint64_t)t, (uint32_t)((uint64_t)t >> 32) };
        uint32_t x[4];
        orc_philox4x32_10(ctr, key, x);
        keys[p] = bits_to_float(x[0] >> 2);     /* a finite float whose bits are the key */
    }
}

typedef struct {
    int32_t N;             /* nodes                                        */
    int32_t r;             /* sketch width                                 */
    int64_t d;             /* per-node vector length                       */
    float eta;             /* EF21M momentum                               */
    int32_t exact;         /* sketch mode (0 Gaussian, 1 exact, test only,  */
                           /* 2 = Rand-K with a shared seed)               */
    uint64_t seed;         /* shared base seed [R7]                         */
    int32_t num_blocks;
    int32_t pad_;
    const orc_block* blocks;  /* tile [0, d) in order                      */
    int32_t wire;             /* value wire: 0 binary32, 1 bfloat16 [R25]  */
    int32_t pad2_;
} orc_cfg;

/* debug outputs, each optional: V concatenated per ARC block ([n_b][r]);
 * sigma per ARC block ([m_b]), both in block order. */
int orc_step(const orc_cfg* cfg, int64_t t,
             const float* const* grad, float* const* h, float* const* g, float* gbar,
             int32_t* sel_out, float* values_out, float* V_out, float* sigma_out)
{
    const int32_t N = cfg->N;
    const float eta = cfg->eta;
    const float one_minus_eta = 1.0f - eta;

    /* eq:ef21m-1: h_t = (1 - eta) h_{t-1} + eta grad, as
     * fma(eta, grad, (1 - eta) h) (ARC-NUM v1 O1, O2) [R11] */
    for (int32_t i = 0; i < N; i++)
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < cfg->d; e++)
            h[i][e] = fmaf(eta, grad[i][e], one_minus_eta * h[i][e]);

    int64_t sel_pos = 0, val_pos = 0, V_pos = 0, sig_pos = 0;
    for (int32_t b = 0; b < cfg->num_blocks; b++) {
        const orc_block* B = &cfg->blocks[b];
        const int64_t m = B->m, n = B->n, K = B->K, len = B->len;

        /* residual Delta_i = h_t - g_{t-1}, the input of C_local in eq:ef21m-2 [R4] */
        float** D = (float**)malloc((size_t)N * sizeof(float*));
        for (int32_t i = 0; i < N; i++) {
            D[i] = (float*)malloc((size_t)len * sizeof(float));
#pragma omp parallel for schedule(static)
            for (int64_t e = 0; e < len; e++) D[i][e] = h[i][B->offset + e] - g[i][B->offset + e];
        }
        int32_t* sel = (int32_t*)malloc((size_t)K * sizeof(int32_t));
        float* Cl = (float*)malloc((size_t)N * K * n * sizeof(float));
        float* Cg = (float*)malloc((size_t)K * n * sizeof(float));

        if (B->kind == 0 && cfg->exact == 2) {
            /* Rand-K: the selection ignores the data */
            float* keys = (float*)malloc((size_t)m * sizeof(float));
            orc_randk_keys(cfg->seed, t, b, m, keys);
            orc_argtop_k(keys, m, K, sel);
            for (int64_t k = 0; k < K; k++) {
                int64_t p = sel[k];
                int64_t nv = row_len(len, n, p);
                for (int64_t q = 0; q < n; q++) {
                    float a = 0.0f;
                    for (int32_t i = 0; i < N; i++) {
                        float c = wire_value((q < nv) ? D[i][p * n + q] : 0.0f, cfg->wire);   /* [R25] */
                        Cl[((size_t)i * K + k) * n + q] = c;
                        a = (i == 0) ? c : a + c;
                    }
                    Cg[(size_t)k * n + q] = a / (float)N;
                }
            }
            if (sigma_out) memcpy(sigma_out + sig_pos, keys, (size_t)m * sizeof(float));
            sig_pos += m;
            V_pos += n * cfg->r;
            free(keys);
        } else if (B->kind == 0) {
            float* V = (float*)malloc((size_t)n * cfg->r * sizeof(float));
            orc_gaussian_V(cfg->seed, t, b, n, cfg->r, V);
            float* sg = (float*)malloc((size_t)m * sizeof(float));
            orc_arc_round(N, len, m, n, K, cfg->r, (const float* const*)D, V, cfg->exact, cfg->wire,
                          NULL, NULL, sg, sel, Cl, Cg);
            if (V_out) memcpy(V_out + V_pos, V, (size_t)n * cfg->r * sizeof(float));
            if (sigma_out) memcpy(sigma_out + sig_pos, sg, (size_t)m * sizeof(float));
            V_pos += n * cfg->r;
            sig_pos += m;
            free(V); free(sg);
        } else {
            /* DENSE block: identity compressor, I = all rows [R20] */
            for (int64_t k = 0; k < K; k++) {
                sel[k] = (int32_t)k;
                int64_t nv = row_len(len, n, k);
                for (int64_t q = 0; q < n; q++) {
                    float a = 0.0f;
                    for (int32_t i = 0; i < N; i++) {
                        float c = wire_value((q < nv) ? D[i][k * n + q] : 0.0f, cfg->wire);   /* [R25] */
                        Cl[((size_t)i * K + k) * n + q] = c;
                        a = (i == 0) ? c : a + c;
                    }
                    Cg[(size_t)k * n + q] = a / (float)N;
                }
            }
        }

        /* eq:ef21m-2: g_t = g_{t-1} + C_local(h_t - g_{t-1}); rows outside I
         * receive + 0 and are left as they are [R12].  gbar += C [R13].
         * With the bfloat16 wire C_local holds what node i sent, bf16(Delta_i),
         * so g_i moves by exactly that and the rounding error stays in the
         * residual h_i - g_i for the next steps (error feedback) [R25].
         * (The rows of I are distinct, so rows may run on any thread.) */
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < K; k++) {
            int64_t p = sel[k];
            int64_t nv = row_len(len, n, p);
            for (int64_t q = 0; q < nv; q++) {
                int64_t e = B->offset + p * n + q;
                for (int32_t i = 0; i < N; i++) g[i][e] = g[i][e] + Cl[((size_t)i * K + k) * n + q];
                gbar[e] = gbar[e] + Cg[(size_t)k * n + q];
            }
        }
        if (sel_out) memcpy(sel_out + sel_pos, sel, (size_t)K * sizeof(int32_t));
        if (values_out) memcpy(values_out + val_pos, Cg, (size_t)K * n * sizeof(float));
        sel_pos += K;
        val_pos += K * n;

        for (int32_t i = 0; i < N; i++) free(D[i]);
        free(D); free(sel); free(Cl); free(Cg);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Baseline: compressed momentum SGD without error feedback (Table II rows     */
/* "(without EF)"; SPEC compressed_msgd_step).  The shared          */
/* ARC-Top-K selection is applied to the gradients themselves,                 */
/* c_i = C_local(grad_i), and the replicated heavy-ball momentum is            */
/*   u_t = beta u_{t-1} + (1/N) sum_i c_i,   beta = cfg->eta [R22]:            */
/* u <- beta * u for every element, then u[I] <- u[I] + A / N.                 */
/* ------------------------------------------------------------------------- */
int orc_step_noef(const orc_cfg* cfg, int64_t t, const float* const* grad, float* u,
                  int32_t* sel_out, float* values_out, float* V_out, float* sigma_out)
{
    const int32_t N = cfg->N;
    const float beta = cfg->eta;
    for (int64_t e = 0; e < cfg->d; e++) u[e] = beta * u[e];

    int64_t sel_pos = 0, val_pos = 0, V_pos = 0, sig_pos = 0;
    const float** G = (const float**)malloc((size_t)N * sizeof(float*));
    for (int32_t b = 0; b < cfg->num_blocks; b++) {
        const orc_block* B = &cfg->blocks[b];
        const int64_t m = B->m, n = B->n, K = B->K, len = B->len;
        for (int32_t i = 0; i < N; i++) G[i] = grad[i] + B->offset;
        int32_t* sel = (int32_t*)malloc((size_t)K * sizeof(int32_t));
        float* Cg = (float*)malloc((size_t)K * n * sizeof(float));
        if (B->kind == 0) {
            float* V = (float*)malloc((size_t)n * cfg->r * sizeof(float));
            orc_gaussian_V(cfg->seed, t, b, n, cfg->r, V);
            float* sg = (float*)malloc((size_t)m * sizeof(float));
            orc_arc_round(N, len, m, n, K, cfg->r, G, V, 0, cfg->wire, NULL, NULL, sg, sel, NULL, Cg);
            if (V_out) memcpy(V_out + V_pos, V, (size_t)n * cfg->r * sizeof(float));
            if (sigma_out) memcpy(sigma_out + sig_pos, sg, (size_t)m * sizeof(float));
            V_pos += n * cfg->r;
            sig_pos += m;
            free(V); free(sg);
        } else {
            /* DENSE block: identity compressor, I = all rows [R20] */
            for (int64_t k = 0; k < K; k++) {
                sel[k] = (int32_t)k;
                int64_t nv = row_len(len, n, k);
                for (int64_t q = 0; q < n; q++) {
                    float a = 0.0f;
                    for (int32_t i = 0; i < N; i++) {
                        float c = wire_value((q < nv) ? G[i][k * n + q] : 0.0f, cfg->wire);   /* [R25] */
                        a = (i == 0) ? c : a + c;
                    }
                    Cg[(size_t)k * n + q] = a / (float)N;
                }
            }
        }
        for (int64_t k = 0; k < K; k++) {
            int64_t p = sel[k];
            int64_t nv = row_len(len, n, p);
            for (int64_t q = 0; q < nv; q++) {
                int64_t e = B->offset + p * n + q;
                u[e] = u[e] + Cg[(size_t)k * n + q];
            }
        }
        if (sel_out) memcpy(sel_out + sel_pos, sel, (size_t)K * sizeof(int32_t));
        if (values_out) memcpy(values_out + val_pos, Cg, (size_t)K * n * sizeof(float));
        sel_pos += K;
        val_pos += K * n;
        free(sel); free(Cg);
    }
    free(G);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Baseline: vanilla EF21M with per-node row Top-K (Table I row "Top-K",      */
/* P:91): node i keeps the K rows of its own residual   */
/* with the largest ||row||^2 (ties -> smaller index), and the global update  */
/* is the average of the N differently supported sparse rows.                 */
/* ------------------------------------------------------------------------- */

/* sel_out: [N][sum K_b] per-node selections (ascending within block);
 * values_out: [N][sum K_b n_b] per-node compact rows C_local_i. */
int orc_step_topk(const orc_cfg* cfg, int64_t t,
                  const float* const* grad, float* const* h, float* const* g, float* gbar,
                  int32_t* sel_out, float* values_out)
{
    (void)t;
    const int32_t N = cfg->N;
    const float eta = cfg->eta;
    const float one_minus_eta = 1.0f - eta;
    for (int32_t i = 0; i < N; i++)
        for (int64_t e = 0; e < cfg->d; e++)
            h[i][e] = fmaf(eta, grad[i][e], one_minus_eta * h[i][e]);   /* [R11] */

    int64_t sumK = 0, sumKn = 0;
    for (int32_t b = 0; b < cfg->num_blocks; b++) { sumK += cfg->blocks[b].K; sumKn += cfg->blocks[b].K * cfg->blocks[b].n; }

    int64_t sel_pos = 0, val_pos = 0;
    for (int32_t b = 0; b < cfg->num_blocks; b++) {
        const orc_block* B = &cfg->blocks[b];
        const int64_t m = B->m, n = B->n, K = B->K, len = B->len;
        int32_t* sel = (int32_t*)malloc((size_t)N * K * sizeof(int32_t));
        float* Cl = (float*)malloc((size_t)N * K * n * sizeof(float));
        float* norms = (float*)malloc((size_t)m * sizeof(float));
        for (int32_t i = 0; i < N; i++) {
            /* node-local row norms ||Delta_i[p,:]||^2, Delta_i = h - g, in the
             * O6 order (the exact sketch of one node) */
            float* row = (float*)malloc((size_t)n * sizeof(float));
            for (int64_t p = 0; p < m; p++) {
                int64_t nv = row_len(len, n, p);
                for (int64_t q = 0; q < nv; q++) {
                    int64_t e = B->offset + p * n + q;
                    row[q] = h[i][e] - g[i][e];
                }
                norms[p] = o6_dot(row, row, 1, nv);
            }
            free(row);
            if (B->kind == 0) orc_argtop_k(norms, m, K, sel + (size_t)i * K);
            else for (int64_t k = 0; k < K; k++) sel[(size_t)i * K + k] = (int32_t)k;
            for (int64_t k = 0; k < K; k++) {
                int64_t p = sel[(size_t)i * K + k];
                int64_t nv = row_len(len, n, p);
                for (int64_t q = 0; q < n; q++) {
                    int64_t e = B->offset + p * n + q;
                    Cl[((size_t)i * K + k) * n + q] = (q < nv) ? (h[i][e] - g[i][e]) : 0.0f;
                }
            }
        }
        /* merge: gbar += (1/N) C_local_j for j ascending; g_i += C_local_i */
        for (int32_t i = 0; i < N; i++) {
            for (int64_t k = 0; k < K; k++) {
                int64_t p = sel[(size_t)i * K + k];
                int64_t nv = row_len(len, n, p);
                for (int64_t q = 0; q < nv; q++) {
                    int64_t e = B->offset + p * n + q;
                    float c = Cl[((size_t)i * K + k) * n + q];
                    g[i][e] = g[i][e] + c;
                    gbar[e] = gbar[e] + c / (float)N;
                }
            }
            if (sel_out) memcpy(sel_out + (size_t)i * sumK + sel_pos, sel + (size_t)i * K, (size_t)K * sizeof(int32_t));
            if (values_out) memcpy(values_out + (size_t)i * sumKn + val_pos, Cl + (size_t)i * K * n, (size_t)K * n * sizeof(float));
        }
        sel_pos += K;
        val_pos += K * n;
        free(sel); free(Cl); free(norms);
    }
    return 0;
}

/* eq:ef21m-1 on one vector: h <- fma(eta, grad, (1 - eta) h) [R11] (used by
 * the multi-process protocol tests). */
void orc_momentum(float* h, const float* grad, int64_t d, float eta)
{
    const float one_minus_eta = 1.0f - eta;
    for (int64_t e = 0; e < d; e++) h[e] = fmaf(eta, grad[e], one_minus_eta * h[e]);
}

/* O8 on given node sums: sigma[p] = s, s = +0; s <- fma(S[p][j], S[p][j], s)
 * for j = 0..r-1 (used by the multi-process protocol tests on row slices). */
void orc_sigma_rows(const float* S, int64_t rows, int32_t r, float* sigma)
{
    for (int64_t p = 0; p < rows; p++) {
        float s = 0.0f;
        for (int32_t j = 0; j < r; j++) s = fmaf(S[p * r + j], S[p * r + j], s);
        sigma[p] = s;
    }
}

/* Array forms of the generator's scalar functions (used by the exhaustive
 * accuracy pins in tests/; a plain loop over the scalar function). */
void orc_ln_array(const float* u, int64_t n, float* out)
{
    for (int64_t i = 0; i < n; i++) out[i] = orc_ln(u[i]);
}
void orc_sincos2pi_array(const float* u, int64_t n, float* s, float* c)
{
    for (int64_t i = 0; i < n; i++) orc_sincos2pi(u[i], &s[i], &c[i]);
}

/* ---------------------------------------------------------------------------
 * The model update that consumes gbar (readings R23, R24).
 * ------------------------------------------------------------------------- */

/* eq:ef21m-3: x_{t+1} = x_t - (gamma/N) sum_i g_i^{(t)} = x_t - gamma gbar_t,
 * gbar being the replicated (1/N) sum_i g_i the step maintains [R13].  Per
 * element, each operation rounded once [R23]: x <- x - (gamma * gbar). */
void orc_apply_sgd(float* x, const float* gbar, int64_t d, float gamma)
{
    for (int64_t e = 0; e < d; e++) x[e] = x[e] - gamma * gbar[e];
}

/* "standard Adam" (Kingma & Ba, Algorithm 1; no weight decay) driven by the
 * EF21M direction gbar, as in the paper's GLUE and C4 experiments (P:572,
 * P:578) [R24].  t >= 1 is Adam's step count.  Per element:
 *   m <- fma(1-b1, gbar, b1 * m)            (the O2 form of eq:ef21m-1)
 *   v <- fma(1-b2, gbar * gbar, b2 * v)
 *   mhat = m / bc1,  vhat = v / bc2,   bc_k = fl32(1 - b_k^t) (pow in double)
 *   x <- x - gamma * (mhat / (sqrt(vhat) + eps))                               */
void orc_apply_adam(float* x, float* m, float* v, const float* gbar, int64_t d, int64_t t,
                    float gamma, float beta1, float beta2, float eps)
{
    const float om1 = 1.0f - beta1, om2 = 1.0f - beta2;
    const float bc1 = (float)(1.0 - pow((double)beta1, (double)t));
    const float bc2 = (float)(1.0 - pow((double)beta2, (double)t));
    for (int64_t e = 0; e < d; e++) {
        const float gb = gbar[e];
        m[e] = fmaf(om1, gb, beta1 * m[e]);
        v[e] = fmaf(om2, gb * gb, beta2 * v[e]);
        const float mhat = m[e] / bc1;
        const float vhat = v[e] / bc2;
        x[e] = x[e] - gamma * (mhat / (sqrtf(vhat) + eps));
    }
}
