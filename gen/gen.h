/* gen.h -- seeded synthetic inputs for the five BASELINE.json configs.
 *
 * This module is TEST/BENCH INPUT, not solver code: it holds none of the
 * method's arithmetic (no SpMV, aggregation, smoothing, Krylov).  Both the
 * oracle harness and the CUDA path consume its output; neither shares any
 * other code (SURVEY.md §8(d) "Synthetic inputs", §1 layer L0).
 *
 * RNG: counter based, so a rank can generate its z-slab
 * independently and bit-identically to the global generation.
 *   mix(z)          = SplitMix64 finaliser
 *   R(stream, idx)  = mix(mix(SEED ^ (stream << 56)) ^ idx)
 *   U01             = (R >> 11) * 2^-53
 *   Uni(a,b)        = a + (b - a) * U01
 *   N01(stream,idx) = Box-Muller, u1 = 1 - U01(stream, 2 idx), u2 = U01(stream, 2 idx + 1),
 *                     z = sqrt(-2 ln u1) cos(2 pi u2)
 * Streams: 1 cfg-1 G entries; 2 uniform RHS; 3 cfg-2 block values; 4 cfg-2 x; 5 Stokes RHS noise.
 *
 * Grid index: I = i + n (j + n k), x fastest, z slowest, so z-slabs are
 * contiguous block-row ranges.  Columns are emitted sorted ascending.
 * All matrices: BSR, 0-based, int32 row_ptr (local, starting at 0) and int32
 * GLOBAL column ids, fp64 row-major b x b blocks.
 */
#ifndef GEN_H
#define GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define GEN_SEED 200606052ULL

enum gen_kind {
  GEN_POISSON3 = 1, /* cfg 1: 7-point vector Poisson, b = 3, + 0.1 G G^T per node */
  GEN_RAND27 = 2,   /* cfg 2: 27-point pattern, N(0,1) blocks, +30 I on the diagonal */
  GEN_STOKES = 3    /* cfg 3-5: stabilised collocated Stokes, b = 4, (u,v,w,p) */
};

enum gen_rhs_kind {
  GEN_RHS_UNIFORM = 0,     /* b_q = Uni(-1,1)(stream 2, q)                    (cfg 1) */
  GEN_RHS_LID = 1,         /* b[4I+0] = 1/h^2 on the k = n-1 layer            (cfg 3) */
  GEN_RHS_FORCE_NOISE = 2, /* f = (sin pi x, cos pi y, 0) + 0.01 N01(5, q)     (cfg 4) */
  GEN_RHS_LID_NOISE = 3,   /* lid term + 0.01 N01(5, q)                        (cfg 5) */
  GEN_X_UNIFORM = 4        /* x_q = Uni(-1,1)(stream 4, q)                     (cfg 2) */
};

uint64_t gen_mix(uint64_t z);
uint64_t gen_rand(uint64_t stream, uint64_t idx);
double gen_u01(uint64_t stream, uint64_t idx);
double gen_uni(uint64_t stream, uint64_t idx, double a, double b);
double gen_n01(uint64_t stream, uint64_t idx);

/* Block size a kind produces (b for RAND27 is the caller's choice: 1..4). */
int gen_block_size(int kind, int b_rand27);

/* Number of stored blocks in block rows [row_begin, row_end) of an n^3 grid. */
int64_t gen_nnzb(int kind, int n, int64_t row_begin, int64_t row_end);

/* Fill ptr[(row_end-row_begin)+1], col[nnzb], val[nnzb*b*b].
 * Returns 0, or -1 on bad arguments. */
int gen_matrix(int kind, int n, int b, int64_t row_begin, int64_t row_end,
               int32_t* ptr, int32_t* col, double* val);

/* Fill out[(row_end-row_begin)*b] with the RHS (or cfg-2 x) of the given kind
 * for block rows [row_begin, row_end); q below is the GLOBAL scalar index. */
int gen_rhs(int rhs_kind, int n, int b, int64_t row_begin, int64_t row_end, double* out);

#ifdef __cplusplus
}
#endif
#endif
