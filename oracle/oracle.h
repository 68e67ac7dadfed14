/* oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded C++17 CPU implementation of the solve phase of
 * the paper's AMG-preconditioned Krylov solver for Stokes systems (Demidov, Mu,
 * Wang, arXiv 2006.06052), written from PAPER.md and the readings in SURVEY.md
 * §8(c) / DESIGN.md "Readings".  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it.  It shares no code, header, table or
 * helper with the CUDA library (paper_2006_06052_b200/) and neither includes
 * nor links the other.
 *
 * Everything is fp64; "fp32 hierarchy" is emulated by rounding matrix values
 * (RNE) at setup and vector values at every store.
 * Compiled with -ffp-contract=off so every product and sum rounds separately,
 * in the order written.
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_CG = 0, ORC_BICGSTAB = 1, ORC_GMRES = 2, ORC_IDRS = 3 };
enum { ORC_PC_AMG = 0, ORC_PC_SCHUR = 1, ORC_PC_NONE = 2 };
enum { ORC_SPAI0 = 0, ORC_JACOBI = 1, ORC_ILU0 = 2, ORC_ILUT = 3 };
enum { ORC_SA = 0, ORC_PLAIN = 1 };

enum {
  ORC_OK = 0, ORC_NOT_CONVERGED = 1, ORC_EINVAL = -1, ORC_EDIM = -2, ORC_EZERODIAG = -3,
  ORC_ESINGULAR_BLOCK = -4, ORC_EBREAKDOWN = -6
};

typedef struct {
  int32_t solver, gmres_m, precond, maxiter;
  int32_t hier_f32;      /* hierarchy values (A_l, P_l, R_l, M_l, coarse, B, B^T, m_S) rounded to fp32 */
  int32_t vec_f32;       /* V-cycle / Schur inner vectors rounded to fp32 at every store */
  int32_t smoother;      /* ORC_SPAI0 | ORC_JACOBI | ORC_ILU0 (block ILU(0), sweep-solved, R20) |
                            ORC_ILUT (block ILUT(tau, p), sweep-solved, R25) */
  double jacobi_omega;   /* 2/3 */
  double sa_omega;       /* 2/3 */
  double eps_strong;     /* 1e-3 */
  int32_t coarse_enough; /* 3000 scalar unknowns */
  int32_t max_levels;    /* 20 */
  int32_t npre, npost;   /* 1, 1 */
  int32_t schur_p_component; /* 3 */
  int32_t nparts;        /* rank-local aggregation: number of contiguous block-row slabs (1 = global) */
  int32_t idrs_s;        /* IDR(s) shadow-space dimension (5, PAPER.md Listing V1-V4 "prm.solver.s = 5") */
  int32_t idrs_seed;     /* IDR(s) shadow-space seed (1234) */
  int32_t schur_u_scalar; /* 1: the U-solver hierarchy is built on the SCALAR expansion of A_u
                             (AMGCL V2, Listing V2); 0: on 3x3 blocks (V3/V4, Listing V3) */
  int32_t coarsening;    /* ORC_SA: smoothed aggregation; ORC_PLAIN: plain
                            aggregation, P = P_tent (Listings V2-V4 "coarsening::aggregation") */
  int32_t schur_shat;    /* P-solver matrix: 0 = C; 1 = Eq. 10 C - diag(B diag(A_u)^-1 B^T)
                            (adjust_p = 1); 2 = the explicitly
                            assembled C - B diag(A_u)^-1 B^T (the PETSc variant) */
  double over_interp;    /* plain aggregation: A_c = (1/over_interp) P^T A P (reading R19, 1.5) */
  int32_t ilu_sweeps;    /* ORC_ILU0 / ORC_ILUT: Jacobi sweeps per triangular solve (>= 1, default 2, R20) */
  int32_t gmres_ortho;   /* GMRES orthogonalisation: 0 CGS2 (default), 1 two-pass Gram/Cholesky
                            (R22), 2 the same with the first pass's dots on the fp32-rounded basis (R23),
                            3 on the fp16-rounded basis at unit-rms scale (R28) */
  double ilut_tau;       /* ORC_ILUT drop tolerance relative to the row's 2-norm (1e-2) */
  int32_t ilut_p;        /* ORC_ILUT fill entries kept per row in each of L and U (2) */
} orc_params;

typedef struct {
  int32_t iters, converged, levels, restarts;
  double relres_true;
} orc_report;

typedef struct orc_mat orc_mat;   /* BSR with square b x b fp64 blocks */
typedef struct orc_solver orc_solver;

void orc_params_default(orc_params* p);

/* ---- C0 containers ---- */
orc_mat* orc_mat_new(int32_t n_rows, int32_t n_cols, int32_t b, const int32_t* ptr,
                     const int32_t* col, const double* val);
void orc_mat_free(orc_mat* A);
/* out[4] = {n_rows, n_cols, b, nnzb} */
void orc_mat_info(const orc_mat* A, int64_t* out);
void orc_mat_export(const orc_mat* A, int32_t* ptr, int32_t* col, double* val);
/* S1 / §4 worked example: scalar CSR (n x m, both divisible by b) -> BSR; absent
 * scalars inside a stored tile become explicit zeros.  NULL if not divisible. */
orc_mat* orc_csr_to_bsr(int32_t n, int32_t m, int32_t b, const int32_t* ptr, const int32_t* col,
                        const double* val);

/* ---- C1 SpMV: y = alpha A x + beta y (beta == 0 overwrites y, NaN included) ---- */
int orc_spmv(const orc_mat* A, double alpha, const double* x, double beta, double* y);

/* Schur pressure correction with a general scalar pressure mask (
 * SPEC.md:631 pmask): pmask[q] != 0 marks scalar unknown q (of n_rows*b) as pressure.  The
 * split is taken on the scalar expansion of A (reading R21); the U-solver hierarchy is
 * scalar (b = 1, as V2).  p->precond must be ORC_PC_SCHUR; schur_shat 0 or 1. */
int orc_setup_pmask(const orc_mat* A, const uint8_t* pmask, const orc_params* p, orc_solver** out);
/* number of pressure unknowns of a Schur solver (the length of the S_hat / m_S vectors) */
int32_t orc_schur_np(const orc_solver* s);

/* ---- smoother pieces (for pins) ---- */
/* x = S_l(f): the pre-smoother of level l from a zero initial guess (SPAI0 / Jacobi:
 * x = M f; ILU(0): the sweep-solved (LU)^-1 f), vectors at the solver's precision. */
int orc_level_smooth(const orc_solver* s, int32_t level, const double* f, double* x);

/* ---- C2 / C3 one-level pieces (for pins) ---- */
/* strength graph after symmetric closure, as CSR without diagonal: returns number of
 * edges; if ptr/col non-NULL they are filled (ptr[n+1], col[edges]). */
int64_t orc_strength(const orc_mat* A, double eps, int32_t nparts, int32_t* ptr, int32_t* col);
/* aggregate id per block row (-1 = isolated); returns number of aggregates, <0 on error. */
int32_t orc_aggregate(const orc_mat* A, double eps, int32_t nparts, int32_t* agg);
/* pass-1 roots flag per row (1 = root) */
int32_t orc_roots(const orc_mat* A, double eps, int32_t nparts, int32_t* is_root);
/* block inverse used by every setup step (Gauss-Jordan, partial pivoting) */
int orc_block_inverse(int32_t b, const double* blk, double* inv);

/* ---- full solver: setup (C2-C10) ---- */
int orc_setup(const orc_mat* A, const orc_params* p, orc_solver** out);
void orc_free(orc_solver* s);
int32_t orc_levels(const orc_solver* s);
/* borrowed level matrices of the AMG hierarchy (on A, or on A_u for Schur); NULL past range.
 * which: 0 = A_l, 1 = P_l, 2 = R_l.  Values are the fp64 setup values (before narrowing). */
const orc_mat* orc_level_mat(const orc_solver* s, int32_t level, int32_t which);
/* aggregates of level l (length n_l), -1 = isolated */
const int32_t* orc_level_agg(const orc_solver* s, int32_t level);
/* smoother blocks M_l (n_l * b * b), fp64 setup values */
const double* orc_level_M(const orc_solver* s, int32_t level);
/* Schur pieces: velocity matrix A_u (3x3 BSR), Shat diagonal (n), m_S (n); NULL if not Schur */
const orc_mat* orc_schur_Au(const orc_solver* s);
/* the matrix the U-solver hierarchy is built on (A_u, or its scalar expansion) */
const orc_mat* orc_schur_Au_amg(const orc_solver* s);
const double* orc_schur_Shat_diag(const orc_solver* s);
const double* orc_schur_mS(const orc_solver* s);

/* ---- applies ---- */
/* one V-cycle of the hierarchy on a vector of the AMG's level-0 size (scalars n_0*b),
 * from zero.  Uses the solver's precision mode. */
int orc_vcycle(const orc_solver* s, const double* f, double* x);
/* one preconditioner application z = M r on the outer vector (AMG or Schur) */
int orc_precond(const orc_solver* s, const double* r, double* z);
/* solve A x = b to relres rtol from the given x (x0), fills rep.  history (optional,
 * length maxiter+1) receives the per-iteration residual estimate ||r||/||b||. */
/* IDR(s) shadow space (tests): s orthonormal vectors [sdim][n] of the counter RNG, stream 6 */
int orc_idrs_shadow(int64_t n, int32_t sdim, int64_t base, double* out);
int orc_solve(const orc_solver* s, const double* b, double* x, double rtol, orc_report* rep,
              double* history);
/* orc_solve with timing instrumentation (no change to the arithmetic): stamps[it] (it < cap)
 * receives the seconds since the call started at which iteration `it` completed (stamps[0] =
 * 0).  Used by bench.py's reference arm to time bounded samples of a full-size solve. */
int orc_solve_timed(const orc_solver* s, const double* b, double* x, double rtol, orc_report* rep,
                    double* stamps, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif
