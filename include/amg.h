/* amg.h -- C ABI of the B200-native solve phase of the AMG-preconditioned Krylov
 * solver for Stokes saddle-point systems of Demidov, Mu & Wang, "Accelerating
 * linear solvers for Stokes problems with C++ metaprogramming" (arXiv 2006.06052).
 *
 * Problem (Listing 3 "Solver S(A, prm)" then apply):
 * given a square sparse block matrix A (BSR), a right-hand side
 * b, an initial guess x0 and a tolerance, return x with ||b - A x||_2 / ||b||_2 <= rtol.
 *
 * Conventions for every entry point
 *  - Pointers are DEVICE pointers unless the comment says "host".
 *  - `stream` is a cudaStream_t passed as void*; every call is stream-ordered on it
 *    (NULL = legacy default stream).  amg_setup / amg_solve synchronise `stream`
 *    before returning (setup reads aggregation flags, solve reads one convergence
 *    scalar per iteration); bsr_spmv never synchronises.
 *  - Every call returns an int status (AMG_OK = 0, AMG_NOT_CONVERGED = 1, negative
 *    codes are errors, see amg_status_string()).  On error nothing the caller owns
 *    is freed; a handle stays valid if it was valid before the call.
 *  - No call throws, no call prints; CUDA/NCCL failures map to AMG_ECUDA / AMG_ENCCL.
 *  - Indices are int32 (nnzb < 2^31), value offsets are 64-bit internally.
 */
#ifndef AMG_B200_H
#define AMG_B200_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---- */
enum {
  AMG_OK = 0,
  AMG_NOT_CONVERGED = 1,       /* x holds the last iterate, report filled */
  AMG_EINVAL = -1,             /* bad argument / unsupported option / coarsening stalled */
  AMG_EDIM = -2,               /* dimension mismatch */
  AMG_EZERODIAG = -3,          /* missing or zero diagonal block */
  AMG_ESINGULAR_BLOCK = -4,    /* a diagonal block is singular */
  AMG_EINDEX_OVERFLOW = -5,    /* nnzb >= 2^31 or n*b overflows int32 */
  AMG_EBREAKDOWN = -6,         /* Krylov breakdown after one restart */
  AMG_ECUDA = -7,
  AMG_ENCCL = -8,
  AMG_ENOMEM = -9
};

typedef enum { AMG_F64 = 0, AMG_F32 = 1 } amg_dtype;
enum { AMG_CG = 0, AMG_BICGSTAB = 1, AMG_GMRES = 2, AMG_IDRS = 3 };
enum { AMG_PC_AMG = 0, AMG_PC_SCHUR = 1, AMG_PC_NONE = 2 };
enum { AMG_SPAI0 = 0, AMG_JACOBI = 1, AMG_ILU0 = 2 /* block ILU(0), Jacobi-sweep solves (R20) */,
       AMG_ILUT = 3 /* block ILUT(tau, p), the paper's U-solver smoother (Listing V2), same solves (R25) */ };
/* coarsening: smoothed aggregation | plain aggregation, P = P_tent
   (Listings V2-V4, "amgcl::coarsening::aggregation") */
enum { AMG_SA = 0, AMG_PLAIN_AGG = 1 };

/* Block-CSR descriptor (PAPER.md:666-672 layout).  Caller-owned; the library never
 * frees or retains it beyond the call (amg_setup deep-copies). */
typedef struct {
  int32_t n_block_rows;   /* rows of this descriptor (local rows when distributed) */
  int32_t n_block_cols;   /* block columns (global) */
  int32_t block_size;     /* b in {1,2,3,4}; the hot path uses 3 and 4 */
  int32_t _pad;
  int64_t nnzb;           /* number of stored blocks, < 2^31 */
  const int32_t* row_ptr; /* [n_block_rows+1], row_ptr[0] = 0, non-decreasing, row_ptr[n] = nnzb */
  const int32_t* col_idx; /* [nnzb], 0-based, strictly increasing within a row; the diagonal
                             block must be present for amg_setup */
  const void* values;     /* [nnzb*b*b] row-major b x b blocks, type `dtype` */
  int32_t dtype;          /* amg_dtype */
  int32_t _pad2;
} amg_bsr;

/* Runtime parameters: a flat version of the paper's nested params structs
 * (Listings 2-3).  Fill with amg_params_default(). */
typedef struct {
  int32_t solver;            /* AMG_CG | AMG_BICGSTAB | AMG_GMRES (flexible GMRES(m)) | AMG_IDRS
                                (IDR(s), the paper's outer solver, Table 1) */
  int32_t gmres_m;           /* restart length, default 30 (PAPER.md:255 shows M = 50) */
  int32_t precond;           /* AMG_PC_AMG (monolithic SA-AMG) | AMG_PC_SCHUR (Eq. 9-10) | AMG_PC_NONE */
  int32_t maxiter;           /* default 1000 */
  int32_t hier_dtype;        /* values of A_l, P_l, R_l, M_l, coarse inverse, B, B^T, m_S:
                                AMG_F32 (default, Listing V4) | AMG_F64 */
  int32_t vcycle_vec_dtype;  /* vectors inside the preconditioner: AMG_F32 (default) | AMG_F64 */
  int32_t smoother;          /* AMG_SPAI0 (default) | AMG_JACOBI | AMG_ILU0 | AMG_ILUT
                                (ILU: single device; the paper's U-solver smoother is ILUT,
                                Listing V2, "AMG with ILU as a smoother has the best
                                performance") */
  int32_t coarse_enough;     /* max scalar unknowns of the coarsest level, default 3000 */
  double jacobi_omega;       /* damped-Jacobi weight, default 2/3 */
  double sa_omega;           /* prolongator damping, default 2/3 (reading R5) */
  double eps_strong;         /* strong-connection threshold, default 1e-3 */
  int32_t max_levels;        /* default 20 */
  int32_t npre, npost;       /* smoothing sweeps, default 1, 1 */
  int32_t schur_p_component; /* pressure component inside a block, default 3 for (u,v,w,p) */
  int32_t use_graphs;        /* 1 (default): replay the preconditioner as a CUDA graph */
  int32_t idrs_s;            /* IDR(s) shadow-space dimension, default 5 (Listings V1-V4 "s = 5") */
  int32_t idrs_seed;         /* IDR(s) shadow-space seed, default 1234 (reading R17) */
  int32_t schur_u_scalar;    /* 1: the Schur U-solver hierarchy is built on the SCALAR expansion of
                                A_u (the paper's V2, Listing V2; R18); 0 (default): on
                                3x3 blocks (V3, Listing V3; fp32 values = V4, Listing V4) */
  int32_t coarsening;        /* AMG_SA (default) | AMG_PLAIN_AGG */
  int32_t schur_shat;        /* matrix of the Schur P-solver's SPAI0: 0 = C; 1 (default) = Eq. 10
                                C - diag(B diag(A_u)^-1 B^T) (adjust_p = 1);
                                2 = the explicitly assembled C - B diag(A_u)^-1 B^T (the PETSc
                                variant) */
  double over_interp;        /* AMG_PLAIN_AGG: A_c = (1/over_interp) P^T A P, default 1.5
                                (over-interpolation, reading R19); ignored for AMG_SA */
  int32_t ilu_sweeps;        /* AMG_ILU0 / AMG_ILUT: Jacobi sweeps per triangular solve, 1..16, default 2 */
  int32_t gmres_ortho;       /* AMG_GMRES orthogonalisation: 3 (default) two-pass Gram/Cholesky with the
                                first pass's dots on an fp16 shadow of the basis at unit-rms scale
                                (R28; +31 fp16 vectors of workspace); 2 the same with an fp32
                                shadow (R23; +31 fp32 vectors); 1 two-pass Gram/Cholesky on the fp64 basis (R22);
                                0 CGS2 (three passes over the basis per step).  1 and 2 reorthogonalise a
                                step whose new direction is still far from orthogonal (R22 safeguard) */
  int32_t fused_presmooth;   /* 1 (default): the pre-smoothing from zero x = M f (K4a) runs in the epilogue of
                                the kernel that produces f (split, B^T update, restriction; DESIGN.md
                                "Fused K4"), bit-identical to 0 (a separate x = M f pass per level) */
  int32_t ilut_p;            /* AMG_ILUT: fill blocks kept per row in each of L and U beyond A's pattern,
                                >= 0, default 2 (the paper gives none) */
  double ilut_tau;           /* AMG_ILUT: drop blocks with ||.||_F < tau ||row of A||_2, >= 0, default 1e-2 */
} amg_params;

typedef struct {
  int32_t iters;        /* Krylov iterations (GMRES: Arnoldi steps; BiCGStab: full steps;
                           IDR(s): products with A, s + 1 per cycle) */
  int32_t converged;    /* 1 iff relres_true <= rtol */
  int32_t levels;       /* AMG levels including the coarsest */
  int32_t restarts;     /* GMRES cycles - 1, or BiCGStab/CG restarts */
  double relres_true;   /* ||b - A x|| / ||b|| recomputed at exit */
  double setup_s;       /* wall seconds of amg_setup (device-synchronised) */
  double solve_s;       /* seconds of this solve: CUDA events on `stream` (max over ranks) */
  double alg_bytes;     /* algorithmic bytes the solve moved */
} amg_report;

struct amg_handle;
struct amg_comm;

int amg_params_default(amg_params* p /* host */);
const char* amg_status_string(int status);

/* Build the solver for A (device descriptor): Schur split + Eq. 10 (if precond =
 * SCHUR), the smoothed-aggregation hierarchy on the GPU, the coarse inverse, the
 * narrowed (fp32) copies and the solve workspace.  A may be freed afterwards. */
int amg_setup(const amg_bsr* A /* host struct, device arrays */, const amg_params* p /* host */,
              void* stream, struct amg_handle** out /* host */);

/* Schur pressure correction with a general scalar pressure mask:
 * pmask (DEVICE, [n_block_rows * block_size] bytes, non-zero = pressure unknown) selects the
 * pressure unknowns among the scalar unknowns of A in any order; the split is taken on the
 * scalar expansion of A and the U-solver hierarchy is scalar (b = 1, as the paper's V2;
 * DESIGN.md reading R21).  p->precond must be AMG_PC_SCHUR, p->schur_shat 0 or 1 (several
 * GPUs: amg_setup_dist_pmask).  The mask may be freed after the call.  Errors as
 * amg_setup; AMG_EINVAL also for an all-velocity or all-pressure mask. */
int amg_setup_pmask(const amg_bsr* A, const uint8_t* pmask, const amg_params* p, void* stream,
                    struct amg_handle** out);

/* Solve A x = b.  b, x: device fp64 [n_block_rows*b]; x is read as x0 and overwritten.
 * Allocates nothing.  ||b|| = 0 returns x = 0, converged, relres 0. */
int amg_solve(struct amg_handle* h, const double* b, double* x, double rtol, void* stream,
              amg_report* rep /* host, may be NULL */);

/* Same as amg_solve with HOST b and x (pageable or pinned); the host<->device copies
 * are part of the call (the bench's end-to-end number). */
int amg_solve_host(struct amg_handle* h, const double* b_host, double* x_host, double rtol,
                   void* stream, amg_report* rep);

/* One application of the preconditioner (z = M r) on outer fp64 device vectors. */
int amg_apply_precond(struct amg_handle* h, const double* r, double* z, void* stream);

/* y = alpha A x + beta y with fp64 accumulation (C1); beta == 0 overwrites y (NaN
 * included).  x, y: device vectors of type xt / yt. */
int bsr_spmv(const amg_bsr* A, double alpha, const void* x, int32_t xt, double beta, void* y,
             int32_t yt, void* stream);

void amg_destroy(struct amg_handle* h);

/* Scalar CSR -> BSR on the device (S1; the §4 worked example PAPER.md:658-672):
 * one b x b block per non-empty tile of the scalar matrix; scalars absent inside a stored
 * tile become explicit zeros; duplicate scalar entries are summed in CSR order.  n and m
 * (scalar rows / columns) must be multiples of b; columns need not be sorted.  Inputs:
 * ptr[n+1], col[nnz], val[nnz] of `dtype` (DEVICE).  Two calls: with bptr == NULL only
 * *nnzb_out (host) is written; then, with caller-allocated DEVICE arrays bptr[n/b+1],
 * bcol[nnzb], bval[nnzb*b*b] (same dtype), the BSR is filled (columns sorted per block
 * row).  Synchronises `stream`.  Errors: AMG_EINVAL (b < 1, n or m not divisible, a
 * column outside [0, m)), AMG_EINDEX_OVERFLOW (nnz >= 2^31), AMG_ENOMEM, AMG_ECUDA. */
int amg_csr_to_bsr(int32_t n, int32_t m, int32_t b, int64_t nnz, const int32_t* ptr, const int32_t* col,
                   const void* val, int32_t dtype, int32_t* bptr, int32_t* bcol, void* bval, int64_t* nnzb_out,
                   void* stream);

/* SpMV plan for repeated products y = alpha A x + beta y (same semantics and errors as
 * bsr_spmv; §4 block layout PAPER.md:644-682).  Creation picks the
 * kernel from the block shape and row length and, for long rows (> 12 blocks per row,
 * enough rows to fill the GPU, square b = 2..4), builds a SLICED copy of A's blocks
 * (32/b consecutive block rows per slice, zero-padded to the slice's longest row) that
 * the plan owns and frees in bsr_plan_destroy (device memory ~= A's values + columns;
 * one stream sync).  The plan also keeps A's device pointers: A's arrays must stay
 * allocated and unchanged while the plan is used.  Errors: AMG_EINVAL (bad A / NULL
 * out), AMG_EINDEX_OVERFLOW (sliced copy beyond 2^31 steps), AMG_ENOMEM, AMG_ECUDA. */
struct bsr_plan;
int bsr_plan_create(const amg_bsr* A /* host struct, device arrays */, void* stream, struct bsr_plan** out);
int bsr_plan_spmv(struct bsr_plan* P, double alpha, const void* x, int32_t xt, double beta, void* y,
                  int32_t yt, void* stream);
void bsr_plan_destroy(struct bsr_plan* P);

/* ---- introspection (used by the parity tests; all outputs HOST) ---- */
/* out[5] = {n_block_rows, block_size, nnzb(A_l), nnzb(P_l) or 0, n_coarse or 0} */
int amg_level_info(struct amg_handle* h, int32_t level, int64_t* out);
/* which: 0 = A_l, 1 = P_l, 2 = R_l (the solve copies in the hierarchy dtype, widened to fp64); 3 = smoother blocks M_l
 * (ptr/col ignored, val = n*b*b; AMG_ILU0: the pivot inverses D^-1); 4 / 5 = the ILU strictly lower / upper
 * factors (AMG_ILU0 / AMG_ILUT only, else AMG_EINVAL; at most nnz(A_l) - n_l blocks, + ilut_p * n_l with
 * AMG_ILUT; ptr[n] gives the count).  Arrays sized
 * from amg_level_info. */
int amg_level_export(struct amg_handle* h, int32_t level, int32_t which, int32_t* ptr, int32_t* col,
                     double* val);
int amg_level_aggregates(struct amg_handle* h, int32_t level, int32_t* agg);
/* Schur vectors: Shat diagonal and m_S (n_block_rows each; amg_setup_pmask: one per pressure
 * unknown, in ascending scalar order), fp64 setup values */
int amg_schur_export(struct amg_handle* h, double* shat_diag, double* m_s);
/* One V-cycle of the hierarchy on fp64 device vectors of the level-0 size. */
int amg_vcycle(struct amg_handle* h, const double* f, double* x, void* stream);
/* device bytes held by the handle (hierarchy + workspace) */
int64_t amg_device_bytes(struct amg_handle* h);
/* Memory footprint per component (the paper's memory comparisons, PAPER.md:717-718,
 * 836-857), bytes, out[n >= 8] (host): [0] outer operator (BSR + sliced copy),
 * [1] hierarchy A_l/P_l/R_l (BSR), [2] their sliced copies, [3] smoother blocks M_l,
 * [4] Schur B, B^T, m_S, [5] coarse inverse, [6] Krylov workspace vectors, [7] total
 * allocated by the handle (includes halo buffers, aggregates, padding).  AMG_EINVAL on a
 * NULL handle / out or n < 8. */
int amg_memory_report(struct amg_handle* h, int64_t* out, int32_t n);

/* Solve counters since setup (host out[n >= 2]): [0] extra orthogonalisation passes the
 * Gram/Cholesky GMRES took where a new direction was still far from orthogonal to the basis
 * (the reorthogonalisation safeguard, reading R22); [1] CUDA graphs instantiated.
 * AMG_EINVAL on a NULL handle / out or n < 2. */
int amg_solve_counters(struct amg_handle* h, int64_t* out, int32_t n);

/* ---- launch accounting / per-kernel timing (diagnostics, host) ---- */
/* number of library kernels launched by this process so far */
int64_t amg_kernel_launches(void);
/* start recording a CUDA-event pair and the algorithmic bytes around every launch */
int amg_profile_begin(void);
/* stop recording; writes a JSON list [{"kernel","bytes","launches","total_ms"}, ...]
 * aggregated per (kernel, bytes per launch) into out (host, capacity cap) and returns the
 * full length.  Synchronises the device. */
int64_t amg_profile_end(char* out, int64_t cap);
/* text of the last error raised on this thread */
const char* amg_last_error(void);

/* ---- multi-GPU: one process per GPU, contiguous block-row slabs ---- */
/* NCCL unique id (128 bytes, host) generated by rank 0 (amg_comm_unique_id) and
 * broadcast by the caller (torch.distributed). */
int amg_comm_unique_id(void* id128 /* host, 128 B */);
int amg_comm_init(const void* id128 /* host */, int32_t nranks, int32_t rank,
                  struct amg_comm** out);
/* A_local: this rank's rows [row_begin, row_begin + n_block_rows) with GLOBAL column
 * ids.  After this call amg_solve takes the LOCAL slices of b and x. */
int amg_setup_dist(const amg_bsr* A_local, int64_t row_begin, int64_t n_global_block_rows,
                   struct amg_comm* c, const amg_params* p, void* stream, struct amg_handle** out);
/* amg_setup_dist with a general scalar pressure mask (R21 on several ranks, R27):
 * pmask_local (DEVICE, [A_local->n_block_rows * block_size] bytes, non-zero = pressure) marks
 * this rank's scalar unknowns; each class is numbered globally in ascending scalar order, so a
 * rank owns a contiguous range of velocity and of pressure unknowns, and the scalar U-solver
 * hierarchy is slab-distributed by those ranges.  p->precond must be AMG_PC_SCHUR,
 * p->schur_shat 0 or 1.  Collective; errors as amg_setup_dist. */
int amg_setup_dist_pmask(const amg_bsr* A_local, const uint8_t* pmask_local, int64_t row_begin,
                         int64_t n_global_block_rows, struct amg_comm* c, const amg_params* p, void* stream,
                         struct amg_handle** out);
void amg_comm_destroy(struct amg_comm* c);
/* Thread-emulated communicator (testing the distributed path on ONE device): a group of
 * nranks host threads of this process, each with its own stream; exchanges are device
 * copies with host barriers (no kernel ever waits on another rank), reductions are
 * summed in rank order.  Same semantics as the NCCL communicator. */
int amg_local_group_create(int32_t nranks, void** group /* host out */);
void amg_local_group_destroy(void* group);
int amg_comm_init_local(void* group, int32_t rank, struct amg_comm** out);

/* Host-staged communicator over a caller's transport (separate PROCESSES, e.g. a
 * torch.distributed gloo group, on one device or several): every exchange is copied to host
 * memory, handed to the callbacks below, and copied back; the stream is synchronised around
 * each call, so no kernel ever waits on another process.  For testing the distributed data
 * plane with real processes where NCCL cannot run (one GPU); the product path is NCCL.
 * Every callback returns 0 on success; any other value fails the call with AMG_ENCCL.  All
 * buffers are HOST memory owned by the library for the duration of the call. */
typedef struct {
  void* ctx;
  /* in-place sum over ranks of n fp64 values */
  int (*allreduce_sum)(void* ctx, double* vals, int32_t n);
  /* all[r * n_each + i] = rank r's mine[i] */
  int (*allgather_i64)(void* ctx, const int64_t* mine, int32_t n_each, int64_t* all);
  /* grouped point-to-point: ns sends (peer, buffer, bytes) and nr receives, completed on return */
  int (*exchange)(void* ctx, int32_t ns, const int32_t* send_peer, const void* const* send_buf,
                  const int64_t* send_bytes, int32_t nr, const int32_t* recv_peer, void* const* recv_buf,
                  const int64_t* recv_bytes);
  int (*barrier)(void* ctx);
} amg_host_comm_ops;
/* flags & 1: stream-ordered mode -- each exchange / reduction becomes device->pinned-host copies,
 * a cudaLaunchHostFunc running the callback, and host->device copies, all on the caller's
 * stream (no host synchronisation, so the solve's CUDA graphs capture them as they capture the
 * NCCL calls); the callbacks then run on CUDA's host-function thread and must not call CUDA.
 * Pinned staging: AMG_HOSTCOMM_POOL_MB (default 256) allocated here. */
int amg_comm_init_host(const amg_host_comm_ops* ops /* host, copied */, int32_t nranks, int32_t rank,
                       int32_t flags, struct amg_comm** out);

#ifdef __cplusplus
}
#endif
#endif
