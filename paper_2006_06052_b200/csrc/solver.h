// solver.h -- the solver handle: hierarchy, Schur pieces, Krylov workspace.
#pragma once

#include <functional>
#include <vector>

#include "blas1.h"
#include "comm.h"
#include "common.cuh"

struct ncclComm;

namespace amgb {

// Ghost exchange plan of one row-distributed square matrix.  Local
// columns are [0, nloc); ghost column g lives at nloc + g, ghosts sorted by global index
// (hence grouped by owner rank).  Vectors read by the matrix carry (nloc + nghost) blocks.
struct Halo {
  int nloc = 0, nghost = 0;
  std::vector<int> peers;
  std::vector<int> send_cnt, send_off, recv_cnt, recv_off;  // per peer, in blocks
  int32_t* send_idx = nullptr;  // device [total_send]: local rows to pack
  int total_send = 0;
  void* send_buf = nullptr;     // device, total_send * 4 doubles
  // rows [int_lo, int_hi) reference no ghost: computed while the exchange is in flight
  // (empty: no overlap)
  int32_t int_lo = 0, int_hi = 0;
};

struct Level {
  Mat A, P, R;                // solve copies, values in hier dtype
  Mat Lf, Uf;                 // AMG_ILU0: strictly lower / upper factor blocks (else empty)
  Halo halo;                  // distributed: ghost plan of A
  void* M = nullptr;          // smoother blocks [n][b][b], hier dtype (AMG_ILU0: pivot inverses)
  void* w[4] = {};            // AMG_ILU0 sweep vectors (y, y', z, z'), vec dtype
  int32_t* agg = nullptr;     // aggregates (device) [n], -1 = isolated
  int32_t nc = 0;
  void *f = nullptr, *x = nullptr, *r = nullptr, *t = nullptr;  // work vectors, vec dtype
};

struct Coarse {
  // distributed: the coarsest level is replicated (its right-hand side allgathered from the
  // ranks' slabs, Handle::lbounds, before the GEMV)
  int32_t N = 0;              // scalar unknowns of the coarsest level
  int32_t n = 0, b = 0;
  void* inv = nullptr;        // dense explicit inverse [N][N], hier dtype
  void *f = nullptr, *x = nullptr;
  Mat A;                      // the coarsest matrix (solve copy, for export)
};


struct PcGraph {
  const double* r;
  void* z;
  int zt;
  const double* sd;
  cudaGraphExec_t exec;
  int64_t kernels;
};

struct Handle {
  amg_params p{};
  int vt = AMG_F32, xt = AMG_F32;  // hier value dtype, V-cycle vector dtype
  Mat A;                           // outer operator, fp64 (library copy)
  int32_t n = 0, b = 0;            // outer block rows / block size
  // Schur: B (1 x nu) and B^T (nu x 1) values on A's pattern, m_S
  bool schur = false;
  int pc = 3, nu = 3;
  void *Bv = nullptr, *BTv = nullptr, *mS = nullptr;
  Mat Bm, BTm;                     // views of B / B^T on A's pattern (1 x nu / nu x 1 blocks)
  double *shat64 = nullptr, *mS64 = nullptr;
  // general scalar pressure mask (amg_setup_pmask, R21): Bm / BTm are then scalar (b = 1)
  // solve copies of B (np x nu) and B^T (nu x np); uidx / pidx the unknowns of each class
  const uint8_t* pmask_in = nullptr;  // setup only
  bool masked = false;
  int32_t np_s = 0, nu_s = 0;
  int32_t *uidx = nullptr, *pidx = nullptr;
  // distributed pressure mask (R27): the ranks' ranges of the velocity / pressure classes
  // (global class numbering; ubounds = the U-solver hierarchy's level-0 slabs) and the ghost
  // plans of the scalar B (velocity ghosts) and B^T (pressure ghosts)
  std::vector<int64_t> ubounds, pbounds;
  Halo haloBu, haloBTp;
  void *ru = nullptr, *rp = nullptr, *us = nullptr, *pp = nullptr, *ru2 = nullptr, *uu = nullptr;
  // AMG hierarchy (on A, or on A_u for Schur)
  int bh = 0;
  std::vector<Level> lv;
  Coarse coarse;
  bool amg_active = false;         // precond != NONE
  // outer-vector workspace (fp64, n*b each)
  int nvec = 0;
  std::vector<double*> vec;
  // GMRES basis (fp64) and preconditioned basis Z (fp32 when the PC output is fp32-exact)
  std::vector<double*> V;
  std::vector<void*> Vs;           // gmres_ortho = 2 / 3: fp32 / fp16 shadow of V for the pass-1 dots (R23 / R28)
  std::vector<void*> Z;
  int zt = AMG_F64;
  // IDR(s) (AMG_IDRS): shadow space, G = A U, U (search directions); shadow seed base
  std::vector<double*> Pi, Gi, Ui;
  uint64_t idrs_base = 0;
  bool idrs_ready = false;
  // reductions
  double* partials = nullptr;      // [kMaxPartials * 32]
  double* dscal = nullptr;         // device scalars [64]
  double* hscal = nullptr;         // pinned host mirror [64]
  // CUDA graphs of the preconditioner application, one per (input, output, dtype, scale)
  std::vector<PcGraph> pc_graphs;
  // one Krylov step as a CUDA graph (BiCGStab, reading R24), per iterate pointer
  std::vector<std::pair<const double*, cudaGraphExec_t>> step_graphs;
  int64_t step_graph_kernels = 0;
  cudaStream_t work = nullptr;     // non-blocking stream the Krylov solve runs on (graph capture)
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  double *stage_b = nullptr, *stage_x = nullptr;  // amg_solve_host's device b / x (alloc_workspace)
  int64_t reorth_passes = 0;       // GMRES Gram/Cholesky: extra orthogonalisation passes taken
  // timing
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double setup_s = 0.0;
  double alg_bytes_precond = 0.0, alg_bytes_spmv = 0.0;
  // distributed (amg_setup_dist): communicator, outer ghost plan, slab bounds per level
  CommBase* comm = nullptr;
  Halo halo0;
  double* x_ext = nullptr;         // fp64 copy of the iterate with ghost space
  cudaStream_t comm_s = nullptr;   // halo exchanges overlapped with the interior rows
  cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
  int64_t row_lo = 0;
  int64_t n_global_rows = 0;       // global block rows (== n when not distributed)
  std::vector<std::vector<int64_t>> lbounds;
  // distributed: levels >= rep_from are replicated on every rank (whole level, no halos); the
  // right-hand side of level rep_from is allgathered from the ranks' slabs (rep_from ==
  // lv.size(): only the coarsest level, the dense inverse)
  size_t rep_from = 0;
  // build the interleaved / sliced solve copies (false for the distributed setup's replicated
  // global handle: every rank slices the BSR arrays and plans its own slabs)
  bool want_copies = true;
  Arena arena;
  ~Handle();
};

// setup.cu
void setup_build(Handle& h, const Mat& A64 /* device fp64 copy owned by h */, const std::vector<int64_t>& bounds,
                 cudaStream_t s);
void alloc_workspace(Handle& h, cudaStream_t s);
// solver.cu: full single-device build on a device matrix view with slab bounds
// workspace = false: hierarchy only (the replicated global handle of amg_setup_dist, whose
// slabs are copied out: no global Krylov basis on every rank)
Handle* build_handle(const Mat& view, const amg_params* p, const std::vector<int64_t>& bounds, cudaStream_t s,
                     bool workspace = true, const uint8_t* pmask = nullptr);
// dist.cu
void halo_exchange(Handle& h, const Halo& H, void* x, int dt, int b, cudaStream_t s);
// launch(r0, r1) over all block rows of A, x's ghosts exchanged first -- on the handle's
// comm stream while the interior rows [H.int_lo, H.int_hi) run, then the
// boundary rows.  Row-lane plans only; otherwise exchange, then one launch.
void halo_overlapped(Handle& h, const Halo& H, const Mat& A, void* x, int dt, int b, cudaStream_t s,
                     const std::function<void(int, int)>& launch);
void dist_allreduce(Handle& h, double* d, int n, cudaStream_t s);
// distributed: allgather the slabs of level l's right-hand side (l == h.rep_from)
void replicated_allgather(Handle& h, size_t l, cudaStream_t s);
// level l's right-hand-side buffer at this rank's slab offset (where R_{l-1} writes)
void* level_f_slab(Handle& h, size_t l);
// vcycle.cu
// V-cycle from level `level` on that level's f buffer; returns the buffer holding x
// pre_done: level `level`'s x = M f was already formed by the producer of f (fused K4a)
// join target of the Schur apply's second U-solve (K9' fused into its last post-smoothing step)
struct JoinOut {
  const void* p;
  void* z;
  int zt;
};
// returns the level's x, or nullptr when `jo` was honoured (z written)
void* vcycle_run(Handle& h, size_t level, cudaStream_t s, bool pre_done = false, const JoinOut* jo = nullptr);
// can the producer of level l's f also form x = M f (fused K4a)?
bool fuse_presmooth(const Handle& h, size_t level);
void* level0_f(Handle& h);
// z = M r (outer fp64 r scaled by `scale` or by *scale_dev when given, z of dtype zt)
// pre (BiCGStab's step graph): form the input r = pre->p = pre->r + beta (pre->p - omega pre->v)
// first (k_bicg_p), fused into the monolithic apply's narrowing where bicg_p_fused(h)
struct BicgPre {
  const double* r;
  const double* v;
  double* p;
  const double* sc;
};
void precond_apply(Handle& h, const double* r, void* z, int zt, cudaStream_t s, double scale = 1.0,
                   const double* scale_dev = nullptr, const BicgPre* pre = nullptr);
bool bicg_p_fused(const Handle& h);
// the same, replayed from a per-(r, z, zt, scale_dev) CUDA graph (s must not be the legacy stream)
void precond_apply_graphed(Handle& h, const double* r, void* z, int zt, cudaStream_t s, const double* scale_dev);
double precond_bytes(const Handle& h);
// krylov.cu
int krylov_solve(Handle& h, const double* b, double* x, double rtol, cudaStream_t s, amg_report* rep);

}  // namespace amgb
