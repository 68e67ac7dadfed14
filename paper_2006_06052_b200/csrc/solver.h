// solver.h -- the solver handle: hierarchy, Schur pieces, Krylov workspace.
#pragma once

#include <vector>

#include "blas1.h"
#include "common.cuh"

struct ncclComm;

namespace amgb {

struct Level {
  Mat A, P, R;                // solve copies, values in hier dtype
  void* M = nullptr;          // smoother blocks [n][b][b], hier dtype
  int32_t* agg = nullptr;     // aggregates (device) [n], -1 = isolated
  int32_t nc = 0;
  void *f = nullptr, *x = nullptr, *r = nullptr, *t = nullptr;  // work vectors, vec dtype
};

struct Coarse {
  int32_t N = 0;              // scalar unknowns of the coarsest level
  int32_t n = 0, b = 0;
  void* inv = nullptr;        // dense explicit inverse [N][N], hier dtype
  void *f = nullptr, *x = nullptr;
  Mat A;                      // the coarsest matrix (solve copy, for export)
};

struct DistInfo;              // dist.cu

struct Handle {
  amg_params p{};
  int vt = AMG_F32, xt = AMG_F32;  // hier value dtype, V-cycle vector dtype
  Mat A;                           // outer operator, fp64 (library copy)
  int32_t n = 0, b = 0;            // outer block rows / block size
  // Schur: B (1 x nu) and B^T (nu x 1) values on A's pattern, m_S
  bool schur = false;
  int pc = 3, nu = 3;
  void *Bv = nullptr, *BTv = nullptr, *mS = nullptr;
  double *shat64 = nullptr, *mS64 = nullptr;
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
  std::vector<void*> Z;
  int zt = AMG_F64;
  // reductions
  double* partials = nullptr;      // [kMaxPartials * 32]
  double* dscal = nullptr;         // device scalars [64]
  double* hscal = nullptr;         // pinned host mirror [64]
  // CUDA graph of one preconditioner application (input/output = fixed buffers)
  cudaGraphExec_t pc_graph = nullptr;
  cudaStream_t pc_graph_stream = nullptr;
  double* pc_in = nullptr;
  double* pc_out = nullptr;
  // timing
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double setup_s = 0.0;
  double alg_bytes_precond = 0.0, alg_bytes_spmv = 0.0;
  DistInfo* dist = nullptr;
  Arena arena;
  ~Handle();
};

// setup.cu
void setup_build(Handle& h, const Mat& A64 /* device fp64 copy owned by h */, int nparts, cudaStream_t s);
// vcycle.cu
// V-cycle from level `level` on that level's f buffer; returns the buffer holding x
void* vcycle_run(Handle& h, size_t level, cudaStream_t s);
void* level0_f(Handle& h);
// z = M r (outer fp64 r scaled by `scale`, z of dtype zt)
void precond_apply(Handle& h, const double* r, void* z, int zt, cudaStream_t s, double scale = 1.0);
double precond_bytes(const Handle& h);
// krylov.cu
int krylov_solve(Handle& h, const double* b, double* x, double rtol, cudaStream_t s, amg_report* rep);

}  // namespace amgb
