// capi.cu -- the C ABI (include/amg.h): argument validation, error mapping, and the
// entry points that need no hierarchy (bsr_spmv, params, status strings).
#include <cstring>

#include "amg.h"
#include "common.cuh"
#include "ops.h"

using namespace amgb;

namespace amgb {
void set_last_error(const std::string& s);

int validate_bsr(const amg_bsr* A, bool square) {
  if (!A) return AMG_EINVAL;
  if (A->block_size < 1 || A->block_size > 4) return AMG_EINVAL;
  if (A->n_block_rows < 0 || A->n_block_cols < 0 || A->nnzb < 0) return AMG_EINVAL;
  if (A->nnzb >= (int64_t(1) << 31)) return AMG_EINDEX_OVERFLOW;
  if ((int64_t)A->n_block_rows * A->block_size >= (int64_t(1) << 31)) return AMG_EINDEX_OVERFLOW;
  if (A->dtype != AMG_F32 && A->dtype != AMG_F64) return AMG_EINVAL;
  if (A->n_block_rows > 0 && (!A->row_ptr || (A->nnzb > 0 && (!A->col_idx || !A->values))))
    return AMG_EINVAL;
  if (square && A->n_block_rows != A->n_block_cols) return AMG_EDIM;
  return AMG_OK;
}

Mat view_of(const amg_bsr* A) {
  Mat M;
  M.n = A->n_block_rows;
  M.m = A->n_block_cols;
  M.b = A->block_size;
  M.nnz = A->nnzb;
  M.ptr = const_cast<int32_t*>(A->row_ptr);
  M.col = const_cast<int32_t*>(A->col_idx);
  M.val = const_cast<void*>(A->values);
  M.vt = A->dtype;
  set_lane_plan(M);
  return M;
}

}  // namespace amgb

#define AMG_GUARD_BEGIN try {
#define AMG_GUARD_END                      \
  }                                        \
  catch (const ::amgb::Error& e) {         \
    ::amgb::set_last_error(e.what);        \
    return e.code;                         \
  }                                        \
  catch (const std::bad_alloc&) {          \
    return AMG_ENOMEM;                     \
  }                                        \
  catch (...) {                            \
    return AMG_EINVAL;                     \
  }

namespace amgb {
static thread_local std::string g_last_error;
void set_last_error(const std::string& s) { g_last_error = s; }
}  // namespace amgb

extern "C" {

const char* amg_last_error(void) { return amgb::g_last_error.c_str(); }

int amg_params_default(amg_params* p) {
  if (!p) return AMG_EINVAL;
  std::memset(p, 0, sizeof(*p));
  p->solver = AMG_GMRES;
  p->gmres_m = 30;
  p->precond = AMG_PC_AMG;
  p->maxiter = 1000;
  p->hier_dtype = AMG_F32;
  p->vcycle_vec_dtype = AMG_F32;
  p->smoother = AMG_SPAI0;
  p->coarse_enough = 3000;
  p->jacobi_omega = 2.0 / 3.0;
  p->sa_omega = 2.0 / 3.0;
  p->eps_strong = 1e-3;
  p->max_levels = 20;
  p->npre = 1;
  p->npost = 1;
  p->schur_p_component = 3;
  p->use_graphs = 1;
  p->idrs_s = 5;
  p->idrs_seed = 1234;
  p->schur_u_scalar = 0;
  p->coarsening = AMG_SA;
  p->schur_shat = 1;
  p->over_interp = 1.5;
  p->ilu_sweeps = 2;
  p->gmres_ortho = 3;  // R28: fp16 shadow for the pass-1 dots
  p->fused_presmooth = 1;
  p->ilut_p = 2;
  p->ilut_tau = 1e-2;
  return AMG_OK;
}

const char* amg_status_string(int s) {
  switch (s) {
    case AMG_OK: return "ok";
    case AMG_NOT_CONVERGED: return "not converged (x holds the last iterate)";
    case AMG_EINVAL: return "invalid argument";
    case AMG_EDIM: return "dimension mismatch";
    case AMG_EZERODIAG: return "missing or zero diagonal block";
    case AMG_ESINGULAR_BLOCK: return "singular diagonal block";
    case AMG_EINDEX_OVERFLOW: return "index overflow (nnzb or n*b >= 2^31)";
    case AMG_EBREAKDOWN: return "Krylov breakdown after one restart";
    case AMG_ECUDA: return "CUDA error";
    case AMG_ENCCL: return "NCCL error";
    case AMG_ENOMEM: return "out of device memory";
    default: return "unknown status";
  }
}

int bsr_spmv(const amg_bsr* A, double alpha, const void* x, int32_t xt, double beta, void* y, int32_t yt,
             void* stream) {
  AMG_GUARD_BEGIN
  int rc = validate_bsr(A, false);
  if (rc != AMG_OK) return rc;
  if ((xt != AMG_F32 && xt != AMG_F64) || (yt != AMG_F32 && yt != AMG_F64)) return AMG_EINVAL;
  if (A->n_block_rows > 0 && (!x || !y)) return AMG_EINVAL;
  launch_spmv(view_of(A), alpha, x, xt, beta, y, yt, (cudaStream_t)stream);
  return AMG_OK;
  AMG_GUARD_END
}

int amg_csr_to_bsr(int32_t n, int32_t m, int32_t b, int64_t nnz, const int32_t* ptr, const int32_t* col,
                   const void* val, int32_t dtype, int32_t* bptr, int32_t* bcol, void* bval, int64_t* nnzb_out,
                   void* stream) {
  AMG_GUARD_BEGIN
  if (!nnzb_out || (n > 0 && !ptr) || (nnz > 0 && (!col || !val)) || nnz < 0) return AMG_EINVAL;
  if (dtype != AMG_F32 && dtype != AMG_F64) return AMG_EINVAL;
  if (bptr && nnz > 0 && (!bcol || !bval)) return AMG_EINVAL;
  *nnzb_out = csr_to_bsr(n, m, b, nnz, ptr, col, val, dtype, bptr, bcol, bval, (cudaStream_t)stream);
  return AMG_OK;
  AMG_GUARD_END
}

struct bsr_plan {
  amgb::Mat A;
  amgb::Arena arena;  // the plan's sliced copy of long-row matrices
};

int bsr_plan_create(const amg_bsr* A, void* stream, struct bsr_plan** out) {
  AMG_GUARD_BEGIN
  int rc = validate_bsr(A, false);
  if (rc != AMG_OK) return rc;
  if (!out) return AMG_EINVAL;
  bsr_plan* p = new bsr_plan;
  p->A = view_of(A);
  try {
    make_tma_plan(p->A, (cudaStream_t)stream, &p->arena);
  } catch (...) {
    delete p;
    throw;
  }
  *out = p;
  return AMG_OK;
  AMG_GUARD_END
}

int bsr_plan_spmv(struct bsr_plan* P, double alpha, const void* x, int32_t xt, double beta, void* y, int32_t yt,
                  void* stream) {
  AMG_GUARD_BEGIN
  if (!P || (xt != AMG_F32 && xt != AMG_F64) || (yt != AMG_F32 && yt != AMG_F64)) return AMG_EINVAL;
  if (P->A.n > 0 && (!x || !y)) return AMG_EINVAL;
  launch_spmv(P->A, alpha, x, xt, beta, y, yt, (cudaStream_t)stream);
  return AMG_OK;
  AMG_GUARD_END
}

void bsr_plan_destroy(struct bsr_plan* P) { delete P; }

}  // extern "C"
