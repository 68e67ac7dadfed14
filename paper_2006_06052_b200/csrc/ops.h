// ops.h -- host launchers of the solve-phase kernels (all stream-ordered, no sync,
// no allocation).  Vector/value types are AMG_F32 / AMG_F64.
#pragma once

#include "common.cuh"

namespace amgb {

// kernel plan of a device matrix: the bsr_lane.cuh variant (host only); with an arena,
// long-row matrices also get the sliced copy (k_bsr_sell, allocated in the arena: one
// sync); the opt-in TMA tile plan (AMG_TMA=1: one reduction + one sync)
void set_lane_plan(Mat& A, bool use_env = true);
void make_tma_plan(Mat& A, cudaStream_t s, Arena* arena = nullptr, bool want_tma = false);
// does A carry an interleaved (k_bsr_sellr) or sliced (k_bsr_sell) copy of its blocks?
bool has_solve_copy(const Mat& A);
// free A's BSR values (A.val = nullptr) when a solve copy carries every product with A; the
// pattern (ptr, col) stays.  No-op otherwise.  One stream sync.
void release_bsr_values(Mat& A, Arena& arena, cudaStream_t s);
// A's BSR values (A.vt, nnz * br * bc) re-materialised from its solve copy into out (device)
void values_from_copy(const Mat& A, void* out, cudaStream_t s);
// the BSR column indices of a matrix whose values are already released go too (its copy carries
// them in its own layout); cols_from_copy re-materialises them (export), given A.ptr
void release_bsr_cols(Mat& A, Arena& arena, cudaStream_t s);
void cols_from_copy(const Mat& A, int32_t* out, cudaStream_t s);

// S1: scalar CSR -> BSR (convert.cu); returns nnzb, fills bptr/bcol/bval when bptr != nullptr
int64_t csr_to_bsr(int32_t n, int32_t m, int32_t b, int64_t nnz, const int32_t* ptr, const int32_t* col,
                   const void* val, int dtype, int32_t* bptr, int32_t* bcol, void* bval, cudaStream_t s);

// K1  y = alpha A x + beta y
// (r0, r1): only block rows [r0, r1) (row-lane plans; r1 < 0 = all rows)
void launch_spmv(const Mat& A, double alpha, const void* x, int xt, double beta, void* y, int yt,
                 cudaStream_t s, int r0 = 0, int r1 = -1);
class CommBase;
// K3  y = A x (fp64 y) with out[j] = w_j . y (w_j == nullptr: y.y), j < nd <= 2, in ONE pass
// (row-lane plans; false: not fused, the caller runs the SpMV and the dots); partials as
// blas1.h (with the ticket); comm: the sums are allreduced
bool launch_spmv_dot(const Mat& A, const void* x, int xt, double* y, const double* w0, const double* w1, int nd,
                     double* partials, double* out, cudaStream_t s, CommBase* comm);
// K2  r = f - A x with out[0] = r.r in one pass (fp64 f, r); false: not fused
bool launch_residual_nrm(const Mat& A, const double* f, const void* x, int xt, double* r, double* partials,
                         double* out, cudaStream_t s, CommBase* comm);
// K2  r = f - A x   (f, x, r of type xt)
void launch_residual(const Mat& A, const void* f, const void* x, void* r, int xt, cudaStream_t s, int r0 = 0,
                     int r1 = -1);
// K5  xo = x + M (f - A x)
void launch_smooth(const Mat& A, const void* M, const void* f, const void* x, void* xo, int xt,
                   cudaStream_t s, int r0 = 0, int r1 = -1);
// ILU(0) U sweep (R20): xo = xb + D^-1 (y - U_s z); xb == nullptr: from zero
void launch_ilu_usweep(const Mat& U, const void* Dinv, const void* y, const void* z, const void* xb, void* xo, int xt,
                       cudaStream_t s);
// the interleaved copy (k_bsr_sellr) runs a row range only on whole unpermuted slices
bool sellr_range_ok(const Mat& A, int r0, int r1);
// K4a x = M f
void launch_apply_M(int32_t n, int b, const void* M, int vt, const void* f, void* x, int xt,
                    cudaStream_t s);
// K4a fused into the producer of f: the producer also stores x = M f
// (M: block-diagonal [n][b][b] of type mvt), bit-identical to the producer + launch_apply_M.
// false: this plan / shape has no fused form (nothing launched; run the pair).
// K6 + K4a  f = A g, x = M f
bool launch_spmv_M(const Mat& A, const void* g, void* f, const void* M, int mvt, void* x, int xt, cudaStream_t s);
// K11 + K4a  ru2 = ru - B^T p, x = M ru2
bool launch_schur_u_M(const Mat& BTm, const void* ru, const void* p, void* ru2, const void* M, int mvt, void* x, int xt,
                      cudaStream_t s);
// K9 + K4a  (b = 4, pc = 3, fp32 vectors) split, xu = M ru
bool launch_split_M(int32_t n, int b, int pc, const double* r, double scale, void* ru, void* rp, int xt, const void* M,
                    int mvt, void* xu, cudaStream_t s, const double* scale_dev = nullptr);
// narrow + K4a  f = narrow(scale r) (n block rows of b), x = M f
// k_bicg_p fused with launch_convert_M (scale 1): p = r + beta (p - omega v), f = narrow(p), x = M f
bool launch_bicg_p_convert_M(int32_t n, int b, const double* r, const double* v, double* p, const double* sc, void* f,
                             int xt, const void* M, int mvt, void* x, cudaStream_t s);
bool launch_convert_M(int32_t n, int b, const double* r, double scale, void* f, int xt, const void* M, int mvt, void* x,
                      cudaStream_t s, const double* scale_dev = nullptr);
// K8  x = Ainv f (dense N x N, values vt, vectors xt)
void launch_dense_gemv(int32_t N, const void* Ainv, int vt, const void* f, void* x, int xt,
                       cudaStream_t s);

// Schur coupling views on the outer pattern: Bm (1 x nu blocks, values Bv [nnz][nu]) and
// BTm (nu x 1 blocks, values BTv [nnz][nu]), with their TMA plans
void make_schur_views(const Mat& A, int nu, const void* Bv, const void* BTv, int vt, Mat& Bm, Mat& BTm,
                      cudaStream_t s,
                      Arena* arena = nullptr);
// K10 p = m_S o (r_p - B u*)
void launch_schur_p(const Mat& Bm, const void* mS, const void* rp, const void* us, void* p, int xt, cudaStream_t s);
// K11 ru2 = r_u - B^T p   (ru2 may alias ru)
void launch_schur_u(const Mat& BTm, const void* ru, const void* p, void* ru2, int xt, cudaStream_t s);

// K9  split the fp64 interleaved outer vector (b comps per cell) into the velocity part
// (nu = b-1 comps, type xt) and the pressure part (type xt), narrowing RNE; optional
// scale (used to fold a GMRES normalisation in).
void launch_split(int32_t n, int b, int pc, const double* r, double scale, void* ru, void* rp, int xt,
                  cudaStream_t s, const double* scale_dev = nullptr);
// K9' join (u, p) -> interleaved fp64 z (exact widening)
void launch_mask_split(int32_t nu, int32_t np, const int32_t* uidx, const int32_t* pidx, const double* r,
                       double scale, void* ru, void* rp, int xt, cudaStream_t s, const double* scale_dev = nullptr);
void launch_mask_join(int32_t nu, int32_t np, const int32_t* uidx, const int32_t* pidx, const void* u, const void* p,
                      int xt, void* z, int zt, cudaStream_t s);
bool smooth_join_ok(const Mat& A, int xt);
// K5 + the monolithic apply's widening: the last post-smoothing step writes z (dtype zt)
bool smooth_widen_ok(const Mat& A, int xt, int zt);
void launch_smooth_widen(const Mat& A, const void* M, const void* f, const void* x, void* z, int zt, int xt,
                         cudaStream_t s, int r0 = 0, int r1 = -1);
void launch_smooth_join(const Mat& A, const void* M, const void* f, const void* x, const void* p, void* z, int zt,
                        int xt, cudaStream_t s, int r0 = 0, int r1 = -1);
void launch_join(int32_t n, int b, int pc, const void* u, const void* p, int xt, void* z, int zt,
                 cudaStream_t s);
// convert a whole vector between dtypes (narrowing RNE / exact widening); scale applied in fp64
// scale_dev (device, optional) replaces scale: graph-replayable scaling
void launch_convert(int64_t N, const void* in, int it, void* out, int ot, double scale, cudaStream_t s,
                    const double* scale_dev = nullptr);

}  // namespace amgb
