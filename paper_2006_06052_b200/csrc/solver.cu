// solver.cu -- C ABI of the solver handle: amg_setup / amg_solve / introspection.
#include <chrono>
#include <cstdlib>
#include <cstring>

#include "amg.h"
#include "ops.h"
#include "solver.h"

namespace amgb {
int validate_bsr(const amg_bsr* A, bool square);
Mat view_of(const amg_bsr* A);
void set_last_error(const std::string& s);

Handle::~Handle() {
  for (PcGraph& G : pc_graphs)
    if (G.exec) cudaGraphExecDestroy(G.exec);
  for (auto& G : step_graphs)
    if (G.second) cudaGraphExecDestroy(G.second);
  if (work) cudaStreamDestroy(work);
  if (comm_s) cudaStreamDestroy(comm_s);
  if (ev_pack) cudaEventDestroy(ev_pack);
  if (ev_halo) cudaEventDestroy(ev_halo);
  if (ev_in) cudaEventDestroy(ev_in);
  if (ev_out) cudaEventDestroy(ev_out);
  for (Level& L : lv)
    if (L.halo.send_buf) L.halo.send_buf = nullptr;  // arena-owned
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (hscal) cudaFreeHost(hscal);
}

void alloc_workspace(Handle& h, cudaStream_t s) {
  const int64_t N = (int64_t)h.n * h.b;
  const int64_t Nx = (int64_t)(h.n + h.halo0.nghost) * h.b;  // SpMV inputs carry ghosts
  // outer work vectors per solver (krylov.cu): CG r z p q, BiCGStab r rh p ph v s sh t, IDR(s)
  // r v vh t; flexible GMRES works in its V / Z bases only
  const int nv = h.p.solver == AMG_BICGSTAB ? 8 : h.p.solver == AMG_GMRES ? 0 : 4;
  for (int i = 0; i < nv; ++i) h.vec.push_back(h.arena.alloc_n<double>(std::max<int64_t>(Nx, 1)));
  // amg_solve_host's device copies of b and x: allocated here so that no solve call allocates
  h.stage_b = h.arena.alloc_n<double>(std::max<int64_t>(N, 1));
  h.stage_x = h.arena.alloc_n<double>(std::max<int64_t>(N, 1));
  if (h.comm) h.x_ext = h.arena.alloc_n<double>(std::max<int64_t>(Nx, 1));
  if (h.p.solver == AMG_GMRES) {
    const int m = h.p.gmres_m;
    // Z is stored in the preconditioner's output precision: the fp32 V-cycle output is
    // exactly representable in fp32, so storing it narrow is lossless.
    h.zt = (h.amg_active && h.xt == AMG_F32) ? AMG_F32 : AMG_F64;
    // one slab for the basis; vector j starts j * (size + stagger) bytes in, so the
    // j-streams the CGS2 kernels read side by side do not share DRAM address bits
    const size_t stagger = (size_t)env_int("AMG_VSTAGGER", 0);
    const size_t vbytes = ((size_t)std::max<int64_t>(N, 1) * 8 + 255) & ~size_t(255);
    char* slab = (char*)h.arena.alloc((vbytes + stagger) * (m + 1) + 256);
    for (int i = 0; i <= m; ++i) h.V.push_back(reinterpret_cast<double*>(slab + (size_t)i * (vbytes + stagger)));
    for (int i = 0; i < m; ++i) h.Z.push_back(h.arena.alloc(std::max<int64_t>(Nx, 1) * dtype_size(h.zt)));
    if (h.p.gmres_ortho == 2)
      for (int i = 0; i <= m; ++i) h.Vs.push_back(h.arena.alloc_n<float>(std::max<int64_t>(N, 1)));
    if (h.p.gmres_ortho == 3)  // fp16: 2 bytes per element, 16-byte aligned rows for the vector loads
      for (int i = 0; i <= m; ++i) h.Vs.push_back(h.arena.alloc(((size_t)std::max<int64_t>(N, 1) * 2 + 15) & ~size_t(15)));
  }
  if (h.p.solver == AMG_IDRS) {
    // IDR(s): shadow space P (N), G (N), U (with ghost space: U_k feeds the SpMV)
    const int sd = h.p.idrs_s;
    for (int i = 0; i < sd; ++i) {
      h.Pi.push_back(h.arena.alloc_n<double>(std::max<int64_t>(N, 1)));
      h.Gi.push_back(h.arena.alloc_n<double>(std::max<int64_t>(N, 1)));
      h.Ui.push_back(h.arena.alloc_n<double>(std::max<int64_t>(Nx, 1)));
    }
  }
  h.partials = h.arena.alloc_n<double>((size_t)kMaxPartials * 32 + 8);  // + ticket (blas1.h)
  AMG_CK(cudaMemset(h.partials + (size_t)kMaxPartials * 32, 0, 8 * sizeof(double)));
  h.dscal = h.arena.alloc_n<double>(256);
  AMG_CK(cudaMallocHost(&h.hscal, sizeof(double) * 256));
  if (h.schur) {
    const size_t xs = dtype_size(h.xt);
    const int np = h.masked ? h.np_s : h.n;
    h.rp = h.arena.alloc(std::max(np, 1) * xs);
    h.pp = h.arena.alloc(std::max(np + std::max(h.halo0.nghost, h.haloBTp.nghost), 1) * xs);
  }
  AMG_CK(cudaStreamCreateWithFlags(&h.work, cudaStreamNonBlocking));
  if (h.comm) {
    AMG_CK(cudaStreamCreateWithFlags(&h.comm_s, cudaStreamNonBlocking));
    AMG_CK(cudaEventCreateWithFlags(&h.ev_pack, cudaEventDisableTiming));
    AMG_CK(cudaEventCreateWithFlags(&h.ev_halo, cudaEventDisableTiming));
  }
  AMG_CK(cudaEventCreateWithFlags(&h.ev_in, cudaEventDisableTiming));
  AMG_CK(cudaEventCreateWithFlags(&h.ev_out, cudaEventDisableTiming));
  AMG_CK(cudaEventCreate(&h.ev0));
  AMG_CK(cudaEventCreate(&h.ev1));
  (void)N;
  (void)s;
}

namespace {

double mat_bytes(const Mat& A, int vt) {
  return (double)A.nnz * (4.0 + (double)A.b * A.b * dtype_size(vt)) + 4.0 * (A.n + 1);
}

}  // namespace

int check_params(const amg_params* p) {
  if (!p) return AMG_EINVAL;
  if (p->solver < AMG_CG || p->solver > AMG_IDRS) return AMG_EINVAL;
  if (p->solver == AMG_IDRS && (p->idrs_s < 1 || p->idrs_s > 8)) return AMG_EINVAL;
  if (p->precond < AMG_PC_AMG || p->precond > AMG_PC_NONE) return AMG_EINVAL;
  if (p->solver == AMG_GMRES && (p->gmres_m < 1 || p->gmres_m > 31)) return AMG_EINVAL;
  if (p->npre < 1 || p->npost < 0 || p->max_levels < 1 || p->maxiter < 0) return AMG_EINVAL;
  if (p->coarsening != AMG_SA && p->coarsening != AMG_PLAIN_AGG) return AMG_EINVAL;
  if (p->schur_shat < 0 || p->schur_shat > 2 || !(p->over_interp > 0.0)) return AMG_EINVAL;
  if (p->smoother < AMG_SPAI0 || p->smoother > AMG_ILUT) return AMG_EINVAL;
  if ((p->smoother == AMG_ILU0 || p->smoother == AMG_ILUT) && (p->ilu_sweeps < 1 || p->ilu_sweeps > 16))
    return AMG_EINVAL;
  if (p->smoother == AMG_ILUT && (p->ilut_p < 0 || !(p->ilut_tau >= 0.0))) return AMG_EINVAL;
  if (p->gmres_ortho < 0 || p->gmres_ortho > 3) return AMG_EINVAL;
  if (p->fused_presmooth < 0 || p->fused_presmooth > 1) return AMG_EINVAL;
  if ((p->hier_dtype != AMG_F32 && p->hier_dtype != AMG_F64) ||
      (p->vcycle_vec_dtype != AMG_F32 && p->vcycle_vec_dtype != AMG_F64))
    return AMG_EINVAL;
  return AMG_OK;
}

Handle* build_handle(const Mat& src, const amg_params* p, const std::vector<int64_t>& bounds, cudaStream_t s,
                     bool workspace, const uint8_t* pmask) {
  auto t0 = std::chrono::steady_clock::now();
  Handle* h = new Handle;
  try {
    h->p = *p;
    h->pmask_in = pmask;
    h->want_copies = workspace;
    h->vt = p->hier_dtype;
    h->xt = p->vcycle_vec_dtype;
    h->n = src.n;
    h->n_global_rows = src.n;
    h->b = src.b;
    h->schur = p->precond == AMG_PC_SCHUR;
    h->pc = p->schur_p_component;
    h->amg_active = p->precond != AMG_PC_NONE;
    if (h->schur && !pmask && (h->pc < 0 || h->pc >= h->b)) fail(AMG_EINVAL, "schur_p_component out of range");
    // library-owned fp64 copy of A (setup in own structures, then moved)
    Mat& M = h->A;
    M = src;
    M.vt = AMG_F64;
    M.ptr = h->arena.alloc_n<int32_t>(M.n + 1);
    M.col = h->arena.alloc_n<int32_t>(std::max<int64_t>(M.nnz, 1));
    M.val = h->arena.alloc_n<double>(std::max<int64_t>(M.nnz, 1) * M.b * M.b);
    AMG_CK(cudaMemcpyAsync(M.ptr, src.ptr, sizeof(int32_t) * (M.n + 1), cudaMemcpyDeviceToDevice, s));
    if (M.nnz > 0) {
      AMG_CK(cudaMemcpyAsync(M.col, src.col, sizeof(int32_t) * M.nnz, cudaMemcpyDeviceToDevice, s));
      launch_convert(M.nnz * M.b * M.b, src.val, src.vt, M.val, AMG_F64, 1.0, s);
    }
    h->alg_bytes_spmv = mat_bytes(M, AMG_F64) + 16.0 * (double)M.n * M.b;
    Arena* copies = workspace ? &h->arena : nullptr;
    make_tma_plan(M, s, copies);
    if (h->amg_active) setup_build(*h, M, bounds, s);
    if (h->schur && !h->masked) make_schur_views(M, h->nu, h->Bv, h->BTv, h->vt, h->Bm, h->BTm, s, copies);
    h->pmask_in = nullptr;
    if (workspace) alloc_workspace(*h, s);
    // single-device solve handle: the interleaved copy carries every solve-phase product with
    // A, so its BSR values (fp64, 15.5 GB at cfg 5) go (the pattern stays: the Schur views
    // use it).  The distributed setup's global handle (workspace == false) keeps them for
    // slicing.
    // single-device solve handle: every solve-phase product with a matrix that has an interleaved
    // or sliced copy runs on the copy, so its BSR values go (the pattern stays: the Schur views
    // and the export use it; amg_level_export re-materialises values from the copy).  Outer A:
    // 15.5 GB fp64 at cfg 5; the fp32 hierarchy A_l / P_l / R_l: 4.7 GB (VERDICT r01 next #6,
    // the paper's memory claim PAPER.md:43-45, 717-718).  The distributed setup's global handle
    // (workspace == false) keeps them for slicing.
    if (workspace && !env_set("AMG_KEEP_VALUES")) {
      release_bsr_values(M, h->arena, s);
      for (Level& L : h->lv) {
        release_bsr_values(L.A, h->arena, s);
        release_bsr_values(L.P, h->arena, s);
        release_bsr_values(L.R, h->arena, s);
        // and their column indices (the copies carry them; the export re-materialises them
        // from the copy and the kept row pointers): 1.3 GB at cfg 5
        release_bsr_cols(L.A, h->arena, s);
        release_bsr_cols(L.P, h->arena, s);
        release_bsr_cols(L.R, h->arena, s);
      }
      // B^T's values behind its interleaved copy (1.4 GB at cfg 5; the outer pattern stays:
      // B runs on the lane kernel over it)
      if (h->schur && !h->masked) {
        release_bsr_values(h->BTm, h->arena, s);
        if (!h->BTm.val) h->BTv = nullptr;
      }
    }
    h->alg_bytes_precond = precond_bytes(*h);
    AMG_CK(cudaStreamSynchronize(s));
  } catch (...) {
    delete h;
    throw;
  }
  h->setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return h;
}

int setup_common(const amg_bsr* A, const amg_params* p, cudaStream_t s, Handle** out) {
  int rc = validate_bsr(A, true);
  if (rc != AMG_OK) return rc;
  if (!out) return AMG_EINVAL;
  rc = check_params(p);
  if (rc != AMG_OK) return rc;
  *out = build_handle(view_of(A), p, {0, (int64_t)A->n_block_rows}, s);
  return AMG_OK;
}

}  // namespace amgb

using namespace amgb;

#define AMG_GUARD_BEGIN try {
#define AMG_GUARD_END                  \
  }                                    \
  catch (const ::amgb::Error& e) {     \
    ::amgb::set_last_error(e.what);    \
    return e.code;                     \
  }                                    \
  catch (const std::bad_alloc&) {      \
    return AMG_ENOMEM;                 \
  }                                    \
  catch (...) {                        \
    return AMG_EINVAL;                 \
  }

extern "C" {

int amg_setup_pmask(const amg_bsr* A, const uint8_t* pmask, const amg_params* p, void* stream,
                    struct amg_handle** out) {
  AMG_GUARD_BEGIN
  if (!A || !p || !out || !pmask) return AMG_EINVAL;
  int rc = validate_bsr(A, true);
  if (rc != AMG_OK) return rc;
  rc = check_params(p);
  if (rc != AMG_OK) return rc;
  if (p->precond != AMG_PC_SCHUR || p->schur_shat == 2) return AMG_EINVAL;
  *out = reinterpret_cast<amg_handle*>(
      build_handle(view_of(A), p, {0, (int64_t)A->n_block_rows}, (cudaStream_t)stream, true, pmask));
  return AMG_OK;
  AMG_GUARD_END
}

int amg_setup(const amg_bsr* A, const amg_params* p, void* stream, struct amg_handle** out) {
  AMG_GUARD_BEGIN
  if (!A || !p || !out) return AMG_EINVAL;
  Handle* h = nullptr;
  int rc = setup_common(A, p, (cudaStream_t)stream, &h);
  if (rc != AMG_OK) return rc;
  *out = reinterpret_cast<amg_handle*>(h);
  return AMG_OK;
  AMG_GUARD_END
}

void amg_destroy(struct amg_handle* hh) {
  Handle* h = reinterpret_cast<Handle*>(hh);
  delete h;
}

int amg_solve(struct amg_handle* hh, const double* b, double* x, double rtol, void* stream, amg_report* rep) {
  AMG_GUARD_BEGIN
  Handle* h = reinterpret_cast<Handle*>(hh);
  if (!h || (!b && h->n > 0) || (!x && h->n > 0) || !(rtol > 0.0)) return AMG_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  amg_report local{};
  amg_report* r = rep ? rep : &local;
  std::memset(r, 0, sizeof(*r));
  AMG_CK(cudaEventRecord(h->ev0, s));
  int st = krylov_solve(*h, b, x, rtol, s, r);
  AMG_CK(cudaEventRecord(h->ev1, s));
  AMG_CK(cudaEventSynchronize(h->ev1));
  float ms = 0.f;
  AMG_CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  r->solve_s = ms * 1e-3;
  r->setup_s = h->setup_s;
  if (st == AMG_OK && !r->converged) st = AMG_NOT_CONVERGED;
  return st;
  AMG_GUARD_END
}

int amg_solve_host(struct amg_handle* hh, const double* b_host, double* x_host, double rtol, void* stream,
                   amg_report* rep) {
  AMG_GUARD_BEGIN
  Handle* h = reinterpret_cast<Handle*>(hh);
  if (!h || !b_host || !x_host) return AMG_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t N = (int64_t)h->n * h->b;
  // device copies of b and x: the handle's staging vectors (alloc_workspace; nothing allocated here)
  AMG_CK(cudaMemcpyAsync(h->stage_b, b_host, sizeof(double) * N, cudaMemcpyHostToDevice, s));
  AMG_CK(cudaMemcpyAsync(h->stage_x, x_host, sizeof(double) * N, cudaMemcpyHostToDevice, s));
  int st = amg_solve(hh, h->stage_b, h->stage_x, rtol, stream, rep);
  if (st < 0) return st;
  AMG_CK(cudaMemcpyAsync(x_host, h->stage_x, sizeof(double) * N, cudaMemcpyDeviceToHost, s));
  AMG_CK(cudaStreamSynchronize(s));
  return st;
  AMG_GUARD_END
}

int amg_apply_precond(struct amg_handle* hh, const double* r, double* z, void* stream) {
  AMG_GUARD_BEGIN
  Handle* h = reinterpret_cast<Handle*>(hh);
  if (!h || ((!r || !z) && h->n > 0)) return AMG_EINVAL;
  precond_apply(*h, r, z, AMG_F64, (cudaStream_t)stream, 1.0);
  return AMG_OK;
  AMG_GUARD_END
}

int amg_vcycle(struct amg_handle* hh, const double* f, double* x, void* stream) {
  AMG_GUARD_BEGIN
  Handle* h = reinterpret_cast<Handle*>(hh);
  if (!h || !h->amg_active) return AMG_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t N0 = h->lv.empty() ? h->coarse.N : (int64_t)h->lv[0].A.n * h->lv[0].A.b;
  launch_convert(N0, f, AMG_F64, level0_f(*h), h->xt, 1.0, s);
  void* out = vcycle_run(*h, 0, s);
  launch_convert(N0, out, h->xt, x, AMG_F64, 1.0, s);
  return AMG_OK;
  AMG_GUARD_END
}

int amg_level_info(struct amg_handle* hh, int32_t level, int64_t* out) {
  Handle* h = reinterpret_cast<Handle*>(hh);
  if (!h || !out || !h->amg_active || level < 0) return AMG_EINVAL;
  if ((size_t)level < h->lv.size()) {
    const Level& L = h->lv[level];
    out[0] = L.A.n, out[1] = L.A.b, out[2] = L.A.nnz, out[3] = L.P.nnz, out[4] = L.nc;
    return AMG_OK;
  }
  if ((size_t)level == h->lv.size()) {
    out[0] = h->coarse.n, out[1] = h->coarse.b, out[2] = h->coarse.A.nnz, out[3] = 0, out[4] = 0;
    return AMG_OK;
  }
  return AMG_EINVAL;
}

int amg_level_export(struct amg_handle* hh, int32_t level, int32_t which, int32_t* ptr, int32_t* col, double* val) {
  AMG_GUARD_BEGIN
  Handle* h = reinterpret_cast<Handle*>(hh);
  if (!h || !val || !h->amg_active || level < 0 || (size_t)level > h->lv.size()) return AMG_EINVAL;
  const bool coarsest = (size_t)level == h->lv.size();
  if (coarsest && !h->coarse.A.ptr) return AMG_EINVAL;  // distributed: coarsest not kept
  if (which == 3) {
    if (coarsest) return AMG_EINVAL;
    const Level& L = h->lv[level];
    const int64_t cnt = (int64_t)L.A.n * L.A.b * L.A.b;
    double* tmp = nullptr;
    AMG_CK(cudaMalloc(&tmp, std::max<int64_t>(cnt, 1) * 8));
    launch_convert(cnt, L.M, h->vt, tmp, AMG_F64, 1.0, nullptr);
    AMG_CK(cudaMemcpy(val, tmp, cnt * 8, cudaMemcpyDeviceToHost));
    cudaFree(tmp);
    return AMG_OK;
  }
  if (which < 0 || which > 5 || (coarsest && which != 0) || !ptr || !col) return AMG_EINVAL;
  if (which >= 4 && !h->lv[level].Lf.ptr) return AMG_EINVAL;  // ILU factors only with AMG_ILU0 / AMG_ILUT
  const Level& LL = h->lv[std::min(level, (int32_t)h->lv.size() - 1)];
  const Mat& M = coarsest ? h->coarse.A
                          : (which == 0 ? LL.A : which == 1 ? LL.P : which == 2 ? LL.R : which == 4 ? LL.Lf : LL.Uf);
  AMG_CK(cudaDeviceSynchronize());
  AMG_CK(cudaMemcpy(ptr, M.ptr, sizeof(int32_t) * (M.n + 1), cudaMemcpyDeviceToHost));
  if (M.nnz > 0 && M.col) AMG_CK(cudaMemcpy(col, M.col, sizeof(int32_t) * M.nnz, cudaMemcpyDeviceToHost));
  if (M.nnz > 0 && !M.col) {  // released column indices: re-materialised from the solve copy
    int32_t* tc = nullptr;
    AMG_CK(cudaMalloc(&tc, sizeof(int32_t) * M.nnz));
    cols_from_copy(M, tc, nullptr);
    AMG_CK(cudaMemcpy(col, tc, sizeof(int32_t) * M.nnz, cudaMemcpyDeviceToHost));
    cudaFree(tc);
  }
  const int64_t cnt = M.nnz * M.b * M.b;
  double* tmp = nullptr;
  void* src = M.val;
  void* mat = nullptr;  // values re-materialised from the solve copy (released BSR values)
  AMG_CK(cudaMalloc(&tmp, std::max<int64_t>(cnt, 1) * 8));
  if (!src && cnt > 0) {
    AMG_CK(cudaMalloc(&mat, cnt * dtype_size(M.vt)));
    values_from_copy(M, mat, nullptr);
    src = mat;
  }
  launch_convert(cnt, src, M.vt, tmp, AMG_F64, 1.0, nullptr);
  AMG_CK(cudaMemcpy(val, tmp, cnt * 8, cudaMemcpyDeviceToHost));
  cudaFree(tmp);
  if (mat) cudaFree(mat);
  return AMG_OK;
  AMG_GUARD_END
}

int amg_level_aggregates(struct amg_handle* hh, int32_t level, int32_t* agg) {
  AMG_GUARD_BEGIN
  Handle* h = reinterpret_cast<Handle*>(hh);
  if (!h || !agg || level < 0 || (size_t)level >= h->lv.size()) return AMG_EINVAL;
  AMG_CK(cudaDeviceSynchronize());
  AMG_CK(cudaMemcpy(agg, h->lv[level].agg, sizeof(int32_t) * h->lv[level].A.n, cudaMemcpyDeviceToHost));
  return AMG_OK;
  AMG_GUARD_END
}

int amg_schur_export(struct amg_handle* hh, double* shat_diag, double* m_s) {
  AMG_GUARD_BEGIN
  Handle* h = reinterpret_cast<Handle*>(hh);
  if (!h || !h->schur || !shat_diag || !m_s) return AMG_EINVAL;
  AMG_CK(cudaDeviceSynchronize());
  const int np = h->masked ? h->np_s : h->n;
  AMG_CK(cudaMemcpy(shat_diag, h->shat64, sizeof(double) * np, cudaMemcpyDeviceToHost));
  AMG_CK(cudaMemcpy(m_s, h->mS64, sizeof(double) * np, cudaMemcpyDeviceToHost));
  return AMG_OK;
  AMG_GUARD_END
}

int64_t amg_device_bytes(struct amg_handle* hh) {
  Handle* h = reinterpret_cast<Handle*>(hh);
  return h ? h->arena.bytes() : 0;
}

int amg_solve_counters(struct amg_handle* hh, int64_t* out, int32_t n) {
  Handle* h = reinterpret_cast<Handle*>(hh);
  if (!h || !out || n < 2) return AMG_EINVAL;
  out[0] = h->reorth_passes;
  out[1] = (int64_t)(h->pc_graphs.size() + h->step_graphs.size());
  return AMG_OK;
}

int amg_memory_report(struct amg_handle* hh, int64_t* out, int32_t n) {
  AMG_GUARD_BEGIN
  Handle* h = reinterpret_cast<Handle*>(hh);
  if (!h || !out || n < 8) return AMG_EINVAL;
  auto mat = [&](const Mat& M) -> int64_t {
    if (!M.ptr) return 0;
    return 4LL * (M.n + 1) +
           M.nnz * ((M.col ? 4LL : 0LL) + (M.val ? (int64_t)M.rows_per_block() * M.cols_per_block() * dtype_size(M.vt) : 0LL));
  };
  auto sell = [&](const Mat& M) -> int64_t {
    if ((M.lane_var != kLaneSell && M.lane_var != kLaneSellR) || !M.sell_ptr) return 0;
    const int C = M.lane_var == kLaneSellR ? 32 : 32 / M.b;
    int32_t last = 0;
    AMG_CK(cudaMemcpy(&last, M.sell_ptr + M.sell_ns, 4, cudaMemcpyDeviceToHost));
    const int64_t steps = last;
    const int64_t perm = M.sell_perm ? 4LL * M.sell_ns * C : 0;
    if (M.lane_var == kLaneSell)
      return 4LL * (M.sell_ns + 1) + steps * C * (4LL + (int64_t)M.b * M.b * dtype_size(M.vt)) + perm;
    int32_t nvec = 0;
    AMG_CK(cudaMemcpy(&nvec, M.sell_vptr + M.sell_ns, 4, cudaMemcpyDeviceToHost));
    return 8LL * (M.sell_ns + 1) + steps * C * 4LL + (int64_t)nvec * C * M.sell_w * dtype_size(M.vt) + perm;
  };
  int64_t v[8] = {};
  v[0] = mat(h->A) + sell(h->A);
  for (const Level& L : h->lv) {
    v[1] += mat(L.A) + mat(L.P) + mat(L.R) + mat(L.Lf) + mat(L.Uf);
    v[2] += sell(L.A) + sell(L.P) + sell(L.R) + sell(L.Lf) + sell(L.Uf);
    v[3] += (int64_t)L.A.n * L.A.b * L.A.b * dtype_size(h->vt);
  }
  if (h->schur && h->masked) v[4] = mat(h->Bm) + mat(h->BTm) + (int64_t)h->np_s * dtype_size(h->vt);
  else if (h->schur)  // B / B^T values on the outer pattern (B^T's released behind its copy), m_S, copies
    v[4] = ((h->Bv ? 1LL : 0LL) + (h->BTv ? 1LL : 0LL)) * h->A.nnz * h->nu * dtype_size(h->vt) +
           (int64_t)h->n * dtype_size(h->vt) + sell(h->Bm) + sell(h->BTm);
  v[5] = (int64_t)h->coarse.N * h->coarse.N * dtype_size(h->vt);
  const int64_t N = (int64_t)h->n * h->b;
  v[6] = (h->p.gmres_ortho == 3 ? 2LL : 4LL) * N * (int64_t)h->Vs.size() + 8LL * N * ((int64_t)h->vec.size() + 2 /* host staging */ + (int64_t)h->V.size() + (int64_t)h->Pi.size() + (int64_t)h->Gi.size() +
                    (int64_t)h->Ui.size()) +
         (int64_t)h->Z.size() * N * dtype_size(h->zt);
  v[7] = h->arena.bytes();
  for (int i = 0; i < 8; ++i) out[i] = v[i];
  return AMG_OK;
  AMG_GUARD_END
}

}  // extern "C"
