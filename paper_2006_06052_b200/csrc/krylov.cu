// krylov.cu -- outer fp64 Krylov solvers: PCG, right-
// preconditioned BiCGStab (van der Vorst), flexible right-preconditioned GMRES(m)
// with CGS2 Arnoldi and Givens rotations, and the paper's IDR(s) (reading R17).  Same
// steps, scalars and stopping rules as the oracle; the host reads the scalars it
// branches on through pinned memory (fused into as few reads per step as the data
// dependencies allow).
#include <cmath>
#include <vector>

#include "blas1.h"
#include "ops.h"
#include "prof.h"
#include "solver.h"

namespace amgb {

namespace {

struct Ctx {
  Handle& h;
  cudaStream_t s;
  int64_t N;
  double bytes = 0.0;  // algorithmic bytes of the solve
  Ctx(Handle& hh, cudaStream_t ss) : h(hh), s(ss), N((int64_t)hh.n * hh.b) {}

  // host copies of device scalars [0, k)
  void read(int k) {
    AMG_CK(cudaMemcpyAsync(h.hscal, h.dscal, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
    AMG_CK(cudaStreamSynchronize(s));
  }
  void dot(const double* a, const double* b, int slot, bool sq = false) {
    launch_dot(N, a, AMG_F64, b, AMG_F64, h.partials, h.dscal + slot, sq, s, h.comm);
    bytes += (a == b ? 8.0 : 16.0) * N;
  }
  // x: a vector with ghost space (workspace / Z basis); ghosts exchanged first
  void spmv(const void* x, int xt, double* y) {
    halo_overlapped(h, h.halo0, h.A, const_cast<void*>(x), xt, h.b, s,
                    [&](int r0, int r1) { launch_spmv(h.A, 1.0, x, xt, 0.0, y, AMG_F64, s, r0, r1); });
    bytes += h.alg_bytes_spmv + N * ((double)dtype_size(xt) - 8.0);
  }
  // x: the caller's iterate (no ghost space): copied into x_ext when distributed
  void residual(const double* b, const double* x, double* r) {
    if (h.comm) {
      AMG_CK(cudaMemcpyAsync(h.x_ext, x, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
      x = h.x_ext;
    }
    halo_overlapped(h, h.halo0, h.A, const_cast<double*>(x), AMG_F64, h.b, s,
                    [&](int r0, int r1) { launch_residual(h.A, b, x, r, AMG_F64, s, r0, r1); });
    bytes += h.alg_bytes_spmv + 8.0 * N;
  }
  // y = A x with dscal[j] = w_j . y (w_j == nullptr: y . y), j < nd: one fused pass when the
  // operator's plan allows it (K3), else the SpMV and the dots
  void spmv_dot(const void* x, int xt, double* y, const double* w0, const double* w1, int nd) {
    if (h.comm) {  // distributed: the exchange overlaps the interior rows, dots separate
      spmv(x, xt, y);
      dot(w0 ? w0 : y, y, 0);
      if (nd > 1) dot(w1 ? w1 : y, y, 1);
      return;
    }
    if (launch_spmv_dot(h.A, x, xt, y, w0, w1, nd, h.partials, h.dscal, s, h.comm)) {
      bytes += h.alg_bytes_spmv + N * ((double)dtype_size(xt) - 8.0) + 8.0 * N * ((w0 ? 1 : 0) + (w1 ? 1 : 0));
      return;
    }
    launch_spmv(h.A, 1.0, x, xt, 0.0, y, AMG_F64, s);
    bytes += h.alg_bytes_spmv + N * ((double)dtype_size(xt) - 8.0);
    dot(w0 ? w0 : y, y, 0);
    if (nd > 1) dot(w1 ? w1 : y, y, 1);
  }
  // r = b - A x with dscal[0] = r . r (K2 fused when the plan allows it)
  void residual_nrm(const double* b, const double* x, double* r) {
    if (h.comm) {  // distributed: overlapped residual, then the norm
      residual(b, x, r);
      dot(r, r, 0);
      return;
    }
    if (launch_residual_nrm(h.A, b, x, AMG_F64, r, h.partials, h.dscal, s, h.comm)) {
      bytes += h.alg_bytes_spmv + 8.0 * N;
      return;
    }
    launch_residual(h.A, b, x, r, AMG_F64, s);
    bytes += h.alg_bytes_spmv + 8.0 * N;
    dot(r, r, 0);
  }
  // scale_dev (device, optional): r is scaled by *scale_dev while narrowing (GMRES's 1/||V_j||)
  void pc(const double* r, void* z, int zt, const double* scale_dev = nullptr) {
    precond_apply_graphed(h, r, z, zt, s, scale_dev);
    bytes += h.alg_bytes_precond + N * ((double)dtype_size(zt) - 8.0);
  }
  void axpby(double a, const double* x, double b, double* y) {
    launch_axpby(N, a, x, b, y, s);
    bytes += (b == 0.0 ? 16.0 : 24.0) * N;
  }
  void axpbypcz(double a, const double* x, double b, const double* y, double c, double* z) {
    launch_axpbypcz(N, a, x, b, y, c, z, s);
    bytes += 32.0 * N;
  }
};

bool finite(double v) { return std::isfinite(v); }

int finish(Ctx& c, const double* b, double* x, double* r, double nb, int status, int iters, int restarts,
           amg_report* rep) {
  c.residual_nrm(b, x, r);
  c.read(1);
  if (rep) {
    rep->iters = iters;
    rep->restarts = restarts;
    rep->relres_true = std::sqrt(c.h.hscal[0]) / nb;
    rep->converged = status == AMG_OK;
    rep->alg_bytes = c.bytes;
  }
  return status;
}

// ---- PCG (cfg 1) ----
int solve_cg(Ctx& c, const double* b, double* x, double rtol, double nb, amg_report* rep) {
  Handle& h = c.h;
  double *r = h.vec[0], *z = h.vec[1], *p = h.vec[2], *q = h.vec[3];
  c.residual_nrm(b, x, r);
  c.read(1);
  int it = 0, status = AMG_NOT_CONVERGED;
  if (std::sqrt(h.hscal[0]) <= rtol * nb) status = AMG_OK;
  bool restart = true;
  double rho = 0.0;
  while (status != AMG_OK && it < h.p.maxiter) {
    if (restart) {
      c.pc(r, z, AMG_F64);
      launch_convert(c.N, z, AMG_F64, p, AMG_F64, 1.0, c.s);
      c.bytes += 16.0 * c.N;
      c.dot(r, z, 0);
      c.read(1);
      rho = h.hscal[0];
      restart = false;
    }
    c.spmv_dot(p, AMG_F64, q, p, nullptr, 1);  // q = A p, p . q
    c.read(1);
    const double pq = h.hscal[0];
    if (pq == 0.0 || !finite(pq)) {
      status = AMG_EBREAKDOWN;
      break;
    }
    const double alpha = rho / pq;
    launch_idr_update(c.N, alpha, q, p, r, x, h.partials, h.dscal, c.s, h.comm);  // r -= a q, x += a p, ||r||
    c.bytes += 48.0 * c.N;
    ++it;
    c.read(1);
    if (h.hscal[0] <= rtol * nb) {
      c.residual_nrm(b, x, r);
      c.read(1);
      if (std::sqrt(h.hscal[0]) <= rtol * nb) {
        status = AMG_OK;
        break;
      }
      restart = true;
      continue;
    }
    c.pc(r, z, AMG_F64);
    c.dot(r, z, 0);
    c.read(1);
    const double rho_new = h.hscal[0];
    const double beta = rho_new / rho;
    c.axpby(1.0, z, beta, p);  // p = z + beta p
    rho = rho_new;
  }
  return finish(c, b, x, r, nb, status, it, 0, rep);
}

// ---- PCG with device-side scalars: one CUDA graph per iteration (reading R24) ----
// q = A p with p.q; r -= alpha q, x += alpha p with ||r|| (alpha = rho / p.q on the device);
// z = M r; r.z; p = z + (r.z / rho) p -- one replay and one read per iteration (the host-driven
// loop has three); the same kernels and expressions, so the iterates are bit-identical.
int solve_cg_graphed(Ctx& c, const double* b, double* x, double rtol, double nb, amg_report* rep) {
  Handle& h = c.h;
  double *r = h.vec[0], *z = h.vec[1], *p = h.vec[2], *q = h.vec[3];
  double* sc = h.dscal + 160;  // [0] rho, [1] p.q, [2] ||r||, [3] r.z
  double* hs = h.hscal + 160;
  c.residual_nrm(b, x, r);
  c.read(1);
  int it = 0, status = AMG_NOT_CONVERGED;
  if (std::sqrt(h.hscal[0]) <= rtol * nb) status = AMG_OK;
  cudaGraphExec_t G = nullptr;
  for (const auto& e : h.step_graphs)
    if (e.first == x) G = e.second;
  if (!G) {
    const int64_t l0 = t_launches;
    cudaGraph_t graph = nullptr;
    AMG_CK(cudaStreamBeginCapture(c.s, cudaStreamCaptureModeThreadLocal));
    try {
      if (h.comm || !launch_spmv_dot(h.A, p, AMG_F64, q, p, nullptr, 1, h.partials, sc + 1, c.s, h.comm)) {
        halo_overlapped(h, h.halo0, h.A, p, AMG_F64, h.b, c.s,
                        [&](int r0, int r1) { launch_spmv(h.A, 1.0, p, AMG_F64, 0.0, q, AMG_F64, c.s, r0, r1); });
        launch_dot(c.N, p, AMG_F64, q, AMG_F64, h.partials, sc + 1, false, c.s, h.comm);
      }
      launch_idr_update(c.N, 0.0, q, p, r, x, h.partials, sc + 2, c.s, h.comm, sc + 0, sc + 1);
      precond_apply(h, r, z, AMG_F64, c.s);
      launch_dot(c.N, r, AMG_F64, z, AMG_F64, h.partials, sc + 3, false, c.s, h.comm);
      launch_cg_p(c.N, z, p, sc + 3, sc + 0, c.s);
    } catch (...) {
      cudaStreamEndCapture(c.s, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    AMG_CK(cudaStreamEndCapture(c.s, &graph));
    h.step_graph_kernels = t_launches - l0;
    t_launches = l0;
    g_launches -= h.step_graph_kernels;
    cudaError_t e = cudaGraphInstantiate(&G, graph, 0);
    cudaGraphDestroy(graph);
    AMG_CK(e);
    h.step_graphs.push_back({x, G});
  }
  const double step_bytes = h.alg_bytes_spmv + 8.0 * c.N + 48.0 * c.N + h.alg_bytes_precond + 16.0 * c.N + 24.0 * c.N;
  bool restart = true;
  double rho = 0.0;
  while (status != AMG_OK && it < h.p.maxiter) {
    if (restart) {
      c.pc(r, z, AMG_F64);
      launch_convert(c.N, z, AMG_F64, p, AMG_F64, 1.0, c.s);
      c.bytes += 16.0 * c.N;
      c.dot(r, z, 0);
      c.read(1);
      rho = h.hscal[0];
      restart = false;
    }
    hs[0] = rho;
    AMG_CK(cudaMemcpyAsync(sc, hs, sizeof(double), cudaMemcpyHostToDevice, c.s));
    AMG_CK(cudaGraphLaunch(G, c.s));
    g_launches += h.step_graph_kernels;
    t_launches += h.step_graph_kernels;
    c.bytes += step_bytes;
    AMG_CK(cudaMemcpyAsync(hs + 1, sc + 1, sizeof(double) * 3, cudaMemcpyDeviceToHost, c.s));
    AMG_CK(cudaStreamSynchronize(c.s));
    const double pq = hs[1];
    if (pq == 0.0 || !finite(pq)) {  // the step left x and r untouched
      status = AMG_EBREAKDOWN;
      break;
    }
    ++it;
    if (hs[2] <= rtol * nb) {
      c.residual_nrm(b, x, r);
      c.read(1);
      if (std::sqrt(h.hscal[0]) <= rtol * nb) {
        status = AMG_OK;
        break;
      }
      restart = true;
      continue;
    }
    rho = hs[3];  // r.z: the step already formed p = z + (r.z / rho) p
  }
  return finish(c, b, x, r, nb, status, it, 0, rep);
}

// ---- BiCGStab (cfg 3) ----
int solve_bicgstab(Ctx& c, const double* b, double* x, double rtol, double nb, amg_report* rep) {
  Handle& h = c.h;
  double *r = h.vec[0], *rh = h.vec[1], *p = h.vec[2], *ph = h.vec[3], *v = h.vec[4], *sv = h.vec[5],
         *sh = h.vec[6], *t = h.vec[7];
  const int64_t N = c.N;
  c.residual_nrm(b, x, r);
  c.read(1);
  int it = 0, restarts = 0, status = AMG_NOT_CONVERGED;
  if (std::sqrt(h.hscal[0]) <= rtol * nb) status = AMG_OK;
  launch_convert(N, r, AMG_F64, rh, AMG_F64, 1.0, c.s);
  bool first = true;
  double rho_old = 1.0, alpha = 1.0, omega = 1.0;
  auto do_restart = [&]() -> bool {
    if (restarts >= 1) return false;
    ++restarts;
    c.residual(b, x, r);
    launch_convert(N, r, AMG_F64, rh, AMG_F64, 1.0, c.s);
    first = true;
    return true;
  };
  auto verify = [&]() -> bool {
    c.residual_nrm(b, x, r);
    c.read(1);
    if (std::sqrt(h.hscal[0]) <= rtol * nb) return true;
    launch_convert(N, r, AMG_F64, rh, AMG_F64, 1.0, c.s);
    first = true;
    return false;
  };
  // rho = rh . r for the next step comes with ||r|| out of the fused r update (one host
  // read per half step instead of two); recomputed after a restart / failed verify
  bool have_rho = false;
  double rho_next = 0.0;
  while (status != AMG_OK && it < h.p.maxiter) {
    if (!have_rho) {
      c.dot(rh, r, 0);
      c.read(1);
      rho_next = h.hscal[0];
    }
    have_rho = false;
    const double rho = rho_next;
    if (!(std::fabs(rho) > 1e-30 * nb * nb) || !finite(rho)) {
      if (do_restart()) continue;
      status = AMG_EBREAKDOWN;
      break;
    }
    if (first) {
      launch_convert(N, r, AMG_F64, p, AMG_F64, 1.0, c.s);
      c.bytes += 16.0 * N;
      first = false;
    } else {
      const double beta = (rho / rho_old) * (alpha / omega);
      // p = r + beta (p - omega v) = r + beta p - beta omega v
      c.axpbypcz(1.0, r, -beta * omega, v, beta, p);
    }
    c.pc(p, ph, AMG_F64);
    c.spmv_dot(ph, AMG_F64, v, rh, nullptr, 1);  // v = A ph, rh . v
    // s = r - (rho / rv) v with rv still on the device, ||s||^2 in the same pass
    launch_sub_div_nrm(N, rho, h.dscal, v, r, sv, h.partials, h.dscal + 1, c.s, h.comm);
    c.bytes += 24.0 * N;
    c.read(2);
    const double rv = h.hscal[0];
    if (rv == 0.0 || !finite(rv)) {
      if (do_restart()) continue;
      status = AMG_EBREAKDOWN;
      break;
    }
    alpha = rho / rv;
    ++it;
    if (std::sqrt(h.hscal[1]) <= rtol * nb) {
      c.axpby(alpha, ph, 1.0, x);
      if (verify()) {
        status = AMG_OK;
        break;
      }
      continue;
    }
    c.pc(sv, sh, AMG_F64);
    c.spmv_dot(sh, AMG_F64, t, nullptr, sv, 2);  // t = A sh, t . t, s . t
    c.read(2);
    const double tt = h.hscal[0];
    if (tt == 0.0 || !finite(tt)) {
      if (do_restart()) continue;
      status = AMG_EBREAKDOWN;
      break;
    }
    omega = h.hscal[1] / tt;
    c.axpbypcz(alpha, ph, omega, sh, 1.0, x);  // x += alpha ph + omega sh
    launch_axpy_2dot(N, omega, t, sv, r, rh, h.partials, h.dscal, c.s, h.comm);  // r = s - omega t; r.r, rh.r
    c.bytes += 32.0 * N;
    c.read(2);
    rho_old = rho;
    const double nr = std::sqrt(h.hscal[0]);
    rho_next = h.hscal[1];
    have_rho = true;
    if (omega == 0.0 || !finite(omega)) {
      if (do_restart()) {
        have_rho = false;
        continue;
      }
      status = AMG_EBREAKDOWN;
      break;
    }
    if (nr <= rtol * nb) {
      if (verify()) {
        status = AMG_OK;
        break;
      }
      have_rho = false;  // r was replaced by the true residual
    }
  }
  return finish(c, b, x, r, nb, status, it, restarts, rep);
}

// ---- BiCGStab with device-side scalars: one CUDA graph per iteration (reading R24) ----
// The whole step -- p update, both preconditioner applications, both fused SpMV + dots, the
// s, x and r updates -- is one graph replay; alpha, beta and omega are formed on the device
// from the scalar block (the host code's own expressions, so the iterates are bit-identical
// to solve_bicgstab's), and the host reads the block once per step: one synchronisation
// instead of three and one graph launch instead of ~8 launches.  The host keeps the control
// flow (breakdown restarts, the half-step exit, the true-residual verification) and writes
// the next step's (rho, rho_old, alpha, omega, first) back with one small copy.
int solve_bicgstab_graphed(Ctx& c, const double* b, double* x, double rtol, double nb, amg_report* rep) {
  Handle& h = c.h;
  double *r = h.vec[0], *rh = h.vec[1], *p = h.vec[2], *ph = h.vec[3], *v = h.vec[4], *sv = h.vec[5],
         *sh = h.vec[6], *t = h.vec[7];
  const int64_t N = c.N;
  double* sc = h.dscal + 160;  // BicgScal block (blas1.h)
  double* hs = h.hscal + 160;
  c.residual_nrm(b, x, r);
  c.read(1);
  int it = 0, restarts = 0, status = AMG_NOT_CONVERGED;
  if (std::sqrt(h.hscal[0]) <= rtol * nb) status = AMG_OK;
  launch_convert(N, r, AMG_F64, rh, AMG_F64, 1.0, c.s);
  bool first = true;
  double rho_old = 1.0, alpha = 1.0, omega = 1.0;
  auto do_restart = [&]() -> bool {
    if (restarts >= 1) return false;
    ++restarts;
    c.residual(b, x, r);
    launch_convert(N, r, AMG_F64, rh, AMG_F64, 1.0, c.s);
    first = true;
    return true;
  };
  auto verify = [&]() -> bool {
    c.residual_nrm(b, x, r);
    c.read(1);
    if (std::sqrt(h.hscal[0]) <= rtol * nb) return true;
    launch_convert(N, r, AMG_F64, rh, AMG_F64, 1.0, c.s);
    first = true;
    return false;
  };
  // the step graph (per iterate pointer x; workspace vectors are the handle's)
  cudaGraphExec_t G = nullptr;
  for (const auto& e : h.step_graphs)
    if (e.first == x) G = e.second;
  // p 32N, rh.v 8N, s 24N, s.t 8N, x + r 64N (p fused into the apply's narrowing: its re-read goes)
  const double step_bytes = 2.0 * h.alg_bytes_precond + 2.0 * (h.alg_bytes_spmv) + 136.0 * N - (bicg_p_fused(h) ? 8.0 * N : 0.0);
  if (!G) {
    const int64_t l0 = t_launches;
    cudaGraph_t graph = nullptr;
    AMG_CK(cudaStreamBeginCapture(c.s, cudaStreamCaptureModeThreadLocal));
    try {
      const BicgPre pre{r, v, p, sc};
      precond_apply(h, p, ph, AMG_F64, c.s, 1.0, nullptr, &pre);             // p; ph = M p
      if (h.comm || !launch_spmv_dot(h.A, ph, AMG_F64, v, rh, nullptr, 1, h.partials, sc + kBicgRv, c.s, h.comm)) {
        halo_overlapped(h, h.halo0, h.A, ph, AMG_F64, h.b, c.s,
                        [&](int r0, int r1) { launch_spmv(h.A, 1.0, ph, AMG_F64, 0.0, v, AMG_F64, c.s, r0, r1); });
        launch_dot(N, rh, AMG_F64, v, AMG_F64, h.partials, sc + kBicgRv, false, c.s, h.comm);
      }
      launch_bicg_s(N, v, r, sv, sc, h.partials, c.s, h.comm);              // s, ||s||^2
      precond_apply(h, sv, sh, AMG_F64, c.s);                                // sh = M s
      if (h.comm || !launch_spmv_dot(h.A, sh, AMG_F64, t, nullptr, sv, 2, h.partials, sc + kBicgTt, c.s, h.comm)) {
        halo_overlapped(h, h.halo0, h.A, sh, AMG_F64, h.b, c.s,
                        [&](int r0, int r1) { launch_spmv(h.A, 1.0, sh, AMG_F64, 0.0, t, AMG_F64, c.s, r0, r1); });
        launch_dot(N, t, AMG_F64, t, AMG_F64, h.partials, sc + kBicgTt, false, c.s, h.comm);
        launch_dot(N, sv, AMG_F64, t, AMG_F64, h.partials, sc + kBicgTs, false, c.s, h.comm);
      }
      launch_bicg_xr(N, ph, sh, t, sv, rh, x, r, sc, h.partials, c.s, h.comm);  // x, r, r.r, rh.r
    } catch (...) {
      cudaStreamEndCapture(c.s, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    AMG_CK(cudaStreamEndCapture(c.s, &graph));
    h.step_graph_kernels = t_launches - l0;
    t_launches = l0;
    g_launches -= h.step_graph_kernels;
    cudaError_t e = cudaGraphInstantiate(&G, graph, 0);
    cudaGraphDestroy(graph);
    AMG_CK(e);
    h.step_graphs.push_back({x, G});
  }
  hs[kBicgTol] = rtol * nb;
  bool have_rho = false;
  double rho_next = 0.0;
  while (status != AMG_OK && it < h.p.maxiter) {
    if (!have_rho) {
      c.dot(rh, r, 0);
      c.read(1);
      rho_next = h.hscal[0];
    }
    have_rho = false;
    const double rho = rho_next;
    if (!(std::fabs(rho) > 1e-30 * nb * nb) || !finite(rho)) {
      if (do_restart()) continue;
      status = AMG_EBREAKDOWN;
      break;
    }
    hs[kBicgRho] = rho, hs[kBicgRhoOld] = rho_old, hs[kBicgAlpha] = alpha, hs[kBicgOmega] = omega;
    hs[kBicgFirst] = first ? 1.0 : 0.0;
    AMG_CK(cudaMemcpyAsync(sc, hs, sizeof(double) * 6, cudaMemcpyHostToDevice, c.s));
    AMG_CK(cudaGraphLaunch(G, c.s));
    g_launches += h.step_graph_kernels;
    t_launches += h.step_graph_kernels;
    c.bytes += step_bytes;
    AMG_CK(cudaMemcpyAsync(hs + kBicgRv, sc + kBicgRv, sizeof(double) * (kBicgSlots - kBicgRv),
                           cudaMemcpyDeviceToHost, c.s));
    AMG_CK(cudaStreamSynchronize(c.s));
    first = false;
    const double rv = hs[kBicgRv];
    if (rv == 0.0 || !finite(rv)) {  // the step left x untouched
      if (do_restart()) continue;
      status = AMG_EBREAKDOWN;
      break;
    }
    alpha = rho / rv;
    ++it;
    if (std::sqrt(hs[kBicgSs]) <= rtol * nb) {  // half-step exit: the step did x += alpha ph only
      if (verify()) {
        status = AMG_OK;
        break;
      }
      continue;
    }
    const double tt = hs[kBicgTt];
    if (tt == 0.0 || !finite(tt)) {  // x untouched
      if (do_restart()) continue;
      status = AMG_EBREAKDOWN;
      break;
    }
    omega = hs[kBicgTs] / tt;
    rho_old = rho;
    const double nr = std::sqrt(hs[kBicgRr]);
    rho_next = hs[kBicgRhoNext];
    have_rho = true;
    if (omega == 0.0 || !finite(omega)) {
      if (do_restart()) {
        have_rho = false;
        continue;
      }
      status = AMG_EBREAKDOWN;
      break;
    }
    if (nr <= rtol * nb) {
      if (verify()) {
        status = AMG_OK;
        break;
      }
      have_rho = false;
    }
  }
  return finish(c, b, x, r, nb, status, it, restarts, rep);
}

// ---- flexible GMRES(m) with CGS2 (cfg 4, 5) ----
// The Arnoldi basis is stored unnormalised, v_j = s_j V_j with s_j = 1/||V_j|| kept on
// the device: the normalisation pass disappears (the preconditioner's split applies
// s_j while narrowing, the Gram-Schmidt kernels apply it in registers), and each CGS2
// step is three passes over the basis: scaled multi-dot, fused update + second
// multi-dot, fused update + norm.
__global__ void k_set_inv(double* dst, const double* src) { *dst = 1.0 / *src; }

int solve_gmres(Ctx& c, const double* b, double* x, double rtol, double nb, amg_report* rep) {
  Handle& h = c.h;
  const int m = h.p.gmres_m;
  const int64_t N = c.N;
  std::vector<double> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1), y(m), hh(m + 1);
  const bool gram = h.p.gmres_ortho >= 1;
  const bool shadow = h.p.gmres_ortho >= 2;  // reading R23 / R28: pass-1 dots on an fp32 / fp16 shadow basis
  const bool half = h.p.gmres_ortho == 3;
  // R28: shadow j holds fp16(V_j sig_j), sig_j the power of two at or below sqrt(N) / ||w|| (w: the
  // pre-update vector the update pass turned into V_j, ||w||^2 from the pass-1 multi-dot; V_0:
  // sig_0 from sqrt(N) s_0); the pass-1 dots scale by m_j = s_j / sig_j
  double* msc = h.dscal + 192;
  const double sqN = std::sqrt((double)std::max<int64_t>(N, 1));
  auto shadow0 = [&]() {  // the shadow of V_0 (the other shadows come out of the update pass)
    if (!shadow) return;
    if (half) {
      launch_to_half_scaled(N, h.V[0], h.dscal + 128, sqN, h.Vs[0], msc, c.s);  // s_0 = 1 / ||V_0||; m_0
      c.bytes += 10.0 * N;
      return;
    }
    launch_convert(N, h.V[0], AMG_F64, h.Vs[0], AMG_F32, 1.0, c.s);
    c.bytes += 12.0 * N;
  };
  std::vector<double> R((size_t)(m + 1) * (m + 1), 0.0), hv(m + 1), cv(m + 1);  // Gram/Cholesky factor
  double* sc = h.dscal + 128;  // s_j
  // r = b - A x straight into V_0
  c.residual(b, x, h.V[0]);
  launch_dot(N, h.V[0], AMG_F64, h.V[0], AMG_F64, h.partials, h.dscal + 64, true, c.s, h.comm);
  c.bytes += 8.0 * N;
  k_set_inv<<<1, 1, 0, c.s>>>(sc, h.dscal + 64);
  AMG_CK_LAUNCH();
  ++g_launches;
  ++t_launches;
  shadow0();
  c.read(65);
  double beta = h.hscal[64];
  int it = 0, cycles = 0, status = AMG_NOT_CONVERGED;
  if (beta <= rtol * nb) status = AMG_OK;
  const double sx = (double)dtype_size(h.zt);
  double s_host = 1.0 / beta;
  while (status != AMG_OK && it < h.p.maxiter) {
    ++cycles;
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    std::fill(R.begin(), R.end(), 0.0);
    R[0] = 1.0;  // t_0 = v_0 = r / beta
    int j = 0;
    bool stop = false;
    for (; j < m && !stop; ++j) {
      c.pc(h.V[j], h.Z[j], h.zt, sc + j);  // z_j = M(v_j), v_j = s_j V_j (s_j on the device)
      double* w = h.V[j + 1];
      c.spmv(h.Z[j], h.zt, w);
      PtrList Vl{};
      for (int i = 0; i <= j; ++i) Vl.p[i] = h.V[i];
      double hn = 0.0;
      if (!gram) {
        launch_mdot_scaled(N, j + 1, Vl, sc, w, h.partials, h.dscal, c.s, h.comm);                 // h1 = v^T w
        launch_cgs_update(N, j + 1, Vl, sc, h.dscal, w, w, true, h.partials, h.dscal + 32, c.s, h.comm);   // w -= v h1; h2 = v^T w
        launch_cgs_update(N, j + 1, Vl, sc, h.dscal + 32, w, w, false, h.partials, h.dscal + 64, c.s, h.comm,
                          sc + j + 1);  // w -= v h2; ||w||; s_{j+1} = 1/||w||
        c.bytes += 8.0 * N * (3.0 * (j + 1) + 5.0);
        c.read(65);
        for (int i = 0; i <= j; ++i) hh[i] = h.hscal[i] + h.hscal[32 + i];
        hn = h.hscal[64];
      } else {
        // two-pass Gram/Cholesky orthogonalisation (reading R22): the stored vectors t_i (once
        // orthogonalised, unit norm) are t = V R with G = t^T t = R^T R.  p = t^T w (pass 1);
        // h = R^-T p = V^T w; w1 = w - t R^-1 h = w - V h (pass 2, with q = t^T w1, ||w1||^2);
        // t_{j+1} = w1 / ||w1||; R's new column from G's (R^-T q / ||w1||);
        // H(:, j) = h + ||w1|| R(:, j+1).
        const int k = j + 1;
        double sig = 1.0;  // R28: the fp16 shadow scale of V_{j+1}
        if (shadow) {
          PtrList Vf{};
          for (int i = 0; i < k; ++i) Vf.p[i] = reinterpret_cast<const double*>(h.Vs[i]);
          if (half) {  // + dscal[k] = ||w||^2 (the shadow scale of V_{j+1})
            launch_mdot_scaled_f16(N, k, Vf, msc, w, h.partials, h.dscal, c.s, h.comm);
            c.bytes += 2.0 * N * k + 8.0 * N;
          } else {
            launch_mdot_scaled_f32(N, k, Vf, sc, w, h.partials, h.dscal, c.s, h.comm);
            c.bytes += 4.0 * N * k + 8.0 * N;
          }
        } else {
          launch_mdot_scaled(N, k, Vl, sc, w, h.partials, h.dscal, c.s, h.comm);
          c.bytes += 8.0 * N * (k + 1.0);
        }
        c.read(half ? k + 1 : k);
        const double wnorm2 = half ? h.hscal[k] : 0.0;
        if (half && wnorm2 > 0.0 && finite(wnorm2)) {
          // a power of two at or below sqrt(N) / ||w||: the scaling is exact, and ||w||'s last
          // bits (its summation order differs between the fused single-device SpMV + dot and the
          // distributed SpMV then dot) do not reach the shadow
          int e = 0;
          std::frexp(sqN / std::sqrt(wnorm2), &e);
          sig = std::ldexp(1.0, e - 1);
        }
        // h = R^-T p (forward substitution), c' = R^-1 h (back substitution); the update pass
        // w -= t c' returns q = t^T w and ||w||^2.  hacc accumulates Q^T w over the passes.
        auto project = [&](const double* pin, double* hout) {
          for (int i = 0; i < k; ++i) {
            double t = pin[i];
            for (int l = 0; l < i; ++l) t -= R[(size_t)l * (m + 1) + i] * hout[l];
            hout[i] = t / R[(size_t)i * (m + 1) + i];
          }
          for (int i = k - 1; i >= 0; --i) {
            double t = hout[i];
            for (int l = i + 1; l < k; ++l) t -= R[(size_t)i * (m + 1) + l] * cv[l];
            cv[i] = t / R[(size_t)i * (m + 1) + i];
          }
          for (int i = 0; i < k; ++i) h.hscal[96 + i] = cv[i];
          h.hscal[96 + k] = sig;  // R28: the fp16 shadow's scale (coef[k] of the update kernel)
          AMG_CK(cudaMemcpyAsync(h.dscal + 96, h.hscal + 96, sizeof(double) * (k + 1), cudaMemcpyHostToDevice, c.s));
          launch_cgs_update_dots_nrm(N, k, Vl, sc, h.dscal + 96, w, w, h.partials, h.dscal + 32, c.s, h.comm,
                                     shadow ? h.Vs[j + 1] : nullptr, half ? AMG_F16 : AMG_F32);
          c.bytes += 8.0 * N * (k + 2.0) + (shadow ? (half ? 2.0 : 4.0) * N : 0.0);  // k vectors and w read, w written
          c.read(32 + k + 1);
        };
        std::vector<double> pin(h.hscal, h.hscal + k), h2(k);
        const bool reorth_always = env_set("AMG_REORTH_ALWAYS");  // test switch: take the extra pass every step
        project(pin.data(), hv.data());
        for (int pass = 0;; ++pass) {
          hn = std::sqrt(std::max(h.hscal[32 + k], 0.0));
          if (!(hn > 0.0 && finite(hn))) break;
          // R(:, k) = R^-T (q / hn), R(k, k) = sqrt(1 - |R(0:k, k)|^2)
          double ss = 0.0;
          for (int i = 0; i < k; ++i) {
            double t = h.hscal[32 + i] / hn;
            for (int l = 0; l < i; ++l) t -= R[(size_t)l * (m + 1) + i] * R[(size_t)l * (m + 1) + k];
            R[(size_t)i * (m + 1) + k] = t / R[(size_t)i * (m + 1) + i];
            ss += R[(size_t)i * (m + 1) + k] * R[(size_t)i * (m + 1) + k];
          }
          const double d2 = 1.0 - ss;
          // Safeguard: when the updated w is still far from orthogonal to span(V) (|Q^T w1|^2
          // above half of |w1|^2), 1 - ss loses its digits to cancellation; orthogonalise w1
          // once more (the pass's q = t^T w1 gives Q^T w1 = R^-T q without another multi-dot)
          // and take the coefficients of both passes -- CGS2's reorthogonalisation, applied
          // only where needed.  At most one extra pass.
          if (pass == 0 && (ss > 0.5 || !(d2 > 1e-8) || reorth_always)) {
            for (int i = 0; i < k; ++i) pin[i] = h.hscal[32 + i];
            project(pin.data(), h2.data());
            for (int i = 0; i < k; ++i) hv[i] += h2[i];
            ++h.reorth_passes;
            continue;
          }
          R[(size_t)k * (m + 1) + k] = d2 > 0.0 ? std::sqrt(d2) : 0.0;
          for (int i = 0; i < k; ++i) hv[i] += hn * R[(size_t)i * (m + 1) + k];
          hn *= R[(size_t)k * (m + 1) + k];
          break;
        }
        h.hscal[100 + m] = 1.0 / std::sqrt(std::max(h.hscal[32 + k], 0.0));  // s_{j+1}: t_{j+1} = s w1
        AMG_CK(cudaMemcpyAsync(sc + j + 1, h.hscal + 100 + m, sizeof(double), cudaMemcpyHostToDevice, c.s));
        if (half) {  // m_{j+1} = s_{j+1} / sig_{j+1}
          h.hscal[223] = h.hscal[100 + m] / sig;
          AMG_CK(cudaMemcpyAsync(msc + j + 1, h.hscal + 223, sizeof(double), cudaMemcpyHostToDevice, c.s));
        }
        for (int i = 0; i < k; ++i) hh[i] = hv[i];
      }
      s_host = 1.0 / hn;
      hh[j + 1] = hn;
      for (int i = 0; i < j; ++i) {
        double t = cs[i] * hh[i] + sn[i] * hh[i + 1];
        hh[i + 1] = -sn[i] * hh[i] + cs[i] * hh[i + 1];
        hh[i] = t;
      }
      const double rr = std::hypot(hh[j], hh[j + 1]);
      if (rr == 0.0 || !finite(rr)) {
        status = AMG_EBREAKDOWN;
        stop = true;
        break;
      }
      cs[j] = hh[j] / rr;
      sn[j] = hh[j + 1] / rr;
      hh[j] = rr;
      hh[j + 1] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = hh[i];
      ++it;
      if (std::fabs(g[j + 1]) <= rtol * nb || it >= h.p.maxiter || hn == 0.0) stop = true;
    }
    if (status == AMG_EBREAKDOWN) break;
    const int k = j;
    for (int i = k - 1; i >= 0; --i) {
      double t = g[i];
      for (int cc = i + 1; cc < k; ++cc) t = t - H[(size_t)i * m + cc] * y[cc];
      y[i] = t / H[(size_t)i * m + i];
    }
    for (int i = 0; i < k; ++i) h.hscal[96 + i] = y[i];
    AMG_CK(cudaMemcpyAsync(h.dscal + 96, h.hscal + 96, sizeof(double) * k, cudaMemcpyHostToDevice, c.s));
    PtrList Zl{};
    for (int i = 0; i < k; ++i) Zl.p[i] = (const double*)h.Z[i];
    launch_zupdate(N, k, Zl, h.zt, h.dscal + 96, x, c.s);
    c.bytes += N * (16.0 + sx * k);
    c.residual(b, x, h.V[0]);  // true residual = next cycle's V_0
    launch_dot(N, h.V[0], AMG_F64, h.V[0], AMG_F64, h.partials, h.dscal + 64, true, c.s, h.comm);
    k_set_inv<<<1, 1, 0, c.s>>>(sc, h.dscal + 64);
    AMG_CK_LAUNCH();
    ++g_launches;
    ++t_launches;
    c.bytes += 8.0 * N;
    shadow0();
    c.read(65);
    beta = h.hscal[64];
    s_host = 1.0 / beta;
    if (beta <= rtol * nb) status = AMG_OK;
  }
  return finish(c, b, x, h.V[0], nb, status, it, cycles > 0 ? cycles - 1 : 0, rep);
}

// ---- IDR(s) (the paper's outer solver, Table 1; reading R17) ----
// Bi-orthogonal IDR(s) (van Gijzen & Sonneveld 2011), right preconditioned, omega by
// "maintaining the convergence" (kappa = 0.7), the oracle's steps and stopping rules
// (oracle.cpp solve_idrs).  The s x s matrix M = P^T G, f = P^T r and all small solves
// live on the host; per inner step the device does: v = r - G c (lincomb), vh = M^-1 v
// (graphed preconditioner), U_k = om vh + U c, G_k = A U_k, one multi-dot P^T G_k (the
// bi-orthogonalisation coefficients follow from it and M by forward substitution, so the
// sequential Gram-Schmidt dots of the oracle need no extra passes), the G_k / U_k / r / x
// updates and ||r||.  Two host reads per inner step.
int solve_idrs(Ctx& c, const double* b, double* x, double rtol, double nb, amg_report* rep) {
  Handle& h = c.h;
  const int sd = h.p.idrs_s;
  const int64_t N = c.N;
  const double kappa = 0.7;
  double *r = h.vec[0], *v = h.vec[1], *vh = h.vec[2], *t = h.vec[3];
  std::vector<double> M((size_t)sd * sd, 0.0), f(sd), cc(sd), al(sd), pg(sd);
  const uint64_t n_global = (uint64_t)h.n_global_rows * h.b, off = (uint64_t)h.row_lo * h.b;
  auto shadow = [&](uint64_t base) {
    idrs_shadow_space(N, sd, base, n_global, off, h.Pi.data(), h.partials, h.dscal + 200, c.s, h.comm);
    c.bytes += 8.0 * N * (1.0 + sd);
  };
  uint64_t base = 64ULL * (uint64_t)h.p.idrs_seed;
  if (!h.idrs_ready || h.idrs_base != base) {  // the shadow space depends only on (seed, n): keep it
    shadow(base);
    h.idrs_base = base;
    h.idrs_ready = true;
  }
  auto reset = [&]() {
    for (int j = 0; j < sd; ++j) {
      AMG_CK(cudaMemsetAsync(h.Gi[j], 0, sizeof(double) * N, c.s));
      AMG_CK(cudaMemsetAsync(h.Ui[j], 0, sizeof(double) * N, c.s));
    }
    std::fill(M.begin(), M.end(), 0.0);
    for (int j = 0; j < sd; ++j) M[(size_t)j * sd + j] = 1.0;
  };
  auto res_nrm = [&]() {  // r = b - A x, ||r||
    c.residual_nrm(b, x, r);
    c.read(1);
    return std::sqrt(h.hscal[0]);
  };
  double nr = res_nrm();
  int it = 0, restarts = 0, status = AMG_NOT_CONVERGED;
  if (nr <= rtol * nb) status = AMG_OK;
  reset();
  double om = 1.0;
  auto converged_true = [&]() -> bool {
    if (res_nrm() <= rtol * nb) return true;
    reset();
    om = 1.0;
    return false;
  };
  auto breakdown = [&]() -> bool {
    if (restarts >= 1) return false;
    ++restarts;
    c.residual(b, x, r);
    base += (uint64_t)sd;
    shadow(base);
    h.idrs_ready = false;  // the handle's next solve regenerates the seed's own space
    reset();
    om = 1.0;
    return true;
  };
  PtrList Pl{};
  for (int j = 0; j < sd; ++j) Pl.p[j] = h.Pi[j];
  while (status != AMG_OK && it < h.p.maxiter) {
    launch_mdot_scaled(N, sd, Pl, nullptr, r, h.partials, h.dscal, c.s, h.comm);  // f = P^T r
    c.bytes += 8.0 * N * (sd + 1);
    c.read(sd);
    for (int i = 0; i < sd; ++i) f[i] = h.hscal[i];
    bool restart_cycle = false;
    for (int k = 0; k < sd && status != AMG_OK && it < h.p.maxiter; ++k) {
      for (int i = k; i < sd; ++i) {  // M[k:s, k:s] c = f[k:s]
        double a = f[i];
        for (int l = k; l < i; ++l) a = a - M[(size_t)i * sd + l] * cc[l];
        cc[i] = a / M[(size_t)i * sd + i];
      }
      LinComb L{};  // v = r - G[k:s] c
      L.n = 0;
      L.c[L.n] = 1.0, L.p[L.n++] = r;
      for (int i = k; i < sd; ++i) L.c[L.n] = -cc[i], L.p[L.n++] = h.Gi[i];
      launch_lincomb(N, L, v, c.s);
      c.bytes += 8.0 * N * (L.n + 1);
      c.pc(v, vh, AMG_F64);
      L.n = 0;  // U_k = om vh + U[k:s] c   (U_k is read before it is written)
      L.c[L.n] = om, L.p[L.n++] = vh;
      for (int i = k; i < sd; ++i) L.c[L.n] = cc[i], L.p[L.n++] = h.Ui[i];
      launch_lincomb(N, L, h.Ui[k], c.s);
      c.bytes += 8.0 * N * (L.n + 1);
      c.spmv(h.Ui[k], AMG_F64, h.Gi[k]);  // G_k = A U_k
      launch_mdot_scaled(N, sd, Pl, nullptr, h.Gi[k], h.partials, h.dscal, c.s, h.comm);  // P^T G_k
      c.bytes += 8.0 * N * (sd + 1);
      c.read(sd);
      for (int i = 0; i < sd; ++i) pg[i] = h.hscal[i];
      // bi-orthogonalise: alpha_i = (P_i.G_k - sum_{l<i} alpha_l M_il) / M_ii, i < k
      for (int i = 0; i < k; ++i) {
        double a = pg[i];
        for (int l = 0; l < i; ++l) a = a - al[l] * M[(size_t)i * sd + l];
        al[i] = a / M[(size_t)i * sd + i];
      }
      if (k > 0) {
        L.n = 0;
        L.c[L.n] = 1.0, L.p[L.n++] = h.Gi[k];
        for (int i = 0; i < k; ++i) L.c[L.n] = -al[i], L.p[L.n++] = h.Gi[i];
        launch_lincomb(N, L, h.Gi[k], c.s);
        L.p[0] = h.Ui[k];
        for (int i = 0; i < k; ++i) L.p[1 + i] = h.Ui[i];
        launch_lincomb(N, L, h.Ui[k], c.s);
        c.bytes += 2.0 * 8.0 * N * (L.n + 1);
      }
      for (int i = k; i < sd; ++i) {  // M[i][k] = P_i . G_k after the update
        double a = pg[i];
        for (int l = 0; l < k; ++l) a = a - al[l] * M[(size_t)i * sd + l];
        M[(size_t)i * sd + k] = a;
      }
      const double mkk = M[(size_t)k * sd + k];
      if (mkk == 0.0 || !finite(mkk)) {
        if (breakdown()) {
          restart_cycle = true;
          break;
        }
        status = AMG_EBREAKDOWN;
        break;
      }
      const double beta = f[k] / mkk;
      launch_idr_update(N, beta, h.Gi[k], h.Ui[k], r, x, h.partials, h.dscal, c.s, h.comm);  // r, x, ||r||
      c.bytes += 8.0 * N * 6;
      c.read(1);
      ++it;
      nr = h.hscal[0];
      if (nr <= rtol * nb) {
        if (converged_true()) status = AMG_OK;
        restart_cycle = true;
        break;
      }
      for (int i = k + 1; i < sd; ++i) f[i] = f[i] - beta * M[(size_t)i * sd + k];
    }
    if (status == AMG_OK || status == AMG_EBREAKDOWN || restart_cycle || it >= h.p.maxiter) continue;
    // dimension reduction: vh = M^-1 r, t = A vh, omega
    c.pc(r, vh, AMG_F64);
    c.spmv(vh, AMG_F64, t);
    PtrList TR{};
    TR.p[0] = t;
    TR.p[1] = r;
    launch_mdot_scaled(N, 2, TR, nullptr, t, h.partials, h.dscal, c.s, h.comm);  // t.t, r.t
    c.bytes += 8.0 * N * 3;
    c.read(2);
    const double tt = h.hscal[0], tr = h.hscal[1], nt = std::sqrt(tt);
    om = tr / tt;
    const double rho = std::fabs(tr) / (nt * nr);
    if (rho < kappa) om = om * kappa / rho;
    if (om == 0.0 || !finite(om)) {
      if (breakdown()) continue;
      status = AMG_EBREAKDOWN;
      break;
    }
    launch_idr_update(N, om, t, vh, r, x, h.partials, h.dscal, c.s, h.comm);  // r -= om t, x += om vh
    c.bytes += 8.0 * N * 6;
    c.read(1);
    ++it;
    nr = h.hscal[0];
    if (nr <= rtol * nb && converged_true()) status = AMG_OK;
  }
  return finish(c, b, x, r, nb, status, it, restarts, rep);
}

}  // namespace

int krylov_solve(Handle& h, const double* b, double* x, double rtol, cudaStream_t caller, amg_report* rep) {
  // the solve runs on the handle's own non-blocking stream (graph capture is not allowed on
  // the legacy default stream), ordered after / before the caller's stream by two events
  cudaStream_t s = h.work ? h.work : caller;
  if (s != caller) {
    AMG_CK(cudaEventRecord(h.ev_in, caller));
    AMG_CK(cudaStreamWaitEvent(s, h.ev_in, 0));
  }
  struct Join {
    Handle& h;
    cudaStream_t s, caller;
    ~Join() {
      if (s != caller) {
        cudaEventRecord(h.ev_out, s);
        cudaStreamWaitEvent(caller, h.ev_out, 0);
      }
    }
  } join{h, s, caller};
  Ctx c(h, s);
  // ||b||; ||b|| = 0 -> x = 0, converged, relres 0
  launch_dot(c.N, b, AMG_F64, b, AMG_F64, h.partials, h.dscal, true, s, h.comm);
  c.read(1);
  const double nb = h.hscal[0];
  if (rep) rep->levels = h.amg_active ? (int)h.lv.size() + 1 : 0;
  if (nb == 0.0) {
    AMG_CK(cudaMemsetAsync(x, 0, sizeof(double) * c.N, s));
    AMG_CK(cudaStreamSynchronize(s));
    if (rep) rep->iters = 0, rep->converged = 1, rep->restarts = 0, rep->relres_true = 0.0, rep->alg_bytes = 0.0;
    return AMG_OK;
  }
  switch (h.p.solver) {
    case AMG_CG:
      if (h.p.use_graphs && !g_prof && !env_set("AMG_NO_GRAPH") && !env_set("AMG_NO_STEP_GRAPH") &&
          (!h.comm || h.comm->capturable()))
        return solve_cg_graphed(c, b, x, rtol, nb, rep);
      return solve_cg(c, b, x, rtol, nb, rep);
    case AMG_BICGSTAB:
      // one graph per step unless graphs are off, the profiler times every launch, or the
      // communicator cannot be captured (the thread-emulated one)
      if (h.p.use_graphs && !g_prof && !env_set("AMG_NO_GRAPH") && !env_set("AMG_NO_STEP_GRAPH") &&
          (!h.comm || h.comm->capturable()))
        return solve_bicgstab_graphed(c, b, x, rtol, nb, rep);
      return solve_bicgstab(c, b, x, rtol, nb, rep);
    case AMG_GMRES: return solve_gmres(c, b, x, rtol, nb, rep);
    case AMG_IDRS: return solve_idrs(c, b, x, rtol, nb, rep);
    default: fail(AMG_EINVAL, "unknown solver");
  }
}

}  // namespace amgb
