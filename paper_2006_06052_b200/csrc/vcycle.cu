// vcycle.cu -- the preconditioner applies: SA V(npre,npost) cycle (C9)
// and the Schur pressure correction (Eq. 9a/9b).  Pure launches on
// one stream; no allocation, no synchronisation (graph-capturable).
#include <cstdlib>
#include <utility>

#include "ops.h"
#include "prof.h"
#include "solver.h"

namespace amgb {

void* level0_f(Handle& h) { return h.lv.empty() ? h.coarse.f : h.lv[0].f; }

// ILU(0) smoothing (reading R20), k = ilu_sweeps Jacobi sweeps per triangular solve:
//   y_0 = g, y_m = g - L_s y_(m-1);  z_0 = D^-1 y_k;  z_m = D^-1 (y_k - U_s z_(m-1)), the last
//   one written as xo = xb + z_k (xb == nullptr: from zero).  2k + 1 launches; single device.
static void ilu_apply(Handle& h, Level& L, const void* g, const void* xb, void* xo, cudaStream_t s) {
  const int xt = h.xt, k = h.p.ilu_sweeps;
  const void* y = g;
  for (int m = 0; m < k; ++m) {
    launch_residual(L.Lf, g, y, L.w[m & 1], xt, s);
    y = L.w[m & 1];
  }
  void* z = L.w[2];
  launch_apply_M(L.A.n, L.A.b, L.M, h.vt, y, z, xt, s);
  for (int m = 1; m <= k; ++m) {
    const bool last = m == k;
    void* zn = last ? xo : (z == L.w[2] ? L.w[3] : L.w[2]);
    launch_ilu_usweep(L.Uf, L.M, y, z, last ? xb : nullptr, zn, xt, s);
    z = zn;
  }
}

// x <- x + (LU)^-1 (f - A x)   (distributed: the residual with the level's halo; the
// factors are slab-local, R26)
static void ilu_step(Handle& h, Level& L, void* x, cudaStream_t s) {
  halo_overlapped(h, L.halo, L.A, x, h.xt, L.A.b, s,
                  [&](int r0, int r1) { launch_residual(L.A, L.f, x, L.r, h.xt, s, r0, r1); });
  ilu_apply(h, L, L.r, x, x, s);
}

// V(l, f):  x = M f;  r = f - A x;  f_c = R r;  x_c = V(l+1, f_c);  x += P x_c;
//           x = x + M (f - A x)            (one kernel per line; fp64 accumulation,
//                                            one rounding on store)
bool fuse_presmooth(const Handle& h, size_t l) {
  return h.p.fused_presmooth && l < h.lv.size() && !h.lv[l].Lf.ptr && !(h.comm && l >= h.rep_from);
}

void* vcycle_run(Handle& h, size_t l, cudaStream_t s, bool pre_done, const JoinOut* jo) {
  const int xt = h.xt, vt = h.vt;
  if (h.comm && l == h.rep_from) replicated_allgather(h, l, s);  // distributed: replicated from here on
  if (l == h.lv.size()) {
    launch_dense_gemv(h.coarse.N, h.coarse.inv, vt, h.coarse.f, h.coarse.x, xt, s);  // K8
    return h.coarse.x;
  }
  Level& L = h.lv[l];
  void* x = L.x;
  void* t = L.t;
  const bool ilu = L.Lf.ptr != nullptr;
  if (ilu) ilu_apply(h, L, L.f, nullptr, x, s);  // K4a with ILU(0): x = (LU)^-1 f (sweeps)
  else if (!pre_done) launch_apply_M(L.A.n, L.A.b, L.M, vt, L.f, x, xt, s);  // K4a: pre-smooth from zero
  for (int k = 1; k < h.p.npre; ++k) {
    if (ilu) {
      ilu_step(h, L, x, s);
      continue;
    }
    halo_overlapped(h, L.halo, L.A, x, xt, L.A.b, s,
                    [&](int r0, int r1) { launch_smooth(L.A, L.M, L.f, x, t, xt, s, r0, r1); });
    std::swap(x, t);
  }
  halo_overlapped(h, L.halo, L.A, x, xt, L.A.b, s,
                  [&](int r0, int r1) { launch_residual(L.A, L.f, x, L.r, xt, s, r0, r1); });  // K4b: r = f - A x
  void* fc = level_f_slab(h, l + 1);
  // K6: f_c = R r (with the next level's K4a x_c = M_c f_c in its epilogue where possible)
  const bool fused = fuse_presmooth(h, l + 1) && launch_spmv_M(L.R, L.r, fc, h.lv[l + 1].M, vt, h.lv[l + 1].x, xt, s);
  if (!fused) launch_spmv(L.R, 1.0, L.r, xt, 0.0, fc, xt, s);
  void* xc = vcycle_run(h, l + 1, s, fused);
  launch_spmv(L.P, 1.0, xc, xt, 1.0, x, xt, s);  // K7: x += P x_c
  for (int k = 0; k < h.p.npost; ++k) {          // K5: post-smooth (double-buffered)
    if (ilu) {
      ilu_step(h, L, x, s);
      continue;
    }
    if (jo && k == h.p.npost - 1 && (jo->p ? smooth_join_ok(L.A, xt) : smooth_widen_ok(L.A, xt, jo->zt))) {
      halo_overlapped(h, L.halo, L.A, x, xt, L.A.b, s, [&](int r0, int r1) {
        if (jo->p) launch_smooth_join(L.A, L.M, L.f, x, jo->p, jo->z, jo->zt, xt, s, r0, r1);  // + K9' (the join)
        else launch_smooth_widen(L.A, L.M, L.f, x, jo->z, jo->zt, xt, s, r0, r1);  // + the output conversion
      });
      return nullptr;
    }
    halo_overlapped(h, L.halo, L.A, x, xt, L.A.b, s,
                    [&](int r0, int r1) { launch_smooth(L.A, L.M, L.f, x, t, xt, s, r0, r1); });
    std::swap(x, t);
  }
  return x;
}

// is the Schur apply's join fused into the second U-solve's last post-smoothing step?
static bool join_fused(const Handle& h) {
  return h.schur && !h.masked && h.amg_active && !h.lv.empty() && h.b == 4 && h.pc == 3 && h.p.npost >= 1 &&
         !h.lv[0].Lf.ptr && !(h.comm && h.rep_from == 0) && smooth_join_ok(h.lv[0].A, h.xt) &&
         !env_int("AMG_NO_JOIN_FUSE", 0);
}

// is the monolithic apply's output conversion fused into level 0's last post-smoothing step?
static bool widen_fused(const Handle& h, int zt) {
  return !h.schur && h.amg_active && !h.lv.empty() && h.p.npost >= 1 && !h.lv[0].Lf.ptr &&
         !(h.comm && h.rep_from == 0) && (int64_t)h.lv[0].A.n * h.lv[0].A.b == (int64_t)h.n * h.b &&
         smooth_widen_ok(h.lv[0].A, h.xt, zt) && !env_int("AMG_NO_WIDEN_FUSE", 0);
}

// z = M r.  Monolithic AMG: narrow r once (RNE), V-cycle, widen exactly (C9).
// Schur (C10): split + narrow; u* = V(r_u); p = m_S o (r_p - B u*); r_u' = r_u - B^T p;
// u = V(r_u'); z = join(u, p).
bool bicg_p_fused(const Handle& h) {
  return !h.schur && h.amg_active && fuse_presmooth(h, 0) && h.lv[0].A.b == h.b && !env_int("AMG_NO_BICGP_FUSE", 0);
}

void precond_apply(Handle& h, const double* r, void* z, int zt, cudaStream_t s, double scale,
                   const double* scale_dev, const BicgPre* pre) {
  const int64_t N = (int64_t)h.n * h.b;
  if (pre && !bicg_p_fused(h)) {  // the direction update on its own (k_bicg_p), then the apply
    launch_bicg_p(N, pre->r, pre->v, pre->p, pre->sc, s);
    pre = nullptr;
  }
  if (!h.amg_active) {
    launch_convert(N, r, AMG_F64, z, zt, scale, s, scale_dev);
    return;
  }
  void* f0 = level0_f(h);
  // level 0's K4a in the producer of f_0 (its blocks are the producer's rows: not the V2
  // scalar U-solver, whose level 0 has 1 x 1 blocks)
  const bool f0M = fuse_presmooth(h, 0) && h.lv[0].A.b == (h.schur ? h.nu : h.b);
  void* x0 = f0M ? h.lv[0].x : nullptr;
  const void* M0 = f0M ? h.lv[0].M : nullptr;
  if (!h.schur) {
    const bool fused =
        f0M && (pre ? launch_bicg_p_convert_M(h.n, h.b, pre->r, pre->v, pre->p, pre->sc, f0, h.xt, M0, h.vt, x0, s)
                    : launch_convert_M(h.n, h.b, r, scale, f0, h.xt, M0, h.vt, x0, s, scale_dev));
    if (!fused) launch_convert(N, r, AMG_F64, f0, h.xt, scale, s, scale_dev);
    const JoinOut jw{nullptr, z, zt};  // p == nullptr: widen into z
    void* x = vcycle_run(h, 0, s, fused, widen_fused(h, zt) ? &jw : nullptr);
    if (x) launch_convert(N, x, h.xt, z, zt, 1.0, s);
    return;
  }
  if (h.masked) {  // general scalar pressure mask (R21): the same steps on the scalar split
    launch_mask_split(h.nu_s, h.np_s, h.uidx, h.pidx, r, scale, f0, h.rp, h.xt, s, scale_dev);
    void* us = vcycle_run(h, 0, s);
    halo_exchange(h, h.haloBu, us, h.xt, 1, s);              // distributed (R27): B's velocity ghosts
    launch_schur_p(h.Bm, h.mS, h.rp, us, h.pp, h.xt, s);     // p = m_S o (r_p - B u*)
    halo_exchange(h, h.haloBTp, h.pp, h.xt, 1, s);           // B^T's pressure ghosts
    launch_residual(h.BTm, f0, h.pp, f0, h.xt, s);           // r_u' = r_u - B^T p (in place)
    void* u = vcycle_run(h, 0, s);
    launch_mask_join(h.nu_s, h.np_s, h.uidx, h.pidx, u, h.pp, h.xt, z, zt, s);
    return;
  }
  // K9 (+ level 0's K4a)
  const bool fs = f0M && launch_split_M(h.n, h.b, h.pc, r, scale, f0, h.rp, h.xt, M0, h.vt, x0, s, scale_dev);
  if (!fs) launch_split(h.n, h.b, h.pc, r, scale, f0, h.rp, h.xt, s, scale_dev);
  void* us = vcycle_run(h, 0, s, fs);                                                          // u* = V(r_u)
  halo_exchange(h, h.halo0, us, h.xt, h.nu, s);
  launch_schur_p(h.Bm, h.mS, h.rp, us, h.pp, h.xt, s);  // K10
  halo_exchange(h, h.halo0, h.pp, h.xt, 1, s);
  // K11 (in place; + level 0's K4a for the second V-cycle).  us (the first V-cycle's output,
  // one of level 0's x / t buffers) is dead after K10, so x_0 may be overwritten here.
  const bool fu = fs && launch_schur_u_M(h.BTm, f0, h.pp, f0, M0, h.vt, x0, h.xt, s);
  if (!fu) launch_schur_u(h.BTm, f0, h.pp, f0, h.xt, s);
  const JoinOut jo{h.pp, z, zt};
  void* u = vcycle_run(h, 0, s, fu, join_fused(h) ? &jo : nullptr);                           // u = V(r_u')
  if (u) launch_join(h.n, h.b, h.pc, u, h.pp, h.xt, z, zt, s);                                 // K9'
}

// The same application replayed from a CUDA graph: one graph per (r, z, zt, scale_dev)
// (the Krylov solvers use a handful of fixed workspace buffers: GMRES(m) has m), captured
// on first use on the handle's work stream and kept for the handle's life.  Eager when a
// communicator is attached (NCCL halo exchanges), while the per-kernel profiler is on, or
// with AMG_NO_GRAPH=1.  The library launch counter advances by the graph's kernel count.
void precond_apply_graphed(Handle& h, const double* r, void* z, int zt, cudaStream_t s, const double* scale_dev) {
  const bool off = env_set("AMG_NO_GRAPH");
  if (off || !h.p.use_graphs || (h.comm && !h.comm->capturable()) || g_prof || h.pc_graphs.size() >= 256) {
    precond_apply(h, r, z, zt, s, 1.0, scale_dev);
    return;
  }
  for (const PcGraph& G : h.pc_graphs)
    if (G.r == r && G.z == z && G.zt == zt && G.sd == scale_dev) {
      AMG_CK(cudaGraphLaunch(G.exec, s));
      g_launches += G.kernels;
      t_launches += G.kernels;
      return;
    }
  PcGraph G{r, z, zt, scale_dev, nullptr, 0};
  const int64_t l0 = t_launches;
  cudaGraph_t graph = nullptr;
  AMG_CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  try {
    precond_apply(h, r, z, zt, s, 1.0, scale_dev);
  } catch (...) {
    cudaStreamEndCapture(s, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  AMG_CK(cudaStreamEndCapture(s, &graph));
  G.kernels = t_launches - l0;  // kernels captured (not launched): undo the count
  t_launches = l0;
  g_launches -= G.kernels;
  cudaError_t e = cudaGraphInstantiate(&G.exec, graph, 0);
  cudaGraphDestroy(graph);
  AMG_CK(e);
  h.pc_graphs.push_back(G);
  AMG_CK(cudaGraphLaunch(G.exec, s));
  g_launches += G.kernels;
  t_launches += G.kernels;
}

// Algorithmic bytes of one preconditioner application:
// every matrix array read once per use, every vector read/written once per kernel.
static double mat_bytes(const Mat& A, int vt) {
  return (double)A.nnz * (4.0 + (double)A.b * A.b * dtype_size(vt)) + 4.0 * (A.n + 1);
}

// does level l's K4a run inside its producer (the launchers' conditions)?
static bool presmooth_fused(const Handle& h, size_t l) {
  if (!fuse_presmooth(h, l)) return false;
  if (l > 0) return h.lv[l - 1].R.tma_grid == 0 && h.lv[l - 1].R.vt == h.vt;
  return !h.masked && h.lv[0].A.b == (h.schur ? h.nu : h.b) && (!h.schur || (h.b == 4 && h.pc == 3 && h.xt == AMG_F32));
}

static double vcycle_bytes(const Handle& h) {
  const double sx = (double)dtype_size(h.xt), sv = (double)dtype_size(h.vt);
  double tot = 0.0;
  for (size_t l = 0; l < h.lv.size(); ++l) {
    const Level& L = h.lv[l];
    const double nb = (double)L.A.n * L.A.b;
    if (L.Lf.ptr) {  // ILU(0): k L sweeps (g, y gathered, y'), z_0 = D^-1 y, k U sweeps (y, z gathered, z' | x rw)
      const double k = h.p.ilu_sweeps, Msz = nb * L.A.b * sv;
      const double app = k * (mat_bytes(L.Lf, h.vt) + 3.0 * nb * sx) + (Msz + 2.0 * nb * sx) +
                         k * (mat_bytes(L.Uf, h.vt) + Msz + 3.0 * nb * sx);
      tot += 2.0 * app + nb * sx;                                 // pre-smooth, post-smooth (+ x read)
      tot += 2.0 * (mat_bytes(L.A, h.vt) + 3.0 * nb * sx);       // K4b and the post-smooth residual
      tot += mat_bytes(L.P, h.vt) + mat_bytes(L.R, h.vt);
      tot += nb * sx * (1 + 2) + (double)L.nc * L.A.b * sx * 2;  // K6 r read; K7 x rw; f_c, x_c
      continue;
    }
    tot += 2.0 * mat_bytes(L.A, h.vt) + mat_bytes(L.P, h.vt) + mat_bytes(L.R, h.vt);
    tot += 2.0 * nb * L.A.b * sv;  // M read twice
    // K4a: f, x (fused into the producer of f: x) | K4b: f, x, r | K6: r, f_c | K7: x_c, x rw | K5: f, x, x'
    tot += nb * sx * ((presmooth_fused(h, l) ? 1 : 2) + 3 + 1 + 2 + 3);
    tot += (double)L.nc * L.A.b * sx * 2;  // f_c write, x_c read
  }
  tot += (double)h.coarse.N * h.coarse.N * sv + 2.0 * h.coarse.N * sx;
  return tot;
}

double precond_bytes(const Handle& h) {
  const int64_t N = (int64_t)h.n * h.b;
  const double sx = (double)dtype_size(h.xt), sv = (double)dtype_size(h.vt);
  if (!h.amg_active) return (double)N * 16.0;
  if (!h.schur)  // convert in, convert out (fused into K5: its x' write and the re-read go)
    return vcycle_bytes(h) + (double)N * (8.0 + sx) * 2.0 - (widen_fused(h, h.p.solver == AMG_GMRES ? h.zt : AMG_F64) ? 2.0 * N * sx : 0.0);
  if (h.masked) {
    const double nu = h.nu_s, np = h.np_s;
    double t = 2.0 * vcycle_bytes(h) + (double)N * (12.0 + sx) + (double)N * (4.0 + sx + 8.0);  // split, join
    t += mat_bytes(h.Bm, h.vt) + np * sv + nu * sx + 2.0 * np * sx;                               // K10
    t += mat_bytes(h.BTm, h.vt) + np * sx + 2.0 * nu * sx;                                        // K11
    return t;
  }
  const double n = (double)h.n, nnz = (double)h.A.nnz;
  double t = 2.0 * vcycle_bytes(h);
  t += (double)N * 8.0 + (double)N * sx;                        // split
  t += nnz * (4.0 + 3.0 * sv) + 4.0 * (n + 1) + n * sv + n * 3 * sx + 2 * n * sx;  // K10
  t += nnz * (4.0 + 3.0 * sv) + 4.0 * (n + 1) + n * sx + 6.0 * n * sx;           // K11
  t += (double)N * sx + (double)N * 8.0;                        // join
  if (join_fused(h)) t -= 6.0 * n * sx;                         // fused: no u write / u read
  return t;
}

}  // namespace amgb
