// blas1.h -- K12 vector kernels (fp64 outer vectors), all stream-ordered.
#pragma once

#include "common.cuh"

namespace amgb {
class CommBase;
}

namespace amgb {

constexpr int kMaxPartials = 148 * 8;

struct PtrList {
  const double* p[32];
};

// out[0] = a . b (or its sqrt); partials: scratch of kMaxPartials doubles
void launch_dot(int64_t n, const void* a, int at, const void* b, int bt, double* partials, double* out,
                bool sqrt_out, cudaStream_t s, CommBase* comm = nullptr);
// out[j] = V_j . w, j < k <= 32; partials: scratch of 32 * kMaxPartials doubles followed
// by one zero-initialised unsigned ticket (the multi-vector kernels finish their own
// reduction in the last block and reset the ticket)
void launch_mdot(int64_t n, int k, const PtrList& V, const double* w, double* partials, double* out, cudaStream_t s);
// out[j] = sc[j] V_j . w   (basis stored unnormalised with scales sc; device)
void launch_mdot_scaled(int64_t n, int k, const PtrList& V, const double* sc, const double* w, double* partials,
                        double* out, cudaStream_t s, CommBase* comm = nullptr);
// w_out = w - sum_j coef[j] sc[j] V_j, plus out[j] = sc[j] V_j . w_out (dot_next) or
// out[0] = ||w_out|| and, if inv_out, *inv_out = 1/||w_out|| -- one pass (CGS2 step of
// flexible GMRES)
void launch_cgs_update(int64_t n, int k, const PtrList& V, const double* sc, const double* coef, const double* w,
                       double* w_out, bool dot_next, double* partials, double* out, cudaStream_t s,
                       CommBase* comm = nullptr, double* inv_out = nullptr);
// the same with the basis read from its fp32 shadow copy (Vf.p[j] are float*; reading R23)
void launch_mdot_scaled_f32(int64_t n, int k, const PtrList& Vf, const double* sc, const double* w, double* partials,
                            double* out, cudaStream_t s, CommBase* comm = nullptr);
// w_out = w - sum_j coef[j] sc[j] V_j, out[j] = sc[j] V_j . w_out (j < k), out[k] = w_out . w_out
// (one pass; the Gram/Cholesky two-pass orthogonalisation of flexible GMRES); wf_out
// (optional): an fp32 copy of w_out written in the same pass (the shadow basis of R23)
void launch_cgs_update_dots_nrm(int64_t n, int k, const PtrList& V, const double* sc, const double* coef,
                                const double* w, double* w_out, double* partials, double* out, cudaStream_t s,
                                CommBase* comm = nullptr, void* wf_out = nullptr, int wf_type = AMG_F32);
// reading R28: the pass-1 multi-dot on an fp16 shadow (Vh.p[j] are __half*) stored at scale
// sig_j; ms[j] = s_j / sig_j (device); out[k] = w . w (k + 1 outputs)
void launch_mdot_scaled_f16(int64_t n, int k, const PtrList& Vh, const double* ms, const double* w, double* partials,
                            double* out, cudaStream_t s, CommBase* comm = nullptr);
// dst (__half) = fp16(src * sig), sig = the power of two at or below mul * *s_dev; *m_out = *s_dev / sig
void launch_to_half_scaled(int64_t n, const double* src, const double* s_dev, double mul, void* dst, double* m_out,
                           cudaStream_t s);
// w -= sum_j coef[j] V_j  (coef: device)
void launch_maxpy(int64_t n, int k, const PtrList& V, const double* coef, double* w, cudaStream_t s);
// x += sum_j y[j] Z_j  (Z of dtype zt, y: device)
void launch_zupdate(int64_t n, int k, const PtrList& Z, int zt, const double* y, double* x, cudaStream_t s);
void launch_axpby(int64_t n, double a, const double* x, double b, double* y, cudaStream_t s);
void launch_axpbypcz(int64_t n, double a, const double* x, double b, const double* y, double c, double* z,
                     cudaStream_t s);
// out = sum_t c[t] p[t]  (t < n <= 12; host coefficients; out may alias an input)
struct LinComb {
  int n;
  double c[12];
  const double* p[12];
};
void launch_lincomb(int64_t n, const LinComb& L, double* out, cudaStream_t s);
// IDR(s) shadow space: P[j] = MGS-orthonormalised N(0,1) draws of the counter RNG
// (stream 6, idx = (base + j) * n_global + off + i); dots over ranks via comm
void idrs_shadow_space(int64_t n, int sdim, uint64_t base, uint64_t n_global, uint64_t off, double* const* P,
                       double* partials, double* dscal, cudaStream_t s, CommBase* comm);
// IDR(s) step: r -= a g; x += a u; out[0] = ||r|| (one pass, deterministic)
// (a_num, a_den: device scalars, a = a_num[0] / a_den[0], no update when a_den[0] is 0 / not finite)
void launch_idr_update(int64_t n, double a, const double* g, const double* u, double* r, double* x,
                       double* partials, double* out, cudaStream_t s, CommBase* comm = nullptr,
                       const double* a_num = nullptr, const double* a_den = nullptr);
// CG: p = z + beta p with beta = rz[0] / rho[0] (device)
void launch_cg_p(int64_t n, const double* z, double* p, const double* rz, const double* rho, cudaStream_t s);
// BiCGStab: out = r - (num / den[0]) v, dst[0] = out.out   (den on the device)
void launch_sub_div_nrm(int64_t n, double num, const double* den, const double* v, const double* r, double* out,
                        double* partials, double* dst, cudaStream_t s, CommBase* comm = nullptr);
// BiCGStab: out = s - c t, dst[0] = out.out, dst[1] = rh.out
void launch_axpy_2dot(int64_t n, double c, const double* t, const double* s_, double* out, const double* rh,
                      double* partials, double* dst, cudaStream_t s, CommBase* comm = nullptr);
// y = x / sdev[0]
void launch_scale_by_inv(int64_t n, const double* x, const double* sdev, double* y, cudaStream_t s);

// BiCGStab with device-side scalars (reading R24): slots of the scalar block `sc`
enum : int {
  kBicgRho = 0,       // rho = rh . r of this iteration
  kBicgRhoOld = 1,    // rho of the previous iteration
  kBicgAlpha = 2,     // alpha of the previous iteration (beta)
  kBicgOmega = 3,     // omega of the previous iteration (beta)
  kBicgFirst = 4,     // 1: p = r (first step after a (re)start)
  kBicgTol = 5,       // rtol ||b||
  kBicgRv = 6,        // rh . v
  kBicgSs = 7,        // s . s
  kBicgTt = 8,        // t . t
  kBicgTs = 9,        // t . s
  kBicgRr = 10,       // r . r (new r)
  kBicgRhoNext = 11,  // rh . r (new r)
  kBicgAlphaNew = 12, // alpha of this iteration
  kBicgOmegaNew = 13, // omega of this iteration
  kBicgSlots = 16
};
// p = r (first) or r + beta (p - omega v), beta = (rho / rho_old) (alpha / omega) from sc
void launch_bicg_p(int64_t n, const double* r, const double* v, double* p, const double* sc, cudaStream_t s);
// alpha = rho / rv -> sc[AlphaNew]; s = r - alpha v; sc[Ss] = s . s
void launch_bicg_s(int64_t n, const double* v, const double* r, double* sv, double* sc, double* partials,
                   cudaStream_t s, CommBase* comm = nullptr);
// omega = ts / tt; x += alpha ph + omega sh (half-step exit: alpha ph; breakdown: nothing);
// r = s - omega t; sc[Rr] = r . r, sc[RhoNext] = rh . r
void launch_bicg_xr(int64_t n, const double* ph, const double* sh, const double* t, const double* sv,
                    const double* rh, double* x, double* r, double* sc, double* partials, cudaStream_t s,
                    CommBase* comm = nullptr);

}  // namespace amgb
