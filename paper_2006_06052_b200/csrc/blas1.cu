// blas1.cu -- K12 Krylov vector kernels: deterministic dot products (two-stage,
// fixed grid for a given length, fixed-order finalisation), multi-dot / multi-axpy
// for the CGS2 Arnoldi step, linear combinations, and the flexible-GMRES update.
#include "blas1.h"
#include "comm.h"
#include "prof.h"

namespace amgb {

namespace {

constexpr int kT = 256;

inline int nblocks_for(int64_t n) {
  int64_t b = (n + kT * 8 - 1) / (kT * 8);
  if (b < 1) b = 1;
  if (b > kMaxPartials) b = kMaxPartials;
  return (int)b;
}

template <int K>
__device__ __forceinline__ void block_reduce_store(double (&acc)[K], int k, double* partials, int nblk) {
  __shared__ double sh[K][kT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (j >= k) break;
    double v = acc[j];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    if (lane == 0) sh[j][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < k) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) v += sh[threadIdx.x][w];
    partials[(int64_t)threadIdx.x * nblk + blockIdx.x] = v;
  }
}

template <typename TA, typename TB>
__global__ void __launch_bounds__(kT) k_dot(int64_t n, const TA* __restrict__ a, const TB* __restrict__ b,
                                            double* partials, int nblk) {
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT)
    acc[0] = fma((double)a[i], (double)b[i], acc[0]);
  block_reduce_store<1>(acc, 1, partials, nblk);
}

// acc[j] = sum_i V_j[i] w[i], j < k <= 32
__global__ void __launch_bounds__(kT) k_mdot(int64_t n, int k, PtrList V, const double* __restrict__ w,
                                             double* partials, int nblk) {
  double acc[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    const double wi = w[i];
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < k) acc[j] = fma(V.p[j][i], wi, acc[j]);
  }
  block_reduce_store<32>(acc, k, partials, nblk);
}

// CGS2 fused update (flexible GMRES).  Basis vectors are stored
// unnormalised with a scale s_j (v_j = s_j V_j): w_out = w - sum_j c_j s_j V_j, and in the
// same pass either the next Gram-Schmidt coefficients acc_j = s_j V_j . w_out (DOT) or
// ||w_out||^2 (acc_0).  V_j[i] is re-read from L1 in the second loop.
template <bool DOT>
__global__ void __launch_bounds__(kT) k_cgs_update(int64_t n, int k, PtrList V, const double* __restrict__ sc,
                                                   const double* __restrict__ coef, const double* w,
                                                   double* w_out, double* partials, int nblk) {
  __shared__ double c[32], sv[32];
  if (threadIdx.x < k) {
    sv[threadIdx.x] = sc[threadIdx.x];
    c[threadIdx.x] = coef[threadIdx.x] * sc[threadIdx.x];
  }
  __syncthreads();
  double acc[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    double v = w[i];
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < k) v = fma(-c[j], V.p[j][i], v);
    w_out[i] = v;
    if constexpr (DOT) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < k) acc[j] = fma(sv[j] * V.p[j][i], v, acc[j]);
    } else {
      acc[0] = fma(v, v, acc[0]);
    }
  }
  block_reduce_store<32>(acc, DOT ? k : 1, partials, nblk);
}

// scaled multi-dot: out[j] = s_j V_j . w
__global__ void __launch_bounds__(kT) k_mdot_scaled(int64_t n, int k, PtrList V, const double* __restrict__ sc,
                                                    const double* __restrict__ w, double* partials, int nblk) {
  double acc[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    const double wi = w[i];
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < k) acc[j] = fma(V.p[j][i], wi, acc[j]);
  }
  __shared__ double s2[32];
  if (threadIdx.x < k) s2[threadIdx.x] = sc[threadIdx.x];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] *= s2[j < k ? j : 0];
  block_reduce_store<32>(acc, k, partials, nblk);
}

// x += sum_j y[j] Z_j ... see k_zupdate; here: out[j] = scale * sum of the nblk partials of reduction j, in a fixed order
__global__ void k_finalize(int k, const double* partials, int nblk, double* out, int sqrt_out) {
  __shared__ double sh[kT];
  for (int j = 0; j < k; ++j) {
    double v = 0.0;
    for (int i = threadIdx.x; i < nblk; i += kT) v += partials[(int64_t)j * nblk + i];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int off = kT / 2; off > 0; off >>= 1) {
      if (threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[j] = sqrt_out ? sqrt(sh[0]) : sh[0];
    __syncthreads();
  }
}

// w -= sum_j coef[j] V_j   (coef on the device)
__global__ void __launch_bounds__(kT) k_maxpy(int64_t n, int k, PtrList V, const double* __restrict__ coef,
                                              double* __restrict__ w) {
  __shared__ double c[32];
  if (threadIdx.x < k) c[threadIdx.x] = coef[threadIdx.x];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    double v = w[i];
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < k) v = fma(-c[j], V.p[j][i], v);
    w[i] = v;
  }
}

// x += sum_j y[j] Z_j  (Z of type T; y on the device)
template <typename T>
__global__ void __launch_bounds__(kT) k_zupdate(int64_t n, int k, PtrList Z, const double* __restrict__ y,
                                                double* __restrict__ x) {
  __shared__ double c[32];
  if (threadIdx.x < k) c[threadIdx.x] = y[threadIdx.x];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    double v = x[i];
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < k) v = fma(c[j], (double)reinterpret_cast<const T*>(Z.p[j])[i], v);
    x[i] = v;
  }
}

// y = a x + b y
__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT)
    y[i] = (b == 0.0) ? a * x[i] : fma(a, x[i], b * y[i]);
}

// z = a x + b y + c z
__global__ void k_axpbypcz(int64_t n, double a, const double* __restrict__ x, double b, const double* __restrict__ y,
                           double c, double* __restrict__ z) {
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT)
    z[i] = fma(a, x[i], fma(b, y[i], c * z[i]));
}

// y = x / s[0]  (s on the device; used to normalise the next Arnoldi vector)
__global__ void k_scale_by_inv(int64_t n, const double* __restrict__ x, const double* __restrict__ s,
                               double* __restrict__ y) {
  const double inv = 1.0 / s[0];
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) y[i] = x[i] * inv;
}

__global__ void k_sqrt_vec(double* d, int n) {
  if (threadIdx.x < n) d[threadIdx.x] = sqrt(d[threadIdx.x]);
}

// distributed: the partials are local; sum over ranks before the square root
inline void finalize_global(CommBase* comm, double* out, int k, bool sqrt_out, cudaStream_t s) {
  if (!comm) return;
  comm->allreduce_sum(out, k, s);
  if (sqrt_out) {
    k_sqrt_vec<<<1, 32, 0, s>>>(out, k);
    AMG_CK_LAUNCH();
  }
}

inline unsigned ew_grid(int64_t n) {
  int64_t g = (n + kT - 1) / kT;
  if (g > kSMs * 16) g = kSMs * 16;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

void launch_dot(int64_t n, const void* a, int at, const void* b, int bt, double* partials, double* out, bool sqrt_out,
                cudaStream_t s, CommBase* comm) {
  const int nb = nblocks_for(n);
  ProfScope ps_(prof_name("dot", 1, at, bt), (double)n * (a == b ? dtype_size(at) : dtype_size(at) + dtype_size(bt)), s);
  if (at == AMG_F64 && bt == AMG_F64)
    k_dot<double, double><<<nb, kT, 0, s>>>(n, (const double*)a, (const double*)b, partials, nb);
  else if (at == AMG_F64 && bt == AMG_F32)
    k_dot<double, float><<<nb, kT, 0, s>>>(n, (const double*)a, (const float*)b, partials, nb);
  else if (at == AMG_F32 && bt == AMG_F64)
    k_dot<float, double><<<nb, kT, 0, s>>>(n, (const float*)a, (const double*)b, partials, nb);
  else
    k_dot<float, float><<<nb, kT, 0, s>>>(n, (const float*)a, (const float*)b, partials, nb);
  AMG_CK_LAUNCH();
  ++g_launches;
  k_finalize<<<1, kT, 0, s>>>(1, partials, nb, out, (sqrt_out && !comm) ? 1 : 0);
  AMG_CK_LAUNCH();
  finalize_global(comm, out, 1, sqrt_out, s);
}

void launch_mdot(int64_t n, int k, const PtrList& V, const double* w, double* partials, double* out, cudaStream_t s) {
  const int nb = nblocks_for(n);
  ProfScope ps_(prof_name("mdot", k, AMG_F64, -1), 8.0 * n * (k + 1), s);
  k_mdot<<<nb, kT, 0, s>>>(n, k, V, w, partials, nb);
  AMG_CK_LAUNCH();
  ++g_launches;
  k_finalize<<<1, kT, 0, s>>>(k, partials, nb, out, 0);
  AMG_CK_LAUNCH();
}

void launch_mdot_scaled(int64_t n, int k, const PtrList& V, const double* sc, const double* w, double* partials,
                        double* out, cudaStream_t s, CommBase* comm) {
  const int nb = nblocks_for(n);
  ProfScope ps_(prof_name("mdot", k, AMG_F64, -1), 8.0 * n * (k + 1), s);
  k_mdot_scaled<<<nb, kT, 0, s>>>(n, k, V, sc, w, partials, nb);
  AMG_CK_LAUNCH();
  ++g_launches;
  k_finalize<<<1, kT, 0, s>>>(k, partials, nb, out, 0);
  AMG_CK_LAUNCH();
  finalize_global(comm, out, k, false, s);
}

void launch_cgs_update(int64_t n, int k, const PtrList& V, const double* sc, const double* coef, const double* w,
                       double* w_out, bool dot_next, double* partials, double* out, cudaStream_t s, CommBase* comm) {
  const int nb = nblocks_for(n);
  ProfScope ps_(prof_name(dot_next ? "cgs_update_dot" : "cgs_update_nrm", k, AMG_F64, -1), 8.0 * n * (k + 2), s);
  if (dot_next) k_cgs_update<true><<<nb, kT, 0, s>>>(n, k, V, sc, coef, w, w_out, partials, nb);
  else k_cgs_update<false><<<nb, kT, 0, s>>>(n, k, V, sc, coef, w, w_out, partials, nb);
  AMG_CK_LAUNCH();
  ++g_launches;
  k_finalize<<<1, kT, 0, s>>>(dot_next ? k : 1, partials, nb, out, (dot_next || comm) ? 0 : 1);
  AMG_CK_LAUNCH();
  finalize_global(comm, out, dot_next ? k : 1, !dot_next, s);
}

void launch_maxpy(int64_t n, int k, const PtrList& V, const double* coef, double* w, cudaStream_t s) {
  ProfScope ps_(prof_name("maxpy", k, AMG_F64, -1), 8.0 * n * (k + 2), s);
  k_maxpy<<<ew_grid(n), kT, 0, s>>>(n, k, V, coef, w);
  AMG_CK_LAUNCH();
}

void launch_zupdate(int64_t n, int k, const PtrList& Z, int zt, const double* y, double* x, cudaStream_t s) {
  ProfScope ps_(prof_name("zupdate", k, zt, -1), (double)n * (16.0 + (double)k * dtype_size(zt)), s);
  if (zt == AMG_F32) k_zupdate<float><<<ew_grid(n), kT, 0, s>>>(n, k, Z, y, x);
  else k_zupdate<double><<<ew_grid(n), kT, 0, s>>>(n, k, Z, y, x);
  AMG_CK_LAUNCH();
}

void launch_axpby(int64_t n, double a, const double* x, double b, double* y, cudaStream_t s) {
  ProfScope ps_(prof_name("axpby", 1, AMG_F64, -1), 8.0 * n * (b == 0.0 ? 2.0 : 3.0), s);
  k_axpby<<<ew_grid(n), kT, 0, s>>>(n, a, x, b, y);
  AMG_CK_LAUNCH();
}

void launch_axpbypcz(int64_t n, double a, const double* x, double b, const double* y, double c, double* z,
                     cudaStream_t s) {
  ProfScope ps_(prof_name("axpbypcz", 1, AMG_F64, -1), 32.0 * n, s);
  k_axpbypcz<<<ew_grid(n), kT, 0, s>>>(n, a, x, b, y, c, z);
  AMG_CK_LAUNCH();
}

void launch_scale_by_inv(int64_t n, const double* x, const double* sdev, double* y, cudaStream_t s) {
  ProfScope ps_(prof_name("scale", 1, AMG_F64, -1), 16.0 * n, s);
  k_scale_by_inv<<<ew_grid(n), kT, 0, s>>>(n, x, sdev, y);
  AMG_CK_LAUNCH();
}

}  // namespace amgb
