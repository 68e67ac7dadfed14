// bsr.cuh -- block-row machinery of every SpMV-type kernel (K1, K2, K4-K7, K10, K11).
//
// Layout: int32 row_ptr[n+1], int32 col[nnzb] sorted, values
// [nnzb][b][b] row-major.  A group of G lanes (G = 8 or 32, a power of two) owns
// one block row.  The row's work is enumerated as items t = (block k, block row r)
// in storage order, so the G lanes of a group read G consecutive b-value segments
// of the value stream: every warp load is contiguous (coalesced) and whole
// sectors are used.  Each lane multiplies its b values with the b entries of x
// at the block's column (the b lanes of one block hit the same x segment: one
// L1 broadcast), accumulating in fp64.  A butterfly inside the group produces the
// b-vector (A x)_I, which the kernel's epilogue consumes.  All arithmetic is fp64
// with one rounding on store.
#pragma once

#include "common.cuh"

namespace amgb {

// ---- b contiguous elements -> fp64 registers (128-bit loads where alignment allows) ----
template <int B, bool STREAM, typename T>
__device__ __forceinline__ void load_b(const T* __restrict__ p, double (&v)[B]) {
  if constexpr (B == 4 && std::is_same_v<T, float>) {
    float4 q = STREAM ? __ldcs(reinterpret_cast<const float4*>(p)) : __ldg(reinterpret_cast<const float4*>(p));
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else if constexpr (B == 4 && std::is_same_v<T, double>) {
    const double2* q = reinterpret_cast<const double2*>(p);
    double2 a = STREAM ? __ldcs(q) : __ldg(q);
    double2 c = STREAM ? __ldcs(q + 1) : __ldg(q + 1);
    v[0] = a.x; v[1] = a.y; v[2] = c.x; v[3] = c.y;
  } else if constexpr (B == 2 && std::is_same_v<T, float>) {
    float2 q = STREAM ? __ldcs(reinterpret_cast<const float2*>(p)) : __ldg(reinterpret_cast<const float2*>(p));
    v[0] = q.x; v[1] = q.y;
  } else if constexpr (B == 2 && std::is_same_v<T, double>) {
    double2 q = STREAM ? __ldcs(reinterpret_cast<const double2*>(p)) : __ldg(reinterpret_cast<const double2*>(p));
    v[0] = q.x; v[1] = q.y;
  } else {
#pragma unroll
    for (int c = 0; c < B; ++c) v[c] = (double)(STREAM ? __ldcs(p + c) : __ldg(p + c));
  }
}

// b contiguous elements in their storage type (keeps fp32 values at 1 register each)
template <int B, bool STREAM, typename T>
__device__ __forceinline__ void load_raw(const T* __restrict__ p, T (&v)[B]) {
  if constexpr (B == 4 && std::is_same_v<T, float>) {
    float4 q = STREAM ? __ldcs(reinterpret_cast<const float4*>(p)) : __ldg(reinterpret_cast<const float4*>(p));
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else if constexpr (B == 4 && std::is_same_v<T, double>) {
    const double2* q = reinterpret_cast<const double2*>(p);
    double2 a = STREAM ? __ldcs(q) : __ldg(q);
    double2 c = STREAM ? __ldcs(q + 1) : __ldg(q + 1);
    v[0] = a.x; v[1] = a.y; v[2] = c.x; v[3] = c.y;
  } else if constexpr (B == 2 && std::is_same_v<T, float>) {
    float2 q = STREAM ? __ldcs(reinterpret_cast<const float2*>(p)) : __ldg(reinterpret_cast<const float2*>(p));
    v[0] = q.x; v[1] = q.y;
  } else if constexpr (B == 2 && std::is_same_v<T, double>) {
    double2 q = STREAM ? __ldcs(reinterpret_cast<const double2*>(p)) : __ldg(reinterpret_cast<const double2*>(p));
    v[0] = q.x; v[1] = q.y;
  } else {
#pragma unroll
    for (int c = 0; c < B; ++c) v[c] = STREAM ? __ldcs(p + c) : __ldg(p + c);
  }
}

// One block-row item: sum_c a[c] x[c], in fp64 (fp32 x fp32 products are exact there).
// FAST (internal V-cycle on the fp32 hierarchy only, Listing V4's float backend,
// PAPER.md:703-704): the b-term chain in fp32 FMA, converted once; the row sum over
// items is still accumulated in fp64 by the caller.
template <int B, typename V, typename X, bool FAST = false>
__device__ __forceinline__ double item_dot(const V (&a)[B], const X (&x)[B]) {
  if constexpr (FAST && std::is_same_v<V, float> && std::is_same_v<X, float>) {
    float s = a[0] * x[0];
#pragma unroll
    for (int c = 1; c < B; ++c) s = fmaf(a[c], x[c], s);
    return (double)s;
  } else {
    double s = (double)a[0] * (double)x[0];
#pragma unroll
    for (int c = 1; c < B; ++c) s = fma((double)a[c], (double)x[c], s);
    return s;
  }
}

template <typename T>
__device__ __forceinline__ T to_out(double v) {
  return (T)v;  // fp32: round-to-nearest-even, once
}

// Partial (A x) of block row `row` for lane gl of its group: one (block, block-row)
// item per lane per iteration, items in storage order.  If G % B == 0 the lane always
// handles block row r = gl % B and accumulates into acc[0]; otherwise acc[r].
template <int B, int G, typename V, typename X>
__device__ __forceinline__ void row_partial(const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                                                   const V* __restrict__ val, const X* __restrict__ x, int row,
                                                   int gl, double (&acc)[B]) {
  const int k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
  const int nitems = (k1 - k0) * B;
#pragma unroll 2
  for (int t = gl; t < nitems; t += G) {
    const int kb = k0 + t / B;
    const int r = (G % B == 0) ? (gl % B) : (t % B);
    const int c = __ldg(col + kb);
    V a[B];
    X xv[B];
    load_raw<B, true>(val + ((int64_t)kb * B + r) * B, a);
    load_raw<B, false>(x + (int64_t)c * B, xv);
    const double s = item_dot<B, V, X>(a, xv);
    if constexpr (G % B == 0) {
      acc[0] += s;
    } else {
#pragma unroll
      for (int rr = 0; rr < B; ++rr)
        if (rr == r) acc[rr] += s;
    }
  }
}

// Group reduction: every lane of the group receives the full b-vector y = (A x)_row.
template <int B, int G>
__device__ __forceinline__ void group_reduce(double (&acc)[B], double (&y)[B]) {
  if constexpr (G % B == 0) {
    double v = acc[0];
#pragma unroll
    for (int off = G / 2; off >= B; off >>= 1) v += __shfl_xor_sync(kFull, v, off, G);
#pragma unroll
    for (int c = 0; c < B; ++c) y[c] = __shfl_sync(kFull, v, c, G);
  } else {
#pragma unroll
    for (int c = 0; c < B; ++c) {
      double v = acc[c];
#pragma unroll
      for (int off = G / 2; off >= 1; off >>= 1) v += __shfl_xor_sync(kFull, v, off, G);
      y[c] = v;
    }
  }
}

template <int B>
__device__ __forceinline__ double pick(const double (&y)[B], int i) {
  double v = y[0];
#pragma unroll
  for (int c = 1; c < B; ++c)
    if (c == i) v = y[c];
  return v;
}

// ---- K1: y = alpha A x + beta y (beta == 0 overwrites) ----
template <int B, int G, typename V, typename X, typename Y>
__global__ void __launch_bounds__(256) k_spmv(int n, const int32_t* __restrict__ ptr,
                                              const int32_t* __restrict__ col, const V* __restrict__ val,
                                              double alpha, const X* __restrict__ x, double beta,
                                              Y* __restrict__ y) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gid / G), gl = threadIdx.x & (G - 1);
  const bool valid = row < n;
  double acc[B] = {};
  if (valid) row_partial<B, G>(ptr, col, val, x, row, gl, acc);
  double yv[B];
  group_reduce<B, G>(acc, yv);
  if (valid && gl < B) {
    const int64_t o = (int64_t)row * B + gl;
    double v = alpha * pick<B>(yv, gl);
    if (beta != 0.0) v = fma(beta, (double)y[o], v);
    y[o] = to_out<Y>(v);
  }
}

// ---- K2: r = f - A x ----
template <int B, int G, typename V, typename X>
__global__ void __launch_bounds__(256) k_residual(int n, const int32_t* __restrict__ ptr,
                                                  const int32_t* __restrict__ col, const V* __restrict__ val,
                                                  const X* __restrict__ f, const X* __restrict__ x,
                                                  X* __restrict__ r) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gid / G), gl = threadIdx.x & (G - 1);
  const bool valid = row < n;
  double acc[B] = {};
  if (valid) row_partial<B, G>(ptr, col, val, x, row, gl, acc);
  double yv[B];
  group_reduce<B, G>(acc, yv);
  if (valid && gl < B) {
    const int64_t o = (int64_t)row * B + gl;
    r[o] = to_out<X>((double)f[o] - pick<B>(yv, gl));
  }
}

// ---- K5: post-smooth xo = x + M (f - A x), every row from the old x (Jacobi-type) ----
template <int B, int G, typename V, typename X>
__global__ void __launch_bounds__(256) k_smooth(int n, const int32_t* __restrict__ ptr,
                                                const int32_t* __restrict__ col, const V* __restrict__ val,
                                                const V* __restrict__ M, const X* __restrict__ f,
                                                const X* __restrict__ x, X* __restrict__ xo) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gid / G), gl = threadIdx.x & (G - 1);
  const bool valid = row < n;
  double acc[B] = {};
  if (valid) row_partial<B, G>(ptr, col, val, x, row, gl, acc);
  double yv[B];
  group_reduce<B, G>(acc, yv);
  if (valid && gl < B) {
    const int64_t o = (int64_t)row * B;
    double res[B];
#pragma unroll
    for (int c = 0; c < B; ++c) res[c] = (double)f[o + c] - yv[c];
    double m[B];
    load_b<B, false>(M + ((int64_t)row * B + gl) * B, m);
    double t = m[0] * res[0];
#pragma unroll
    for (int c = 1; c < B; ++c) t = fma(m[c], res[c], t);
    xo[o + gl] = to_out<X>((double)x[o + gl] + t);
  }
}

// ---- K4 (first half): x = M f (pre-smoothing from a zero initial guess) ----
template <int B, typename V, typename X>
__global__ void __launch_bounds__(256) k_apply_M(int n, const V* __restrict__ M, const X* __restrict__ f,
                                                 X* __restrict__ x) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * B) return;
  const int64_t row = t / B;
  const int r = (int)(t % B);
  double m[B], fv[B];
  load_b<B, false>(M + (row * B + r) * B, m);
  load_b<B, false>(f + row * B, fv);
  double s = m[0] * fv[0];
#pragma unroll
  for (int c = 1; c < B; ++c) s = fma(m[c], fv[c], s);
  x[t] = to_out<X>(s);
}

}  // namespace amgb
