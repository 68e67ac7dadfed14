// bsr.cuh -- shared device helpers of the SpMV-type kernels (bsr_lane.cuh, bsr_tma.cuh):
// b-element loads, the block-row dot item_dot, the fp64 -> storage rounding, and the
// K4a pre-smoother x = M f.  Layout: int32 row_ptr[n+1], int32
// col[nnzb] sorted, values [nnzb][b][b] row-major.  All arithmetic is fp64 with one
// rounding on store.
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

// Three consecutive fp32 values (a 3x3 fp32 block row, or x of one block column) in TWO
// loads instead of three: one 8-byte load at the even-aligned pair and one 4-byte load
// for the remaining value.  Every lane issues the same two instructions; only the
// addresses depend on the parity of p.
template <bool NC>
__device__ __forceinline__ void ld3f(const float* __restrict__ p, float (&v)[3]) {
  const bool even = ((reinterpret_cast<uintptr_t>(p) >> 2) & 1) == 0;
  const float2* q2 = reinterpret_cast<const float2*>(even ? p : p + 1);
  const float* q1 = even ? p + 2 : p;
  const float2 a = NC ? __ldg(q2) : __ldcs(q2);
  const float b = NC ? __ldg(q1) : __ldcs(q1);
  v[0] = even ? a.x : b;
  v[1] = even ? a.y : a.x;
  v[2] = even ? b : a.y;
}

// b values -> fp64 registers; 3 fp32 values in two loads (ld3f)
template <int B, typename T>
__device__ __forceinline__ void load_bd(const T* __restrict__ p, double (&v)[B]) {
  if constexpr (B == 3 && std::is_same_v<T, float>) {
    float f[3];
    ld3f<true>(p, f);
    v[0] = f[0]; v[1] = f[1]; v[2] = f[2];
  } else {
    load_b<B, false>(p, v);
  }
}

template <typename T>
__device__ __forceinline__ T to_out(double v) {
  return (T)v;  // fp32: round-to-nearest-even, once
}

template <int B>
__device__ __forceinline__ double pick(const double (&y)[B], int i) {
  double v = y[0];
#pragma unroll
  for (int c = 1; c < B; ++c)
    if (c == i) v = y[c];
  return v;
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
