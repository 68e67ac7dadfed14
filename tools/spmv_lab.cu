// spmv_lab.cu -- standalone kernel-design lab for long-row BSR SpMV (cfg 2 27-point and
// coarse-level shapes).  Not part of the library: builds a synthetic pattern on the GPU,
// times candidate kernels with CUDA events and checks them against a plain reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/lab tools/spmv_lab.cu
//   /tmp/lab <n> <b> <stencil 7|27> <vt 0=f64,1=f32> <xt>
#include <cuda_runtime.h>

#include "bsr_lane.cuh"

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);        \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

__host__ __device__ inline uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ inline double u11(uint64_t i) { return ((mix(i) >> 11) * 0x1.0p-53) * 2.0 - 1.0; }

__global__ void k_rowlen(int n, int st, int* len) {
  int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (I >= (int64_t)n * n * n) return;
  int i = I % n, j = (I / n) % n, k = I / ((int64_t)n * n);
  int c = 0;
  if (st == 27) {
    for (int dk = -1; dk <= 1; ++dk)
      for (int dj = -1; dj <= 1; ++dj)
        for (int di = -1; di <= 1; ++di)
          c += (i + di >= 0 && i + di < n && j + dj >= 0 && j + dj < n && k + dk >= 0 && k + dk < n);
  } else {
    c = 1 + (i > 0) + (i < n - 1) + (j > 0) + (j < n - 1) + (k > 0) + (k < n - 1);
  }
  len[I] = c;
}
template <typename V>
__global__ void k_fill(int n, int st, int b, const int* ptr, int* col, V* val) {
  int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (I >= (int64_t)n * n * n) return;
  int i = I % n, j = (I / n) % n, k = I / ((int64_t)n * n);
  int64_t e = ptr[I];
  for (int dk = -1; dk <= 1; ++dk)
    for (int dj = -1; dj <= 1; ++dj)
      for (int di = -1; di <= 1; ++di) {
        if (st == 7 && (abs(di) + abs(dj) + abs(dk)) > 1) continue;
        if (!(i + di >= 0 && i + di < n && j + dj >= 0 && j + dj < n && k + dk >= 0 && k + dk < n)) continue;
        int64_t J = (i + di) + n * ((j + dj) + (int64_t)n * (k + dk));
        col[e] = (int)J;
        for (int q = 0; q < b * b; ++q) val[e * b * b + q] = (V)(u11(e * 16 + q) + ((J == I && q % (b + 1) == 0) ? 30.0 : 0.0));
        ++e;
      }
}

// reference: thread per row, fp64
template <int B, typename V, typename X>
__global__ void k_ref(int n, const int* ptr, const int* col, const V* val, const X* x, double* y) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  double acc[B] = {};
  for (int k = ptr[I]; k < ptr[I + 1]; ++k)
    for (int r = 0; r < B; ++r)
      for (int c = 0; c < B; ++c) acc[r] += (double)val[(int64_t)k * B * B + r * B + c] * (double)x[(int64_t)col[k] * B + c];
  for (int r = 0; r < B; ++r) y[(int64_t)I * B + r] = acc[r];
}

template <int B, typename T>
__device__ __forceinline__ void ldx(const T* p, T (&v)[B]) {
  if constexpr (B == 4 && sizeof(T) == 8) {
    double2 a = __ldg(reinterpret_cast<const double2*>(p)), c = __ldg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = c.x; v[3] = c.y;
  } else if constexpr (B == 4 && sizeof(T) == 4) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  } else {
#pragma unroll
    for (int c = 0; c < B; ++c) v[c] = __ldg(p + c);
  }
}
__device__ int g_nc;  // unused
template <int B, typename T>
__device__ __forceinline__ void ldv_nc(const T* p, T (&v)[B]) {  // L1-allocating
#pragma unroll
  for (int c = 0; c < B; ++c) v[c] = __ldg(p + c);
}
template <int B, typename T>
__device__ __forceinline__ void ldv(const T* p, T (&v)[B]) {  // streaming
  if constexpr (B == 4 && sizeof(T) == 4) {
    float4 a = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  } else if constexpr (B == 4 && sizeof(T) == 8) {
    double2 a = __ldcs(reinterpret_cast<const double2*>(p)), c = __ldcs(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = c.x; v[3] = c.y;
  } else {
#pragma unroll
    for (int c = 0; c < B; ++c) v[c] = __ldcs(p + c);
  }
}

// A: 4 lanes per row, lane r < B owns y[row][r]; U blocks per iteration, loads first
template <int B, int U, typename V, typename X>
__global__ void __launch_bounds__(256) k_lane_r(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                                const V* __restrict__ val, const X* __restrict__ x, double* __restrict__ y) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int row = (int)(gid >> 2), r = (int)(gid & 3);
  if (row >= n) return;
  const int k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
  const int rr = r < B ? r : B - 1;
  double acc = 0.0;
  int k = k0;
  for (; k + U <= k1; k += U) {
    int c[U];
    V a[U][B];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = __ldg(col + k + u);
      ldv<B>(val + ((int64_t)(k + u) * B + rr) * B, a[u]);
    }
    X xv[U][B];
#pragma unroll
    for (int u = 0; u < U; ++u) ldx<B>(x + (int64_t)c[u] * B, xv[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < B; ++q) acc = fma((double)a[u][q], (double)xv[u][q], acc);
  }
  for (; k < k1; ++k) {
    V a[B];
    X xv[B];
    ldv<B>(val + ((int64_t)k * B + rr) * B, a);
    ldx<B>(x + (int64_t)__ldg(col + k) * B, xv);
#pragma unroll
    for (int q = 0; q < B; ++q) acc = fma((double)a[q], (double)xv[q], acc);
  }
  if (r < B) y[(int64_t)row * B + r] = acc;
}

// B: warp per row, (block,row) items, 32 lanes; loads first, unroll U passes
template <int B, int U, typename V, typename X>
__global__ void __launch_bounds__(256) k_warp(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                              const V* __restrict__ val, const X* __restrict__ x, double* __restrict__ y) {
  static_assert(32 % B == 0, "B | 32");
  constexpr int BPP = 32 / B;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int row = (int)(gid >> 5), lane = threadIdx.x & 31, r = lane % B;
  if (row >= n) return;
  const int k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
  double acc = 0.0;
  for (int kb = k0 + lane / B; kb < k1; kb += BPP * U) {
    int c[U];
    V a[U][B];
    X xv[U][B];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = kb + u * BPP;
      c[u] = k < k1 ? __ldg(col + k) : -1;
      if (k < k1) ldv<B>(val + ((int64_t)k * B + r) * B, a[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c[u] >= 0) ldx<B>(x + (int64_t)c[u] * B, xv[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c[u] >= 0)
#pragma unroll
        for (int q = 0; q < B; ++q) acc = fma((double)a[u][q], (double)xv[u][q], acc);
  }
#pragma unroll
  for (int off = 16; off >= B; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane < B) y[(int64_t)row * B + lane] = acc;
}

// C: B lanes per row (32/B rows per warp, 32 % B lanes idle), lane r owns y[row][r]
template <int B, int U, typename V, typename X>
__global__ void __launch_bounds__(256) k_lane_b(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                                const V* __restrict__ val, const X* __restrict__ x, double* __restrict__ y) {
  constexpr int RPW = 32 / B;
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  const int row = warp * RPW + lane / B, r = lane % B;
  if (lane >= RPW * B || row >= n) return;
  const int k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
  double acc = 0.0;
  int k = k0;
  for (; k + U <= k1; k += U) {
    int c[U];
    V a[U][B];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = __ldg(col + k + u);
      ldv<B>(val + ((int64_t)(k + u) * B + r) * B, a[u]);
    }
    X xv[U][B];
#pragma unroll
    for (int u = 0; u < U; ++u) ldx<B>(x + (int64_t)c[u] * B, xv[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < B; ++q) acc = fma((double)a[u][q], (double)xv[u][q], acc);
  }
  for (; k < k1; ++k) {
    V a[B];
    X xv[B];
    ldv<B>(val + ((int64_t)k * B + r) * B, a);
    ldx<B>(x + (int64_t)__ldg(col + k) * B, xv);
#pragma unroll
    for (int q = 0; q < B; ++q) acc = fma((double)a[q], (double)xv[q], acc);
  }
  y[(int64_t)row * B + r] = acc;
}

// C2: as C with L1-allocating value loads (3x3 fp32: the lanes' 12-B pieces share sectors)
template <int B, int U, typename V, typename X>
__global__ void __launch_bounds__(256) k_lane_bnc(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                                  const V* __restrict__ val, const X* __restrict__ x, double* __restrict__ y) {
  constexpr int RPW = 32 / B;
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  const int row = warp * RPW + lane / B, r = lane % B;
  if (lane >= RPW * B || row >= n) return;
  const int k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
  double acc = 0.0;
  int k = k0;
  for (; k + U <= k1; k += U) {
    int c[U];
    V a[U][B];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = __ldg(col + k + u);
      ldv_nc<B>(val + ((int64_t)(k + u) * B + r) * B, a[u]);
    }
    X xv[U][B];
#pragma unroll
    for (int u = 0; u < U; ++u) ldx<B>(x + (int64_t)c[u] * B, xv[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < B; ++q) acc = fma((double)a[u][q], (double)xv[u][q], acc);
  }
  for (; k < k1; ++k) {
    V a[B];
    X xv[B];
    ldv_nc<B>(val + ((int64_t)k * B + r) * B, a);
    ldx<B>(x + (int64_t)__ldg(col + k) * B, xv);
#pragma unroll
    for (int q = 0; q < B; ++q) acc = fma((double)a[q], (double)xv[q], acc);
  }
  y[(int64_t)row * B + r] = acc;
}

// E: B lanes per row, lane r holds COLUMN r of each block (coalesced 9-word block reads
// across the row's lanes) and x[col][r]; per-row transpose-reduce among the B lanes
template <int B, int U, typename V, typename X, bool NC>
__global__ void __launch_bounds__(256) k_lane_col(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                                  const V* __restrict__ val, const X* __restrict__ x, double* __restrict__ y) {
  constexpr int RPW = 32 / B;
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  const int g = lane / B, r = lane % B;
  const int row = warp * RPW + g;
  const bool valid = lane < RPW * B && row < n;
  int k0 = 0, k1 = 0;
  if (valid) k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
  double acc[B] = {};
  int k = k0;
  for (; k + U <= k1; k += U) {
    int c[U];
    V a[U][B];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = __ldg(col + k + u);
#pragma unroll
      for (int i = 0; i < B; ++i) a[u][i] = NC ? __ldg(val + (int64_t)(k + u) * B * B + i * B + r) : __ldcs(val + (int64_t)(k + u) * B * B + i * B + r);
    }
    X xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = __ldg(x + (int64_t)c[u] * B + r);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < B; ++i) acc[i] = fma((double)a[u][i], (double)xv[u], acc[i]);
  }
  for (; k < k1; ++k) {
    const int c = __ldg(col + k);
    const X xv = __ldg(x + (int64_t)c * B + r);
#pragma unroll
    for (int i = 0; i < B; ++i) acc[i] = fma((double)(NC ? __ldg(val + (int64_t)k * B * B + i * B + r) : __ldcs(val + (int64_t)k * B * B + i * B + r)), (double)xv, acc[i]);
  }
  // y[r] = sum over the row's lanes l of acc_l[r]
  const int base = lane - r;
  double s = acc[0];
#pragma unroll
  for (int i = 1; i < B; ++i)
    if (i == r) s = acc[i];
#pragma unroll
  for (int d = 1; d < B; ++d) {
    const int want = (r + B - d) % B;  // the entry my receiver (lane base + want) needs... sender view
    double v = acc[0];
#pragma unroll
    for (int i = 1; i < B; ++i)
      if (i == want) v = acc[i];
    const int src = base + (r + d) % B;
    s += __shfl_sync(0xffffffffu, v, src < 32 ? src : lane);
  }
  if (valid) y[(int64_t)row * B + r] = s;
}

// G: B lanes per row, whole short row (<= UMAX blocks) loaded in ONE round: predicated
// col/value loads, then predicated x gathers; MINB = min blocks/SM for the register budget
template <int B, int UMAX, int MINB, typename V, typename X>
__global__ void __launch_bounds__(256, MINB) k_lane_pre(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                                   const V* __restrict__ val, const X* __restrict__ x, double* __restrict__ y) {
  constexpr int RPW = 32 / B;
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  const int row = warp * RPW + lane / B, r = lane % B;
  if (lane >= RPW * B || row >= n) return;
  const int k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
  double acc = 0.0;
  for (int k = k0; k < k1; k += UMAX) {
    int c[UMAX];
    V a[UMAX][B];
#pragma unroll
    for (int u = 0; u < UMAX; ++u) {
      const bool ok = k + u < k1;
      c[u] = ok ? __ldg(col + k + u) : 0;
#pragma unroll
      for (int q = 0; q < B; ++q) a[u][q] = ok ? __ldg(val + ((int64_t)(k + u) * B + r) * B + q) : V(0);
    }
    X xv[UMAX][B];
#pragma unroll
    for (int u = 0; u < UMAX; ++u)
#pragma unroll
      for (int q = 0; q < B; ++q) xv[u][q] = (k + u < k1) ? __ldg(x + (int64_t)c[u] * B + q) : X(0);
#pragma unroll
    for (int u = 0; u < UMAX; ++u) {
      float s2 = 0.f;
#pragma unroll
      for (int q = 0; q < B; ++q) s2 = fmaf((float)a[u][q], (float)xv[u][q], s2);
      acc += (double)s2;
    }
  }
  y[(int64_t)row * B + r] = acc;
}

// D: lane_r with the col/val loads of the next U-chunk issued before the current chunk's
// x gathers are consumed (software pipelined)
template <int B, int U, typename V, typename X>
__global__ void __launch_bounds__(256) k_lane_p(int n, const int* __restrict__ ptr, const int* __restrict__ col,
                                                const V* __restrict__ val, const X* __restrict__ x, double* __restrict__ y) {
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int row = (int)(gid >> 2), r = (int)(gid & 3);
  if (row >= n) return;
  const int k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
  const int rr = r < B ? r : B - 1;
  double acc = 0.0;
  int c[U];
  V a[U][B];
  auto ld = [&](int k) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = k + u < k1;
      c[u] = ok ? __ldg(col + k + u) : -1;
      if (ok) ldv<B>(val + ((int64_t)(k + u) * B + rr) * B, a[u]);
    }
  };
  ld(k0);
  for (int k = k0; k < k1; k += U) {
    X xv[U][B];
    V ac[U][B];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (c[u] >= 0) ldx<B>(x + (int64_t)c[u] * B, xv[u]);
#pragma unroll
      for (int q = 0; q < B; ++q) ac[u][q] = a[u][q];
    }
    int cc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cc[u] = c[u];
    ld(k + U);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (cc[u] >= 0)
#pragma unroll
        for (int q = 0; q < B; ++q) acc = fma((double)ac[u][q], (double)xv[u][q], acc);
  }
  if (r < B) y[(int64_t)row * B + r] = acc;
}

// F: sliced BSR (SELL-C, C = 32/B rows per warp) + COLS: step j of slice s holds
// [i][g][r] = A_{row g, block j}[i][r] (i < B block rows, g < C rows, r < B columns):
// every value load of a warp is 4 * C * B contiguous bytes.  scol[s][j][g].
template <int B, int U, typename V, typename X>
__global__ void __launch_bounds__(256) k_sell_col(int n, int nslices, const int* __restrict__ sptr /*[nslices+1] steps offset*/,
                                                  const int* __restrict__ scol, const V* __restrict__ sval,
                                                  const X* __restrict__ x, double* __restrict__ y) {
  constexpr int C = 32 / B;
  const int lane = threadIdx.x & 31;
  const int s = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (s >= nslices) return;
  const int g = lane / B, r = lane - g * B;
  const bool act = g < C;
  const int j0 = __ldg(sptr + s), j1 = __ldg(sptr + s + 1);
  double acc[B] = {};
  const int L = act ? lane : 0;
  int j = j0;
#pragma unroll 1
  for (; j + U <= j1; j += U) {
    int c[U];
    V a[U][B];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = __ldg(scol + (int64_t)(j + u) * C + (act ? g : 0));
#pragma unroll
      for (int i = 0; i < B; ++i) a[u][i] = __ldcs(sval + ((int64_t)(j + u) * B + i) * (C * B) + L);
    }
    X xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = __ldg(x + (int64_t)c[u] * B + r);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < B; ++i) acc[i] = fma((double)a[u][i], (double)xv[u], acc[i]);
  }
#pragma unroll 1
  for (; j < j1; ++j) {
    const int c = __ldg(scol + (int64_t)j * C + (act ? g : 0));
    const X xv = __ldg(x + (int64_t)c * B + r);
#pragma unroll
    for (int i = 0; i < B; ++i) acc[i] = fma((double)__ldcs(sval + ((int64_t)j * B + i) * (C * B) + L), (double)xv, acc[i]);
  }
  const int base = lane - r;
  double sum = acc[0];
#pragma unroll
  for (int i = 1; i < B; ++i)
    if (i == r) sum = acc[i];
#pragma unroll
  for (int d = 1; d < B; ++d) {
    const int want = (r + B - d) % B;
    double v = acc[0];
#pragma unroll
    for (int i = 1; i < B; ++i)
      if (i == want) v = acc[i];
    sum += __shfl_sync(0xffffffffu, v, base + (r + d) % B);
  }
  const int row = s * C + g;
  if (act && row < n) y[(int64_t)row * B + r] = sum;
}

// H: sliced copy with ROW layout: step j of slice s stores the C blocks [g][B][B] row-major
// (the BSR blocks of the slice's rows, contiguous); lane (g, r) reads row r of its block with
// the two-load triple (fp32 B = 3) and x_col with the same trick
template <int B, int U, typename V, typename X>
__global__ void __launch_bounds__(256) k_sell_rows(int n, int nslices, const int* __restrict__ sptr,
                                                   const int* __restrict__ scol, const V* __restrict__ sval,
                                                   const X* __restrict__ x, double* __restrict__ y) {
  constexpr int C = 32 / B;
  const int lane = threadIdx.x & 31;
  const int s = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (s >= nslices) return;
  const int g = lane / B, r = lane - g * B;
  const bool act = g < C;
  const int gg = act ? g : 0;
  const int j0 = __ldg(sptr + s), j1 = __ldg(sptr + s + 1);
  double acc = 0.0;
  int j = j0;
#pragma unroll 1
  for (; j + U <= j1; j += U) {
    int c[U];
    V a[U][B];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = __ldg(scol + (int64_t)(j + u) * C + gg);
      amgb::ld_row<B, false>(sval + ((int64_t)(j + u) * C + gg) * B * B + r * B, a[u]);
    }
    X xv[U][B];
#pragma unroll
    for (int u = 0; u < U; ++u) amgb::ld_x<B>(x + (int64_t)c[u] * B, xv[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float s2 = 0.f;
#pragma unroll
      for (int q = 0; q < B; ++q) s2 = fmaf((float)a[u][q], (float)xv[u][q], s2);
      acc += (double)s2;
    }
  }
#pragma unroll 1
  for (; j < j1; ++j) {
    const int c = __ldg(scol + (int64_t)j * C + gg);
    V a[B];
    X xv[B];
    amgb::ld_row<B, false>(sval + ((int64_t)j * C + gg) * B * B + r * B, a);
    amgb::ld_x<B>(x + (int64_t)c * B, xv);
    float s2 = 0.f;
#pragma unroll
    for (int q = 0; q < B; ++q) s2 = fmaf((float)a[q], (float)xv[q], s2);
    acc += (double)s2;
  }
  const int row = s * C + g;
  if (act && row < n) y[(int64_t)row * B + r] = acc;
}

template <class F>
float timeit(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  std::vector<float> t;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    t.push_back(ms);
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

template <int B, typename V, typename X>
void run(int n, int st) {
  const int64_t N = (int64_t)n * n * n;
  int *len, *ptr, *col;
  CK(cudaMalloc(&len, N * 4));
  CK(cudaMalloc(&ptr, (N + 1) * 4));
  k_rowlen<<<(N + 255) / 256, 256>>>(n, st, len);
  std::vector<int> hl(N), hp(N + 1, 0);
  CK(cudaMemcpy(hl.data(), len, N * 4, cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < N; ++i) hp[i + 1] = hp[i] + hl[i];
  const int64_t Z = hp[N];
  CK(cudaMemcpy(ptr, hp.data(), (N + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&col, Z * 4));
  V* val;
  CK(cudaMalloc(&val, Z * B * B * sizeof(V)));
  k_fill<V><<<(N + 255) / 256, 256>>>(n, st, B, ptr, col, val);
  X* x;
  CK(cudaMalloc(&x, N * B * sizeof(X)));
  std::vector<X> hx(N * B);
  for (int64_t i = 0; i < N * B; ++i) hx[i] = (X)(((mix(i + 777) >> 11) * 0x1.0p-53) * 2 - 1);
  CK(cudaMemcpy(x, hx.data(), N * B * sizeof(X), cudaMemcpyHostToDevice));
  double *y0, *y1;
  CK(cudaMalloc(&y0, N * B * 8));
  CK(cudaMalloc(&y1, N * B * 8));
  CK(cudaDeviceSynchronize());
  const double bytes = 4.0 * (N + 1) + Z * (4.0 + B * B * sizeof(V)) + N * B * sizeof(X) + N * B * 8.0;
  printf("n=%d st=%d B=%d V=%zu X=%zu: rows %lld blocks %lld (%.2f/row), alg %.3f GB\n", n, st, B, sizeof(V), sizeof(X),
         (long long)N, (long long)Z, (double)Z / N, bytes / 1e9);
  auto check = [&](const char* name, float ms) {
    std::vector<double> a(N * B), b(N * B);
    CK(cudaMemcpy(a.data(), y0, N * B * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), y1, N * B * 8, cudaMemcpyDeviceToHost));
    double num = 0, den = 0;
    for (int64_t i = 0; i < N * B; ++i) num += (a[i] - b[i]) * (a[i] - b[i]), den += a[i] * a[i];
    printf("  %-24s %8.3f ms  %7.0f GB/s  relerr %.1e\n", name, ms, bytes / ms / 1e6, sqrt(num / den));
  };
  float t = timeit([&] { k_ref<B, V, X><<<(N + 255) / 256, 256>>>(N, ptr, col, val, x, y0); }, 10);
  check("ref (thread/row)", t);
#define LANE(U)                                                                                          \
  t = timeit([&] { k_lane_r<B, U, V, X><<<(N * 4 + 255) / 256, 256>>>(N, ptr, col, val, x, y1); }, 20); \
  check("lane_r U=" #U, t);
  LANE(2) LANE(8)
#define LANEB(U)                                                                                              \
  t = timeit([&] { k_lane_b<B, U, V, X><<<((N + 32 / B - 1) / (32 / B) * 32 + 255) / 256, 256>>>(N, ptr, col, val, x, y1); }, 20); \
  check("lane_b U=" #U, t);
  LANEB(2) LANEB(4) LANEB(8)
  {
    amgb::LEpiSpmv<double> e{1.0, 0.0, y1};
    t = timeit([&] { amgb::k_bsr_lane<B, B, 4, false, false, V, X, false, amgb::LEpiSpmv<double>><<<((N + 32 / B - 1) / (32 / B) * 32 + 255) / 256, 256>>>(N, ptr, col, val, x, e); }, 20);
    check("lib lane RC4", t);
    t = timeit([&] { amgb::k_bsr_lane<B, B, 2, false, false, V, X, false, amgb::LEpiSpmv<double>><<<((N + 32 / B - 1) / (32 / B) * 32 + 255) / 256, 256>>>(N, ptr, col, val, x, e); }, 20);
    check("lib lane RC2", t);
  }
  {
    constexpr int C = 32 / B;
    const int64_t ns = (N + C - 1) / C;
    std::vector<int> hcol(Z);
    CK(cudaMemcpy(hcol.data(), col, Z * 4, cudaMemcpyDeviceToHost));
    std::vector<V> hval((size_t)Z * B * B);
    CK(cudaMemcpy(hval.data(), val, (size_t)Z * B * B * sizeof(V), cudaMemcpyDeviceToHost));
    std::vector<int> sp(ns + 1, 0);
    for (int64_t s2 = 0; s2 < ns; ++s2) {
      int mx = 0;
      for (int g = 0; g < C && s2 * C + g < N; ++g) mx = std::max(mx, hp[s2 * C + g + 1] - hp[s2 * C + g]);
      sp[s2 + 1] = sp[s2] + mx;
    }
    const int64_t steps = sp[ns];
    std::vector<int> sc((size_t)steps * C, 0);
    std::vector<V> sv((size_t)steps * B * C * B, V(0));
    for (int64_t s2 = 0; s2 < ns; ++s2)
      for (int g = 0; g < C; ++g) {
        const int64_t row = s2 * C + g;
        const int len = row < N ? hp[row + 1] - hp[row] : 0;
        for (int j = 0; j < sp[s2 + 1] - sp[s2]; ++j) {
          const int64_t st = sp[s2] + j;
          if (j < len) {
            const int64_t k = hp[row] + j;
            sc[st * C + g] = hcol[k];
            for (int i = 0; i < B; ++i)
              for (int r = 0; r < B; ++r) sv[(st * B + i) * (C * B) + g * B + r] = hval[k * B * B + i * B + r];
          } else {
            sc[st * C + g] = row < N ? (int)row : 0;
          }
        }
      }
    int *dsp, *dsc;
    V* dsv;
    CK(cudaMalloc(&dsp, (ns + 1) * 4));
    CK(cudaMalloc(&dsc, steps * C * 4));
    CK(cudaMalloc(&dsv, steps * B * C * B * sizeof(V)));
    CK(cudaMemcpy(dsp, sp.data(), (ns + 1) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dsc, sc.data(), steps * C * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dsv, sv.data(), steps * B * C * B * sizeof(V), cudaMemcpyHostToDevice));
    printf("  SELL: %lld steps, padding %.1f%%\n", (long long)steps, 100.0 * ((double)steps * C / Z - 1.0));
    t = timeit([&] { k_sell_col<B, 2, V, X><<<(ns * 32 + 255) / 256, 256>>>(N, ns, dsp, dsc, dsv, x, y1); }, 20);
    check("sell_col U=2", t);
    t = timeit([&] { k_sell_col<B, 4, V, X><<<(ns * 32 + 255) / 256, 256>>>(N, ns, dsp, dsc, dsv, x, y1); }, 20);
    check("sell_col U=4", t);
    t = timeit([&] { k_sell_col<B, 7, V, X><<<(ns * 32 + 255) / 256, 256>>>(N, ns, dsp, dsc, dsv, x, y1); }, 20);
    check("sell_col U=7", t);
    t = timeit([&] { k_sell_col<B, 8, V, X><<<(ns * 32 + 255) / 256, 256>>>(N, ns, dsp, dsc, dsv, x, y1); }, 20);
    check("sell_col U=8", t);
    // row-layout slice steps: [step][g][B][B]
    std::vector<V> sv2((size_t)steps * C * B * B, V(0));
    for (int64_t s2 = 0; s2 < ns; ++s2)
      for (int g = 0; g < C; ++g) {
        const int64_t row = s2 * C + g;
        const int len = row < N ? hp[row + 1] - hp[row] : 0;
        for (int j = 0; j < sp[s2 + 1] - sp[s2] && j < len; ++j) {
          const int64_t st = sp[s2] + j, k = hp[row] + j;
          for (int q = 0; q < B * B; ++q) sv2[(st * C + g) * B * B + q] = hval[k * B * B + q];
        }
      }
    CK(cudaMemcpy(dsv, sv2.data(), steps * B * C * B * sizeof(V), cudaMemcpyHostToDevice));
    if constexpr (sizeof(V) == 4 && sizeof(X) == 4) {
      t = timeit([&] { k_sell_rows<B, 2, V, X><<<(ns * 32 + 255) / 256, 256>>>(N, ns, dsp, dsc, dsv, x, y1); }, 20);
      check("sell_rows U=2", t);
      t = timeit([&] { k_sell_rows<B, 4, V, X><<<(ns * 32 + 255) / 256, 256>>>(N, ns, dsp, dsc, dsv, x, y1); }, 20);
      check("sell_rows U=4", t);
      t = timeit([&] { k_sell_rows<B, 7, V, X><<<(ns * 32 + 255) / 256, 256>>>(N, ns, dsp, dsc, dsv, x, y1); }, 20);
      check("sell_rows U=7", t);
    }
    cudaFree(dsp); cudaFree(dsc); cudaFree(dsv);
  }
#define LANEPRE(U, M)                                                                                              \
  t = timeit([&] { k_lane_pre<B, U, M, V, X><<<((N + 32 / B - 1) / (32 / B) * 32 + 255) / 256, 256>>>(N, ptr, col, val, x, y1); }, 20); \
  check("lane_pre U=" #U " minb=" #M, t);
  LANEPRE(4, 8) LANEPRE(4, 4) LANEPRE(8, 4) LANEPRE(8, 2) LANEPRE(7, 4)
#define LANEBNC(U)                                                                                              \
  t = timeit([&] { k_lane_bnc<B, U, V, X><<<((N + 32 / B - 1) / (32 / B) * 32 + 255) / 256, 256>>>(N, ptr, col, val, x, y1); }, 20); \
  check("lane_bnc U=" #U, t);
  LANEBNC(2) LANEBNC(4)
#define LANECOL(U, NC)                                                                                              \
  t = timeit([&] { k_lane_col<B, U, V, X, NC><<<((N + 32 / B - 1) / (32 / B) * 32 + 255) / 256, 256>>>(N, ptr, col, val, x, y1); }, 20); \
  check("lane_col U=" #U " nc=" #NC, t);
  LANECOL(2, false) LANECOL(4, false) LANECOL(2, true) LANECOL(4, true)
#define LANEP(U)                                                                                          \
  t = timeit([&] { k_lane_p<B, U, V, X><<<(N * 4 + 255) / 256, 256>>>(N, ptr, col, val, x, y1); }, 20); \
  check("lane_p U=" #U, t);

  if constexpr (32 % B == 0) {
#define WARP(U)                                                                                         \
  t = timeit([&] { k_warp<B, U, V, X><<<(N * 32 + 255) / 256, 256>>>(N, ptr, col, val, x, y1); }, 20); \
  check("warp U=" #U, t);
    WARP(2)
  }
  cudaFree(len); cudaFree(ptr); cudaFree(col); cudaFree(val); cudaFree(x); cudaFree(y0); cudaFree(y1);
}

int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 128, b = argc > 2 ? atoi(argv[2]) : 4, st = argc > 3 ? atoi(argv[3]) : 27;
  int vt = argc > 4 ? atoi(argv[4]) : 1, xt = argc > 5 ? atoi(argv[5]) : 0;
#define GO(BB, VV, XX) run<BB, VV, XX>(n, st)
  if (b == 4 && vt == 1 && xt == 0) GO(4, float, double);
  else if (b == 4 && vt == 1 && xt == 1) GO(4, float, float);
  else if (b == 4 && vt == 0) GO(4, double, double);
  else if (b == 3 && vt == 1 && xt == 0) GO(3, float, double);
  else if (b == 3 && vt == 1 && xt == 1) GO(3, float, float);
  else if (b == 3 && vt == 0) GO(3, double, double);
  return 0;
}
