// blas1.cu -- K12 Krylov vector kernels: deterministic dot products (two-stage,
// fixed grid for a given length, fixed-order finalisation), multi-dot / multi-axpy
// for the CGS2 Arnoldi step, linear combinations, and the flexible-GMRES update.
#include "blas1.h"
#include "reduce.cuh"
#include "comm.h"
#include "prof.h"

#include <cuda_fp16.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>

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

// ---- multi-vector kernels of the CGS2 Arnoldi step (flexible GMRES) ----
// K (the number of basis vectors, 1..32) is a template parameter: every loop over the
// basis unrolls without predication and the thread's K values of V stay in registers
// between the update and the dot of the same pass (no L1 re-read).  Each thread handles
// U elements per grid-stride step (U loads of every vector in flight for small K).  The
// grid is persistent (occupancy x 148 SMs); block partials are reduced by the LAST block
// to finish (ticket), in a fixed order -- deterministic, and no second launch.
constexpr int kTM = 128;

template <int K>
constexpr int cgs_unroll() { return K <= 2 ? 8 : (K <= 4 ? 4 : (K <= 10 ? 2 : 1)); }

template <int K>
__device__ __forceinline__ void reduce_finish(double (&acc)[K], int kout, double* partials, unsigned* ticket,
                                              double* out, int post, double* inv) {
  block_reduce_finish<K, kTM>(acc, kout, partials, ticket, out, post, inv);
}

// MODE 0: out[j] = s_j V_j . w                                   (scaled multi-dot)
// MODE 1: w_out = w - sum_j c_j s_j V_j;  out[j] = s_j V_j . w_out   (update + next dot)
// MODE 2: w_out = w - sum_j c_j s_j V_j;  out[0] = ||w_out||        (update + norm)
// MODE 3: w_out = w - sum_j c_j s_j V_j;  out[j] = s_j V_j . w_out, out[k] = w_out . w_out
//         (update + next dots + squared norm: the two-pass Gram/Cholesky orthogonalisation)
// (v_j = s_j V_j: the basis is stored unnormalised with device scales sc)
// TV: element type of the basis as read (double; float for the fp32 shadow copy the GMRES
// pass-1 multi-dot of reading R23 reads); wf (MODE 3, optional): fp32 copy of w_out
// the shadow copy of w_out written by MODE 3: fp32 as is (R23), or fp16 scaled by sig (R28:
// sig = sqrt(N) / ||w||, the pre-update norm, so every entry of the shadow is <= sqrt(N) in
// magnitude and its rms is ||w_out|| / ||w|| <= 1)
template <typename WF>
__device__ __forceinline__ WF to_shadow(double v, double sig) {
  if constexpr (std::is_same_v<WF, __half>) return __double2half(v * sig);
  else return (float)v;
}

template <int K, int MODE, typename TV = double, typename WF = float>
__global__ void __launch_bounds__(kTM) k_cgs(int64_t n, PtrList V, const double* __restrict__ sc,
                                             const double* __restrict__ coef, const double* w, double* w_out,
                                             double* partials, unsigned* ticket, double* out, int post,
                                             double* inv, WF* wf) {
  constexpr int U = cgs_unroll<K>();
  __shared__ double c[K], sv[K];
  __shared__ double sig;
  if (threadIdx.x < K) {
    sv[threadIdx.x] = sc ? sc[threadIdx.x] : 1.0;
    c[threadIdx.x] = (MODE == 0) ? 0.0 : coef[threadIdx.x] * sv[threadIdx.x];
  }
  if (threadIdx.x == 0) sig = (MODE == 3 && std::is_same_v<WF, __half> && wf) ? coef[K] : 1.0;
  __syncthreads();
  constexpr bool H16 = MODE == 0 && std::is_same_v<TV, __half>;  // R28's multi-dot: + w . w in acc[K]
  constexpr int KA = (MODE == 2) ? 1 : ((MODE == 3 || H16) ? K + 1 : K);
  double acc[KA];
#pragma unroll
  for (int j = 0; j < KA; ++j) acc[j] = 0.0;
  if constexpr (H16) {
    // fp16 shadow basis (reading R28): four consecutive elements per thread, one 8-byte load per
    // vector, each vector's values widened as its load is consumed; w . w on the side
    const int64_t n4 = n / 4;
    for (int64_t i4 = (int64_t)blockIdx.x * kTM + threadIdx.x; i4 < n4; i4 += (int64_t)gridDim.x * kTM) {
      uint2 hr[K];
#pragma unroll
      for (int j = 0; j < K; ++j) hr[j] = __ldcs(reinterpret_cast<const uint2*>(V.p[j]) + i4);
      const double2 w0 = __ldcs(reinterpret_cast<const double2*>(w) + 2 * i4);
      const double2 w1 = __ldcs(reinterpret_cast<const double2*>(w) + 2 * i4 + 1);
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&hr[j].x));
        const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&hr[j].y));
        acc[j] = fma((double)a.x, w0.x, acc[j]);
        acc[j] = fma((double)a.y, w0.y, acc[j]);
        acc[j] = fma((double)b.x, w1.x, acc[j]);
        acc[j] = fma((double)b.y, w1.y, acc[j]);
      }
      acc[K] = fma(w0.x, w0.x, acc[K]);
      acc[K] = fma(w0.y, w0.y, acc[K]);
      acc[K] = fma(w1.x, w1.x, acc[K]);
      acc[K] = fma(w1.y, w1.y, acc[K]);
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * kTM + threadIdx.x; i < n; i += (int64_t)gridDim.x * kTM) {
      const double wi = w[i];
#pragma unroll
      for (int j = 0; j < K; ++j) acc[j] = fma((double)__half2float(reinterpret_cast<const __half*>(V.p[j])[i]), wi, acc[j]);
      acc[K] = fma(wi, wi, acc[K]);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] *= sv[j];
    reduce_finish<KA>(acc, KA, partials, ticket, out, post, inv);
    return;
  } else if constexpr (MODE == 0 && std::is_same_v<TV, float>) {
    // fp32 shadow basis (reading R23): four consecutive elements per thread, one 16-byte load
    // per vector (the scalar form kept one 4-byte load per vector in flight: 2-4 TB/s)
    const int64_t n4 = n / 4;
    for (int64_t i4 = (int64_t)blockIdx.x * kTM + threadIdx.x; i4 < n4; i4 += (int64_t)gridDim.x * kTM) {
      float4 raw[K];
#pragma unroll
      for (int j = 0; j < K; ++j) raw[j] = __ldcs(reinterpret_cast<const float4*>(V.p[j]) + i4);
      const double2 w0 = __ldcs(reinterpret_cast<const double2*>(w) + 2 * i4);
      const double2 w1 = __ldcs(reinterpret_cast<const double2*>(w) + 2 * i4 + 1);
#pragma unroll
      for (int j = 0; j < K; ++j) {
        acc[j] = fma((double)raw[j].x, w0.x, acc[j]);
        acc[j] = fma((double)raw[j].y, w0.y, acc[j]);
        acc[j] = fma((double)raw[j].z, w1.x, acc[j]);
        acc[j] = fma((double)raw[j].w, w1.y, acc[j]);
      }
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * kTM + threadIdx.x; i < n; i += (int64_t)gridDim.x * kTM) {
      const double wi = w[i];
#pragma unroll
      for (int j = 0; j < K; ++j) acc[j] = fma((double)reinterpret_cast<const TV*>(V.p[j])[i], wi, acc[j]);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] *= sv[j];
    reduce_finish<KA>(acc, KA, partials, ticket, out, post, inv);
    return;
  }
  const int64_t step = (int64_t)gridDim.x * kTM * U;
  for (int64_t i0 = (int64_t)blockIdx.x * kTM * U + threadIdx.x; i0 < n; i0 += step) {
    double wv[U], vv[U][K];
    if constexpr (std::is_same_v<TV, double>) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + (int64_t)u * kTM;
        const bool ok = i < n;
        wv[u] = ok ? w[i] : 0.0;
#pragma unroll
        for (int j = 0; j < K; ++j) vv[u][j] = ok ? __ldcs(V.p[j] + i) : 0.0;
      }
    } else {
      // fp32 basis: unpredicated loads (clamped index) all issued before the widening, which
      // a predicated load + F2F pair would serialise (SASS: one LDG in flight)
      TV raw[U][K];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = min(i0 + (int64_t)u * kTM, n - 1);
#pragma unroll
        for (int j = 0; j < K; ++j) raw[u][j] = __ldcs(reinterpret_cast<const TV*>(V.p[j]) + i);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + (int64_t)u * kTM;
        const bool ok = i < n;
        wv[u] = ok ? w[i] : 0.0;
#pragma unroll
        for (int j = 0; j < K; ++j) vv[u][j] = ok ? (double)raw[u][j] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + (int64_t)u * kTM;
      if constexpr (MODE == 0) {
#pragma unroll
        for (int j = 0; j < K; ++j) acc[j] = fma(vv[u][j], wv[u], acc[j]);
      } else {
        double v = wv[u];
#pragma unroll
        for (int j = 0; j < K; ++j) v = fma(-c[j], vv[u][j], v);
        if (i < n) w_out[i] = v;
        if (MODE == 3 && wf && i < n) wf[i] = to_shadow<WF>(v, sig);
        if constexpr (MODE == 1 || MODE == 3) {
#pragma unroll
          for (int j = 0; j < K; ++j) acc[j] = fma(sv[j] * vv[u][j], v, acc[j]);
          if constexpr (MODE == 3) acc[K] = fma(v, v, acc[K]);
        } else {
          acc[0] = fma(v, v, acc[0]);
        }
      }
    }
  }
  if constexpr (MODE == 0) {
#pragma unroll
    for (int j = 0; j < K; ++j) acc[j] *= sv[j];
  }
  reduce_finish<KA>(acc, KA, partials, ticket, out, post, inv);
}

// ---- wide variant for many basis vectors (k > 12) ----
// The K-templated k_cgs keeps all k values of an element in one thread: past k ~ 13 the
// compiler no longer issues all loads before the arithmetic (measured 2.6-4.5 TB/s at
// k = 16..29).  Here the 8 warps of a 256-thread block split the VECTORS (warp w owns
// j = w + 8q, q < NJ) and the block walks chunks of 256 elements: every lane holds NJ x 8
// values in registers, each load of a warp is 256 contiguous bytes, and the update
// sum_j c_j s_j V_j is combined across warps through shared memory in a fixed order.
constexpr int kTW = 256, kCW = 256;  // threads, elements per chunk

__device__ __forceinline__ void finish_partials(int kout, double* partials, unsigned* ticket, double* out, int post,
                                                double* inv) {
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblk = gridDim.x;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == (unsigned)nblk - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int j = warp; j < kout; j += blockDim.x / 32) {
    double v = 0.0;
    for (int i = lane; i < nblk; i += 32) v += __ldcg(partials + (int64_t)j * nblk + i);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    if (lane == 0) {
      if (post >= 1) v = sqrt(v);
      out[j] = v;
      if (post == 2 && j == 0) inv[0] = 1.0 / v;
    }
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

template <int NJ, int MODE, typename TV = double, typename WF = float>
__global__ void __launch_bounds__(kTW, (NJ <= 3 ? 3 : 2)) k_cgs_wide(int64_t n, int k, PtrList V, const double* __restrict__ sc,
                                                     const double* __restrict__ coef, const double* w, double* w_out,
                                                     double* partials, unsigned* ticket, double* out, int post,
                                                     double* inv, WF* wf) {
  constexpr int T = kCW / 32;  // elements per lane per chunk
  __shared__ double c[32], sv[32];
  __shared__ double part[8][kCW + 1];
  __shared__ __align__(16) double vs[kCW];
  __shared__ double sig;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < k) {
    sv[threadIdx.x] = sc ? sc[threadIdx.x] : 1.0;
    c[threadIdx.x] = (MODE == 0) ? 0.0 : coef[threadIdx.x] * sv[threadIdx.x];
  }
  if (threadIdx.x == 0) sig = (MODE == 3 && std::is_same_v<WF, __half> && wf) ? coef[k] : 1.0;
  __syncthreads();
  const TV* vp[NJ];
  bool own[NJ];
#pragma unroll
  for (int q = 0; q < NJ; ++q) {
    const int j = warp + 8 * q;
    own[q] = j < k;
    vp[q] = reinterpret_cast<const TV*>(own[q] ? V.p[j] : V.p[0]);
  }
  double acc[NJ];
#pragma unroll
  for (int q = 0; q < NJ; ++q) acc[q] = 0.0;
  double nrm = 0.0;
  for (int64_t i0 = (int64_t)blockIdx.x * kCW; i0 < n; i0 += (int64_t)gridDim.x * kCW) {
    const bool full = i0 + kCW <= n;
    if constexpr (MODE == 0 && std::is_same_v<TV, float>) {
      // fp32 shadow basis (reading R23): lane owns elements i0 + 128 h + 4 lane + e (h, e < 2, 4)
      // -- two 16-byte loads per vector and four for w (L1 serves the other warps' reads of
      // the same w chunk), so a warp keeps as many bytes in flight as the fp64 kernel
      if (full) {
        float4 raw[NJ][2];
#pragma unroll
        for (int q = 0; q < NJ; ++q)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
            raw[q][hh] = __ldcs(reinterpret_cast<const float4*>(vp[q] + i0 + 128 * hh + 4 * lane));
        double2 wv[2][2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            wv[hh][e] = __ldg(reinterpret_cast<const double2*>(w + i0 + 128 * hh + 4 * lane) + e);
#pragma unroll
        for (int q = 0; q < NJ; ++q)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            acc[q] = fma((double)raw[q][hh].x, wv[hh][0].x, acc[q]);
            acc[q] = fma((double)raw[q][hh].y, wv[hh][0].y, acc[q]);
            acc[q] = fma((double)raw[q][hh].z, wv[hh][1].x, acc[q]);
            acc[q] = fma((double)raw[q][hh].w, wv[hh][1].y, acc[q]);
          }
#pragma unroll
        for (int q = 0; q < NJ; ++q)
          if (!own[q]) acc[q] = 0.0;
      } else {
        for (int hh = 0; hh < 2; ++hh)
          for (int e = 0; e < 4; ++e) {
            const int64_t i = i0 + 128 * hh + 4 * lane + e;
            if (i < n) {
              const double wi = w[i];
#pragma unroll
              for (int q = 0; q < NJ; ++q)
                if (own[q]) acc[q] = fma((double)vp[q][i], wi, acc[q]);
            }
          }
      }
      continue;
    }
    double val[NJ][T];
    if constexpr (std::is_same_v<TV, double>) {
#pragma unroll
      for (int q = 0; q < NJ; ++q)
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int64_t i = i0 + lane + 32 * t;
          val[q][t] = (own[q] && (full || i < n)) ? __ldcs(vp[q] + i) : 0.0;
        }
    } else {  // fp32 basis: unpredicated loads first, then the widening (see k_cgs)
      TV raw[NJ][T];
#pragma unroll
      for (int q = 0; q < NJ; ++q)
#pragma unroll
        for (int t = 0; t < T; ++t) raw[q][t] = __ldcs(vp[q] + min(i0 + lane + 32 * t, n - 1));
#pragma unroll
      for (int q = 0; q < NJ; ++q)
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int64_t i = i0 + lane + 32 * t;
          val[q][t] = (own[q] && (full || i < n)) ? (double)raw[q][t] : 0.0;
        }
    }
    const int64_t it = i0 + threadIdx.x;
    const double wv = (it < n) ? w[it] : 0.0;
    if constexpr (MODE == 0) {
      vs[threadIdx.x] = wv;
      __syncthreads();
#pragma unroll
      for (int q = 0; q < NJ; ++q)
#pragma unroll
        for (int t = 0; t < T; ++t) acc[q] = fma(val[q][t], vs[lane + 32 * t], acc[q]);
      __syncthreads();
    } else {
      // partial update of this warp's vectors, element e = lane + 32 t
#pragma unroll
      for (int t = 0; t < T; ++t) {
        double p = 0.0;
#pragma unroll
        for (int q = 0; q < NJ; ++q) p = fma(c[own[q] ? warp + 8 * q : 0] * (own[q] ? 1.0 : 0.0), val[q][t], p);
        part[warp][lane + 32 * t] = p;
      }
      __syncthreads();
      double v = wv;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) v -= part[ww][threadIdx.x];
      if (it < n) w_out[it] = v;
      if (MODE == 3 && wf && it < n) wf[it] = to_shadow<WF>(v, sig);
      if constexpr (MODE == 2 || MODE == 3) nrm = fma(v, v, nrm);
      if constexpr (MODE != 2) {
        vs[threadIdx.x] = v;
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NJ; ++q)
#pragma unroll
          for (int t = 0; t < T; ++t) acc[q] = fma(val[q][t], vs[lane + 32 * t], acc[q]);
      }
      __syncthreads();  // part / vs reused by the next chunk
    }
  }
  if constexpr (MODE == 2) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) nrm += __shfl_xor_sync(kFull, nrm, off);
    if (lane == 0) part[0][warp] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
#pragma unroll
      for (int ww = 0; ww < 8; ++ww) s += part[0][ww];
      partials[blockIdx.x] = s;
    }
    finish_partials(1, partials, ticket, out, post, inv);
  } else {
#pragma unroll
    for (int q = 0; q < NJ; ++q) {
      double v = acc[q];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
      const int j = warp + 8 * q;
      if (lane == 0 && own[q]) partials[(int64_t)j * gridDim.x + blockIdx.x] = v * sv[j];
    }
    if constexpr (MODE == 3) {
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) nrm += __shfl_xor_sync(kFull, nrm, off);
      __syncthreads();
      if (lane == 0) part[0][warp] = nrm;
      __syncthreads();
      if (threadIdx.x == 0) {
        double s = 0.0;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) s += part[0][ww];
        partials[(int64_t)k * gridDim.x + blockIdx.x] = s;
      }
    }
    finish_partials(MODE == 3 ? k + 1 : k, partials, ticket, out, post, inv);
  }
}

// R28's pass-1 multi-dot for k > 12: out[j] = ms_j (h_j . w) over the fp16 shadows h_j, the
// wide kernel's layout (warp w owns vectors w + 8q; lane owns elements i0 + 128 hh + 4 lane +
// e of each 256-element chunk, one 8-byte load per vector and hh) at <= 64 registers so that
// more blocks per SM keep the loads in flight (the shared template held 107 registers and ran
// two blocks per SM: 3-4.5 TB/s; this one 5.2-6.3 at 8 blocks per SM).  Measured and dropped
// (run r02m): 40 / 48 registers for NJ = 2 / 3 (6 / 5 resident blocks) -- 0.87 -> 1.30 ms at
// k = 13, 1.11 -> 1.22 at k = 17; the time per launch is flat inside an NJ group, with or
// without the loads of the slots a warp does not own (run r02l).
template <int NJ>
__global__ void __launch_bounds__(kTW, 4) k_mdot16_wide(int64_t n, int k, PtrList V, const double* __restrict__ ms,
                                                        const double* w, double* partials, unsigned* ticket,
                                                        double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const __half* vp[NJ];
  bool own[NJ];
#pragma unroll
  for (int q = 0; q < NJ; ++q) {
    const int j = warp + 8 * q;
    own[q] = j < k;
    vp[q] = reinterpret_cast<const __half*>(own[q] ? V.p[j] : V.p[0]);
  }
  double acc[NJ];
#pragma unroll
  for (int q = 0; q < NJ; ++q) acc[q] = 0.0;
  double ww = 0.0;  // w . w (warp 0, whose lanes cover the whole chunk): the next shadow's scale
  for (int64_t i0 = (int64_t)blockIdx.x * kCW; i0 < n; i0 += (int64_t)gridDim.x * kCW) {
    if (i0 + kCW <= n) {
      uint2 hr[NJ][2];
#pragma unroll
      for (int q = 0; q < NJ; ++q)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)  // a warp without a q-th vector (k < 8 (q + 1)) loads nothing for it
          hr[q][hh] = own[q] ? __ldcs(reinterpret_cast<const uint2*>(vp[q] + i0 + 128 * hh + 4 * lane)) : make_uint2(0u, 0u);
      double2 wv[2][2];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
#pragma unroll
        for (int e = 0; e < 2; ++e) wv[hh][e] = __ldg(reinterpret_cast<const double2*>(w + i0 + 128 * hh + 4 * lane) + e);
#pragma unroll
      for (int q = 0; q < NJ; ++q)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&hr[q][hh].x));
          const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&hr[q][hh].y));
          acc[q] = fma((double)a.x, wv[hh][0].x, acc[q]);
          acc[q] = fma((double)a.y, wv[hh][0].y, acc[q]);
          acc[q] = fma((double)b.x, wv[hh][1].x, acc[q]);
          acc[q] = fma((double)b.y, wv[hh][1].y, acc[q]);
        }
      if (warp == 0)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          ww = fma(wv[hh][0].x, wv[hh][0].x, ww);
          ww = fma(wv[hh][0].y, wv[hh][0].y, ww);
          ww = fma(wv[hh][1].x, wv[hh][1].x, ww);
          ww = fma(wv[hh][1].y, wv[hh][1].y, ww);
        }
    } else {
      for (int hh = 0; hh < 2; ++hh)
        for (int e = 0; e < 4; ++e) {
          const int64_t i = i0 + 128 * hh + 4 * lane + e;
          if (i < n) {
            const double wi = w[i];
#pragma unroll
            for (int q = 0; q < NJ; ++q) acc[q] = fma((double)__half2float(vp[q][i]), wi, acc[q]);
            if (warp == 0) ww = fma(wi, wi, ww);
          }
        }
    }
  }
#pragma unroll
  for (int q = 0; q < NJ; ++q) {
    double v = own[q] ? acc[q] : 0.0;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    const int j = warp + 8 * q;
    if (lane == 0 && own[q]) partials[(int64_t)j * gridDim.x + blockIdx.x] = v * ms[j];
  }
  if (warp == 0) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) ww += __shfl_xor_sync(kFull, ww, off);
    if (lane == 0) partials[(int64_t)k * gridDim.x + blockIdx.x] = ww;
  }
  finish_partials(k + 1, partials, ticket, out, 0, nullptr);  // out[k] = w . w
}

template <int KMAX, int K = 1, class F>
void dispatch_k_upto(int k, F&& f) {
  if (k == K) f(std::integral_constant<int, K>{});
  else if constexpr (K < KMAX) dispatch_k_upto<KMAX, K + 1>(k, f);
  else fail(AMG_EINVAL, "multi-vector kernel: too many vectors for this variant");
}

template <int K = 1, class F>
void dispatch_k(int k, F&& f) {
  if (k == K) f(std::integral_constant<int, K>{});
  else if constexpr (K < 32) dispatch_k<K + 1>(k, f);
  else fail(AMG_EINVAL, "multi-vector kernels take 1..32 vectors");
}

template <int MODE, typename TV = double, typename WF = float>
void launch_cgs(int64_t n, int k, const PtrList& V, const double* sc, const double* coef, const double* w,
                double* w_out, double* partials, double* out, int post, double* inv, cudaStream_t s,
                WF* wf = nullptr) {
  unsigned* ticket = reinterpret_cast<unsigned*>(partials + (size_t)kMaxPartials * 32);
  if constexpr (MODE == 0 && std::is_same_v<TV, __half>) {  // R28: the fp16 multi-dot (+ w . w)
    if (k < std::min(env_int("AMG_F16_WIDE", 11), 13)) {  // K-templated (k = 11 / 12 there: 4.8 / 3.2 TB/s)
      dispatch_k_upto<12>(k, [&](auto Kc) {
        constexpr int K = decltype(Kc)::value;
        static int occ = 0;
        if (occ == 0) {
          AMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cgs<K, 0, __half, float>, kTM, 0));
          occ = std::max(occ, 1);
        }
        const int64_t work = (n + (int64_t)kTM * 4 - 1) / ((int64_t)kTM * 4);
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)occ * kSMs, (int64_t)kMaxPartials, work}));
        k_cgs<K, 0, __half, float><<<g, kTM, 0, s>>>(n, V, sc, coef, w, w_out, partials, ticket, out, post, inv,
                                                      (float*)nullptr);
      });
      AMG_CK_LAUNCH();
      return;
    }
    const int64_t work = (n + kCW - 1) / kCW;
    const int g16 = (int)std::max<int64_t>(
        1, std::min<int64_t>({(int64_t)env_int("AMG_F16_BLOCKS", 8) * kSMs, (int64_t)kMaxPartials, work}));
    auto go16 = [&](auto kern) { kern<<<g16, kTW, 0, s>>>(n, k, V, sc, w, partials, ticket, out); };
    if (k <= 16) go16(k_mdot16_wide<2>);
    else if (k <= 24) go16(k_mdot16_wide<3>);
    else go16(k_mdot16_wide<4>);
    AMG_CK_LAUNCH();
    return;
  } else {
  const int wide_from = env_int("AMG_CGS_WIDE", 13);  // first k served by k_cgs_wide (tests force both)
  if (k >= wide_from) {
    const int64_t work = (n + kCW - 1) / kCW;
    // two or three vectors per warp (k <= 24) fit three blocks per SM at 80 registers: the
    // third hides the idle slots of the warps that own one vector fewer (AMG_CGS_BPS2 /
    // AMG_CGS_BPS3 = 2: the two-block grid, A/B).  Four vectors per warp spill 160 bytes at 80
    // registers and run at 4.2-4.6 TB/s against 6.2-6.5 with two blocks of 126 registers.
    const int bps = k <= 16 ? std::min(std::max(env_int("AMG_CGS_BPS2", 3), 1), 3)
                    : k <= 24 ? std::min(std::max(env_int("AMG_CGS_BPS3", 3), 1), 3) : 2;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)bps * kSMs, (int64_t)kMaxPartials, work}));
    auto go = [&](auto kern) {
      kern<<<g, kTW, 0, s>>>(n, k, V, sc, coef, w, w_out, partials, ticket, out, post, inv, wf);
    };
    if (k <= 16) go(k_cgs_wide<2, MODE, TV, WF>);
    else if (k <= 24) go(k_cgs_wide<3, MODE, TV, WF>);
    else go(k_cgs_wide<4, MODE, TV, WF>);
    AMG_CK_LAUNCH();
    return;
  }
  dispatch_k(k, [&](auto Kc) {
    constexpr int K = decltype(Kc)::value;
    constexpr int U = cgs_unroll<K>();
    static int occ = 0;  // per (K, MODE, TV, WF) instantiation
    if (occ == 0) {
      AMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cgs<K, MODE, TV, WF>, kTM, 0));
      occ = std::max(occ, 1);
    }
    const int64_t work = (n + (int64_t)kTM * U - 1) / ((int64_t)kTM * U);
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)occ * kSMs, (int64_t)kMaxPartials, work}));
    k_cgs<K, MODE, TV, WF><<<g, kTM, 0, s>>>(n, V, sc, coef, w, w_out, partials, ticket, out, post, inv, wf);
  });
  AMG_CK_LAUNCH();
  }
}

// out[j] = sum of the nblk partials of reduction j, in a fixed order
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

// x += sum_j y[j] Z_j  (Z of type T; y on the device); K-templated like k_cgs
template <int K, typename T>
constexpr int zupdate_unroll() { return (sizeof(T) == 4 && K > 10) ? 2 : cgs_unroll<K>(); }

template <int K, typename T>
__global__ void __launch_bounds__(kTM) k_zupdate(int64_t n, PtrList Z, const double* __restrict__ y,
                                                 double* __restrict__ x) {
  constexpr int U = zupdate_unroll<K, T>();
  __shared__ double c[K];
  if (threadIdx.x < K) c[threadIdx.x] = y[threadIdx.x];
  __syncthreads();
  const int64_t step = (int64_t)gridDim.x * kTM * U;
  for (int64_t i0 = (int64_t)blockIdx.x * kTM * U + threadIdx.x; i0 < n; i0 += step) {
    double xv[U];
    T zv[U][K];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + (int64_t)u * kTM;
      const bool ok = i < n;
      xv[u] = ok ? x[i] : 0.0;
#pragma unroll
      for (int j = 0; j < K; ++j) zv[u][j] = ok ? __ldcs(reinterpret_cast<const T*>(Z.p[j]) + i) : T(0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + (int64_t)u * kTM;
      double v = xv[u];
#pragma unroll
      for (int j = 0; j < K; ++j) v = fma(c[j], (double)zv[u][j], v);
      if (i < n) x[i] = v;
    }
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

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

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
  ++t_launches;
  k_finalize<<<1, kT, 0, s>>>(1, partials, nb, out, (sqrt_out && !comm) ? 1 : 0);
  AMG_CK_LAUNCH();
  finalize_global(comm, out, 1, sqrt_out, s);
}

void launch_mdot(int64_t n, int k, const PtrList& V, const double* w, double* partials, double* out, cudaStream_t s) {
  ProfScope ps_(prof_name("mdot", k, AMG_F64, -1), 8.0 * n * (k + 1), s);
  launch_cgs<0>(n, k, V, nullptr, nullptr, w, nullptr, partials, out, 0, nullptr, s);
}

void launch_mdot_scaled(int64_t n, int k, const PtrList& V, const double* sc, const double* w, double* partials,
                        double* out, cudaStream_t s, CommBase* comm) {
  ProfScope ps_(prof_name("mdot", k, AMG_F64, -1), 8.0 * n * (k + 1), s);
  launch_cgs<0>(n, k, V, sc, nullptr, w, nullptr, partials, out, 0, nullptr, s);
  finalize_global(comm, out, k, false, s);
}

void launch_mdot_scaled_f32(int64_t n, int k, const PtrList& Vf, const double* sc, const double* w, double* partials,
                            double* out, cudaStream_t s, CommBase* comm) {
  ProfScope ps_(prof_name("mdot", k, AMG_F32, -1), 4.0 * n * k + 8.0 * n, s);
  launch_cgs<0, float>(n, k, Vf, sc, nullptr, w, nullptr, partials, out, 0, nullptr, s);
  finalize_global(comm, out, k, false, s);
}

void launch_mdot_scaled_f16(int64_t n, int k, const PtrList& Vh, const double* ms, const double* w, double* partials,
                            double* out, cudaStream_t s, CommBase* comm) {
  if (k + 1 > 32) fail(AMG_EINVAL, "fp16 multi-dot: at most 31 vectors");
  ProfScope ps_(prof_name("mdot", k, AMG_F16, -1), 2.0 * n * k + 8.0 * n, s);
  launch_cgs<0, __half>(n, k, Vh, ms, nullptr, w, nullptr, partials, out, 0, nullptr, s);
  finalize_global(comm, out, k + 1, false, s);
}

// dst = fp16(src * sig), sig the power of two at or below mul * *s_dev (the fp16 shadow of V_0 at
// about unit rms: mul = sqrt(N), s_dev = 1 / ||V_0||); *m_out = *s_dev / sig
__global__ void k_to_half_scaled(int64_t n, const double* __restrict__ src, const double* __restrict__ s_dev,
                                 double mul, __half* __restrict__ dst, double* m_out) {
  int e = 0;
  frexp(mul * *s_dev, &e);
  const double sig = ldexp(1.0, e - 1);
  if (blockIdx.x == 0 && threadIdx.x == 0) *m_out = *s_dev / sig;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT)
    dst[i] = __double2half(src[i] * sig);
}

void launch_to_half_scaled(int64_t n, const double* src, const double* s_dev, double mul, void* dst, double* m_out,
                           cudaStream_t s) {
  ProfScope ps_(prof_name("convert", 1, AMG_F16, AMG_F64), 10.0 * n, s);
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, (int64_t)kSMs * 16));
  k_to_half_scaled<<<g, kT, 0, s>>>(n, src, s_dev, mul, (__half*)dst, m_out);
  AMG_CK_LAUNCH();
}

__global__ void k_set_inv1(double* dst, const double* src) { *dst = 1.0 / *src; }

void launch_cgs_update_dots_nrm(int64_t n, int k, const PtrList& V, const double* sc, const double* coef,
                                const double* w, double* w_out, double* partials, double* out, cudaStream_t s,
                                CommBase* comm, void* wf_out, int wf_type) {
  if (k + 1 > 32) fail(AMG_EINVAL, "update + dots + norm: at most 31 vectors");
  {
    const double ws = wf_out ? (wf_type == AMG_F16 ? 2.0 : 4.0) : 0.0;
    ProfScope ps_(prof_name("cgs_update_dots_nrm", k, AMG_F64, -1), 8.0 * n * (k + 2) + ws * n, s);
    if (wf_out && wf_type == AMG_F16)
      launch_cgs<3, double, __half>(n, k, V, sc, coef, w, w_out, partials, out, 0, nullptr, s, (__half*)wf_out);
    else
      launch_cgs<3>(n, k, V, sc, coef, w, w_out, partials, out, 0, nullptr, s, (float*)wf_out);
  }
  finalize_global(comm, out, k + 1, false, s);
}

void launch_cgs_update(int64_t n, int k, const PtrList& V, const double* sc, const double* coef, const double* w,
                       double* w_out, bool dot_next, double* partials, double* out, cudaStream_t s, CommBase* comm,
                       double* inv_out) {
  ProfScope ps_(prof_name(dot_next ? "cgs_update_dot" : "cgs_update_nrm", k, AMG_F64, -1), 8.0 * n * (k + 2), s);
  if (dot_next) {
    launch_cgs<1>(n, k, V, sc, coef, w, w_out, partials, out, 0, nullptr, s);
    finalize_global(comm, out, k, false, s);
    return;
  }
  const int post = comm ? 0 : (inv_out ? 2 : 1);
  launch_cgs<2>(n, k, V, sc, coef, w, w_out, partials, out, post, inv_out, s);
  finalize_global(comm, out, 1, true, s);
  if (comm && inv_out) {
    k_set_inv1<<<1, 1, 0, s>>>(inv_out, out);
    AMG_CK_LAUNCH();
  }
}

void launch_maxpy(int64_t n, int k, const PtrList& V, const double* coef, double* w, cudaStream_t s) {
  ProfScope ps_(prof_name("maxpy", k, AMG_F64, -1), 8.0 * n * (k + 2), s);
  k_maxpy<<<ew_grid(n), kT, 0, s>>>(n, k, V, coef, w);
  AMG_CK_LAUNCH();
}

void launch_zupdate(int64_t n, int k, const PtrList& Z, int zt, const double* y, double* x, cudaStream_t s) {
  ProfScope ps_(prof_name("zupdate", k, zt, -1), (double)n * (16.0 + (double)k * dtype_size(zt)), s);
  dispatch_k(k, [&](auto Kc) {
    constexpr int K = decltype(Kc)::value;
    auto go = [&](auto T) {
      using TT = decltype(T);
      constexpr int U = zupdate_unroll<K, TT>();
      static int occ = 0;  // per instantiation
      if (occ == 0) {
        AMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_zupdate<K, TT>, kTM, 0));
        occ = std::max(occ, 1);
      }
      const int64_t work = (n + (int64_t)kTM * U - 1) / ((int64_t)kTM * U);
      const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)kSMs * occ, work));
      k_zupdate<K, TT><<<g, kTM, 0, s>>>(n, Z, y, x);
    };
    if (zt == AMG_F32) go(float{});
    else go(double{});
  });
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

// ---- IDR(s) helpers ----
// out = sum_t c_t in_t  (t < L.n <= 12 terms, host coefficients; out may alias an input:
// every element is read before it is written, by the same thread)
// N a template parameter (all N loads of an element pair issued before the FMAs) and two
// elements per thread as one 16-byte load per vector: 4.9-5.5 -> 6+ TB/s for IDR(s)'s
// v = r - G c and U updates (the generic loop kept one load in flight per thread)
template <int N, bool VEC>
__global__ void __launch_bounds__(kT) k_lincomb(int64_t n, LinComb L, double* out) {
  if constexpr (!VEC) {  // a pointer not 16-byte aligned (a user vector at an odd offset)
    for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
      double q[N];
#pragma unroll
      for (int t = 0; t < N; ++t) q[t] = L.p[t][i];
      double v = L.c[0] * q[0];
#pragma unroll
      for (int t = 1; t < N; ++t) v = fma(L.c[t], q[t], v);
      out[i] = v;
    }
    return;
  }
  const int64_t n2 = n / 2;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n2; i += (int64_t)gridDim.x * kT) {
    double2 q[N];
#pragma unroll
    for (int t = 0; t < N; ++t) q[t] = reinterpret_cast<const double2*>(L.p[t])[i];
    double2 v = make_double2(L.c[0] * q[0].x, L.c[0] * q[0].y);
#pragma unroll
    for (int t = 1; t < N; ++t) v.x = fma(L.c[t], q[t].x, v.x), v.y = fma(L.c[t], q[t].y, v.y);
    reinterpret_cast<double2*>(out)[i] = v;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    double v = L.c[0] * L.p[0][n - 1];
#pragma unroll
    for (int t = 1; t < N; ++t) v = fma(L.c[t], L.p[t][n - 1], v);
    out[n - 1] = v;
  }
}

void launch_lincomb(int64_t n, const LinComb& L, double* out, cudaStream_t s) {
  if (n == 0 || L.n == 0) return;
  ProfScope ps_(prof_name("lincomb", L.n, AMG_F64, -1), 8.0 * n * (L.n + 1), s);
  if (L.n > 12) fail(AMG_EINVAL, "lincomb: at most 12 vectors");
  bool vec = aligned16(out);
  for (int t = 0; t < L.n; ++t) vec = vec && aligned16(L.p[t]);
  const unsigned g = ew_grid(vec ? (n + 1) / 2 : n);
  switch (L.n) {
#define AMG_LC(N)                                                  \
  case N:                                                          \
    if (vec) k_lincomb<N, true><<<g, kT, 0, s>>>(n, L, out);      \
    else k_lincomb<N, false><<<g, kT, 0, s>>>(n, L, out);         \
    break;
    AMG_LC(1) AMG_LC(2) AMG_LC(3) AMG_LC(4) AMG_LC(5) AMG_LC(6) AMG_LC(7) AMG_LC(8) AMG_LC(9) AMG_LC(10) AMG_LC(11)
    AMG_LC(12)
#undef AMG_LC
  }
  AMG_CK_LAUNCH();
}

// IDR(s) shadow vector: p[i] = N01(stream 6, idx = row * n_global + off + i) with the
// counter RNG of SURVEY.md §8(d): SplitMix64 finaliser mix, R = mix(mix(SEED ^ (6 << 56)) ^ idx),
// U01 = (R >> 11) 2^-53, Box-Muller on (1 - U01(2 idx), U01(2 idx + 1))
__device__ __forceinline__ uint64_t rng_mix_d(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double rng_u01_d(uint64_t key, uint64_t idx) {
  return (double)(rng_mix_d(key ^ idx) >> 11) * (1.0 / 9007199254740992.0);
}
__global__ void k_shadow(int64_t n, uint64_t row, uint64_t n_global, uint64_t off, double* p) {
  const uint64_t key = rng_mix_d(200606052ULL ^ (6ULL << 56));
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) {
    const uint64_t idx = row * n_global + off + (uint64_t)i;
    const double u1 = 1.0 - rng_u01_d(key, 2 * idx), u2 = rng_u01_d(key, 2 * idx + 1);
    p[i] = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
  }
}

__global__ void k_axpy_dev(int64_t n, const double* __restrict__ d, const double* __restrict__ x, double* y) {
  const double a = d[0];
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT) y[i] = y[i] - a * x[i];
}

void idrs_shadow_space(int64_t n, int sdim, uint64_t base, uint64_t n_global, uint64_t off, double* const* P,
                       double* partials, double* dscal, cudaStream_t s, CommBase* comm) {
  for (int j = 0; j < sdim; ++j) {
    k_shadow<<<ew_grid(n), kT, 0, s>>>(n, base + (uint64_t)j, n_global, off, P[j]);
    AMG_CK_LAUNCH();
    for (int l = 0; l < j; ++l) {  // modified Gram-Schmidt
      launch_dot(n, P[l], AMG_F64, P[j], AMG_F64, partials, dscal, false, s, comm);
      k_axpy_dev<<<ew_grid(n), kT, 0, s>>>(n, dscal, P[l], P[j]);
      AMG_CK_LAUNCH();
    }
    launch_dot(n, P[j], AMG_F64, P[j], AMG_F64, partials, dscal, true, s, comm);
    launch_scale_by_inv(n, P[j], dscal, P[j], s);
  }
}

// IDR(s) step update in one pass: r -= a g; x += a u; out[0] = ||r||  (deterministic
// block partials + last-block finish, as k_cgs)
template <bool VEC>
__global__ void __launch_bounds__(kTM) k_idr_update(int64_t n, double a, const double* __restrict__ g,
                                                    const double* __restrict__ u, double* r, double* x,
                                                    double* partials, unsigned* ticket, double* out, int post,
                                                    const double* a_num = nullptr, const double* a_den = nullptr) {
  // a_num / a_den (device, optional): a = a_num[0] / a_den[0] (CG's alpha = rho / p.q formed on
  // the device, reading R24); the update is skipped when the denominator broke down
  if (a_num) {
    const double den = a_den[0];
    a = a_num[0] / den;
    if (den == 0.0 || !isfinite(den)) n = 0;
  }
  // two elements per thread as 16-byte loads (all four loads in flight): 5.0 -> 6+ TB/s
  double acc[1] = {0.0};
  const int64_t n2 = VEC ? n / 2 : 0;
  for (int64_t i = (int64_t)blockIdx.x * kTM + threadIdx.x; i < n2; i += (int64_t)gridDim.x * kTM) {
    const double2 gi = reinterpret_cast<const double2*>(g)[i], ri0 = reinterpret_cast<const double2*>(r)[i];
    const double2 ui = reinterpret_cast<const double2*>(u)[i], xi = reinterpret_cast<const double2*>(x)[i];
    const double2 ri = make_double2(fma(-a, gi.x, ri0.x), fma(-a, gi.y, ri0.y));
    reinterpret_cast<double2*>(r)[i] = ri;
    reinterpret_cast<double2*>(x)[i] = make_double2(fma(a, ui.x, xi.x), fma(a, ui.y, xi.y));
    acc[0] = fma(ri.x, ri.x, acc[0]);
    acc[0] = fma(ri.y, ri.y, acc[0]);
  }
  // the scalar remainder: the odd last element, or everything when a pointer is unaligned
  for (int64_t i = 2 * n2 + (int64_t)blockIdx.x * kTM + threadIdx.x; i < n; i += (int64_t)gridDim.x * kTM) {
    const double ri = fma(-a, g[i], r[i]);
    r[i] = ri;
    x[i] = fma(a, u[i], x[i]);
    acc[0] = fma(ri, ri, acc[0]);
  }
  reduce_finish<1>(acc, 1, partials, ticket, out, post, nullptr);
}

void launch_idr_update(int64_t n, double a, const double* g, const double* u, double* r, double* x,
                       double* partials, double* out, cudaStream_t s, CommBase* comm, const double* a_num,
                       const double* a_den) {
  ProfScope ps_(prof_name("idr_update", 1, AMG_F64, -1), 8.0 * n * 6, s);
  unsigned* ticket = reinterpret_cast<unsigned*>(partials + (size_t)kMaxPartials * 32);
  const int64_t work = (n + kTM - 1) / kTM;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)kMaxPartials, work));
  if (aligned16(g) && aligned16(u) && aligned16(r) && aligned16(x))
    k_idr_update<true><<<grid, kTM, 0, s>>>(n, a, g, u, r, x, partials, ticket, out, comm ? 0 : 1, a_num, a_den);
  else
    k_idr_update<false><<<grid, kTM, 0, s>>>(n, a, g, u, r, x, partials, ticket, out, comm ? 0 : 1, a_num, a_den);
  AMG_CK_LAUNCH();
  finalize_global(comm, out, 1, true, s);
}

// CG: p = z + beta p, beta = rz / rho from the device scalars (k_axpby's expression)
__global__ void __launch_bounds__(kT) k_cg_p(int64_t n, const double* __restrict__ z, double* __restrict__ p,
                                             const double* __restrict__ rz, const double* __restrict__ rho) {
  const double beta = rz[0] / rho[0];
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT)
    p[i] = (beta == 0.0) ? z[i] : fma(1.0, z[i], __dmul_rn(beta, p[i]));  // __dmul_rn: no contraction
}

void launch_cg_p(int64_t n, const double* z, double* p, const double* rz, const double* rho, cudaStream_t s) {
  ProfScope ps_(prof_name("axpby", 1, AMG_F64, -1), 24.0 * n, s);
  k_cg_p<<<ew_grid(n), kT, 0, s>>>(n, z, p, rz, rho);
  AMG_CK_LAUNCH();
}

// ---- BiCGStab fused steps (one pass, deterministic reductions, last-block finish) ----
// out = r - (num / den[0]) v;  dst[0] = out . out          (s = r - alpha v, alpha on the device)
__global__ void __launch_bounds__(kTM) k_sub_div_nrm(int64_t n, double num, const double* __restrict__ den,
                                                     const double* __restrict__ v, const double* __restrict__ r,
                                                     double* __restrict__ out, double* partials, unsigned* ticket,
                                                     double* dst) {
  const double a = num / den[0];
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * kTM + threadIdx.x; i < n; i += (int64_t)gridDim.x * kTM) {
    const double o = fma(-a, v[i], r[i]);
    out[i] = o;
    acc[0] = fma(o, o, acc[0]);
  }
  reduce_finish<1>(acc, 1, partials, ticket, dst, 0, nullptr);
}

// out = s - c t;  dst[0] = out . out,  dst[1] = rh . out     (r = s - omega t, next rho)
__global__ void __launch_bounds__(kTM) k_axpy_2dot(int64_t n, double c, const double* __restrict__ t,
                                                   const double* __restrict__ s, double* __restrict__ out,
                                                   const double* __restrict__ rh, double* partials, unsigned* ticket,
                                                   double* dst) {
  double acc[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * kTM + threadIdx.x; i < n; i += (int64_t)gridDim.x * kTM) {
    const double o = fma(-c, t[i], s[i]);
    out[i] = o;
    acc[0] = fma(o, o, acc[0]);
    acc[1] = fma(rh[i], o, acc[1]);
  }
  reduce_finish<2>(acc, 2, partials, ticket, dst, 0, nullptr);
}

static int fused_grid(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)kMaxPartials, (n + kTM - 1) / kTM));
}

void launch_sub_div_nrm(int64_t n, double num, const double* den, const double* v, const double* r, double* out,
                        double* partials, double* dst, cudaStream_t s, CommBase* comm) {
  ProfScope ps_(prof_name("sub_div_nrm", 1, AMG_F64, -1), 8.0 * n * 3, s);
  unsigned* ticket = reinterpret_cast<unsigned*>(partials + (size_t)kMaxPartials * 32);
  k_sub_div_nrm<<<fused_grid(n), kTM, 0, s>>>(n, num, den, v, r, out, partials, ticket, dst);
  AMG_CK_LAUNCH();
  finalize_global(comm, dst, 1, false, s);
}

void launch_axpy_2dot(int64_t n, double c, const double* t, const double* s_, double* out, const double* rh,
                      double* partials, double* dst, cudaStream_t s, CommBase* comm) {
  ProfScope ps_(prof_name("axpy_2dot", 2, AMG_F64, -1), 8.0 * n * 4, s);
  unsigned* ticket = reinterpret_cast<unsigned*>(partials + (size_t)kMaxPartials * 32);
  k_axpy_2dot<<<fused_grid(n), kTM, 0, s>>>(n, c, t, s_, out, rh, partials, ticket, dst);
  AMG_CK_LAUNCH();
  finalize_global(comm, dst, 2, false, s);
}


// ---- BiCGStab with device-side scalars (one CUDA graph per iteration, reading R24) ----
// Every scalar the iteration needs lives in BicgScal (device); the kernels compute alpha,
// beta and omega from it with the host code's own expressions, so the iterates are
// bit-identical to the host-driven loop.
__global__ void __launch_bounds__(kT) k_bicg_p(int64_t n, const double* __restrict__ r, const double* __restrict__ v,
                                               double* __restrict__ p, const double* __restrict__ sc) {
  const bool first = sc[kBicgFirst] != 0.0;
  const double beta = (sc[kBicgRho] / sc[kBicgRhoOld]) * (sc[kBicgAlpha] / sc[kBicgOmega]);
  const double b2 = -beta * sc[kBicgOmega];
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kT)
    p[i] = first ? r[i] : fma(1.0, r[i], fma(b2, v[i], beta * p[i]));
}

// alpha = rho / rv; s = r - alpha v; ss = s.s
__global__ void __launch_bounds__(kTM) k_bicg_s(int64_t n, const double* __restrict__ v, const double* __restrict__ r,
                                                double* __restrict__ sv, double* sc, double* partials,
                                                unsigned* ticket) {
  const double a = sc[kBicgRho] / sc[kBicgRv];
  double acc[1] = {0.0};
  for (int64_t i = (int64_t)blockIdx.x * kTM + threadIdx.x; i < n; i += (int64_t)gridDim.x * kTM) {
    const double o = fma(-a, v[i], r[i]);
    sv[i] = o;
    acc[0] = fma(o, o, acc[0]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) sc[kBicgAlphaNew] = a;
  reduce_finish<1>(acc, 1, partials, ticket, sc + kBicgSs, 0, nullptr);
}

// omega = ts / tt; x += alpha ph + omega sh (alpha ph only on the half-step exit ||s|| <=
// tol; nothing when rv or tt broke down); r = s - omega t with r.r and rh.r
__global__ void __launch_bounds__(kTM) k_bicg_xr(int64_t n, const double* __restrict__ ph,
                                                 const double* __restrict__ sh, const double* __restrict__ t,
                                                 const double* __restrict__ sv, const double* __restrict__ rh,
                                                 double* __restrict__ x, double* __restrict__ r, double* sc,
                                                 double* partials, unsigned* ticket) {
  const double rv = sc[kBicgRv], tt = sc[kBicgTt];
  const double alpha = sc[kBicgAlphaNew];
  const bool rv_ok = rv != 0.0 && isfinite(rv);
  const bool half = rv_ok && sqrt(sc[kBicgSs]) <= sc[kBicgTol];
  const bool tt_ok = tt != 0.0 && isfinite(tt);
  const double omega = sc[kBicgTs] / tt;
  double acc[2] = {0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * kTM + threadIdx.x; i < n; i += (int64_t)gridDim.x * kTM) {
    if (half) {
      x[i] = fma(alpha, ph[i], 1.0 * x[i]);
    } else if (rv_ok && tt_ok) {
      x[i] = fma(alpha, ph[i], fma(omega, sh[i], 1.0 * x[i]));
      const double o = fma(-omega, t[i], sv[i]);
      r[i] = o;
      acc[0] = fma(o, o, acc[0]);
      acc[1] = fma(rh[i], o, acc[1]);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && rv_ok && tt_ok && !half) sc[kBicgOmegaNew] = omega;
  reduce_finish<2>(acc, 2, partials, ticket, sc + kBicgRr, 0, nullptr);
}

void launch_bicg_p(int64_t n, const double* r, const double* v, double* p, const double* sc, cudaStream_t s) {
  ProfScope ps_(prof_name("bicg_p", 1, AMG_F64, -1), 32.0 * n, s);
  k_bicg_p<<<ew_grid(n), kT, 0, s>>>(n, r, v, p, sc);
  AMG_CK_LAUNCH();
}

void launch_bicg_s(int64_t n, const double* v, const double* r, double* sv, double* sc, double* partials,
                   cudaStream_t s, CommBase* comm) {
  ProfScope ps_(prof_name("sub_div_nrm", 1, AMG_F64, -1), 8.0 * n * 3, s);
  unsigned* ticket = reinterpret_cast<unsigned*>(partials + (size_t)kMaxPartials * 32);
  k_bicg_s<<<fused_grid(n), kTM, 0, s>>>(n, v, r, sv, sc, partials, ticket);
  AMG_CK_LAUNCH();
  finalize_global(comm, sc + kBicgSs, 1, false, s);
}

void launch_bicg_xr(int64_t n, const double* ph, const double* sh, const double* t, const double* sv,
                    const double* rh, double* x, double* r, double* sc, double* partials, cudaStream_t s,
                    CommBase* comm) {
  ProfScope ps_(prof_name("bicg_xr", 2, AMG_F64, -1), 8.0 * n * 8, s);
  unsigned* ticket = reinterpret_cast<unsigned*>(partials + (size_t)kMaxPartials * 32);
  k_bicg_xr<<<fused_grid(n), kTM, 0, s>>>(n, ph, sh, t, sv, rh, x, r, sc, partials, ticket);
  AMG_CK_LAUNCH();
  finalize_global(comm, sc + kBicgRr, 2, false, s);
}

}  // namespace amgb
