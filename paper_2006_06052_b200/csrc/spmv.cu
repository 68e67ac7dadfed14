// spmv.cu -- instantiation + dispatch of the SpMV-type solve kernels (K1, K2, K4, K5,
// K8, K9, K10, K11).  See bsr.cuh for the block-row design.
#include <cstdlib>

#include "bsr.cuh"
#include "ops.h"
#include "prof.h"

namespace amgb {

int64_t g_schur_nnz = 0;  // nnz of the Schur B / B^T pattern (set by setup)

namespace {

constexpr int kBlock = 256;

template <typename F>
void dispatch_t(int dt, F&& f) {
  if (dt == AMG_F32) f(float{});
  else if (dt == AMG_F64) f(double{});
  else fail(AMG_EINVAL, "bad dtype");
}

template <typename F>
void dispatch_b(int b, F&& f) {
  switch (b) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    default: fail(AMG_EINVAL, "block size must be 1..4");
  }
}

template <typename F>
void dispatch_g(int G, F&& f) {
  if (G == 32) f(std::integral_constant<int, 32>{});
  else f(std::integral_constant<int, 8>{});
}

double mat_bytes(const Mat& A) {  // algorithmic bytes of one pass over A
  return (double)A.nnz * (4.0 + (double)A.b * A.b * dtype_size(A.vt)) + 4.0 * (A.n + 1);
}

}  // namespace

void launch_spmv(const Mat& A, double alpha, const void* x, int xt, double beta, void* y, int yt,
                 cudaStream_t s) {
  if (A.n == 0) return;
  ProfScope ps_(prof_name("spmv", A.b, A.vt, xt),
                mat_bytes(A) + (double)A.m * A.b * dtype_size(xt) +
                    (double)A.n * A.b * dtype_size(yt) * (beta != 0.0 ? 2.0 : 1.0), s);
  dispatch_b(A.b, [&](auto Bc) {
    constexpr int B = decltype(Bc)::value;
    dispatch_g(A.G, [&](auto Gc) {
      constexpr int G = decltype(Gc)::value;
      dispatch_t(A.vt, [&](auto v) {
        using V = decltype(v);
        dispatch_t(xt, [&](auto xx) {
          using X = decltype(xx);
          dispatch_t(yt, [&](auto yy) {
            using Y = decltype(yy);
            static int variant = getenv("AMG_SPMV_V") ? atoi(getenv("AMG_SPMV_V")) : 0;
            if (variant == 1)
              k_spmv<B, G, V, X, Y, 1><<<grid_for((int64_t)A.n * G, kBlock), kBlock, 0, s>>>(
                  A.n, A.ptr, A.col, (const V*)A.val, alpha, (const X*)x, beta, (Y*)y);
            else
              k_spmv<B, G, V, X, Y, 0><<<grid_for((int64_t)A.n * G, kBlock), kBlock, 0, s>>>(
                  A.n, A.ptr, A.col, (const V*)A.val, alpha, (const X*)x, beta, (Y*)y);
          });
        });
      });
    });
  });
  AMG_CK_LAUNCH();
}

void launch_residual(const Mat& A, const void* f, const void* x, void* r, int xt, cudaStream_t s) {
  if (A.n == 0) return;
  ProfScope ps_(prof_name("residual", A.b, A.vt, xt),
                mat_bytes(A) + (double)A.m * A.b * dtype_size(xt) + 2.0 * A.n * A.b * dtype_size(xt), s);
  dispatch_b(A.b, [&](auto Bc) {
    constexpr int B = decltype(Bc)::value;
    dispatch_g(A.G, [&](auto Gc) {
      constexpr int G = decltype(Gc)::value;
      dispatch_t(A.vt, [&](auto v) {
        using V = decltype(v);
        dispatch_t(xt, [&](auto xx) {
          using X = decltype(xx);
          k_residual<B, G, V, X><<<grid_for((int64_t)A.n * G, kBlock), kBlock, 0, s>>>(
              A.n, A.ptr, A.col, (const V*)A.val, (const X*)f, (const X*)x, (X*)r);
        });
      });
    });
  });
  AMG_CK_LAUNCH();
}

void launch_smooth(const Mat& A, const void* M, const void* f, const void* x, void* xo, int xt,
                   cudaStream_t s) {
  if (A.n == 0) return;
  ProfScope ps_(prof_name("smooth", A.b, A.vt, xt),
                mat_bytes(A) + (double)A.n * A.b * A.b * dtype_size(A.vt) + 3.0 * A.n * A.b * dtype_size(xt), s);
  dispatch_b(A.b, [&](auto Bc) {
    constexpr int B = decltype(Bc)::value;
    dispatch_g(A.G, [&](auto Gc) {
      constexpr int G = decltype(Gc)::value;
      dispatch_t(A.vt, [&](auto v) {
        using V = decltype(v);
        dispatch_t(xt, [&](auto xx) {
          using X = decltype(xx);
          k_smooth<B, G, V, X><<<grid_for((int64_t)A.n * G, kBlock), kBlock, 0, s>>>(
              A.n, A.ptr, A.col, (const V*)A.val, (const V*)M, (const X*)f, (const X*)x, (X*)xo);
        });
      });
    });
  });
  AMG_CK_LAUNCH();
}

void launch_apply_M(int32_t n, int b, const void* M, int vt, const void* f, void* x, int xt,
                    cudaStream_t s) {
  if (n == 0) return;
  ProfScope ps_(prof_name("apply_M", b, vt, xt), (double)n * b * b * dtype_size(vt) + 2.0 * n * b * dtype_size(xt), s);
  dispatch_b(b, [&](auto Bc) {
    constexpr int B = decltype(Bc)::value;
    dispatch_t(vt, [&](auto v) {
      using V = decltype(v);
      dispatch_t(xt, [&](auto xx) {
        using X = decltype(xx);
        k_apply_M<B, V, X><<<grid_for((int64_t)n * B, kBlock), kBlock, 0, s>>>(n, (const V*)M, (const X*)f,
                                                                              (X*)x);
      });
    });
  });
  AMG_CK_LAUNCH();
}

// ---- K8: coarse solve as a dense GEMV with the explicit inverse (one warp per row) ----
template <typename V, typename X>
__global__ void __launch_bounds__(256) k_dense_gemv(int N, const V* __restrict__ A, const X* __restrict__ f,
                                                    X* __restrict__ x) {
  const int warp = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (warp >= N) return;
  const V* row = A + (int64_t)warp * N;
  double s = 0.0;
  for (int j = lane; j < N; j += 32) s = fma((double)__ldg(row + j), (double)__ldg(f + j), s);
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
  if (lane == 0) x[warp] = to_out<X>(s);
}

void launch_dense_gemv(int32_t N, const void* Ainv, int vt, const void* f, void* x, int xt,
                       cudaStream_t s) {
  if (N == 0) return;
  ProfScope ps_(prof_name("coarse_gemv", 1, vt, xt), (double)N * N * dtype_size(vt) + 2.0 * N * dtype_size(xt), s);
  dispatch_t(vt, [&](auto v) {
    using V = decltype(v);
    dispatch_t(xt, [&](auto xx) {
      using X = decltype(xx);
      k_dense_gemv<V, X><<<grid_for((int64_t)N * 32, 256), 256, 0, s>>>(N, (const V*)Ainv, (const X*)f, (X*)x);
    });
  });
  AMG_CK_LAUNCH();
}

// ---- K10: p = m_S o (r_p - B u*) ; items = blocks of the row, NU values each ----
template <int NU, int G, typename V, typename X>
__global__ void __launch_bounds__(256) k_schur_p(int n, const int32_t* __restrict__ ptr,
                                                 const int32_t* __restrict__ col, const V* __restrict__ Bv,
                                                 const V* __restrict__ mS, const X* __restrict__ rp,
                                                 const X* __restrict__ us, X* __restrict__ p) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gid / G), gl = threadIdx.x & (G - 1);
  const bool valid = row < n;
  double acc = 0.0;
  if (valid) {
    const int k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
    for (int k = k0 + gl; k < k1; k += G) {
      const int c = __ldg(col + k);
      double bv[NU], uv[NU];
      load_b<NU, true>(Bv + (int64_t)k * NU, bv);
      load_b<NU, false>(us + (int64_t)c * NU, uv);
#pragma unroll
      for (int d = 0; d < NU; ++d) acc = fma(bv[d], uv[d], acc);
    }
  }
#pragma unroll
  for (int off = G / 2; off >= 1; off >>= 1) acc += __shfl_xor_sync(kFull, acc, off, G);
  if (valid && gl == 0) p[row] = to_out<X>((double)mS[row] * ((double)rp[row] - acc));
}

// ---- K11: r_u' = r_u - B^T p ; items = (block k, velocity comp d), one value each ----
template <int NU, int G, typename V, typename X>
__global__ void __launch_bounds__(256) k_schur_u(int n, const int32_t* __restrict__ ptr,
                                                 const int32_t* __restrict__ col, const V* __restrict__ BTv,
                                                 const X* ru, const X* __restrict__ p,
                                                 X* ru2) {  // ru2 may alias ru (in-place update)
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gid / G), gl = threadIdx.x & (G - 1);
  const bool valid = row < n;
  double acc[NU] = {};
  if (valid) {
    const int k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
    const int nitems = (k1 - k0) * NU;
    for (int t = gl; t < nitems; t += G) {
      const int k = k0 + t / NU, d = t % NU;
      const double v = (double)__ldcs(BTv + (int64_t)k0 * NU + t) * (double)__ldg(p + __ldg(col + k));
#pragma unroll
      for (int dd = 0; dd < NU; ++dd)
        if (dd == d) acc[dd] += v;
    }
  }
  double y[NU];
#pragma unroll
  for (int d = 0; d < NU; ++d) {
    double v = acc[d];
#pragma unroll
    for (int off = G / 2; off >= 1; off >>= 1) v += __shfl_xor_sync(kFull, v, off, G);
    y[d] = v;
  }
  if (valid && gl < NU) {
    const int64_t o = (int64_t)row * NU + gl;
    double yy = y[0];
#pragma unroll
    for (int d = 1; d < NU; ++d)
      if (d == gl) yy = y[d];
    ru2[o] = to_out<X>((double)ru[o] - yy);
  }
}

void launch_schur_p(int32_t n, int nu, const int32_t* ptr, const int32_t* col, const void* Bv,
                    const void* mS, int vt, const void* rp, const void* us, void* p, int xt, int G,
                    cudaStream_t s) {
  if (n == 0) return;
  if (nu != 3) fail(AMG_EINVAL, "Schur split supports 3 velocity components");
  ProfScope ps_(prof_name("schur_p", 3, vt, xt),
                ((double)g_schur_nnz * (4.0 + 3.0 * dtype_size(vt)) + 4.0 * (n + 1)) + (double)n * dtype_size(vt) + 5.0 * n * dtype_size(xt), s);
  dispatch_g(G, [&](auto Gc) {
    constexpr int GG = decltype(Gc)::value;
    dispatch_t(vt, [&](auto v) {
      using V = decltype(v);
      dispatch_t(xt, [&](auto xx) {
        using X = decltype(xx);
        k_schur_p<3, GG, V, X><<<grid_for((int64_t)n * GG, 256), 256, 0, s>>>(
            n, ptr, col, (const V*)Bv, (const V*)mS, (const X*)rp, (const X*)us, (X*)p);
      });
    });
  });
  AMG_CK_LAUNCH();
}

void launch_schur_u(int32_t n, int nu, const int32_t* ptr, const int32_t* col, const void* BTv, int vt,
                    const void* ru, const void* p, void* ru2, int xt, int G, cudaStream_t s) {
  if (n == 0) return;
  if (nu != 3) fail(AMG_EINVAL, "Schur split supports 3 velocity components");
  ProfScope ps_(prof_name("schur_u", 3, vt, xt), ((double)g_schur_nnz * (4.0 + 3.0 * dtype_size(vt)) + 4.0 * (n + 1)) + 7.0 * n * dtype_size(xt), s);
  dispatch_g(G, [&](auto Gc) {
    constexpr int GG = decltype(Gc)::value;
    dispatch_t(vt, [&](auto v) {
      using V = decltype(v);
      dispatch_t(xt, [&](auto xx) {
        using X = decltype(xx);
        k_schur_u<3, GG, V, X><<<grid_for((int64_t)n * GG, 256), 256, 0, s>>>(
            n, ptr, col, (const V*)BTv, (const X*)ru, (const X*)p, (X*)ru2);
      });
    });
  });
  AMG_CK_LAUNCH();
}

// ---- K9: split / join of the interleaved outer vector ----
template <typename X>
__global__ void k_split(int n, int b, int pc, const double* __restrict__ r, double scale, X* __restrict__ ru,
                        X* __restrict__ rp) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * b) return;
  const int64_t I = t / b;
  const int c = (int)(t % b);
  const double v = r[t] * scale;
  if (c == pc) rp[I] = to_out<X>(v);
  else ru[I * (b - 1) + (c < pc ? c : c - 1)] = to_out<X>(v);
}

template <typename X, typename Z>
__global__ void k_join(int n, int b, int pc, const X* __restrict__ u, const X* __restrict__ p,
                       Z* __restrict__ z) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * b) return;
  const int64_t I = t / b;
  const int c = (int)(t % b);
  z[t] = (Z)((c == pc) ? p[I] : u[I * (b - 1) + (c < pc ? c : c - 1)]);
}

template <typename I, typename O>
__global__ void k_convert(int64_t N, const I* __restrict__ in, O* __restrict__ out, double scale) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = to_out<O>((double)in[t] * scale);
}

void launch_split(int32_t n, int b, int pc, const double* r, double scale, void* ru, void* rp, int xt,
                  cudaStream_t s) {
  if (n == 0) return;
  ProfScope ps_(prof_name("split", b, AMG_F64, xt), (double)n * b * (8.0 + dtype_size(xt)), s);
  dispatch_t(xt, [&](auto xx) {
    using X = decltype(xx);
    k_split<X><<<grid_for((int64_t)n * b, 256), 256, 0, s>>>(n, b, pc, r, scale, (X*)ru, (X*)rp);
  });
  AMG_CK_LAUNCH();
}

void launch_join(int32_t n, int b, int pc, const void* u, const void* p, int xt, void* z, int zt, cudaStream_t s) {
  if (n == 0) return;
  ProfScope ps_(prof_name("join", b, zt, xt), (double)n * b * (dtype_size(zt) + dtype_size(xt)), s);
  dispatch_t(xt, [&](auto xx) {
    using X = decltype(xx);
    dispatch_t(zt, [&](auto zz) {
      using Z = decltype(zz);
      k_join<X, Z><<<grid_for((int64_t)n * b, 256), 256, 0, s>>>(n, b, pc, (const X*)u, (const X*)p, (Z*)z);
    });
  });
  AMG_CK_LAUNCH();
}

void launch_convert(int64_t N, const void* in, int it, void* out, int ot, double scale, cudaStream_t s) {
  if (N == 0) return;
  ProfScope ps_(prof_name("convert", 1, ot, it), (double)N * (dtype_size(it) + dtype_size(ot)), s);
  unsigned g = grid_for(N, 256);
  if (g > 148u * 16u) g = 148u * 16u;
  dispatch_t(it, [&](auto ii) {
    using I = decltype(ii);
    dispatch_t(ot, [&](auto oo) {
      using O = decltype(oo);
      k_convert<I, O><<<g, 256, 0, s>>>(N, (const I*)in, (O*)out, scale);
    });
  });
  AMG_CK_LAUNCH();
}

}  // namespace amgb
