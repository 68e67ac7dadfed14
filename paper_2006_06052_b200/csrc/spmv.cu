// spmv.cu -- instantiation + dispatch of the SpMV-type solve kernels (K1, K2, K4, K5,
// K8, K9, K10, K11).  See bsr.cuh for the block-row design.
#include <algorithm>
#include <cstdlib>

#include "bsr.cuh"
#include "bsr_tma.cuh"
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


// ---------------------------------------------------------------- TMA tile plans
__global__ void k_tile_max(int n, int tr, const int32_t* ptr, int* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t * (int64_t)tr >= n) return;
  const int r0 = t * tr, r1 = min(r0 + tr, n);
  atomicMax(out, ptr[r1] - ptr[r0]);
}

template <int B, int G, typename V, typename X, bool FAST, class EPI>
static void launch_tma_f(const Mat& A, const X* x, EPI epi, cudaStream_t s) {
  TmaArgs a{A.n, A.tma_tr, A.tma_ntiles, A.tma_ns, A.tma_stage, A.tma_col_off, A.tma_val_off};
  const int smem = A.tma_ns * A.tma_stage;
  if (A.tma_rows) {
    static int configured_r = 48 * 1024;
    if (smem > configured_r) {
      AMG_CK(cudaFuncSetAttribute(k_bsr_tma_rows<B, V, X, FAST, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      configured_r = smem;
    }
    k_bsr_tma_rows<B, V, X, FAST, EPI><<<A.tma_grid, A.tma_tr, smem, s>>>(a, A.ptr, A.col, (const V*)A.val, x, epi);
    return;
  }
  static int configured = 48 * 1024;
  if (smem > configured) {
    AMG_CK(cudaFuncSetAttribute(k_bsr_tma<B, G, V, X, FAST, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = smem;
  }
  k_bsr_tma<B, G, V, X, FAST, EPI><<<A.tma_grid, 256, smem, s>>>(a, A.ptr, A.col, (const V*)A.val, x, epi);
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

void make_tma_plan(Mat& A, cudaStream_t s) {
  A.tma_grid = 0;
  A.tma_rows = false;
  if (A.n < 2048 || env_int("AMG_NO_TMA", 0)) return;
  if (A.vt == AMG_F64 && !env_int("AMG_TMA_F64", 0)) return;  // direct kernels stream fp64 blocks at ~95 %
  const double bb = (double)A.b * A.b * dtype_size(A.vt) + 4.0;
  const double row_bytes = std::max(1.0, (double)A.nnz / A.n * bb);
  // row-per-lane mode for short rows (<= 12 blocks) when a 128-row tile fits a stage
  const int mode_rows = env_int("AMG_TMA_ROWS", 1) && (double)A.nnz / A.n <= 12.0 && 128 * row_bytes <= 40 * 1024;
  int tr = 4;
  while (tr < 256 && tr * 2 * row_bytes <= env_int("AMG_TMA_TILE_BYTES", 16384)) tr *= 2;
  if (mode_rows) tr = env_int("AMG_TMA_ROWS_TR", 128);
  const int ntiles = (int)((A.n + tr - 1) / tr);
  int* d = nullptr;
  AMG_CK(cudaMallocAsync((void**)&d, sizeof(int), s));
  AMG_CK(cudaMemsetAsync(d, 0, sizeof(int), s));
  k_tile_max<<<grid_for(ntiles, 256), 256, 0, s>>>(A.n, tr, A.ptr, d);
  AMG_CK_LAUNCH();
  int mx = 0;
  AMG_CK(cudaMemcpyAsync(&mx, d, sizeof(int), cudaMemcpyDeviceToHost, s));
  AMG_CK(cudaFreeAsync(d, s));
  AMG_CK(cudaStreamSynchronize(s));
  auto a16 = [](int64_t v) { return (int)((v + 15) & ~int64_t(15)); };
  const int pbytes = a16(4LL * (tr + 1) + 32);
  const int cbytes = a16(4LL * mx + 32);
  const int64_t vbytes64 = (int64_t)mx * A.b * A.b * dtype_size(A.vt) + 32;
  if (vbytes64 > 96 * 1024) return;  // pathological rows: direct kernels
  const int stage = pbytes + cbytes + a16(vbytes64);
  const int ns = env_int("AMG_TMA_NS", mode_rows ? 3 : (stage > 40 * 1024 ? 2 : 3));
  const int budget = 220 * 1024;
  int per_sm = budget / (ns * stage);
  const int cap = mode_rows ? std::min(32, 2048 / tr) : 4;
  if (per_sm > cap) per_sm = cap;
  if (per_sm < 1) return;
  A.tma_rows = mode_rows;
  A.tma_tr = tr;
  A.tma_ntiles = ntiles;
  A.tma_ns = ns;
  A.tma_stage = stage;
  A.tma_col_off = pbytes;
  A.tma_val_off = pbytes + cbytes;
  A.tma_grid = std::min(ntiles, kSMs * per_sm);
}

template <int B, int G, typename V, typename X, class EPI>
static void launch_tma(const Mat& A, const X* x, EPI epi, cudaStream_t s) {
  if (A.fast32) launch_tma_f<B, G, V, X, true>(A, x, epi, s);
  else launch_tma_f<B, G, V, X, false>(A, x, epi, s);
}

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
            if (A.tma_grid > 0)
              launch_tma<B, G, V, X>(A, (const X*)x, EpiSpmv<B, Y>{alpha, beta, (Y*)y}, s);
            else
              k_spmv<B, G, V, X, Y><<<grid_for((int64_t)A.n * G, kBlock), kBlock, 0, s>>>(
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
          if (A.tma_grid > 0)
            launch_tma<B, G, V, X>(A, (const X*)x, EpiResidual<B, X>{(const X*)f, (X*)r}, s);
          else
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
          if (A.tma_grid > 0)
            launch_tma<B, G, V, X>(A, (const X*)x, EpiSmooth<B, V, X>{(const V*)M, (const X*)f, (const X*)x, (X*)xo}, s);
          else
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
