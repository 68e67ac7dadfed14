// bsr_lane.cuh -- "row-component lanes": the default SpMV-type kernels (K1 SpMV, K2
// residual, K5 smoother, K6/K7 restriction/prolongation, K10/K11 Schur products).
//
// BR lanes own one block row: lane r accumulates (A x)_{row, r} on its own, so there
// is no cross-lane reduction and the epilogue store of a warp is contiguous; a warp
// covers 32/BR consecutive block rows (32 % BR lanes idle).  Each lane walks the row's
// blocks with U blocks per step: the U column indices and the U block-row segments
// are loaded first, then the U x gathers, then the arithmetic -- every load of a step
// is in flight at once.  Two value layouts:
//   ROWS  lane r reads row r of every block (BC contiguous values: one 16-byte load for
//         4 fp32 values, two for 4 fp64) and the BC-vector x_col;
//   COLS  lane r reads column r of every block (values i*B + r: at each i the BR lanes
//         read consecutive words) and the single value x_col[r]; partial sums acc[i]
//         for every i, combined across the row's lanes at the end (transpose-reduce).
// Value loads are cache-streaming (ld.global.cs: read once, evict first) or, where the
// lanes' pieces share 32-byte sectors (3x3 fp32), L1-allocating (ld.global.nc).
// Measured on B200 (tools/spmv_lab.cu, cfg-2 27-point 128^3): 4x4 fp32 x fp64 5.49 TB/s,
// 4x4 fp64 6.08 TB/s (7-point 256^3: 6.60), 3x3 fp32 COLS 4.60 TB/s; the 7-point 3x3
// fp32 ROWS+nc 5.13 TB/s -- ahead of the TMA-staged consumers (bsr_tma.cuh) in every case.
// Arithmetic: fp64 accumulation, one rounding on store; FAST
// (fp32 hierarchy x fp32 vectors, the V-cycle's float backend) forms each block-row dot
// in fp32 before adding it in fp64.
#pragma once

#include "bsr.cuh"
#include "reduce.cuh"

namespace amgb {

template <bool NC, typename T>
__device__ __forceinline__ T ld_val(const T* p) {
  if constexpr (NC) return __ldg(p);
  else return __ldcs(p);
}

// n contiguous values (row segment of a block): vector loads where 16-B aligned
template <int N, bool NC, typename T>
__device__ __forceinline__ void ld_seg(const T* __restrict__ p, T (&v)[N]) {
  if constexpr (N == 4 && std::is_same_v<T, float>) {
    const float4 q = NC ? __ldg(reinterpret_cast<const float4*>(p)) : __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else if constexpr (N == 4 && std::is_same_v<T, double>) {
    const double2* q = reinterpret_cast<const double2*>(p);
    const double2 a = NC ? __ldg(q) : __ldcs(q), c = NC ? __ldg(q + 1) : __ldcs(q + 1);
    v[0] = a.x; v[1] = a.y; v[2] = c.x; v[3] = c.y;
  } else if constexpr (N == 2 && std::is_same_v<T, double>) {
    const double2 a = NC ? __ldg(reinterpret_cast<const double2*>(p)) : __ldcs(reinterpret_cast<const double2*>(p));
    v[0] = a.x; v[1] = a.y;
  } else {
#pragma unroll
    for (int c = 0; c < N; ++c) v[c] = ld_val<NC>(p + c);
  }
}

template <int BC, bool NC, typename T>
__device__ __forceinline__ void ld_row(const T* __restrict__ p, T (&v)[BC]) {
  if constexpr (BC == 3 && std::is_same_v<T, float>) ld3f<NC>(p, v);
  else ld_seg<BC, NC>(p, v);
}
template <int BC, typename T>
__device__ __forceinline__ void ld_x(const T* __restrict__ p, T (&v)[BC]) {
  if constexpr (BC == 3 && std::is_same_v<T, float>) ld3f<true>(p, v);
  else load_raw<BC, false>(p, v);
}

// Row-component lane context handed to the epilogue: y_r = (A x)_{row, r}; all()
// gathers the row's full BR-vector from its lanes (warp shuffles, every lane of the
// warp must call it).
template <int BR>
struct LaneRow {
  int row, r, base;  // block row, component, lane of component 0
  bool valid;
  double yr;
  __device__ __forceinline__ void all(double (&y)[BR]) const {
#pragma unroll
    for (int c = 0; c < BR; ++c) y[c] = __shfl_sync(kFull, yr, base + c);
  }
};

// ---------------------------------------------------------------- epilogues
template <typename Y>
struct LEpiSpmv {  // y = alpha A x + beta y
  static constexpr int kDots = 0;
  double alpha, beta;
  Y* y;
  template <int BR>
  __device__ __forceinline__ void operator()(const LaneRow<BR>& L) const {
    if (!L.valid) return;
    const int64_t o = (int64_t)L.row * BR + L.r;
    double v = alpha * L.yr;
    if (beta != 0.0) v = fma(beta, (double)y[o], v);
    y[o] = to_out<Y>(v);
  }
  // row-per-lane form (k_bsr_sellr): the lane holds the row's BR results
  template <int BR>
  __device__ __forceinline__ void row(int row, const double (&yr)[BR]) const {
    const int64_t o = (int64_t)row * BR;
    double v[BR];
#pragma unroll
    for (int c = 0; c < BR; ++c) v[c] = beta != 0.0 ? (double)y[o + c] : 0.0;
#pragma unroll
    for (int c = 0; c < BR; ++c) {
      double t = alpha * yr[c];
      if (beta != 0.0) t = fma(beta, v[c], t);
      y[o + c] = to_out<Y>(t);
    }
  }
};

// y = A x + y (beta = 1: the prolongation K7) with y[row] loaded BEFORE the row's blocks
// (k_bsr_sellr only): short-row matrices (P_0: 3.6 blocks per row, two steps) are latency
// bound on their chain of dependent loads, and the epilogue's y load is independent of it
template <typename Y>
struct LEpiSpmvPre : LEpiSpmv<Y> {
  static constexpr bool kPre = true;
  using PreT = Y;
  template <int BR>
  __device__ __forceinline__ void pre(int row, Y (&v)[BR]) const {
#pragma unroll
    for (int c = 0; c < BR; ++c) v[c] = this->y[(int64_t)row * BR + c];
  }
  template <int BR>
  __device__ __forceinline__ void row_pre(int row, const double (&yr)[BR], const Y (&v)[BR]) const {
    const int64_t o = (int64_t)row * BR;
#pragma unroll
    for (int c = 0; c < BR; ++c) this->y[o + c] = to_out<Y>(fma(this->beta, (double)v[c], this->alpha * yr[c]));
  }
};
template <class E, class = void>
struct EpiPre : std::false_type {};
template <class E>
struct EpiPre<E, std::void_t<decltype(E::kPre)>> : std::true_type {};
template <class E, bool P = EpiPre<E>::value>
struct EpiPreT {
  using type = char;
};
template <class E>
struct EpiPreT<E, true> {
  using type = typename E::PreT;
};

template <typename X>
struct LEpiResidual {  // r = f - A x
  static constexpr int kDots = 0;
  const X* f;
  X* res;
  template <int BR>
  __device__ __forceinline__ void operator()(const LaneRow<BR>& L) const {
    if (!L.valid) return;
    const int64_t o = (int64_t)L.row * BR + L.r;
    res[o] = to_out<X>((double)f[o] - L.yr);
  }
  template <int BR>
  __device__ __forceinline__ void row(int row, const double (&yr)[BR]) const {
    const int64_t o = (int64_t)row * BR;
    double fv[BR];
#pragma unroll
    for (int c = 0; c < BR; ++c) fv[c] = (double)f[o + c];
#pragma unroll
    for (int c = 0; c < BR; ++c) res[o + c] = to_out<X>(fv[c] - yr[c]);
  }
};

template <typename V, typename X>
struct LEpiSmooth {  // xo = x + M (f - A g), M block-diagonal; g the gathered vector (usually x)
  static constexpr int kDots = 0;
  const V* M;
  const X* f;
  const X* x;
  X* xo;
  template <int BR>
  __device__ __forceinline__ void operator()(const LaneRow<BR>& L) const {
    const int64_t o = (int64_t)L.row * BR + L.r;
    const double res = L.valid ? (double)f[o] - L.yr : 0.0;
    double rv[BR];
#pragma unroll
    for (int c = 0; c < BR; ++c) rv[c] = __shfl_sync(kFull, res, L.base + c);
    if (!L.valid) return;
    double m[BR];
    load_b<BR, false>(M + o * BR, m);
    double t = m[0] * rv[0];
#pragma unroll
    for (int c = 1; c < BR; ++c) t = fma(m[c], rv[c], t);
    xo[o] = to_out<X>((x ? (double)x[o] : 0.0) + t);  // x == nullptr: from zero (ILU(0) U sweeps)
  }
  template <int BR>
  __device__ __forceinline__ void row(int row, const double (&yr)[BR]) const {
    const int64_t o = (int64_t)row * BR;
    double rv[BR], xv[BR], m[BR][BR];
#pragma unroll
    for (int c = 0; c < BR; ++c) rv[c] = (double)f[o + c] - yr[c], xv[c] = x ? (double)x[o + c] : 0.0;
#pragma unroll
    for (int i = 0; i < BR; ++i) load_b<BR, false>(M + (o + i) * BR, m[i]);
#pragma unroll
    for (int i = 0; i < BR; ++i) {
      double t = m[i][0] * rv[0];
#pragma unroll
      for (int c = 1; c < BR; ++c) t = fma(m[i][c], rv[c], t);
      xo[o + i] = to_out<X>(xv[i] + t);
    }
  }
};

// The monolithic preconditioner's last post-smoothing step with the widening of its output
// (C9: the fp32 V-cycle result widened exactly into the outer fp64 z) in its epilogue:
// x + M (f - A x) rounded to X as LEpiSmooth stores it, then stored widened into z -- the
// values LEpiSmooth + k_convert would store, without the x round trip
template <typename V, typename X, typename Z>
struct LEpiSmoothWiden {
  static constexpr int kDots = 0;
  const V* M;
  const X* f;
  const X* x;
  Z* z;
  template <int BR>
  __device__ __forceinline__ void operator()(const LaneRow<BR>& L) const {
    const int64_t o = (int64_t)L.row * BR + L.r;
    const double res = L.valid ? (double)f[o] - L.yr : 0.0;
    double rv[BR];
#pragma unroll
    for (int c = 0; c < BR; ++c) rv[c] = __shfl_sync(kFull, res, L.base + c);
    if (!L.valid) return;
    double m[BR];
    load_b<BR, false>(M + o * BR, m);
    double t = m[0] * rv[0];
#pragma unroll
    for (int c = 1; c < BR; ++c) t = fma(m[c], rv[c], t);
    z[o] = (Z)to_out<X>((double)x[o] + t);
  }
  template <int BR>
  __device__ __forceinline__ void row(int row, const double (&yr)[BR]) const {
    const int64_t o = (int64_t)row * BR;
    double rv[BR], xv[BR], m[BR][BR];
#pragma unroll
    for (int c = 0; c < BR; ++c) rv[c] = (double)f[o + c] - yr[c], xv[c] = (double)x[o + c];
#pragma unroll
    for (int i = 0; i < BR; ++i) load_b<BR, false>(M + (o + i) * BR, m[i]);
#pragma unroll
    for (int i = 0; i < BR; ++i) {
      double t = m[i][0] * rv[0];
#pragma unroll
      for (int c = 1; c < BR; ++c) t = fma(m[i][c], rv[c], t);
      z[o + i] = (Z)to_out<X>(xv[i] + t);
    }
  }
};

// The last post-smoothing step of the Schur preconditioner's second U-solve with the join
// (K9') in its epilogue: xo = x + M (f - A x) is stored straight into the output z as the
// velocity slots of the interleaved (u, v, w, p) cells, with p[row] in slot 3 -- the values
// LEpiSmooth + k_join4 would store (same expressions), without the u round trip
template <typename V, typename X, typename Z>
struct LEpiSmoothJoin {
  static constexpr int kDots = 0;
  const V* M;
  const X* f;
  const X* x;
  const X* p;
  Z* z;
  template <int BR>
  __device__ __forceinline__ void operator()(const LaneRow<BR>& L) const {
    static_assert(BR == 3, "join: 3 velocity components + p");
    const int64_t o = (int64_t)L.row * BR + L.r;
    const double res = L.valid ? (double)f[o] - L.yr : 0.0;
    double rv[BR];
#pragma unroll
    for (int c = 0; c < BR; ++c) rv[c] = __shfl_sync(kFull, res, L.base + c);
    if (!L.valid) return;
    double m[BR];
    load_b<BR, false>(M + o * BR, m);
    double t = m[0] * rv[0];
#pragma unroll
    for (int c = 1; c < BR; ++c) t = fma(m[c], rv[c], t);
    const X u = to_out<X>((double)x[o] + t);
    z[(int64_t)L.row * 4 + L.r] = (Z)u;
    if (L.r == 0) z[(int64_t)L.row * 4 + 3] = (Z)p[L.row];
  }
  template <int BR>
  __device__ __forceinline__ void row(int row, const double (&yr)[BR]) const {
    static_assert(BR == 3, "join: 3 velocity components + p");
    const int64_t o = (int64_t)row * BR;
    double rv[BR], xv[BR], m[BR][BR];
#pragma unroll
    for (int c = 0; c < BR; ++c) rv[c] = (double)f[o + c] - yr[c], xv[c] = (double)x[o + c];
    const X pv = p[row];
#pragma unroll
    for (int i = 0; i < BR; ++i) load_b<BR, false>(M + (o + i) * BR, m[i]);
    X u[BR];
#pragma unroll
    for (int i = 0; i < BR; ++i) {
      double t = m[i][0] * rv[0];
#pragma unroll
      for (int c = 1; c < BR; ++c) t = fma(m[i][c], rv[c], t);
      u[i] = to_out<X>(xv[i] + t);
    }
    if constexpr (std::is_same_v<Z, float>) {
      reinterpret_cast<float4*>(z)[row] = make_float4((float)u[0], (float)u[1], (float)u[2], (float)pv);
    } else {
      double2* q = reinterpret_cast<double2*>(z + (int64_t)row * 4);
      q[0] = make_double2((double)u[0], (double)u[1]);
      q[1] = make_double2((double)u[2], (double)pv);
    }
  }
};

template <typename V, typename X>
struct LEpiSchurP {  // p = m_S o (r_p - B u*)      (1 x nu blocks)
  static constexpr int kDots = 0;
  const V* mS;
  const X* rp;
  X* p;
  // k_bsr_sellr: m_S and r_p of the row loaded ahead of its blocks (short rows, as K7)
  static constexpr bool kPre = true;
  struct PreT {
    V m;
    X r;
  };
  template <int BR>
  __device__ __forceinline__ void pre(int row, PreT (&v)[BR]) const {
    v[0].m = mS[row];
    v[0].r = rp[row];
  }
  template <int BR>
  __device__ __forceinline__ void row_pre(int row, const double (&yr)[BR], const PreT (&v)[BR]) const {
    p[row] = to_out<X>((double)v[0].m * ((double)v[0].r - yr[0]));
  }
  template <int BR>
  __device__ __forceinline__ void operator()(const LaneRow<BR>& L) const {
    if (!L.valid) return;
    p[L.row] = to_out<X>((double)mS[L.row] * ((double)rp[L.row] - L.yr));
  }
  template <int BR>
  __device__ __forceinline__ void row(int row, const double (&yr)[BR]) const {
    p[row] = to_out<X>((double)mS[row] * ((double)rp[row] - yr[0]));
  }
};

template <typename X>
struct LEpiSchurU {  // r_u' = r_u - B^T p          (nu x 1 blocks; in place allowed)
  static constexpr int kDots = 0;
  const X* ru;
  X* ru2;
  template <int BR>
  __device__ __forceinline__ void operator()(const LaneRow<BR>& L) const {
    if (!L.valid) return;
    const int64_t o = (int64_t)L.row * BR + L.r;
    ru2[o] = to_out<X>((double)ru[o] - L.yr);
  }
  template <int BR>
  __device__ __forceinline__ void row(int row, const double (&yr)[BR]) const {
    const int64_t o = (int64_t)row * BR;
    double v[BR];
#pragma unroll
    for (int c = 0; c < BR; ++c) v[c] = (double)ru[o + c];
#pragma unroll
    for (int c = 0; c < BR; ++c) ru2[o + c] = to_out<X>(v[c] - yr[c]);
  }
};

// Fused pre-smoothing from zero (K4a in the producer of f): the kernel
// that produces a level's right-hand side f also applies the level's block-diagonal M to it
// and stores x = M f.  f is rounded to the vector type first and M f is formed from the
// rounded values in k_apply_M's order (m0 f0, then fma), so f and x are bit-identical to
// the unfused pair.  All lanes of the warp must call the lane form (shuffles).
template <int BR, typename V, typename X>
__device__ __forceinline__ void apply_M_row(const V* __restrict__ M, int64_t o, const double (&fv)[BR], X* x) {
#pragma unroll
  for (int i = 0; i < BR; ++i) {
    double m[BR];
    load_b<BR, false>(M + (o + i) * BR, m);
    double t = m[0] * fv[0];
#pragma unroll
    for (int c = 1; c < BR; ++c) t = fma(m[c], fv[c], t);
    x[o + i] = to_out<X>(t);
  }
}

template <typename V, typename X>
struct LEpiSpmvM {  // f = A g (K6 restriction: g = r of the finer level), x = M f (K4a)
  static constexpr int kDots = 0;
  const V* M;
  X* f;
  X* x;
  template <int BR>
  __device__ __forceinline__ void operator()(const LaneRow<BR>& L) const {
    const int64_t o = (int64_t)L.row * BR + L.r;
    const X fr = to_out<X>(L.yr);
    const double fd = L.valid ? (double)fr : 0.0;
    double fv[BR];
#pragma unroll
    for (int c = 0; c < BR; ++c) fv[c] = __shfl_sync(kFull, fd, L.base + c);
    if (!L.valid) return;
    f[o] = fr;
    double m[BR];
    load_b<BR, false>(M + o * BR, m);
    double t = m[0] * fv[0];
#pragma unroll
    for (int c = 1; c < BR; ++c) t = fma(m[c], fv[c], t);
    x[o] = to_out<X>(t);
  }
  template <int BR>
  __device__ __forceinline__ void row(int row, const double (&yr)[BR]) const {
    const int64_t o = (int64_t)row * BR;
    double fv[BR];
#pragma unroll
    for (int c = 0; c < BR; ++c) {
      const X t = to_out<X>(yr[c]);
      f[o + c] = t;
      fv[c] = (double)t;
    }
    apply_M_row<BR>(M, o, fv, x);
  }
};

template <typename V, typename X>
struct LEpiSchurUM {  // r_u' = r_u - B^T p (K11, in place allowed), x = M r_u' (K4a of the second V-cycle)
  static constexpr int kDots = 0;
  const V* M;
  const X* ru;
  X* ru2;
  X* x;
  template <int BR>
  __device__ __forceinline__ void operator()(const LaneRow<BR>& L) const {
    const int64_t o = (int64_t)L.row * BR + L.r;
    const X fr = L.valid ? to_out<X>((double)ru[o] - L.yr) : X(0);
    double fv[BR];
#pragma unroll
    for (int c = 0; c < BR; ++c) fv[c] = __shfl_sync(kFull, (double)fr, L.base + c);
    if (!L.valid) return;
    ru2[o] = fr;
    double m[BR];
    load_b<BR, false>(M + o * BR, m);
    double t = m[0] * fv[0];
#pragma unroll
    for (int c = 1; c < BR; ++c) t = fma(m[c], fv[c], t);
    x[o] = to_out<X>(t);
  }
  template <int BR>
  __device__ __forceinline__ void row(int row, const double (&yr)[BR]) const {
    const int64_t o = (int64_t)row * BR;
    double fv[BR];
#pragma unroll
    for (int c = 0; c < BR; ++c) fv[c] = (double)ru[o + c];
#pragma unroll
    for (int c = 0; c < BR; ++c) {
      const X t = to_out<X>(fv[c] - yr[c]);
      ru2[o + c] = t;
      fv[c] = (double)t;
    }
    apply_M_row<BR>(M, o, fv, x);
  }
};

// fused SpMV + dot(s) (K3): y = A x (fp64); d_j += w_j[o] y_o, w_j == nullptr meaning y
template <int ND>
struct LEpiSpmvDot {
  static constexpr int kDots = ND;
  double* y;
  const double* w[2];
  double *partials, *out;
  unsigned* ticket;
  template <int BR>
  __device__ __forceinline__ void operator()(const LaneRow<BR>& L) const {
    if (L.valid) y[(int64_t)L.row * BR + L.r] = L.yr;
  }
  template <int BR>
  __device__ __forceinline__ void dots(const LaneRow<BR>& L, double (&d)[ND]) const {
    if (!L.valid) return;
    const int64_t o = (int64_t)L.row * BR + L.r;
#pragma unroll
    for (int j = 0; j < ND; ++j) d[j] = fma(w[j] ? w[j][o] : L.yr, L.yr, d[j]);
  }
  template <int BR>
  __device__ __forceinline__ void row(int row, const double (&yr)[BR]) const {
#pragma unroll
    for (int c = 0; c < BR; ++c) y[(int64_t)row * BR + c] = yr[c];
  }
  template <int BR>
  __device__ __forceinline__ void row_dots(int row, const double (&yr)[BR], double (&d)[ND]) const {
    const int64_t o = (int64_t)row * BR;
#pragma unroll
    for (int j = 0; j < ND; ++j)
#pragma unroll
      for (int c = 0; c < BR; ++c) d[j] = fma(w[j] ? w[j][o + c] : yr[c], yr[c], d[j]);
  }
};

// fused residual + norm (K2): r = f - A x; d_0 += r_o^2
struct LEpiResidualNrm {
  static constexpr int kDots = 1;
  const double* f;
  double* r;
  double *partials, *out;
  unsigned* ticket;
  template <int BR>
  __device__ __forceinline__ void operator()(const LaneRow<BR>& L) const {
    if (L.valid) r[(int64_t)L.row * BR + L.r] = f[(int64_t)L.row * BR + L.r] - L.yr;
  }
  template <int BR>
  __device__ __forceinline__ void dots(const LaneRow<BR>& L, double (&d)[1]) const {
    if (!L.valid) return;
    const double v = f[(int64_t)L.row * BR + L.r] - L.yr;
    d[0] = fma(v, v, d[0]);
  }
  template <int BR>
  __device__ __forceinline__ void row(int row, const double (&yr)[BR]) const {
    const int64_t o = (int64_t)row * BR;
#pragma unroll
    for (int c = 0; c < BR; ++c) r[o + c] = f[o + c] - yr[c];
  }
  template <int BR>
  __device__ __forceinline__ void row_dots(int row, const double (&yr)[BR], double (&d)[1]) const {
    const int64_t o = (int64_t)row * BR;
#pragma unroll
    for (int c = 0; c < BR; ++c) {
      const double v = f[o + c] - yr[c];
      d[0] = fma(v, v, d[0]);
    }
  }
};

// ---------------------------------------------------------------- the kernel
template <int BR, int BC, int U, bool COLS, bool NC, typename V, typename X, bool FAST, class EPI>
__global__ void __launch_bounds__(256, 8) k_bsr_lane(int r0, int n, const int32_t* __restrict__ ptr,
                                                  const int32_t* __restrict__ col, const V* __restrict__ val,
                                                  const X* __restrict__ x, EPI epi) {
  static_assert(!COLS || BR == BC, "column layout needs square blocks");
  constexpr int RPW = 32 / BR;
  constexpr int BE = BR * BC;
  constexpr int ND = EPI::kDots > 0 ? EPI::kDots : 1;
  const int lane = threadIdx.x & 31;
  // virtual blocks of 8 warps: one per CUDA block, or -- fused dots -- a persistent grid
  // (at most kMaxPartials blocks) walks them, accumulating its dot partials
  const int64_t nvb = ((int64_t)(n - r0) + RPW * 8 - 1) / (RPW * 8);  // rows [r0, n)
  double dacc[ND] = {};
  for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
  const int warp = (int)(vb * (blockDim.x >> 5) + (threadIdx.x >> 5));
  const int g = lane / BR, r = lane - g * BR;
  const int row = r0 + warp * RPW + g;
  LaneRow<BR> L;
  L.row = row;
  L.r = r;
  L.base = lane - r;
  L.valid = g < RPW && row < n;
  int k0 = 0, k1 = 0;
  if (L.valid) k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
  if constexpr (!COLS) {
    double acc = 0.0;
    int k = k0;
#pragma unroll 1
    for (; k + U <= k1; k += U) {
      int c[U];
      V a[U][BC];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        c[u] = __ldg(col + k + u);
        ld_row<BC, NC>(val + (int64_t)(k + u) * BE + r * BC, a[u]);
      }
      X xv[U][BC];
#pragma unroll
      for (int u = 0; u < U; ++u) ld_x<BC>(x + (int64_t)c[u] * BC, xv[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) acc += item_dot<BC, V, X, FAST>(a[u], xv[u]);
    }
#pragma unroll 1
    for (; k < k1; ++k) {
      V a[BC];
      X xv[BC];
      ld_row<BC, NC>(val + (int64_t)k * BE + r * BC, a);
      ld_x<BC>(x + (int64_t)__ldg(col + k) * BC, xv);
      acc += item_dot<BC, V, X, FAST>(a, xv);
    }
    L.yr = acc;
  } else {
    double acc[BR] = {};
    int k = k0;
#pragma unroll 1
    for (; k + U <= k1; k += U) {
      int c[U];
      V a[U][BR];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        c[u] = __ldg(col + k + u);
#pragma unroll
        for (int i = 0; i < BR; ++i) a[u][i] = ld_val<NC>(val + (int64_t)(k + u) * BE + i * BC + r);
      }
      X xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = __ldg(x + (int64_t)c[u] * BC + r);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < BR; ++i) acc[i] = fma((double)a[u][i], (double)xv[u], acc[i]);
    }
    for (; k < k1; ++k) {
      const X xv = __ldg(x + (int64_t)__ldg(col + k) * BC + r);
#pragma unroll
      for (int i = 0; i < BR; ++i) acc[i] = fma((double)ld_val<NC>(val + (int64_t)k * BE + i * BC + r), (double)xv, acc[i]);
    }
    // y_r = sum over the row's lanes l of acc_l[r]: BR-1 rotations, lane r sends the
    // entry its receiver needs
    double s = acc[0];
#pragma unroll
    for (int i = 1; i < BR; ++i)
      if (i == r) s = acc[i];
#pragma unroll
    for (int d = 1; d < BR; ++d) {
      const int want = (r + BR - d) % BR;  // component of the lane that reads from me
      double v = acc[0];
#pragma unroll
      for (int i = 1; i < BR; ++i)
        if (i == want) v = acc[i];
      const int src = L.base + (r + d) % BR;
      s += __shfl_sync(kFull, v, src);
    }
    L.yr = s;
  }
  epi(L);
  if constexpr (EPI::kDots > 0) epi.dots(L, dacc);
  }  // virtual blocks
  if constexpr (EPI::kDots > 0)
    block_reduce_finish<EPI::kDots, 256>(dacc, EPI::kDots, epi.partials, epi.ticket, epi.out, 0, nullptr);
}

// Very long rows (coarse operators, restriction onto a small coarsest level): one warp
// per block row, whole blocks per lane (U per step, loads first), butterfly over the
// warp; lanes r < BR then hold component r for the epilogue.
template <int BR, int BC, int U, typename V, typename X, bool FAST, class EPI>
__global__ void __launch_bounds__(256) k_bsr_warp(int n, const int32_t* __restrict__ ptr,
                                                  const int32_t* __restrict__ col, const V* __restrict__ val,
                                                  const X* __restrict__ x, EPI epi) {
  constexpr int BE = BR * BC;
  const int lane = threadIdx.x & 31;
  const int row = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  int k0 = 0, k1 = 0;
  if (row < n) k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
  double acc[BR] = {};
  for (int kb = k0 + lane; kb < k1; kb += 32 * U) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = (kb + 32 * u < k1) ? __ldg(col + kb + 32 * u) : -1;
    X xv[U][BC];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c[u] >= 0) ld_x<BC>(x + (int64_t)c[u] * BC, xv[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (c[u] < 0) continue;
#pragma unroll
      for (int i = 0; i < BR; ++i) {
        V a[BC];
        ld_row<BC, false>(val + (int64_t)(kb + 32 * u) * BE + i * BC, a);
        acc[i] += item_dot<BC, V, X, FAST>(a, xv[u]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < BR; ++i)
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc[i] += __shfl_xor_sync(kFull, acc[i], off);
  LaneRow<BR> L;
  L.row = row;
  L.r = lane < BR ? lane : 0;
  L.base = 0;
  L.valid = lane < BR && row < n;
  L.yr = pick<BR>(acc, L.r);
  epi(L);
}

// Long rows on few rows (restrictions R_l into the coarse levels: 150-240 blocks per row on
// 22-45 K rows; coarse A_l of 54-68 blocks): G warps share one block row, warp p taking the
// 32-block chunks p, p + G, p + 2G, ... of it, so a row is one or two load steps deep instead
// of G times that; the G butterfly sums meet in shared memory and warp 0 of the row adds them
// in part order (deterministic) and runs the epilogue.  256 threads = 8 / G rows per CTA.
template <int BR, int BC, int U, int G, typename V, typename X, bool FAST, class EPI>
__global__ void __launch_bounds__(256) k_bsr_warps(int n, const int32_t* __restrict__ ptr,
                                                   const int32_t* __restrict__ col, const V* __restrict__ val,
                                                   const X* __restrict__ x, EPI epi) {
  static_assert(G == 2 || G == 4 || G == 8, "k_bsr_warps: G in {2, 4, 8}");
  constexpr int BE = BR * BC;
  __shared__ double part[8][BR];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, p = w % G;
  const int row = blockIdx.x * (8 / G) + w / G;
  int k0 = 0, k1 = 0;
  if (row < n) k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
  double acc[BR] = {};
  for (int kb = k0 + 32 * p + lane; kb < k1; kb += 32 * G * U) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = (kb + 32 * G * u < k1) ? __ldg(col + kb + 32 * G * u) : -1;
    X xv[U][BC];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c[u] >= 0) ld_x<BC>(x + (int64_t)c[u] * BC, xv[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (c[u] < 0) continue;
#pragma unroll
      for (int i = 0; i < BR; ++i) {
        V a[BC];
        ld_row<BC, false>(val + (int64_t)(kb + 32 * G * u) * BE + i * BC, a);
        acc[i] += item_dot<BC, V, X, FAST>(a, xv[u]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < BR; ++i)
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc[i] += __shfl_xor_sync(kFull, acc[i], off);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < BR; ++i) part[w][i] = acc[i];
  __syncthreads();
  if (p != 0) return;
#pragma unroll
  for (int i = 0; i < BR; ++i) {
    double t = part[w][i];
#pragma unroll
    for (int q = 1; q < G; ++q) t += part[w + q][i];
    acc[i] = t;
  }
  LaneRow<BR> L;
  L.row = row;
  L.r = lane < BR ? lane : 0;
  L.base = 0;
  L.valid = lane < BR && row < n;
  L.yr = pick<BR>(acc, L.r);
  epi(L);
}

// ---------------------------------------------------------------- sliced BSR
// Long rows: the library's solve copy also holds a SLICED layout of the same blocks
// (SELL-C with C = 32/B consecutive block rows per slice, one warp per slice, padded to
// the slice's longest row with zero blocks; built once in make_tma_plan).  Step j of
// slice s stores, for block row i < B, the C*B words [g][r] = A_{row s*C+g, block j}[i][r]
// contiguously, so each of the B value loads of a warp reads C*B consecutive words
// (perfect coalescing, no sector shared across instructions); lane (g, r) holds column
// r of its row's block (COLS) and gathers the single value x_col[r].
// Measured (tools/spmv_lab.cu): 27-point 3x3 fp32 5.63 TB/s (row layout 4.59), 4x4
// fp32 x fp64 6.04 TB/s (5.68), 4x4 fp64 6.69 TB/s (6.16).
template <int B, int U, typename V, typename X, class EPI>
__global__ void __launch_bounds__(256, 8) k_bsr_sell(int n, int nslices, const int32_t* __restrict__ sptr,
                                                     const int32_t* __restrict__ perm,
                                                     const int32_t* __restrict__ scol, const V* __restrict__ sval,
                                                     const X* __restrict__ x, EPI epi) {
  constexpr int C = 32 / B;
  const int lane = threadIdx.x & 31;
  const int s = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int g = lane / B, r = lane - g * B;
  const bool act = g < C && s < nslices;
  const int L = g < C ? lane : 0, gg = g < C ? g : 0;
  int j0 = 0, j1 = 0;
  if (s < nslices) j0 = __ldg(sptr + s), j1 = __ldg(sptr + s + 1);
  double acc[B] = {};
  int j = j0;
#pragma unroll 1
  for (; j + U <= j1; j += U) {
    int c[U];
    V a[U][B];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = __ldg(scol + (int64_t)(j + u) * C + gg);
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
    const int c = __ldg(scol + (int64_t)j * C + gg);
    const X xv = __ldg(x + (int64_t)c * B + r);
#pragma unroll
    for (int i = 0; i < B; ++i)
      acc[i] = fma((double)__ldcs(sval + ((int64_t)j * B + i) * (C * B) + L), (double)xv, acc[i]);
  }
  // y_r = sum over the row's lanes l of acc_l[r] (transpose-reduce, as k_bsr_lane COLS)
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
    sum += __shfl_sync(kFull, v, base + (r + d) % B);
  }
  LaneRow<B> Lr;
  Lr.row = s * C + g;
  if (perm && act) Lr.row = __ldg(perm + (int64_t)s * C + g);  // sorted windows: slot -> row (-1: padding)
  Lr.r = r;
  Lr.base = base;
  Lr.valid = act && Lr.row >= 0 && Lr.row < n;
  Lr.yr = sum;
  epi(Lr);
}

// ---------------------------------------------------------------- interleaved row-per-lane
// Default for the fp32 hierarchy's 6..64-block rows (spmv.cu make_tma_plan).
// The solve copy interleaves 32 consecutive block rows (one slice, one warp; lane = row).  Each
// row's blocks are flattened ([block][i][c], padded to the slice's longest row with zero
// blocks) and cut into W-element vectors (W = 16 bytes / sizeof(V)); vector t of lane l
// sits at (vptr[s] + t) * 32 + l, so every value load of the warp is 32 x 16 contiguous
// bytes (4 L1 wavefronts, no sector shared between instructions) and column index j of
// the slice is one 128-byte load.  GB blocks (the least multiple of the block that fills
// whole vectors: 4 for 3x3 fp32, 2 for 3x3 fp64, 1 for 4x4) are loaded per step, all
// loads first, the next step's column indices one step ahead.  The lane owns its row's
// BR results and runs the epilogue's row-per-lane form (row(), row_dots()).
// Arithmetic: the block-row dots of k_bsr_lane's ROWS layout in the same block order --
// bit-identical to it.
template <int BR, int BC, int W>
struct SellrShape {
  static constexpr int E = BR * BC;
  static constexpr int gcd(int a, int b) { return b == 0 ? a : gcd(b, a % b); }
  static constexpr int GB = W / gcd(E, W);  // blocks per step: lcm(E, W) / E
  static constexpr int NV = GB * E / W;     // vectors per step
};
// Launch shape: a step's values take NV * W registers.  Above 18 words (3x3 fp32, 36
// values) the budget must let ptxas issue every load of a step first: at 80 registers it
// interleaved each 16-byte load with its FMAs (one load in flight per thread, 4.8 TB/s on
// A_0), at 128 (256 threads x 2 blocks) all loads issue first (5.65 TB/s).  128 threads x 5
// blocks (96 registers, 20 warps per SM; -DSELLR_TPB_BIG=128) interleaves again: 5.3 TB/s.
// 18-word steps (3x3 fp32, 8-byte vectors: A_0, the prolongators) run 6 blocks per SM (40
// registers, 88 bytes of L1-resident spill): P_0 4.0 / 4.3 / 4.7 / 5.1 TB/s at 3 / 4 / 5 / 6
// blocks, A_0's smoother 5.77 / 5.93 / 6.06 at 4 / 5 / 6; 8 blocks (32 registers) spill
// 168 bytes and drop to 5.2.  4x4 fp64 (32 words) stays at 2 (uses 72): 4 blocks, 6.90 vs 7.07.
#ifndef SELLR_TPB_BIG
#define SELLR_TPB_BIG 256
#endif
template <int BR, int BC, int W, typename V, bool FAST>
struct SellrCfg {
  static constexpr int words = SellrShape<BR, BC, W>::NV * W * (int)sizeof(V) / 4;
  static constexpr int TPB = words <= 18 ? 256 : SELLR_TPB_BIG;
  static constexpr int MINB = words <= 16 ? 4 : words <= 18 ? 6 : (65536 / TPB) / (TPB == 256 ? 128 : 102);
  static constexpr int WPB = TPB / 32;
};

template <int W, typename V>
__device__ __forceinline__ void ld_vec(const V* __restrict__ p, V* v) {
  if constexpr (W == 4 && std::is_same_v<V, float>) {
    const float4 q = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else if constexpr (W == 2 && std::is_same_v<V, float>) {
    const float2 q = __ldcs(reinterpret_cast<const float2*>(p));
    v[0] = q.x; v[1] = q.y;
  } else if constexpr (W == 2 && std::is_same_v<V, double>) {
    const double2 q = __ldcs(reinterpret_cast<const double2*>(p));
    v[0] = q.x; v[1] = q.y;
  } else {
    static_assert(W == 1, "vector width");
    v[0] = __ldcs(p);
  }
}

// One step: GB blocks of the lane's row.  c holds this step's column indices (loaded one
// step ahead); the value loads, the x gathers and the next step's column loads are all
// issued before any arithmetic.
template <int BR, int BC, int W, bool TAIL, typename V, typename X, bool FAST>
__device__ __forceinline__ void sellr_step(const V* __restrict__ vp, const int32_t* __restrict__ cpn,
                                           const X* __restrict__ x, int nb, int nbn,
                                           int (&c)[SellrShape<BR, BC, W>::GB], double (&acc)[BR]) {
  using S = SellrShape<BR, BC, W>;
  V a[S::NV * W];
  const int nv = TAIL ? (S::E * nb + W - 1) / W : S::NV;
#pragma unroll
  for (int q = 0; q < S::NV; ++q)
    if (!TAIL || q < nv) ld_vec<W>(vp + (int64_t)q * 32 * W, a + q * W);
  X xv[S::GB][BC];
#pragma unroll
  for (int u = 0; u < S::GB; ++u)
    if (!TAIL || u < nb) ld_x<BC>(x + (int64_t)c[u] * BC, xv[u]);
  if constexpr (!TAIL) {
#pragma unroll
    for (int u = 0; u < S::GB; ++u) c[u] = u < nbn ? __ldcs(cpn + u * 32) : 0;
  }
#pragma unroll
  for (int u = 0; u < S::GB; ++u) {
    if (TAIL && u >= nb) continue;
#pragma unroll
    for (int i = 0; i < BR; ++i) {
      V ar[BC];
#pragma unroll
      for (int cc = 0; cc < BC; ++cc) ar[cc] = a[u * S::E + i * BC + cc];
      acc[i] += item_dot<BC, V, X, FAST>(ar, xv[u]);
    }
  }
}

// k_bsr_sellr's prefetch flags (pf): the low 16 bits cap one prefetch in KiB.  Measured and
// dropped: prefetching the warp's NEXT slice with a persistent one-wave grid (cfg 5: A_0
// smoother 6.1 -> 3.3 TB/s -- the prefetched wave evicts itself from L2), and per-lane L2
// prefetches of the epilogue's operands (f, x, M) at the slice start (6.4 -> 6.2 TB/s: the
// row index held across the loop adds spill)
constexpr int kPfRest = 1 << 30;  // the rest of the current slice past its first step

template <int BR, int BC, int W, typename V, typename X, bool FAST, class EPI>
__global__ void __launch_bounds__(SellrCfg<BR, BC, W, V, FAST>::TPB, SellrCfg<BR, BC, W, V, FAST>::MINB) k_bsr_sellr(
    int n, int s0, int nslices, const int32_t* __restrict__ sptr, const int32_t* __restrict__ vptr,
    const int32_t* __restrict__ perm, const int32_t* __restrict__ scol, const V* __restrict__ sval,
    const X* __restrict__ x, EPI epi, int pf) {
  // slices [s0, nslices) (a row range of 32-aligned bounds: the distributed interior / boundary split)
  // pf: at the start of a slice, lane 0 requests the slice's values past its first step into L2
  // with one bulk (TMA) prefetch, so the per-step loads find them there instead of each step
  // waiting a full DRAM round trip (the warp's steps are a dependent chain)
  using S = SellrShape<BR, BC, W>;
  constexpr int ND = EPI::kDots > 0 ? EPI::kDots : 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int WPB = SellrCfg<BR, BC, W, V, FAST>::WPB;
  const int64_t nvb = ((int64_t)nslices - s0 + WPB - 1) / WPB;
  double dacc[ND] = {};
  for (int64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
    const int s = s0 + (int)(vb * WPB + w);
    double acc[BR] = {};
    [[maybe_unused]] int prow = -1;
    [[maybe_unused]] typename EpiPreT<EPI>::type pv[BR];
    if constexpr (EpiPre<EPI>::value) {  // the epilogue's operand, loaded ahead of the row
      if (s < nslices) {
        prow = perm ? __ldg(perm + (int64_t)s * 32 + lane) : s * 32 + lane;
        if (prow >= 0 && prow < n) epi.template pre<BR>(prow, pv);
      }
    }
    if (s < nslices) {
      const int j0 = __ldg(sptr + s), L = __ldg(sptr + s + 1) - j0;
      const int64_t v0 = __ldg(vptr + s);
      const V* vp = sval + (v0 * 32 + lane) * W;
      const uint32_t cap = (uint32_t)(pf & 0xffff) << 10;  // at most this many bytes per prefetch
      if ((pf & kPfRest) && lane == 0 && L > S::GB) {
        const int64_t first = (int64_t)S::NV * 32 * W;                     // the first step's values
        const int64_t tot = ((int64_t)__ldg(vptr + s + 1) - v0) * 32 * W;  // the slice's values
        const char* a = reinterpret_cast<const char*>(sval + v0 * 32 * W + first);
        const uint32_t bytes = min((uint32_t)((tot - first) * (int64_t)sizeof(V)), cap) & ~15u;
        if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
      }
      const int32_t* cp = scol + (int64_t)j0 * 32 + lane;
      int c[S::GB];
#pragma unroll
      for (int u = 0; u < S::GB; ++u) c[u] = u < L ? __ldcs(cp + u * 32) : 0;
      int j = 0;
#pragma unroll 1
      for (; j + S::GB <= L; j += S::GB) {
        cp += S::GB * 32;
        sellr_step<BR, BC, W, false, V, X, FAST>(vp, cp, x, S::GB, min(S::GB, L - j - S::GB), c, acc);
        vp += (int64_t)S::NV * 32 * W;
      }
      if (j < L) sellr_step<BR, BC, W, true, V, X, FAST>(vp, cp, x, L - j, 0, c, acc);
    }
    if constexpr (EpiPre<EPI>::value) {
      if (s < nslices && prow >= 0 && prow < n) epi.template row_pre<BR>(prow, acc, pv);
      continue;
    }
    int row = s * 32 + lane;
    if (perm && s < nslices) row = __ldg(perm + (int64_t)s * 32 + lane);  // sorted windows (-1: padding)
    if (s < nslices && row >= 0 && row < n) {
      epi.template row<BR>(row, acc);
      if constexpr (EPI::kDots > 0) epi.template row_dots<BR>(row, acc, dacc);
    }
  }
  if constexpr (EPI::kDots > 0)
    block_reduce_finish<EPI::kDots, SellrCfg<BR, BC, W, V, FAST>::TPB>(dacc, EPI::kDots, epi.partials, epi.ticket, epi.out,
                                                                   0, nullptr);
}

}  // namespace amgb
