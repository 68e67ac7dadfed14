// bsr_tma.cuh -- persistent, TMA-staged BSR kernels (K1 SpMV, K2 residual, K5 smoother,
// K10/K11 Schur coupling products).
//
// The direct kernels in bsr.cuh are latency bound: every group walks ptr -> col -> x
// with only a few hundred bytes in flight (ncu: 81 % of stall cycles on L1TEX
// scoreboard, profiles/r01_ncu_spmv_direct_b4_f32xf64.csv).  Here each CTA owns a
// set of row tiles (tr consecutive block rows).  A tile's row_ptr slice, its column
// indices and its block values are each ONE contiguous byte range of global memory,
// so thread 0 moves them into a shared-memory stage with three bulk async copies
// (cp.async.bulk, TMA engine) completing on the stage's mbarrier.  `ns` stages are in
// flight per CTA while the CTA's threads compute the current tile out of shared
// memory; HBM streams the matrix continuously and only the x gather latency is
// exposed in compute.
//
// Tile order (TmaArgs::wave): 0 = each CTA owns a contiguous tile range; 1 = tile i of
// CTA c is c + i*grid, so all CTAs sweep the matrix together and the x entries a
// banded (stencil-ordered) matrix gathers -- rows within +-n^2 of the sweep front --
// stay L2-resident instead of being re-read from HBM.
//
// Consumer: k_bsr_tma_rows, one thread per block row (short rows, <= 12 blocks); x
// gathers of the next tile in flight while the current one is computed; rectangular
// BR x BC blocks (Schur B: 1 x 3, B^T: 3 x 1).
//
// Status: opt-in (AMG_TMA=1).  The row-component lane kernels of bsr_lane.cuh measured
// faster on B200 for every shape of the path (tools/spmv_lab.cu); two
// further TMA consumers (a warp-per-row group consumer and a thread-per-block consumer
// with a shared-memory segmented sum) were measured at 2.0-4.0 TB/s and removed.
#pragma once

#include "bsr.cuh"

namespace amgb {

constexpr int kTmaMaxStages = 4;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared (TMA), completes tx bytes on `bar`; 16-B aligned, size % 16 == 0.
// The matrix is streamed exactly once per launch: L2 evict-first keeps x resident.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// b contiguous values from shared memory; 16-byte vector reads when a block row is a
// multiple of 16 bytes (then the staged tile is 16-byte aligned: blocks of b*b*s_v bytes
// start the tile, and the bulk copy's 16-byte rounding shift is zero)
template <int B, typename V>
__device__ __forceinline__ void lds_b(const V* p, V (&v)[B]) {
  if constexpr (B == 4 && std::is_same_v<V, float>) {
    float4 q = *reinterpret_cast<const float4*>(p);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else if constexpr (B == 4 && std::is_same_v<V, double>) {
    double2 a = reinterpret_cast<const double2*>(p)[0], c = reinterpret_cast<const double2*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = c.x; v[3] = c.y;
  } else if constexpr (B == 2 && std::is_same_v<V, double>) {
    double2 a = *reinterpret_cast<const double2*>(p);
    v[0] = a.x; v[1] = a.y;
  } else if constexpr (B == 2 && std::is_same_v<V, float>) {
    float2 a = *reinterpret_cast<const float2*>(p);
    v[0] = a.x; v[1] = a.y;
  } else {
#pragma unroll
    for (int c = 0; c < B; ++c) v[c] = p[c];
  }
}

// ---------------------------------------------------------------- epilogues
// called by the owner of `row` with the full row vector y = (A x)_row, once per
// component gl < BR (the row kernels call it for every gl with the same y)
template <int B, typename Y>
struct EpiSpmv {
  double alpha, beta;
  Y* y;
  __device__ __forceinline__ void operator()(int row, int gl, const double (&yv)[B]) const {
    const int64_t o = (int64_t)row * B + gl;
    double v = alpha * pick<B>(yv, gl);
    if (beta != 0.0) v = fma(beta, (double)y[o], v);
    y[o] = to_out<Y>(v);
  }
};

template <int B, typename X>
struct EpiResidual {
  const X* f;
  X* r;
  __device__ __forceinline__ void operator()(int row, int gl, const double (&yv)[B]) const {
    const int64_t o = (int64_t)row * B + gl;
    r[o] = to_out<X>((double)f[o] - pick<B>(yv, gl));
  }
};

template <int B, typename V, typename X>
struct EpiSmooth {  // xo = x + M (f - A x)
  const V* M;
  const X* f;
  const X* x;
  X* xo;
  __device__ __forceinline__ void operator()(int row, int gl, const double (&yv)[B]) const {
    const int64_t o = (int64_t)row * B;
    double res[B], m[B];
#pragma unroll
    for (int c = 0; c < B; ++c) res[c] = (double)f[o + c] - yv[c];
    load_b<B, false>(M + ((int64_t)row * B + gl) * B, m);
    double t = m[0] * res[0];
#pragma unroll
    for (int c = 1; c < B; ++c) t = fma(m[c], res[c], t);
    xo[o + gl] = to_out<X>((x ? (double)x[o + gl] : 0.0) + t);  // x == nullptr: from zero
  }
};

// K10 epilogue (1 x nu blocks of B): p = m_S o (r_p - B u*)
template <typename V, typename X>
struct EpiSchurP {
  const V* mS;
  const X* rp;
  X* p;
  __device__ __forceinline__ void operator()(int row, int, const double (&yv)[1]) const {
    p[row] = to_out<X>((double)mS[row] * ((double)rp[row] - yv[0]));
  }
};

// K11 epilogue (nu x 1 blocks of B^T): r_u' = r_u - B^T p   (in place allowed: each
// element is read and written by its own thread)
template <int NU, typename X>
struct EpiSchurU {
  const X* ru;
  X* ru2;
  __device__ __forceinline__ void operator()(int row, int gl, const double (&yv)[NU]) const {
    const int64_t o = (int64_t)row * NU + gl;
    ru2[o] = to_out<X>((double)ru[o] - pick<NU>(yv, gl));
  }
};

// r_u' = r_u - B^T p and x = M r_u' (the fused pre-smoothing of the second V-cycle; the
// consumer calls gl = 0..NU-1 in order with the row's whole result, the last call does all)
template <int NU, typename V, typename X>
struct EpiSchurUM {
  const V* M;
  const X* ru;
  X* ru2;
  X* x;
  __device__ __forceinline__ void operator()(int row, int gl, const double (&yv)[NU]) const {
    if (gl != NU - 1) return;
    const int64_t o = (int64_t)row * NU;
    double fv[NU];
#pragma unroll
    for (int c = 0; c < NU; ++c) fv[c] = (double)ru[o + c];
#pragma unroll
    for (int c = 0; c < NU; ++c) {
      const X t = to_out<X>(fv[c] - yv[c]);
      ru2[o + c] = t;
      fv[c] = (double)t;
    }
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      double m[NU];
      load_b<NU, false>(M + (o + i) * NU, m);
      double t = m[0] * fv[0];
#pragma unroll
      for (int c = 1; c < NU; ++c) t = fma(m[c], fv[c], t);
      x[o + i] = to_out<X>(t);
    }
  }
};

// ---------------------------------------------------------------- staging
struct TmaArgs {
  int n, tr, ntiles, ns;
  int stage_bytes, col_off, val_off;  // stage layout: [ptr | col | val]
  int wave;                           // tile order (see top)
  int part_off, max_blk;              // seg consumer: partial sums [BR][max_blk] doubles after the stages
};

// Producer side of the pipeline: one elected thread issues the three bulk copies of a
// tile; consumers read the tile through Tile views.
template <int BE, typename V>  // BE = elements per block (BR * BC)
struct TmaPipe {
  const TmaArgs& a;
  const int32_t* __restrict__ ptr;
  const int32_t* __restrict__ col;
  const V* __restrict__ val;
  unsigned char* smem;
  uint64_t* full;
  int (*meta)[4];  // per stage: ptr shift, col shift, val shift (bytes), k0
  int t_begin, my_tiles;
  uint64_t pol;

  __device__ TmaPipe(const TmaArgs& aa, const int32_t* p, const int32_t* c, const V* v, unsigned char* sm,
                     uint64_t* fu, int (*me)[4])
      : a(aa), ptr(p), col(c), val(v), smem(sm), full(fu), meta(me) {
    if (a.wave) {
      t_begin = 0;
      my_tiles = (a.ntiles > (int)blockIdx.x) ? (a.ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    } else {
      const int per = (a.ntiles + gridDim.x - 1) / gridDim.x;
      t_begin = blockIdx.x * per;
      my_tiles = max(0, min(per, a.ntiles - t_begin));
    }
    pol = policy_evict_first();
  }
  __device__ __forceinline__ int tile(int i) const { return a.wave ? (int)blockIdx.x + i * (int)gridDim.x : t_begin + i; }
  __device__ __forceinline__ int row0(int i) const { return tile(i) * a.tr; }
  __device__ __forceinline__ void kpair(int i, int& k0, int& k1) const {
    const int R0 = row0(i);
    k0 = __ldg(ptr + R0);
    k1 = __ldg(ptr + min(R0 + a.tr, a.n));
  }
  __device__ void issue(int i, int s, int k0, int k1) {
    const int R0 = row0(i), R1 = min(R0 + a.tr, a.n);
    unsigned char* st = smem + (size_t)s * a.stage_bytes;
    const uintptr_t pa = (uintptr_t)(ptr + R0), pe = (uintptr_t)(ptr + R1 + 1);
    const uintptr_t ca = (uintptr_t)(col + k0), ce = (uintptr_t)(col + k1);
    const uintptr_t va = (uintptr_t)(val + (int64_t)k0 * BE), ve = (uintptr_t)(val + (int64_t)k1 * BE);
    const uintptr_t pa16 = pa & ~uintptr_t(15), ca16 = ca & ~uintptr_t(15), va16 = va & ~uintptr_t(15);
    const unsigned pb = (unsigned)(((pe + 15) & ~uintptr_t(15)) - pa16);
    const unsigned cb = (k1 > k0) ? (unsigned)(((ce + 15) & ~uintptr_t(15)) - ca16) : 0u;
    const unsigned vb = (k1 > k0) ? (unsigned)(((ve + 15) & ~uintptr_t(15)) - va16) : 0u;
    meta[s][0] = (int)(pa - pa16);
    meta[s][1] = (int)(ca - ca16);
    meta[s][2] = (int)(va - va16);
    meta[s][3] = k0;
    mbar_arrive_expect_tx(&full[s], pb + cb + vb);
    tma_load_1d(st, (const void*)pa16, pb, &full[s], pol);
    if (cb) tma_load_1d(st + a.col_off, (const void*)ca16, cb, &full[s], pol);
    if (vb) tma_load_1d(st + a.val_off, (const void*)va16, vb, &full[s], pol);
  }
  // thread 0: prologue, first min(ns, my_tiles) tiles; returns the k-pair of tile ns
  __device__ void prologue(int& nk0, int& nk1) {
    const int pro = min(a.ns, my_tiles);
    for (int i = 0; i < pro; ++i) {
      int k0, k1;
      kpair(i, k0, k1);
      issue(i, i, k0, k1);
    }
    if (a.ns < my_tiles) kpair(a.ns, nk0, nk1);
  }
  // thread 0, after stage s (tile i) is consumed: refill it with tile i + ns
  __device__ void refill(int i, int s, int& nk0, int& nk1) {
    if (i + a.ns < my_tiles) {
      issue(i + a.ns, s, nk0, nk1);
      if (i + a.ns + 1 < my_tiles) kpair(i + a.ns + 1, nk0, nk1);
    }
  }
  __device__ __forceinline__ void wait(int i) { mbar_wait(&full[i % a.ns], (unsigned)((i / a.ns) & 1)); }
  // shared-memory views of tile i
  __device__ __forceinline__ void view(int i, const int32_t*& sp, const int32_t*& sc, const V*& sv, int& k0, int& nr,
                                       int& R0) const {
    const int s = i % a.ns;
    const unsigned char* st = smem + (size_t)s * a.stage_bytes;
    sp = reinterpret_cast<const int32_t*>(st + meta[s][0]);
    sc = reinterpret_cast<const int32_t*>(st + a.col_off + meta[s][1]);
    sv = reinterpret_cast<const V*>(st + a.val_off + meta[s][2]);
    k0 = meta[s][3];
    R0 = row0(i);
    nr = min(a.tr, a.n - R0);
  }
};

#define AMGB_TMA_PROLOGUE(BE, V)                                              \
  extern __shared__ __align__(128) unsigned char smem[];                      \
  __shared__ __align__(8) uint64_t full[kTmaMaxStages];                      \
  __shared__ int meta[kTmaMaxStages][4];                                      \
  const int tid = threadIdx.x;                                                \
  TmaPipe<BE, V> pipe(a, ptr, col, val, smem, full, meta);                    \
  if (tid == 0) {                                                             \
    for (int s_ = 0; s_ < a.ns; ++s_) mbar_init(&full[s_], 1);                \
    mbar_fence_init();                                                        \
  }                                                                           \
  __syncthreads();                                                            \
  int nk0 = 0, nk1 = 0;                                                       \
  if (tid == 0) pipe.prologue(nk0, nk1);

// ---------------------------------------------------------------- row per lane
// One THREAD per block row (tile = blockDim rows).  For short rows in a banded /
// stencil ordering the lanes of a warp then gather x at the same block slot of 32
// consecutive rows, i.e. contiguous addresses (coalesced), while the row-strided block
// values are read from shared memory (a row of 7 3x3 fp32 blocks is 63 words: odd
// stride, conflict-free).  No shuffles; the thread owns the whole BR-vector of its row.
// Blocks are BR x BC (square BSR: BR = BC = b).
template <int BR, int BC, typename V, typename X, bool FAST, class EPI>
__global__ void __launch_bounds__(256) k_bsr_tma_rows(TmaArgs a, const int32_t* __restrict__ ptr,
                                                      const int32_t* __restrict__ col, const V* __restrict__ val,
                                                      const X* __restrict__ x, EPI epi) {
  AMGB_TMA_PROLOGUE(BR * BC, V)
  // software pipeline: while tile i is computed, the x gathers of this thread's row of
  // tile i+1 are already in flight (tile i+1 landed: ns >= 3 stages)
  constexpr int U = (BC <= 3) ? 8 : 4;
  auto prefetch = [&](int i, X (&xb)[U][BC]) {
    const int32_t *sp, *sc;
    const V* sv;
    int k0, nr, R0;
    pipe.view(i, sp, sc, sv, k0, nr, R0);
    int kb0 = 0, kb1 = 0;
    if (tid < nr) kb0 = sp[tid] - k0, kb1 = sp[tid + 1] - k0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (kb0 + u < kb1) {
        load_raw<BC, false>(x + (int64_t)sc[kb0 + u] * BC, xb[u]);
      } else {
#pragma unroll
        for (int c = 0; c < BC; ++c) xb[u][c] = X(0);
      }
    }
  };
  X xa[U][BC], xb[U][BC];
  if (pipe.my_tiles > 0) {
    pipe.wait(0);
    prefetch(0, xa);
  }
  for (int i = 0; i < pipe.my_tiles; ++i) {
    if (i + 1 < pipe.my_tiles) {
      pipe.wait(i + 1);
      prefetch(i + 1, xb);
    }
    const int32_t *sp, *sc;
    const V* sv;
    int k0, nr, R0;
    pipe.view(i, sp, sc, sv, k0, nr, R0);
    if (tid < nr) {
      const int kb0 = sp[tid] - k0, kb1 = sp[tid + 1] - k0;
      double acc[BR] = {};
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (kb0 + u < kb1) {
          const V* blk = sv + (int64_t)(kb0 + u) * BR * BC;
#pragma unroll
          for (int r = 0; r < BR; ++r) {
            V av[BC];
#pragma unroll
            for (int c = 0; c < BC; ++c) av[c] = blk[r * BC + c];
            acc[r] += item_dot<BC, V, X, FAST>(av, xa[u]);
          }
        }
      }
      for (int kb = kb0 + U; kb < kb1; ++kb) {  // long rows: the rest loaded in place
        X xv[BC];
        load_raw<BC, false>(x + (int64_t)sc[kb] * BC, xv);
        const V* blk = sv + (int64_t)kb * BR * BC;
#pragma unroll
        for (int r = 0; r < BR; ++r) {
          V av[BC];
#pragma unroll
          for (int c = 0; c < BC; ++c) av[c] = blk[r * BC + c];
          acc[r] += item_dot<BC, V, X, FAST>(av, xv);
        }
      }
#pragma unroll
      for (int c = 0; c < BR; ++c) epi(R0 + tid, c, acc);
    }
    __syncthreads();
    if (tid == 0) pipe.refill(i, i % a.ns, nk0, nk1);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < BC; ++c) xa[u][c] = xb[u][c];
  }
}

}  // namespace amgb
