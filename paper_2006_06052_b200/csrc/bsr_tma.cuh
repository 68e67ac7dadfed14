// bsr_tma.cuh -- persistent, TMA-staged BSR kernels (K1 SpMV, K2 residual, K5 smoother).
//
// The direct kernels in bsr.cuh are latency bound: every group walks ptr -> col -> x
// with only a few hundred bytes in flight (ncu: 81 % of stall cycles on L1TEX
// scoreboard, profiles/r01_ncu_spmv_direct_b4_f32xf64.csv).  Here each CTA owns a
// strided set of row tiles (tr consecutive block rows).  A tile's row_ptr slice, its
// column indices and its block values are each ONE contiguous byte range of global
// memory, so thread 0 moves them into a shared-memory stage with three bulk async
// copies (cp.async.bulk, TMA engine) completing on the stage's mbarrier.  `ns` stages
// are in flight per CTA while the CTA's 8 warps compute the current tile out of
// shared memory: G lanes per block row, (block, block row) items, fp64
// accumulation, x gathered from L2, group butterfly, epilogue functor.  HBM streams
// the matrix continuously; only the x gather latency is exposed in compute.
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
// 1-D bulk copy global -> shared (TMA), completes tx bytes on `bar`; 16-B aligned, size % 16 == 0
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
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
// called by lanes gl < B of the group owning `row` with the full row vector y = (A x)_row
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
    xo[o + gl] = to_out<X>((double)x[o + gl] + t);
  }
};

// ---------------------------------------------------------------- the kernel
struct TmaArgs {
  int n, tr, ntiles, ns;
  int stage_bytes, col_off, val_off;  // stage layout: [ptr | col | val]
};

template <int B, int G, typename V, typename X, bool FAST, class EPI>
__global__ void __launch_bounds__(256) k_bsr_tma(TmaArgs a, const int32_t* __restrict__ ptr,
                                                 const int32_t* __restrict__ col, const V* __restrict__ val,
                                                 const X* __restrict__ x, EPI epi) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kTmaMaxStages];
  __shared__ int meta[kTmaMaxStages][4];  // ptr shift (B), col shift (B), val shift (B), k0
  const int tid = threadIdx.x;
  // contiguous tile range per CTA: consecutive tiles stay on one SM, so the x entries
  // of the +-1 and +-n neighbours of a 3-D stencil row are L1 hits
  const int per = (a.ntiles + gridDim.x - 1) / gridDim.x;
  const int t_begin = blockIdx.x * per;
  const int my_tiles = max(0, min(per, a.ntiles - t_begin));
  if (tid == 0) {
    for (int s = 0; s < a.ns; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();

  // thread 0 is the producer: stage the tile's ptr slice, columns and values
  auto issue = [&](int i, int s, int k0, int k1) {
    const int t = t_begin + i;
    const int R0 = t * a.tr, R1 = min(R0 + a.tr, a.n);
    unsigned char* st = smem + (size_t)s * a.stage_bytes;
    const uintptr_t pa = (uintptr_t)(ptr + R0), pe = (uintptr_t)(ptr + R1 + 1);
    const uintptr_t ca = (uintptr_t)(col + k0), ce = (uintptr_t)(col + k1);
    const uintptr_t va = (uintptr_t)(val + (int64_t)k0 * B * B), ve = (uintptr_t)(val + (int64_t)k1 * B * B);
    const uintptr_t pa16 = pa & ~uintptr_t(15), ca16 = ca & ~uintptr_t(15), va16 = va & ~uintptr_t(15);
    const unsigned pb = (unsigned)(((pe + 15) & ~uintptr_t(15)) - pa16);
    const unsigned cb = (k1 > k0) ? (unsigned)(((ce + 15) & ~uintptr_t(15)) - ca16) : 0u;
    const unsigned vb = (k1 > k0) ? (unsigned)(((ve + 15) & ~uintptr_t(15)) - va16) : 0u;
    meta[s][0] = (int)(pa - pa16);
    meta[s][1] = (int)(ca - ca16);
    meta[s][2] = (int)(va - va16);
    meta[s][3] = k0;
    mbar_arrive_expect_tx(&full[s], pb + cb + vb);
    tma_load_1d(st, (const void*)pa16, pb, &full[s]);
    if (cb) tma_load_1d(st + a.col_off, (const void*)ca16, cb, &full[s]);
    if (vb) tma_load_1d(st + a.val_off, (const void*)va16, vb, &full[s]);
  };
  int nk0 = 0, nk1 = 0;  // producer's prefetched ptr pair of the next tile to issue
  if (tid == 0) {
    const int pro = min(a.ns, my_tiles);
    for (int i = 0; i < pro; ++i) {
      const int t = t_begin + i;
      issue(i, i, __ldg(ptr + t * a.tr), __ldg(ptr + min(t * a.tr + a.tr, a.n)));
    }
    if (a.ns < my_tiles) {
      const int t = t_begin + a.ns;
      nk0 = __ldg(ptr + t * a.tr);
      nk1 = __ldg(ptr + min(t * a.tr + a.tr, a.n));
    }
  }

  const int g = tid / G, gl = tid & (G - 1);
  constexpr int NG = 256 / G;
  const unsigned gmask = (G == 32) ? kFull : (((1u << G) - 1u) << ((tid & 31) & ~(G - 1)));
  for (int i = 0; i < my_tiles; ++i) {
    const int s = i % a.ns;
    mbar_wait(&full[s], (unsigned)((i / a.ns) & 1));
    const int t = t_begin + i;
    const int R0 = t * a.tr, nr = min(a.tr, a.n - R0);
    const unsigned char* st = smem + (size_t)s * a.stage_bytes;
    const int32_t* sp = reinterpret_cast<const int32_t*>(st + meta[s][0]);
    const int32_t* sc = reinterpret_cast<const int32_t*>(st + a.col_off + meta[s][1]);
    const V* sv = reinterpret_cast<const V*>(st + a.val_off + meta[s][2]);
    const int k0 = meta[s][3];
    for (int lr = g; lr < nr + (NG - 1) - ((nr + NG - 1) % NG); lr += NG) {
      // every group of the CTA runs the same number of passes (shuffles stay converged)
      const bool valid = lr < nr;
      // block per lane: lane gl handles blocks kb0 + gl, kb0 + gl + G, ...; x is
      // gathered once per block (b loads) and the b x b block is read from shared memory
      double acc[B] = {};
      if (valid) {
        const int kb0 = sp[lr] - k0, kb1 = sp[lr + 1] - k0;
        for (int kb = kb0 + gl; kb < kb1; kb += G) {
          X xv[B];
          load_raw<B, false>(x + (int64_t)sc[kb] * B, xv);
          const V* blk = sv + (int64_t)kb * B * B;
#pragma unroll
          for (int q = 0; q < B; ++q) {
            // rotate the block-row order per lane: 16-byte rows of neighbouring lanes fall
            // in different shared-memory bank groups
            const int r = (B == 4) ? ((q + gl) & 3) : q;
            V av[B];
            lds_b<B, V>(blk + r * B, av);
            const double d = item_dot<B, V, X, FAST>(av, xv);
#pragma unroll
            for (int rr = 0; rr < B; ++rr)
              if (rr == r) acc[rr] += d;
          }
        }
      }
      double yv[B];
#pragma unroll
      for (int c = 0; c < B; ++c) {
        double v = acc[c];
#pragma unroll
        for (int off = G / 2; off >= 1; off >>= 1) v += __shfl_xor_sync(gmask, v, off, G);
        yv[c] = v;
      }
      if (valid && gl < B) epi(R0 + lr, gl, yv);
    }
    __syncthreads();  // stage s fully consumed
    if (tid == 0 && i + a.ns < my_tiles) {
      issue(i + a.ns, s, nk0, nk1);
      if (i + a.ns + 1 < my_tiles) {
        const int tn = t_begin + i + a.ns + 1;
        nk0 = __ldg(ptr + tn * a.tr);
        nk1 = __ldg(ptr + min(tn * a.tr + a.tr, a.n));
      }
    }
  }
}

}  // namespace amgb

namespace amgb {

// ---------------------------------------------------------------- row per lane
// Same TMA staging as k_bsr_tma, but one THREAD per block row (tile = blockDim rows).
// For short rows in a banded / stencil ordering the lanes of a warp then gather x at
// the same block slot of 32 consecutive rows, i.e. contiguous addresses (coalesced),
// while the row-strided block values are read from shared memory (a row of 7 3x3 fp32
// blocks is 63 words: odd stride, conflict-free).  No shuffles; the thread owns the
// whole b-vector of its row.
template <int B, typename V, typename X, bool FAST, class EPI>
__global__ void __launch_bounds__(256) k_bsr_tma_rows(TmaArgs a, const int32_t* __restrict__ ptr,
                                                      const int32_t* __restrict__ col, const V* __restrict__ val,
                                                      const X* __restrict__ x, EPI epi) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kTmaMaxStages];
  __shared__ int meta[kTmaMaxStages][4];
  const int tid = threadIdx.x;
  const int per = (a.ntiles + gridDim.x - 1) / gridDim.x;
  const int t_begin = blockIdx.x * per;
  const int my_tiles = max(0, min(per, a.ntiles - t_begin));
  if (tid == 0) {
    for (int s = 0; s < a.ns; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](int i, int s, int k0, int k1) {
    const int t = t_begin + i;
    const int R0 = t * a.tr, R1 = min(R0 + a.tr, a.n);
    unsigned char* st = smem + (size_t)s * a.stage_bytes;
    const uintptr_t pa = (uintptr_t)(ptr + R0), pe = (uintptr_t)(ptr + R1 + 1);
    const uintptr_t ca = (uintptr_t)(col + k0), ce = (uintptr_t)(col + k1);
    const uintptr_t va = (uintptr_t)(val + (int64_t)k0 * B * B), ve = (uintptr_t)(val + (int64_t)k1 * B * B);
    const uintptr_t pa16 = pa & ~uintptr_t(15), ca16 = ca & ~uintptr_t(15), va16 = va & ~uintptr_t(15);
    const unsigned pb = (unsigned)(((pe + 15) & ~uintptr_t(15)) - pa16);
    const unsigned cb = (k1 > k0) ? (unsigned)(((ce + 15) & ~uintptr_t(15)) - ca16) : 0u;
    const unsigned vb = (k1 > k0) ? (unsigned)(((ve + 15) & ~uintptr_t(15)) - va16) : 0u;
    meta[s][0] = (int)(pa - pa16);
    meta[s][1] = (int)(ca - ca16);
    meta[s][2] = (int)(va - va16);
    meta[s][3] = k0;
    mbar_arrive_expect_tx(&full[s], pb + cb + vb);
    tma_load_1d(st, (const void*)pa16, pb, &full[s]);
    if (cb) tma_load_1d(st + a.col_off, (const void*)ca16, cb, &full[s]);
    if (vb) tma_load_1d(st + a.val_off, (const void*)va16, vb, &full[s]);
  };
  int nk0 = 0, nk1 = 0;
  if (tid == 0) {
    const int pro = min(a.ns, my_tiles);
    for (int i = 0; i < pro; ++i) {
      const int t = t_begin + i;
      issue(i, i, __ldg(ptr + t * a.tr), __ldg(ptr + min(t * a.tr + a.tr, a.n)));
    }
    if (a.ns < my_tiles) {
      const int t = t_begin + a.ns;
      nk0 = __ldg(ptr + t * a.tr);
      nk1 = __ldg(ptr + min(t * a.tr + a.tr, a.n));
    }
  }
  // software pipeline: while tile i is computed, the x gathers of this thread's row of
  // tile i+1 are already in flight (tile i+1 landed: ns >= 3 stages)
  constexpr int U = (B <= 3) ? 8 : 4;
  auto tile_info = [&](int i, const int32_t*& sp, const int32_t*& sc, const V*& sv, int& k0, int& nr, int& R0) {
    const int s = i % a.ns;
    const unsigned char* st = smem + (size_t)s * a.stage_bytes;
    sp = reinterpret_cast<const int32_t*>(st + meta[s][0]);
    sc = reinterpret_cast<const int32_t*>(st + a.col_off + meta[s][1]);
    sv = reinterpret_cast<const V*>(st + a.val_off + meta[s][2]);
    k0 = meta[s][3];
    R0 = (t_begin + i) * a.tr;
    nr = min(a.tr, a.n - R0);
  };
  auto prefetch = [&](int i, X (&xb)[U][B]) {
    const int32_t *sp, *sc;
    const V* sv;
    int k0, nr, R0;
    tile_info(i, sp, sc, sv, k0, nr, R0);
    const int lr = tid;
    int kb0 = 0, kb1 = 0;
    if (lr < nr) kb0 = sp[lr] - k0, kb1 = sp[lr + 1] - k0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (kb0 + u < kb1) {
        load_raw<B, false>(x + (int64_t)sc[kb0 + u] * B, xb[u]);
      } else {
#pragma unroll
        for (int c = 0; c < B; ++c) xb[u][c] = X(0);
      }
    }
  };
  X xa[U][B], xb[U][B];
  if (my_tiles > 0) {
    mbar_wait(&full[0], 0u);
    prefetch(0, xa);
  }
  for (int i = 0; i < my_tiles; ++i) {
    if (i + 1 < my_tiles) {
      mbar_wait(&full[(i + 1) % a.ns], (unsigned)(((i + 1) / a.ns) & 1));
      prefetch(i + 1, xb);
    }
    const int32_t *sp, *sc;
    const V* sv;
    int k0, nr, R0;
    tile_info(i, sp, sc, sv, k0, nr, R0);
    const int lr = tid;
    if (lr < nr) {
      const int kb0 = sp[lr] - k0, kb1 = sp[lr + 1] - k0;
      double acc[B] = {};
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (kb0 + u < kb1) {
          const V* blk = sv + (int64_t)(kb0 + u) * B * B;
#pragma unroll
          for (int r = 0; r < B; ++r) {
            V av[B];
#pragma unroll
            for (int c = 0; c < B; ++c) av[c] = blk[r * B + c];
            acc[r] += item_dot<B, V, X, FAST>(av, xa[u]);
          }
        }
      }
      for (int kb = kb0 + U; kb < kb1; ++kb) {  // long rows: the rest loaded in place
        X xv[B];
        load_raw<B, false>(x + (int64_t)sc[kb] * B, xv);
        const V* blk = sv + (int64_t)kb * B * B;
#pragma unroll
        for (int r = 0; r < B; ++r) {
          V av[B];
#pragma unroll
          for (int c = 0; c < B; ++c) av[c] = blk[r * B + c];
          acc[r] += item_dot<B, V, X, FAST>(av, xv);
        }
      }
#pragma unroll
      for (int c = 0; c < B; ++c) epi(R0 + lr, c, acc);
    }
    __syncthreads();
    const int s = i % a.ns;
    if (tid == 0 && i + a.ns < my_tiles) {
      issue(i + a.ns, s, nk0, nk1);
      if (i + a.ns + 1 < my_tiles) {
        const int tn = t_begin + i + a.ns + 1;
        nk0 = __ldg(ptr + tn * a.tr);
        nk1 = __ldg(ptr + min(tn * a.tr + a.tr, a.n));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < B; ++c) xa[u][c] = xb[u][c];
  }
}

}  // namespace amgb
