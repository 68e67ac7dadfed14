// reduce.cuh -- deterministic grid reduction used by the fused kernels: every block writes
// its partial sums, the LAST block to finish (atomic ticket) adds the gridDim.x partials of
// each output in a fixed order -- bit-reproducible for a fixed grid, one launch, and the
// ticket is reset for the next launch (CUDA-graph safe).  partials: [K][gridDim.x].
#pragma once

#include "common.cuh"

namespace amgb {

// acc[j] (j < kout) of every thread -> partials[j * gridDim.x + block]; the last block sums
// the gridDim.x partials of each output in a fixed order: out[j] = post(sum_j).
// post: 0 = plain, 1 = sqrt, 2 = sqrt and inv[0] = 1 / sqrt
template <int K, int THREADS>
__device__ __forceinline__ void block_reduce_finish(double (&acc)[K], int kout, double* partials, unsigned* ticket,
                                              double* out, int post, double* inv) {
  __shared__ double sh[K][THREADS / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nblk = gridDim.x;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (j < kout) {
      double v = acc[j];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
      if (lane == 0) sh[j][warp] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < kout) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < THREADS / 32; ++w) v += sh[threadIdx.x][w];
    partials[(int64_t)threadIdx.x * nblk + blockIdx.x] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == (unsigned)nblk - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int j = warp; j < kout; j += THREADS / 32) {
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
  if (threadIdx.x == 0) *ticket = 0u;  // ready for the next launch (graph-safe)
}

}  // namespace amgb
