// convert.cu -- S1: scalar CSR -> BSR on the device (the §4 worked example, PAPER.md:
// 658-672).  One block per non-empty b x b tile; absent
// scalars inside a stored tile are explicit zeros; duplicate scalar
// entries are summed in CSR order (row, then position), the order the oracle sums in.
//
// Device algorithm: every scalar entry gets the key (I = row / b, J = col / b); a stable
// radix sort by key groups a tile's entries (keeping CSR order inside a tile); the first
// entry of each key run opens a block; one thread per block accumulates its entries
// sequentially.  Blocks come out sorted by (I, J): row_ptr by count + scan.
#include <cub/cub.cuh>

#include "amg.h"
#include "common.cuh"
#include "prof.h"

namespace amgb {

namespace {

constexpr int kT = 256;

__global__ void k_entry_keys(int32_t n, int b, int64_t nbc, const int32_t* __restrict__ ptr,
                             const int32_t* __restrict__ col, int64_t* __restrict__ key, int32_t* __restrict__ idx,
                             int* __restrict__ err, int32_t m) {
  const int32_t row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  for (int32_t k = ptr[row]; k < ptr[row + 1]; ++k) {
    const int32_t c = col[k];
    if (c < 0 || c >= m) atomicExch(err, 1);
    key[k] = (int64_t)(row / b) * nbc + (c / b);
    idx[k] = k;
  }
}

// first entry of each key run -> 1
__global__ void k_run_heads(int64_t E, const int64_t* __restrict__ key, int32_t* __restrict__ head) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  head[e] = (e == 0 || key[e] != key[e - 1]) ? 1 : 0;
}

// blocks: bcol, per-row counts, run start of every block
__global__ void k_blocks(int64_t E, int64_t nbc, const int64_t* __restrict__ key, const int32_t* __restrict__ head,
                         const int32_t* __restrict__ bid, int32_t* __restrict__ bcol, int32_t* __restrict__ rowcnt,
                         int32_t* __restrict__ start) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E || !head[e]) return;
  const int32_t u = bid[e];
  bcol[u] = (int32_t)(key[e] % nbc);
  start[u] = (int32_t)e;
  atomicAdd(rowcnt + key[e] / nbc, 1);  // integer count: order-free
}

template <typename T>
__global__ void k_block_values(int64_t nb, int64_t E, int b, const int32_t* __restrict__ start,
                               const int32_t* __restrict__ idx, const int64_t* __restrict__ key,
                               const int32_t* __restrict__ ptr_rows /* scalar row of entry via rowof */,
                               const int32_t* __restrict__ col, const T* __restrict__ val, T* __restrict__ bval) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= nb) return;
  const int32_t s0 = start[u];
  const int32_t s1 = (u + 1 < nb) ? start[u + 1] : (int32_t)E;
  T* blk = bval + u * b * b;
  for (int q = 0; q < b * b; ++q) blk[q] = T(0);
  for (int32_t e = s0; e < s1; ++e) {  // CSR order inside the tile (stable sort)
    const int32_t k = idx[e];
    const int r = ptr_rows[k] % b, c = col[k] % b;
    blk[r * b + c] = blk[r * b + c] + val[k];
  }
}

__global__ void k_row_of(int32_t n, const int32_t* __restrict__ ptr, int32_t* __restrict__ rowof) {
  const int32_t row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  for (int32_t k = ptr[row]; k < ptr[row + 1]; ++k) rowof[k] = row;
}

}  // namespace

// returns nnzb; fills the arrays when bptr != nullptr
int64_t csr_to_bsr(int32_t n, int32_t m, int32_t b, int64_t nnz, const int32_t* ptr, const int32_t* col,
                   const void* val, int dtype, int32_t* bptr, int32_t* bcol, void* bval, cudaStream_t s) {
  if (b < 1 || n < 0 || m < 0 || n % b || m % b) fail(AMG_EINVAL, "csr_to_bsr: n and m must be multiples of b");
  if (nnz >= (int64_t(1) << 31)) fail(AMG_EINDEX_OVERFLOW, "csr_to_bsr: nnz >= 2^31");
  const int32_t nbr = n / b;
  const int64_t nbc = std::max<int64_t>(m / b, 1);
  Arena t;
  const int64_t E = nnz;
  int* err = t.alloc_n<int>(1);
  AMG_CK(cudaMemsetAsync(err, 0, sizeof(int), s));
  int64_t *key = t.alloc_n<int64_t>(std::max<int64_t>(E, 1)), *key2 = t.alloc_n<int64_t>(std::max<int64_t>(E, 1));
  int32_t *idx = t.alloc_n<int32_t>(std::max<int64_t>(E, 1)), *idx2 = t.alloc_n<int32_t>(std::max<int64_t>(E, 1));
  if (n > 0) k_entry_keys<<<grid_for(n, kT), kT, 0, s>>>(n, b, nbc, ptr, col, key, idx, err, m);
  AMG_CK_LAUNCH();
  int herr = 0;
  AMG_CK(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s));
  AMG_CK(cudaStreamSynchronize(s));
  if (herr) fail(AMG_EINVAL, "csr_to_bsr: column index out of range");
  int64_t nb = 0;
  int32_t* rowcnt = t.alloc_n<int32_t>(nbr + 1);
  AMG_CK(cudaMemsetAsync(rowcnt, 0, sizeof(int32_t) * (nbr + 1), s));
  if (E > 0) {
    // stable LSD radix sort by key (only the bits the keys use)
    int bits = 1;
    while (bits < 63 && ((int64_t)nbr * nbc) >> bits) ++bits;
    size_t need = 0;
    AMG_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, key, key2, idx, idx2, (int)E, 0, bits, s));
    void* tmp = t.alloc(need);
    AMG_CK(cub::DeviceRadixSort::SortPairs(tmp, need, key, key2, idx, idx2, (int)E, 0, bits, s));
    int32_t* head = t.alloc_n<int32_t>(E + 1);
    k_run_heads<<<grid_for(E, kT), kT, 0, s>>>(E, key2, head);
    AMG_CK_LAUNCH();
    int32_t* bid = t.alloc_n<int32_t>(E + 1);
    need = 0;
    AMG_CK(cub::DeviceScan::ExclusiveSum(nullptr, need, head, bid, (int)E + 1, s));
    void* tmp2 = t.alloc(need);
    AMG_CK(cudaMemsetAsync(head + E, 0, sizeof(int32_t), s));
    AMG_CK(cub::DeviceScan::ExclusiveSum(tmp2, need, head, bid, (int)E + 1, s));
    int32_t nb32 = 0;
    AMG_CK(cudaMemcpyAsync(&nb32, bid + E, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    AMG_CK(cudaStreamSynchronize(s));
    nb = nb32;
    if (bptr) {
      int32_t* start = t.alloc_n<int32_t>(std::max<int64_t>(nb, 1));
      k_blocks<<<grid_for(E, kT), kT, 0, s>>>(E, nbc, key2, head, bid, bcol, rowcnt, start);
      AMG_CK_LAUNCH();
      int32_t* rowof = t.alloc_n<int32_t>(E);
      k_row_of<<<grid_for(n, kT), kT, 0, s>>>(n, ptr, rowof);
      AMG_CK_LAUNCH();
      if (dtype == AMG_F32)
        k_block_values<float><<<grid_for(nb, kT), kT, 0, s>>>(nb, E, b, start, idx2, key2, rowof, col,
                                                              (const float*)val, (float*)bval);
      else
        k_block_values<double><<<grid_for(nb, kT), kT, 0, s>>>(nb, E, b, start, idx2, key2, rowof, col,
                                                               (const double*)val, (double*)bval);
      AMG_CK_LAUNCH();
    }
  }
  if (bptr) {
    size_t need = 0;
    AMG_CK(cub::DeviceScan::ExclusiveSum(nullptr, need, rowcnt, bptr, nbr + 1, s));
    void* tmp3 = t.alloc(std::max<size_t>(need, 16));
    AMG_CK(cub::DeviceScan::ExclusiveSum(tmp3, need, rowcnt, bptr, nbr + 1, s));
  }
  AMG_CK(cudaStreamSynchronize(s));  // the temporaries are freed on return
  return nb;
}

}  // namespace amgb
