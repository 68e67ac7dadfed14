// common.cuh -- shared host/device plumbing of the B200 library (no method arithmetic).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "amg.h"

namespace amgb {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

// Internal error: thrown inside the library, converted to a status code at the C ABI.
struct Error {
  int code;
  std::string what;
};

[[noreturn]] inline void fail(int code, const std::string& what) { throw Error{code, what}; }

#define AMG_CK(expr)                                                                       \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      ::amgb::fail(e_ == cudaErrorMemoryAllocation ? AMG_ENOMEM : AMG_ECUDA,               \
                   std::string(#expr) + ": " + cudaGetErrorString(e_));                    \
  } while (0)

#define AMG_CK_LAUNCH() AMG_CK(cudaGetLastError())

// internal element type (not a public amg_dtype): the GMRES pass-1 fp16 shadow basis (R28)
constexpr int AMG_F16 = 2;
inline size_t dtype_size(int dt) { return dt == AMG_F32 ? 4 : (dt == AMG_F16 ? 2 : 8); }

// Lab / test switches (AMG_*): read from the environment whenever a plan is made or an
// apply starts, never cached, so a test can A/B a kernel variant within one process.  None
// changes the arithmetic of the default path; DESIGN.md §6 lists them.
inline int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}
inline bool env_set(const char* name) { return std::getenv(name) != nullptr; }

// Owning device allocation list: every buffer of a handle lives here and is freed
// by the destructor.  Solve-phase code never allocates.
class Arena {
 public:
  Arena() = default;
  Arena(const Arena&) = delete;
  Arena& operator=(const Arena&) = delete;
  ~Arena() { release(); }
  void* alloc(size_t bytes) {
    if (bytes == 0) bytes = 16;
    bytes = (bytes + 255) & ~size_t(255);
    void* p = nullptr;
    AMG_CK(cudaMalloc(&p, bytes));
    ptrs_.push_back(p);
    sizes_.push_back((int64_t)bytes);
    total_ += (int64_t)bytes;
    return p;
  }
  template <class T>
  T* alloc_n(size_t n) {
    return static_cast<T*>(alloc(n * sizeof(T)));
  }
  void release() {
    for (void* p : ptrs_) cudaFree(p);
    ptrs_.clear();
    sizes_.clear();
    total_ = 0;
  }
  // free one allocation of this arena early (no-op for foreign pointers)
  void release_one(void* p) {
    for (size_t i = 0; i < ptrs_.size(); ++i)
      if (ptrs_[i] == p) {
        cudaFree(p);
        total_ -= sizes_[i];
        ptrs_.erase(ptrs_.begin() + i);
        sizes_.erase(sizes_.begin() + i);
        return;
      }
  }
  int64_t bytes() const { return total_; }

 private:
  std::vector<void*> ptrs_;
  std::vector<int64_t> sizes_;
  int64_t total_ = 0;
};

enum { kTmaNone = 0, kTmaGroup = 1, kTmaRows = 2, kTmaSeg = 3 };
// bsr_lane.cuh variants: R/C = ROWS/COLS layout, C/N = streaming / L1-allocating loads, U
enum { kLaneRC2 = 0, kLaneRC4 = 1, kLaneRN2 = 2, kLaneRN4 = 3, kLaneCN2 = 4, kLaneCN4 = 5, kLaneW = 6 /* warp per row */, kLaneSell = 7 /* sliced copy */,
       kLaneSellR = 8 /* interleaved row-per-lane copy */ };

// Device BSR matrix with b x b blocks (PAPER.md:666-672 layout); the Schur coupling
// views use rectangular br x bc blocks on the outer pattern.
struct Mat {
  int32_t n = 0, m = 0, b = 1;
  int64_t nnz = 0;
  int32_t* ptr = nullptr;
  int32_t* col = nullptr;
  void* val = nullptr;
  int vt = AMG_F64;
  int br = 0, bc = 0;  // rectangular blocks (0: b)
  // TMA-staged tile plan (bsr_tma.cuh); tma_grid == 0 -> direct kernels
  int tma_mode = kTmaNone;
  int tma_tr = 0, tma_ntiles = 0, tma_ns = 0, tma_stage = 0, tma_col_off = 0, tma_val_off = 0, tma_grid = 0;
  int tma_wave = 1, tma_part_off = 0, tma_max_blk = 0, tma_smem = 0;
  int lane_var = kLaneRC2;  // bsr_lane.cuh variant (make_tma_plan)
  int warp_g = 1;           // kLaneW: warps per block row (k_bsr_warps; set_lane_plan, by row length)
  // sliced copy of the blocks (kLaneSell; bsr_lane.cuh k_bsr_sell), owned by the builder's arena
  int32_t sell_ns = 0;
  int32_t* sell_ptr = nullptr;  // [sell_ns + 1] step offsets
  int32_t* sell_col = nullptr;  // [steps][C]
  void* sell_val = nullptr;     // [steps][b][C][b]
  int32_t* sell_perm = nullptr; // [sell_ns * C] slot -> row (-1: padding slot), or nullptr (in order)
  // kLaneSellR (k_bsr_sellr, C = 32): sell_col [steps][32], sell_val [vectors][32][sell_w],
  // sell_vptr [sell_ns + 1] vector offsets
  int32_t* sell_vptr = nullptr;
  int sell_w = 0;
  int sell_pf = 0;      // k_bsr_sellr bulk L2 prefetch flags (bsr_lane.cuh kPfRest | KiB cap)
  bool fast32 = false;  // internal fp32-hierarchy matrices: fp32 block-row dots (bsr.cuh item_dot)
  int rows_per_block() const { return br ? br : b; }
  int cols_per_block() const { return bc ? bc : b; }
};

inline unsigned grid_for(int64_t threads, int block) {
  int64_t g = (threads + block - 1) / block;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace amgb
