// spmv.cu -- instantiation + dispatch of the SpMV-type solve kernels (K1, K2, K4, K5,
// K8, K9, K10, K11).  See bsr.cuh for the block-row design.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "bsr.cuh"
#include "bsr_lane.cuh"
#include "bsr_tma.cuh"
#include "blas1.h"
#include "comm.h"
#include "ops.h"
#include "prof.h"

namespace amgb {


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

// dynamic shared memory already enabled per kernel (host-side, per function)
// (thread safe: ranks of the thread-emulated communicator launch concurrently)
static void ensure_smem(const void* kern, int smem) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> m;
  std::lock_guard<std::mutex> lk(mu);
  auto it = m.find(kern);
  if (it == m.end()) it = m.emplace(kern, 48 * 1024).first;
  if (smem > it->second) {
    AMG_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    it->second = smem;
  }
}

template <int BR, int BC, typename V, typename X, bool FAST, class EPI>
static void launch_tma_rows(const Mat& A, const X* x, EPI epi, cudaStream_t s) {
  if (!A.val && A.nnz > 0) fail(AMG_EINVAL, "BSR values released: no TMA plan on the BSR arrays");
  TmaArgs a{A.n, A.tma_tr, A.tma_ntiles, A.tma_ns, A.tma_stage, A.tma_col_off, A.tma_val_off,
            A.tma_wave, A.tma_part_off, A.tma_max_blk};
  const int smem = A.tma_smem;
  auto kern = k_bsr_tma_rows<BR, BC, V, X, FAST, EPI>;
  ensure_smem((const void*)kern, smem);
  kern<<<A.tma_grid, A.tma_tr, smem, s>>>(a, A.ptr, A.col, (const V*)A.val, x, epi);
}


// Kernel plan of a device matrix (bsr_lane.cuh variants, measured in tools/spmv_lab.cu):
//   4 x 4 (and b <= 2):     ROWS, streaming loads, U = 4 for long rows (> 12 blocks), else 2
//   3 x 3 fp32 values:      long rows COLS + L1-allocating loads, U = 4; short rows ROWS + nc, U = 2
//   3 x 3 fp64, rectangular: ROWS, U = 2 (nc for fp32 values)
// AMG_TMA=1 switches short-row fp32 matrices to the TMA-staged row-per-lane consumer
// (bsr_tma.cuh) for comparison.  One reduction + one sync only in that case.
void set_lane_plan(Mat& A, bool use_env) {
  const int br = A.rows_per_block(), bc = A.cols_per_block();
  const double per_row = A.n > 0 ? (double)A.nnz / A.n : 0.0;
  const bool f32 = A.vt == AMG_F32;
  int var = kLaneRC2;
  if (br == 4 && bc == 4) var = per_row > 12.0 ? kLaneRC4 : kLaneRC2;
  else if (br == 3 && bc == 3 && f32)  // very short rows (prolongators, ~3.6 blocks): COLS lanes
    var = per_row > 12.0 ? kLaneCN4 : (per_row < 6.5 ? kLaneCN2 : kLaneRN2);
  else if (br == 3 && bc == 3) var = per_row > 12.0 ? kLaneCN4 : kLaneCN2;
  else if (br == bc) var = kLaneRN4;
  else var = f32 ? kLaneRN2 : kLaneRC2;
  // very long rows, or long rows on a matrix too small to fill the GPU with row-lane
  // warps (coarse levels): one warp per row
  const double lane_warps = (double)A.n / (32 / std::max(br, 1));
  if (per_row > 64.0 || (per_row > 12.0 && lane_warps < (double)env_int("AMG_LANEW_WARPS", kSMs * 64))) var = kLaneW;
  A.lane_var = use_env ? env_int("AMG_LANE_VAR", var) : var;
  // warp-per-row matrices with long rows: G warps per row (k_bsr_warps), by the row length
  // (one or two 32-block chunks per warp)
  // and only where the level has at most one wave of row warps (n <= kSMs * 64: cfg 3 levels
  // 2-3, cfg 5 level 3; on 44 K-row levels the split loses, cfg 5 895 -> 914 ms)
  const int g = A.n > (int64_t)kSMs * 64 ? 1 : per_row >= 160.0 ? 8 : (per_row >= 80.0 ? 4 : (per_row >= 40.0 ? 2 : 1));
  A.warp_g = use_env && env_int("AMG_WARP_G", 0) > 0 ? env_int("AMG_WARP_G", 0) : g;
  if (A.warp_g != 1 && A.warp_g != 2 && A.warp_g != 4 && A.warp_g != 8) fail(AMG_EINVAL, "AMG_WARP_G: 1, 2, 4 or 8");
  // a forced sliced / interleaved variant needs its copy (make_tma_plan builds it)
  if ((A.lane_var == kLaneSell && !A.sell_ptr) || (A.lane_var == kLaneSellR && !A.sell_vptr)) A.lane_var = var;
}

// ---- sliced copy (k_bsr_sell) ----
template <typename V>
__global__ void k_sell_fill(int n, int b, int C, int ns, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                            const V* __restrict__ val, const int32_t* __restrict__ sptr, const int32_t* __restrict__ perm,
                            int32_t* __restrict__ scol, V* __restrict__ sval) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)ns * C) return;
  const int s = (int)(t / C), g = (int)(t % C);
  int64_t row = (int64_t)s * C + g;
  if (perm) row = perm[t] >= 0 ? perm[t] : n;  // slot -> row (sorted windows), n = padding slot
  const int k0 = row < n ? ptr[row] : 0, len = row < n ? ptr[row + 1] - k0 : 0;
  const int pad_col = row < n ? (int)row : 0;
  for (int j = 0; j < sptr[s + 1] - sptr[s]; ++j) {
    const int64_t st = sptr[s] + j;
    scol[st * C + g] = j < len ? col[k0 + j] : (len > 0 ? col[k0] : pad_col);
    for (int i = 0; i < b; ++i)
      for (int r = 0; r < b; ++r)
        sval[(st * b + i) * ((int64_t)C * b) + g * b + r] = j < len ? val[((int64_t)(k0 + j) * b + i) * b + r] : V(0);
  }
}

// Rows are taken in order, or -- when that cuts the zero padding by more than 3 % of the
// blocks -- sorted by length (descending, stable) inside windows of 32 slices (SELL-C-sigma,
// sigma = 32 C): a slot -> row permutation kept on the device, the epilogue writes row
// perm[slot].  Only rows inside one window are reordered, so the output stays local.
struct Slicing {
  int ns = 0;
  std::vector<int32_t> h, perm;  // steps per slice; slot -> row (empty: in order)
};

static Slicing slice_rows(const Mat& A, int C, cudaStream_t s) {
  Slicing out;
  const int ns = (int)((A.n + C - 1) / C);
  out.ns = ns;
  std::vector<int32_t> hp((size_t)A.n + 1);
  AMG_CK(cudaMemcpyAsync(hp.data(), A.ptr, sizeof(int32_t) * (A.n + 1), cudaMemcpyDeviceToHost, s));
  AMG_CK(cudaStreamSynchronize(s));
  auto len_of = [&](int64_t r) { return r < A.n ? hp[r + 1] - hp[r] : 0; };
  std::vector<int32_t> h(ns);
  int64_t pad_plain = 0;
  for (int i = 0; i < ns; ++i) {
    int mx = 0;
    for (int g = 0; g < C; ++g) mx = std::max(mx, len_of((int64_t)i * C + g));
    h[i] = mx;
    pad_plain += (int64_t)mx * C;
  }
  const int W = 32 * C;
  std::vector<int32_t> perm((size_t)ns * C, -1), hs(ns);
  int64_t pad_sorted = 0;
  for (int64_t w0 = 0; w0 < (int64_t)ns * C; w0 += W) {
    const int64_t w1 = std::min<int64_t>(w0 + W, (int64_t)ns * C);
    std::vector<int32_t> rows;
    for (int64_t r = w0; r < std::min<int64_t>(w1, A.n); ++r) rows.push_back((int32_t)r);
    std::stable_sort(rows.begin(), rows.end(), [&](int32_t a, int32_t b) { return len_of(a) > len_of(b); });
    for (size_t q = 0; q < rows.size(); ++q) perm[w0 + q] = rows[q];
    for (int64_t sl = w0 / C; sl < w1 / C; ++sl) {
      int mx = 0;
      for (int g = 0; g < C; ++g) {
        const int32_t r = perm[sl * C + g];
        if (r >= 0) mx = std::max(mx, len_of(r));
      }
      hs[sl] = mx;
      pad_sorted += (int64_t)mx * C;
    }
  }
  const bool sorted = (double)(pad_plain - pad_sorted) > 0.03 * (double)std::max<int64_t>(A.nnz, 1) &&
                      !env_int("AMG_SELL_NO_SORT", 0);
  out.h = sorted ? hs : h;
  if (sorted) out.perm = std::move(perm);
  return out;
}

static std::vector<int32_t> prefix32(const std::vector<int32_t>& h, const char* what) {
  std::vector<int32_t> sp(h.size() + 1, 0);
  for (size_t i = 0; i < h.size(); ++i) {
    if ((int64_t)sp[i] + h[i] > INT32_MAX) fail(AMG_EINDEX_OVERFLOW, what);
    sp[i + 1] = sp[i] + h[i];
  }
  return sp;
}

static int32_t* upload_perm(const Slicing& sl, int C, Arena& arena, cudaStream_t s) {
  if (sl.perm.empty()) return nullptr;
  int32_t* d = arena.alloc_n<int32_t>((size_t)sl.ns * C);
  AMG_CK(cudaMemcpyAsync(d, sl.perm.data(), sizeof(int32_t) * sl.ns * C, cudaMemcpyHostToDevice, s));
  return d;
}

static void build_sell(Mat& A, Arena& arena, cudaStream_t s) {
  const int C = 32 / A.b;
  const Slicing sl = slice_rows(A, C, s);
  const int ns = sl.ns;
  const std::vector<int32_t> sp = prefix32(sl.h, "sliced copy: too many steps");
  const int64_t steps = sp[ns];
  A.sell_ns = ns;
  A.sell_ptr = arena.alloc_n<int32_t>(ns + 1);
  A.sell_col = arena.alloc_n<int32_t>(std::max<int64_t>(steps * C, 1));
  A.sell_val = arena.alloc(std::max<int64_t>(steps * C * A.b * A.b, 1) * dtype_size(A.vt));
  AMG_CK(cudaMemcpyAsync(A.sell_ptr, sp.data(), sizeof(int32_t) * (ns + 1), cudaMemcpyHostToDevice, s));
  A.sell_perm = upload_perm(sl, C, arena, s);
  dispatch_t(A.vt, [&](auto v) {
    using V = decltype(v);
    k_sell_fill<V><<<grid_for((int64_t)ns * C, 256), 256, 0, s>>>(A.n, A.b, C, ns, A.ptr, A.col, (const V*)A.val,
                                                                   A.sell_ptr, A.sell_perm, A.sell_col, (V*)A.sell_val);
  });
  AMG_CK_LAUNCH();
  AMG_CK(cudaStreamSynchronize(s));  // sp (host) must outlive the copy
  A.lane_var = kLaneSell;
}

// inverse of k_sell_fill: the BSR values back from the sliced copy (padding skipped)
template <typename V>
__global__ void k_sell_unfill(int n, int b, int C, int ns, const int32_t* __restrict__ ptr,
                              const int32_t* __restrict__ sptr, const int32_t* __restrict__ perm,
                              const V* __restrict__ sval, V* __restrict__ val) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)ns * C) return;
  const int s = (int)(t / C), g = (int)(t % C);
  int64_t row = (int64_t)s * C + g;
  if (perm) row = perm[t] >= 0 ? perm[t] : n;
  if (row >= n) return;
  const int k0 = ptr[row], len = ptr[row + 1] - k0;
  for (int j = 0; j < len; ++j) {
    const int64_t st = sptr[s] + j;
    for (int i = 0; i < b; ++i)
      for (int r = 0; r < b; ++r)
        val[((int64_t)(k0 + j) * b + i) * b + r] = sval[(st * b + i) * ((int64_t)C * b) + g * b + r];
  }
}

// ---- interleaved row-per-lane copy (k_bsr_sellr) ----
template <typename V>
__global__ void k_sellr_fill(int n, int E, int W, int ns, const int32_t* __restrict__ ptr,
                             const int32_t* __restrict__ col, const V* __restrict__ val,
                             const int32_t* __restrict__ sptr, const int32_t* __restrict__ vptr,
                             const int32_t* __restrict__ perm, int32_t* __restrict__ scol, V* __restrict__ sval) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)ns * 32) return;
  const int s = (int)(t / 32), g = (int)(t % 32);
  int64_t row = t;
  if (perm) row = perm[t] >= 0 ? perm[t] : n;
  const int k0 = row < n ? ptr[row] : 0, len = row < n ? ptr[row + 1] - k0 : 0;
  for (int j = 0; j < sptr[s + 1] - sptr[s]; ++j)  // padding: a column the row reads anyway (or 0)
    scol[((int64_t)sptr[s] + j) * 32 + g] = j < len ? col[k0 + j] : (len > 0 ? col[k0] : 0);
  const int64_t nv = vptr[s + 1] - vptr[s];
  for (int64_t e = 0; e < nv * W; ++e) {
    const int64_t q = e / W, jb = e / E;
    sval[(((int64_t)vptr[s] + q) * 32 + g) * W + (e % W)] = jb < len ? val[(k0 + jb) * E + (e % E)] : V(0);
  }
}

// inverse of k_sellr_fill
template <typename V>
__global__ void k_sellr_unfill(int n, int E, int W, int ns, const int32_t* __restrict__ ptr,
                               const int32_t* __restrict__ vptr, const int32_t* __restrict__ perm,
                               const V* __restrict__ sval, V* __restrict__ val) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)ns * 32) return;
  const int s = (int)(t / 32), g = (int)(t % 32);
  int64_t row = t;
  if (perm) row = perm[t] >= 0 ? perm[t] : n;
  if (row >= n) return;
  const int k0 = ptr[row], len = ptr[row + 1] - k0;
  for (int64_t e = 0; e < (int64_t)len * E; ++e) {
    const int64_t q = e / W, jb = e / E;
    val[(k0 + jb) * E + (e % E)] = sval[(((int64_t)vptr[s] + q) * 32 + g) * W + (e % W)];
  }
}

static void build_sellr(Mat& A, Arena& arena, cudaStream_t s) {
  // 16-byte vectors; square 3x3 fp32 rows of < 12 blocks (A_0: 7, prolongators: 3.6) take
  // 8-byte ones -- GB = 2 blocks per step at 48 registers and 5 blocks per SM instead of 4
  // blocks per step at 128 registers and 2 (A_0 5.65 -> 6.0, P_0 3.3 -> 4.7 TB/s); long rows
  // keep 16-byte vectors (A_1 / R_0 6.4-6.5 vs 5.8-6.3)
  const double per_row = A.n > 0 ? (double)A.nnz / A.n : 0.0;
  const bool short3 = A.br == 0 && A.bc == 0 && A.b == 3 && per_row < 12.0;
  const int W = env_int("AMG_SELLR_W", A.vt == AMG_F32 && !short3 ? 4 : 2);
  if (!(W == 4 && A.vt == AMG_F32) && W != 2) fail(AMG_EINVAL, "AMG_SELLR_W: 4 (fp32) or 2");
  const int E = A.rows_per_block() * A.cols_per_block();
  const Slicing sl = slice_rows(A, 32, s);
  const int ns = sl.ns;
  const std::vector<int32_t> sp = prefix32(sl.h, "interleaved copy: too many steps");
  std::vector<int32_t> nvec(ns);
  for (int i = 0; i < ns; ++i) nvec[i] = (int32_t)(((int64_t)E * sl.h[i] + W - 1) / W);
  const std::vector<int32_t> vp = prefix32(nvec, "interleaved copy: too many vectors");
  A.sell_ns = ns;
  A.sell_w = W;
  A.sell_ptr = arena.alloc_n<int32_t>(ns + 1);
  A.sell_vptr = arena.alloc_n<int32_t>(ns + 1);
  A.sell_col = arena.alloc_n<int32_t>(std::max<int64_t>((int64_t)sp[ns] * 32, 1));
  A.sell_val = arena.alloc(std::max<int64_t>((int64_t)vp[ns] * 32 * W, 1) * dtype_size(A.vt));
  AMG_CK(cudaMemcpyAsync(A.sell_ptr, sp.data(), sizeof(int32_t) * (ns + 1), cudaMemcpyHostToDevice, s));
  AMG_CK(cudaMemcpyAsync(A.sell_vptr, vp.data(), sizeof(int32_t) * (ns + 1), cudaMemcpyHostToDevice, s));
  A.sell_perm = upload_perm(sl, 32, arena, s);
  dispatch_t(A.vt, [&](auto v) {
    using V = decltype(v);
    k_sellr_fill<V><<<grid_for((int64_t)ns * 32, 256), 256, 0, s>>>(A.n, E, W, ns, A.ptr, A.col, (const V*)A.val,
                                                                     A.sell_ptr, A.sell_vptr, A.sell_perm, A.sell_col,
                                                                     (V*)A.sell_val);
  });
  AMG_CK_LAUNCH();
  AMG_CK(cudaStreamSynchronize(s));
  A.lane_var = kLaneSellR;
  // bulk L2 prefetch of each slice past its first step (kPfRest): the 8-byte-vector 3x3 fp32
  // rows of >= 5 blocks -- 2-4 dependent steps per slice at 40 registers (cfg 5 A_0: smoother
  // 6.08 -> 6.42-6.53, residual 5.95 -> 6.39-6.42 TB/s); the 16-byte-vector / fp64 shapes lose
  // 1-3 % with it (outer 4x4 fp64 7.07 -> 6.97, R_0 6.34 -> 6.07-6.16 TB/s)
  A.sell_pf = (short3 && W == 2 && per_row >= 5.0) ? (kPfRest | 64) : 0;
}

void make_tma_plan(Mat& A, cudaStream_t s, Arena* arena, bool want_tma) {
  A.tma_grid = 0;
  A.tma_mode = kTmaNone;
  set_lane_plan(A);
  {
    const double per_row = A.n > 0 ? (double)A.nnz / A.n : 0.0;
    const bool square = A.br == 0 && A.bc == 0 && A.b >= 2 && A.b <= 4;
    // Schur B^T (nu x 1 blocks): interleaved copy 5.4 vs 5.15 TB/s (TMA rows); B (1 x nu) stays on
    // the lane kernel (5.1 vs 4.1 interleaved)
    const bool rect = (A.br > 0 || A.bc > 0) && (A.rows_per_block() > 1 || env_int("AMG_SCHUR_B_SELLR", 0)) &&
                      A.rows_per_block() <= 4 && A.cols_per_block() <= 4;
    const int forced = env_set("AMG_LANE_VAR") ? env_int("AMG_LANE_VAR", 0) : -1;
    // interleaved row-per-lane copy (k_bsr_sellr): 0 never, 1 (default) square-block matrices with
    // 3..64 blocks per row on >= 64 slices per SM, 2 every square matrix with an arena.  Measured
    // (cfg 5 / cfg 2): A_0 5.65, A_1 / R_0 6.4-6.5, outer 4x4 fp64 7.07, cfg-2 4x4 fp32 x fp64
    // 6.85, fp64 7.03 TB/s vs 4.8 / 5.4 / 6.74 / 6.07 / 6.70 for the row lanes / sliced copy;
    // the 3.6-block prolongators with 8-byte vectors 4.0 vs 3.9 for the COLS lanes
    const int sellr_mode = env_int("AMG_SELLR", 1);
    const double sellr_min_row = env_int("AMG_SELLR_MIN_ROW", 3);
    // sliced copies need the builder's arena and square b x b blocks
    if (arena && rect && forced < 0 && sellr_mode >= 1 && per_row >= 3 && per_row <= 64 &&
        (int64_t)A.n / 32 >= env_int("AMG_SELLR_MIN_SLICES", 4096)) {
      build_sellr(A, *arena, s);  // Schur coupling views (1 x nu, nu x 1 blocks on A's pattern)
    } else if (arena && square && forced == kLaneSellR) {
      build_sellr(A, *arena, s);
    } else if (arena && square && forced == kLaneSell) {
      build_sell(A, *arena, s);
    } else if (arena && square && forced < 0) {
      const double lo = env_int("AMG_SELL_MIN_ROW", 12), hi = env_int("AMG_SELL_MAX_ROW", 64);
      // >= 64 slices per SM: below that the per-slice step chains are latency bound and
      // the warp-per-row kernel (set_lane_plan) is faster (cfg 3 level 1: 41 us vs ~10 us)
      const int64_t min_slices = env_int("AMG_SELL_MIN_SLICES", kSMs * 64);
      // the interleaved copy pays from >= 4096 slices of 32 rows (cfg 4 level 1, 8,236 slices:
      // 4.8 -> 5.5-5.6 TB/s; 1024 slices lose at cfg 3)
      const bool many = (int64_t)A.n / 32 >= env_int("AMG_SELLR_MIN_SLICES", 4096);
      if (sellr_mode == 2 || (sellr_mode == 1 && many && per_row >= sellr_min_row && per_row <= hi))
        build_sellr(A, *arena, s);
      else if (per_row > lo && per_row <= hi && (int64_t)A.n / (32 / A.b) >= min_slices && !env_int("AMG_NO_SELL", 0))
        build_sell(A, *arena, s);
    }
  }
  if (A.lane_var == kLaneSellR) return;  // the interleaved copy replaces the TMA consumer
  const int br = A.rows_per_block(), bc = A.cols_per_block();
  const double per_row = A.n > 0 ? (double)A.nnz / A.n : 0.0;
  if (!(want_tma || env_int("AMG_TMA", 0)) || A.n < 2048 || A.vt != AMG_F32) return;
  const double bb = (double)br * bc * dtype_size(A.vt) + 4.0;
  const double row_bytes = std::max(1.0, per_row * bb);
  if (!(per_row <= 12.0 && 128 * row_bytes <= 40 * 1024)) return;
  const int tr = env_int("AMG_TMA_ROWS_TR", 128);
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
  const int64_t vbytes64 = (int64_t)mx * br * bc * dtype_size(A.vt) + 32;
  if (vbytes64 > 96 * 1024) return;
  const int stage = pbytes + cbytes + a16(vbytes64);
  const int ns = env_int("AMG_TMA_NS", 3);
  int per_sm = (220 * 1024) / (ns * stage);
  per_sm = std::min(per_sm, std::min(8, 2048 / tr));
  if (per_sm < 1) return;
  A.tma_mode = kTmaRows;
  A.tma_tr = tr;
  A.tma_ntiles = ntiles;
  A.tma_ns = ns;
  A.tma_stage = stage;
  A.tma_col_off = pbytes;
  A.tma_val_off = pbytes + cbytes;
  A.tma_part_off = ns * stage;
  A.tma_max_blk = std::max(mx, 1);
  A.tma_smem = ns * stage;
  A.tma_wave = env_int("AMG_TMA_WAVE", 1);
  A.tma_grid = std::min(ntiles, kSMs * per_sm);
}

// lane-kernel variant -> compile-time (U, COLS, NC); only the variants a block shape uses
// are instantiated
template <int BR, int BC, class F>
static void dispatch_lane(int var, F&& f) {
  auto go = [&](auto U, auto COLS, auto NC) { f(U, COLS, NC); };
  using I2 = std::integral_constant<int, 2>;
  using I4 = std::integral_constant<int, 4>;
  using T = std::true_type;
  using Fa = std::false_type;
  if constexpr (BR == 3 && BC == 3) {
    if (var == kLaneCN4) go(I4{}, T{}, T{});
    else if (var == kLaneCN2) go(I2{}, T{}, T{});
    else if (var == kLaneRN4) go(I4{}, Fa{}, T{});
    else if (var == kLaneRC2) go(I2{}, Fa{}, Fa{});
    else go(I2{}, Fa{}, T{});
  } else if constexpr (BR == 4 && BC == 4) {
    if (var == kLaneRC4) go(I4{}, Fa{}, Fa{});
    else if (var == kLaneRN2) go(I2{}, Fa{}, T{});
    else go(I2{}, Fa{}, Fa{});
  } else {
    if (var == kLaneRC2) go(I2{}, Fa{}, Fa{});
    else if (var == kLaneRN2) go(I2{}, Fa{}, T{});
    else go(I4{}, Fa{}, T{});
  }
}

bool sellr_range_ok(const Mat& A, int r0, int r1) {
  return A.lane_var == kLaneSellR && !A.sell_perm && r0 % 32 == 0 && (r1 >= A.n || r1 % 32 == 0);
}

// grid: one virtual block per WPB slices (the kernel's launch shape, SellrCfg); fused dots:
// a persistent grid of at most kMaxPartials blocks
template <int BR, int BC, typename V, typename X, class EPI>
static void launch_sellr(const Mat& A, const X* x, EPI epi, cudaStream_t s, bool fast, bool dots, int s0 = 0,
                         int s1 = -1) {
  if (s1 < 0) s1 = A.sell_ns;
  if (s1 <= s0) return;
  // L2 prefetches (plan: Mat::sell_pf; AMG_SELLR_PF overrides): kPfRest | KiB cap
  const int pf = env_set("AMG_SELLR_PF") ? env_int("AMG_SELLR_PF", 0) : A.sell_pf;
  auto go = [&](auto Wc) {
    constexpr int W = decltype(Wc)::value;
    constexpr bool can_fast = std::is_same_v<V, float> && std::is_same_v<X, float>;
    auto run = [&](auto Fc) {
      constexpr bool F = decltype(Fc)::value;
      using Cfg = SellrCfg<BR, BC, W, V, F>;
      int64_t g = ((int64_t)s1 - s0 + Cfg::WPB - 1) / Cfg::WPB;
      if (dots) g = std::min<int64_t>(g, kMaxPartials);
      k_bsr_sellr<BR, BC, W, V, X, F, EPI><<<(unsigned)std::max<int64_t>(g, 1), Cfg::TPB, 0, s>>>(
          A.n, s0, s1, A.sell_ptr, A.sell_vptr, A.sell_perm, A.sell_col, (const V*)A.sell_val, x, epi, pf);
    };
    if (can_fast && fast) run(std::integral_constant<bool, can_fast>{});
    else run(std::false_type{});
  };
  if constexpr (std::is_same_v<V, float>) {
    if (A.sell_w == 4) go(std::integral_constant<int, 4>{});
    else go(std::integral_constant<int, 2>{});
  } else {
    go(std::integral_constant<int, 2>{});
  }
}

template <int BR, int BC, typename V, typename X, class EPI>
static void launch_lane(const Mat& A, const X* x, EPI epi, cudaStream_t s, int r0 = 0, int r1 = -1) {
  if (r1 < 0) r1 = A.n;
  if (r1 <= r0) return;
  const bool ranged = r0 > 0 || r1 < A.n;
  if (ranged && A.lane_var == kLaneSellR && !sellr_range_ok(A, r0, r1))
    fail(AMG_EINVAL, "interleaved copy: row ranges must be 32-aligned and unpermuted");
  if (ranged && ((A.lane_var > kLaneCN4 && A.lane_var != kLaneSellR) || A.tma_grid > 0))
    fail(AMG_EINVAL, "row ranges need a row-lane plan");
  constexpr bool can_fast = std::is_same_v<V, float> && std::is_same_v<X, float>;
  if constexpr (BR != BC || BR >= 2) {
    if (A.lane_var == kLaneSellR) {
      const int s0 = r0 / 32, s1 = r1 >= A.n ? A.sell_ns : r1 / 32;
      launch_sellr<BR, BC, V, X>(A, x, epi, s, can_fast && A.fast32, false, s0, s1);
      return;
    }
  }
  if constexpr (BR == BC && BR >= 2) {
    if (A.lane_var == kLaneSell) {
      constexpr int U = (BR * BR * sizeof(V) <= 36) ? 4 : 2;
      const unsigned grid = grid_for((int64_t)A.sell_ns * 32, kBlock);
      k_bsr_sell<BR, U, V, X, EPI><<<grid, kBlock, 0, s>>>(A.n, A.sell_ns, A.sell_ptr, A.sell_perm, A.sell_col,
                                                          (const V*)A.sell_val, x, epi);
      return;
    }
  }
  if (!A.val && A.nnz > 0)
    fail(AMG_EINVAL, "BSR values released: this matrix runs on its interleaved / sliced copy only");
  if (A.lane_var == kLaneW && A.warp_g > 1) {
    auto go = [&](auto Gc) {
      constexpr int G = decltype(Gc)::value;
      const unsigned grid = (unsigned)(((int64_t)A.n + 8 / G - 1) / (8 / G));
      if (can_fast && A.fast32)
        k_bsr_warps<BR, BC, 2, G, V, X, can_fast, EPI><<<grid, 256, 0, s>>>(A.n, A.ptr, A.col, (const V*)A.val, x, epi);
      else
        k_bsr_warps<BR, BC, 2, G, V, X, false, EPI><<<grid, 256, 0, s>>>(A.n, A.ptr, A.col, (const V*)A.val, x, epi);
    };
    if (A.warp_g == 2) go(std::integral_constant<int, 2>{});
    else if (A.warp_g == 4) go(std::integral_constant<int, 4>{});
    else go(std::integral_constant<int, 8>{});
    return;
  }
  if (A.lane_var == kLaneW) {
    const unsigned grid = grid_for((int64_t)A.n * 32, kBlock);
    if (can_fast && A.fast32)
      k_bsr_warp<BR, BC, 2, V, X, can_fast, EPI><<<grid, kBlock, 0, s>>>(A.n, A.ptr, A.col, (const V*)A.val, x, epi);
    else
      k_bsr_warp<BR, BC, 2, V, X, false, EPI><<<grid, kBlock, 0, s>>>(A.n, A.ptr, A.col, (const V*)A.val, x, epi);
    return;
  }
  constexpr int RPW = 32 / BR;
  const int64_t warps = ((int64_t)(r1 - r0) + RPW - 1) / RPW;
  const unsigned grid = grid_for(warps * 32, kBlock);
  dispatch_lane<BR, BC>(A.lane_var, [&](auto Uc, auto Cc, auto Nc) {
    constexpr int U = decltype(Uc)::value;
    constexpr bool COLS = decltype(Cc)::value, NC = decltype(Nc)::value;
    if (can_fast && A.fast32)
      k_bsr_lane<BR, BC, U, COLS, NC, V, X, can_fast, EPI><<<grid, kBlock, 0, s>>>(r0, r1, A.ptr, A.col, (const V*)A.val, x, epi);
    else
      k_bsr_lane<BR, BC, U, COLS, NC, V, X, false, EPI><<<grid, kBlock, 0, s>>>(r0, r1, A.ptr, A.col, (const V*)A.val, x, epi);
  });
}

void launch_spmv(const Mat& A, double alpha, const void* x, int xt, double beta, void* y, int yt,
                 cudaStream_t s, int r0, int r1) {
  if (r1 < 0) r1 = A.n;
  if (A.n == 0 || r1 <= r0) return;
  const double frac = (double)(r1 - r0) / A.n;
  ProfScope ps_(prof_name("spmv", A.b, A.vt, xt),
                frac * (mat_bytes(A) + (double)A.m * A.b * dtype_size(xt) +
                        (double)A.n * A.b * dtype_size(yt) * (beta != 0.0 ? 2.0 : 1.0)), s);
  dispatch_b(A.b, [&](auto Bc) {
    constexpr int B = decltype(Bc)::value;
    dispatch_t(A.vt, [&](auto v) {
      using V = decltype(v);
      dispatch_t(xt, [&](auto xx) {
        using X = decltype(xx);
        dispatch_t(yt, [&](auto yy) {
          using Y = decltype(yy);
          if (A.tma_grid > 0) {
            if (A.fast32) launch_tma_rows<B, B, V, X, true>(A, (const X*)x, EpiSpmv<B, Y>{alpha, beta, (Y*)y}, s);
            else launch_tma_rows<B, B, V, X, false>(A, (const X*)x, EpiSpmv<B, Y>{alpha, beta, (Y*)y}, s);
          } else {
            // K7 on short-row interleaved copies (the prolongators): y loaded ahead of the row
            const bool pre = beta != 0.0 && A.lane_var == kLaneSellR && A.sell_pf == 0 && env_int("AMG_SPMV_PRE", 1);
            if (pre)
              launch_lane<B, B, V, X>(A, (const X*)x, LEpiSpmvPre<Y>{{alpha, beta, (Y*)y}}, s, r0, r1);
            else
              launch_lane<B, B, V, X>(A, (const X*)x, LEpiSpmv<Y>{alpha, beta, (Y*)y}, s, r0, r1);
          }
        });
      });
    });
  });
  AMG_CK_LAUNCH();
}

// K3 / K2 fused forms (row-lane plans only; false -> the caller runs the unfused pair)
template <class EPI>
static bool launch_lane_dot(const Mat& A, const void* x, int xt, EPI epi, cudaStream_t s) {
  if (A.tma_grid > 0 || A.n == 0) return false;
  if (A.lane_var == kLaneSellR) {
    bool done = false;
    dispatch_b(A.b, [&](auto Bc) {
      constexpr int B = decltype(Bc)::value;
      if constexpr (B >= 2) {
        done = true;
        dispatch_t(A.vt, [&](auto v) {
          using V = decltype(v);
          dispatch_t(xt, [&](auto xx) {
            using X = decltype(xx);
            launch_sellr<B, B, V, X>(A, (const X*)x, epi, s, false, true);
          });
        });
      }
    });
    AMG_CK_LAUNCH();
    return done;
  }
  if (A.lane_var > kLaneCN4) return false;
  if (!A.val && A.nnz > 0)
    fail(AMG_EINVAL, "BSR values released: this matrix runs on its interleaved / sliced copy only");
  bool done = false;
  dispatch_b(A.b, [&](auto Bc) {
    constexpr int B = decltype(Bc)::value;
    constexpr int RPW = 32 / B;
    const int64_t nvb = ((int64_t)A.n + RPW * 8 - 1) / (RPW * 8);
    const unsigned grid = (unsigned)std::min<int64_t>(nvb, kMaxPartials);
    dispatch_t(A.vt, [&](auto v) {
      using V = decltype(v);
      dispatch_t(xt, [&](auto xx) {
        using X = decltype(xx);
        dispatch_lane<B, B>(A.lane_var, [&](auto Uc, auto Cc, auto Nc) {
          constexpr int U = decltype(Uc)::value;
          constexpr bool COLS = decltype(Cc)::value, NC = decltype(Nc)::value;
          k_bsr_lane<B, B, U, COLS, NC, V, X, false, EPI><<<grid, kBlock, 0, s>>>(0, A.n, A.ptr, A.col,
                                                                                  (const V*)A.val, (const X*)x, epi);
          done = true;
        });
      });
    });
  });
  AMG_CK_LAUNCH();
  return done;
}

bool launch_spmv_dot(const Mat& A, const void* x, int xt, double* y, const double* w0, const double* w1, int nd,
                     double* partials, double* out, cudaStream_t s, CommBase* comm) {
  if (nd < 1 || nd > 2) return false;
  const double mb = mat_bytes(A) + (double)A.m * A.b * dtype_size(xt) + (double)A.n * A.b * 8.0 * (1 + nd);
  unsigned* ticket = reinterpret_cast<unsigned*>(partials + (size_t)kMaxPartials * 32);
  bool ok;
  {
    ProfScope ps_(prof_name("spmv_dot", A.b, A.vt, xt), mb, s);
    if (nd == 1) ok = launch_lane_dot(A, x, xt, LEpiSpmvDot<1>{y, {w0, nullptr}, partials, out, ticket}, s);
    else ok = launch_lane_dot(A, x, xt, LEpiSpmvDot<2>{y, {w0, w1}, partials, out, ticket}, s);
  }
  if (ok && comm) comm->allreduce_sum(out, nd, s);
  return ok;
}

bool launch_residual_nrm(const Mat& A, const double* f, const void* x, int xt, double* r, double* partials,
                         double* out, cudaStream_t s, CommBase* comm) {
  const double mb = mat_bytes(A) + (double)A.m * A.b * dtype_size(xt) + (double)A.n * A.b * 16.0;
  unsigned* ticket = reinterpret_cast<unsigned*>(partials + (size_t)kMaxPartials * 32);
  bool ok;
  {
    ProfScope ps_(prof_name("residual_nrm", A.b, A.vt, xt), mb, s);
    ok = launch_lane_dot(A, x, xt, LEpiResidualNrm{f, r, partials, out, ticket}, s);
  }
  if (ok && comm) comm->allreduce_sum(out, 1, s);
  return ok;
}

void launch_residual(const Mat& A, const void* f, const void* x, void* r, int xt, cudaStream_t s, int r0, int r1) {
  if (r1 < 0) r1 = A.n;
  if (A.n == 0 || r1 <= r0) return;
  const double frac = (double)(r1 - r0) / A.n;
  ProfScope ps_(prof_name("residual", A.b, A.vt, xt),
                frac * (mat_bytes(A) + (double)A.m * A.b * dtype_size(xt) + 2.0 * A.n * A.b * dtype_size(xt)), s);
  dispatch_b(A.b, [&](auto Bc) {
    constexpr int B = decltype(Bc)::value;
    dispatch_t(A.vt, [&](auto v) {
      using V = decltype(v);
      dispatch_t(xt, [&](auto xx) {
        using X = decltype(xx);
        if (A.tma_grid > 0) {
          if (A.fast32) launch_tma_rows<B, B, V, X, true>(A, (const X*)x, EpiResidual<B, X>{(const X*)f, (X*)r}, s);
          else launch_tma_rows<B, B, V, X, false>(A, (const X*)x, EpiResidual<B, X>{(const X*)f, (X*)r}, s);
        } else {
          launch_lane<B, B, V, X>(A, (const X*)x, LEpiResidual<X>{(const X*)f, (X*)r}, s, r0, r1);
        }
      });
    });
  });
  AMG_CK_LAUNCH();
}

// xo = xb + M (f - A g): the smoother (g = xb = x) and the ILU(0) U sweeps (g = z, xb = the
// smoothed iterate on the last sweep, else nullptr = from zero)
static void launch_smooth_g(const char* label, const Mat& A, const void* M, const void* f, const void* g,
                            const void* xb, void* xo, int xt, cudaStream_t s, int r0, int r1) {
  if (r1 < 0) r1 = A.n;
  if (A.n == 0 || r1 <= r0) return;
  const double frac = (double)(r1 - r0) / A.n;
  ProfScope ps_(prof_name(label, A.b, A.vt, xt),
                frac * (mat_bytes(A) + (double)A.n * A.b * A.b * dtype_size(A.vt) +
                        (2.0 + (xb ? 1.0 : 0.0)) * A.n * A.b * dtype_size(xt) + (double)A.m * A.b * dtype_size(xt) -
                        (g == xb ? (double)A.n * A.b * dtype_size(xt) : 0.0)),
                s);
  dispatch_b(A.b, [&](auto Bc) {
    constexpr int B = decltype(Bc)::value;
    dispatch_t(A.vt, [&](auto v) {
      using V = decltype(v);
      dispatch_t(xt, [&](auto xx) {
        using X = decltype(xx);
        if (A.tma_grid > 0) {
          auto e = EpiSmooth<B, V, X>{(const V*)M, (const X*)f, (const X*)xb, (X*)xo};
          if (A.fast32) launch_tma_rows<B, B, V, X, true>(A, (const X*)g, e, s);
          else launch_tma_rows<B, B, V, X, false>(A, (const X*)g, e, s);
        } else {
          launch_lane<B, B, V, X>(A, (const X*)g, LEpiSmooth<V, X>{(const V*)M, (const X*)f, (const X*)xb, (X*)xo}, s,
                                  r0, r1);
        }
      });
    });
  });
  AMG_CK_LAUNCH();
}

void launch_smooth(const Mat& A, const void* M, const void* f, const void* x, void* xo, int xt,
                   cudaStream_t s, int r0, int r1) {
  launch_smooth_g("smooth", A, M, f, x, x, xo, xt, s, r0, r1);
}

// K5 + K9': the second U-solve's last post-smoothing step writes z = join(u, p) directly
// (LEpiSmoothJoin; 3x3 fp32 velocity levels of the interleaved 4x4 Stokes layout)
bool smooth_join_ok(const Mat& A, int xt) { return A.b == 3 && A.br == 0 && A.bc == 0 && A.tma_grid == 0 && xt == AMG_F32; }

void launch_smooth_join(const Mat& A, const void* M, const void* f, const void* x, const void* p, void* z, int zt,
                        int xt, cudaStream_t s, int r0, int r1) {
  if (!smooth_join_ok(A, xt)) fail(AMG_EINVAL, "fused smooth + join: 3x3 fp32 velocity level only");
  if (r1 < 0) r1 = A.n;
  if (A.n == 0 || r1 <= r0) return;
  const double frac = (double)(r1 - r0) / A.n;
  // matrix, M, f and x read, x gathered (once: g == x), p read, z written
  ProfScope ps_(prof_name("smooth_join", A.b, A.vt, zt),
                frac * (mat_bytes(A) + (double)A.n * 9 * dtype_size(A.vt) + (double)A.n * 3 * 4 +
                        (double)A.m * 3 * 4 + (double)A.n * 4 + (double)A.n * 4 * dtype_size(zt)),
                s);
  dispatch_t(A.vt, [&](auto v) {
    using V = decltype(v);
    dispatch_t(zt, [&](auto zz) {
      using Z = decltype(zz);
      launch_lane<3, 3, V, float>(
          A, (const float*)x,
          LEpiSmoothJoin<V, float, Z>{(const V*)M, (const float*)f, (const float*)x, (const float*)p, (Z*)z}, s, r0,
          r1);
    });
  });
  AMG_CK_LAUNCH();
}

// K5 + the monolithic apply's output conversion (LEpiSmoothWiden): 3x3 / 4x4 levels on the
// lane kernels; fp32 vectors widened into fp64 z, or z of the vectors' own dtype (the plain
// smoother writing z)
bool smooth_widen_ok(const Mat& A, int xt, int zt) {
  return A.br == 0 && A.bc == 0 && A.tma_grid == 0 && (A.b == 3 || A.b == 4) &&
         (xt == zt || (xt == AMG_F32 && zt == AMG_F64));
}

void launch_smooth_widen(const Mat& A, const void* M, const void* f, const void* x, void* z, int zt, int xt,
                         cudaStream_t s, int r0, int r1) {
  if (!smooth_widen_ok(A, xt, zt)) fail(AMG_EINVAL, "fused smooth + widen: 3x3 / 4x4 lane-kernel level only");
  if (xt == zt) return launch_smooth_g("smooth", A, M, f, x, x, z, xt, s, r0, r1);
  if (r1 < 0) r1 = A.n;
  if (A.n == 0 || r1 <= r0) return;
  const double frac = (double)(r1 - r0) / A.n;
  // matrix, M, f and x read, x gathered (once), z written (fp64)
  ProfScope ps_(prof_name("smooth_widen", A.b, A.vt, zt),
                frac * (mat_bytes(A) + (double)A.n * A.b * A.b * dtype_size(A.vt) + 2.0 * A.n * A.b * 4 +
                        (double)A.m * A.b * 4 + (double)A.n * A.b * 8),
                s);
  dispatch_t(A.vt, [&](auto v) {
    using V = decltype(v);
    auto go = [&](auto Bc) {
      constexpr int B = decltype(Bc)::value;
      launch_lane<B, B, V, float>(
          A, (const float*)x, LEpiSmoothWiden<V, float, double>{(const V*)M, (const float*)f, (const float*)x, (double*)z},
          s, r0, r1);
    };
    if (A.b == 3) go(std::integral_constant<int, 3>{});
    else go(std::integral_constant<int, 4>{});
  });
  AMG_CK_LAUNCH();
}

void launch_ilu_usweep(const Mat& U, const void* Dinv, const void* y, const void* z, const void* xb, void* xo, int xt,
                       cudaStream_t s) {
  launch_smooth_g("ilu_u", U, Dinv, y, z, xb, xo, xt, s, 0, -1);
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

// ---- K4a fused into the producer of f ----
// K6 + K4a: f = A g, x = M f (A: the restriction R_l; M, f, x: level l+1's)
bool launch_spmv_M(const Mat& A, const void* g, void* f, const void* M, int mvt, void* x, int xt, cudaStream_t s) {
  if (A.tma_grid > 0 || mvt != A.vt || A.br != A.bc) return false;
  if (A.n == 0) return true;
  ProfScope ps_(prof_name("spmv_M", A.b, A.vt, xt),
                mat_bytes(A) + (double)A.m * A.b * dtype_size(xt) + 2.0 * A.n * A.b * dtype_size(xt) +
                    (double)A.n * A.b * A.b * dtype_size(mvt),
                s);
  dispatch_b(A.b, [&](auto Bc) {
    constexpr int B = decltype(Bc)::value;
    dispatch_t(A.vt, [&](auto v) {
      using V = decltype(v);
      dispatch_t(xt, [&](auto xx) {
        using X = decltype(xx);
        launch_lane<B, B, V, X>(A, (const X*)g, LEpiSpmvM<V, X>{(const V*)M, (X*)f, (X*)x}, s);
      });
    });
  });
  AMG_CK_LAUNCH();
  return true;
}

// K11 + K4a: ru2 = ru - B^T p, x = M ru2 (M, x: level 0's)
bool launch_schur_u_M(const Mat& BTm, const void* ru, const void* p, void* ru2, const void* M, int mvt, void* x, int xt,
                      cudaStream_t s) {
  const int n = BTm.n, vt = BTm.vt;
  if (BTm.br != 3 || mvt != vt) return false;
  if (n == 0) return true;
  ProfScope ps_(prof_name("schur_u_M", 3, vt, xt),
                ((double)BTm.nnz * (4.0 + 3.0 * dtype_size(vt)) + 4.0 * (n + 1)) + 10.0 * n * dtype_size(xt) +
                    9.0 * n * dtype_size(mvt),
                s);
  dispatch_t(vt, [&](auto v) {
    using V = decltype(v);
    dispatch_t(xt, [&](auto xx) {
      using X = decltype(xx);
      if (BTm.tma_grid > 0)
        launch_tma_rows<3, 1, V, X, false>(BTm, (const X*)p, EpiSchurUM<3, V, X>{(const V*)M, (const X*)ru, (X*)ru2, (X*)x},
                                           s);
      else
        launch_lane<3, 1, V, X>(BTm, (const X*)p, LEpiSchurUM<V, X>{(const V*)M, (const X*)ru, (X*)ru2, (X*)x}, s);
    });
  });
  AMG_CK_LAUNCH();
  return true;
}

// K9 + K4a, hot shape (b = 4, pressure component 3, fp32 vectors): k_split4 that also forms
// x_u = M u for the cell's velocity triple.  The cell's M block (9 values) and the x triples
// are staged through shared memory (16-byte global accesses, 256 cells per block).
template <typename V>
__global__ void __launch_bounds__(256) k_split4_M(int n, const double* __restrict__ r, double scale_v,
                                                  const double* scale_d, float* __restrict__ ru, float* __restrict__ rp,
                                                  const V* __restrict__ M, float* __restrict__ xu) {
  const double scale = scale_d ? *scale_d : scale_v;
  __shared__ __align__(16) float su[3 * 256];
  __shared__ __align__(16) float sx[3 * 256];
  __shared__ __align__(16) V sm[9 * 256];
  const int64_t c0 = (int64_t)blockIdx.x * 256;
  const int64_t c = c0 + threadIdx.x;
  const int nc = (int)min((int64_t)256, (int64_t)n - c0);
  {  // the block's M values: 9 * nc contiguous V (16-byte aligned: c0 * 9 * sizeof(V) % 16 == 0)
    const V* src = M + c0 * 9;
    if (nc == 256) {
      constexpr int NV = 9 * 256 * (int)sizeof(V) / 16;
      for (int i = threadIdx.x; i < NV; i += 256)
        reinterpret_cast<float4*>(sm)[i] = __ldcs(reinterpret_cast<const float4*>(src) + i);
    } else {
      for (int i = threadIdx.x; i < 9 * nc; i += 256) sm[i] = src[i];
    }
  }
  float u[3] = {};
  if (c < n) {
    const double2* q = reinterpret_cast<const double2*>(r + c * 4);
    const double2 a = __ldcs(q), b = __ldcs(q + 1);
    u[0] = (float)(a.x * scale);
    u[1] = (float)(a.y * scale);
    u[2] = (float)(b.x * scale);
    su[3 * threadIdx.x + 0] = u[0];
    su[3 * threadIdx.x + 1] = u[1];
    su[3 * threadIdx.x + 2] = u[2];
    rp[c] = (float)(b.y * scale);
  }
  __syncthreads();
  if (c < n) {
    const V* m = sm + 9 * threadIdx.x;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double t = (double)m[3 * i] * (double)u[0];
      t = fma((double)m[3 * i + 1], (double)u[1], t);
      t = fma((double)m[3 * i + 2], (double)u[2], t);
      sx[3 * threadIdx.x + i] = (float)t;
    }
  }
  __syncthreads();
  float* dst = ru + c0 * 3;
  float* dx = xu + c0 * 3;
  if (nc == 256) {
    if (threadIdx.x < 192) {
      reinterpret_cast<float4*>(dst)[threadIdx.x] = reinterpret_cast<const float4*>(su)[threadIdx.x];
      reinterpret_cast<float4*>(dx)[threadIdx.x] = reinterpret_cast<const float4*>(sx)[threadIdx.x];
    }
  } else {
    for (int i = threadIdx.x; i < 3 * nc; i += 256) dst[i] = su[i], dx[i] = sx[i];
  }
}

bool launch_split_M(int32_t n, int b, int pc, const double* r, double scale, void* ru, void* rp, int xt, const void* M,
                    int mvt, void* xu, cudaStream_t s, const double* scale_dev) {
  if (!(b == 4 && pc == 3 && xt == AMG_F32)) return false;
  if (n == 0) return true;
  ProfScope ps_(prof_name("split_M", b, AMG_F64, xt), (double)n * (4 * 8.0 + 7 * 4.0 + 9.0 * dtype_size(mvt)), s);
  if (mvt == AMG_F32)
    k_split4_M<float><<<grid_for(n, 256), 256, 0, s>>>(n, r, scale, scale_dev, (float*)ru, (float*)rp,
                                                        (const float*)M, (float*)xu);
  else
    k_split4_M<double><<<grid_for(n, 256), 256, 0, s>>>(n, r, scale, scale_dev, (float*)ru, (float*)rp,
                                                         (const double*)M, (float*)xu);
  AMG_CK_LAUNCH();
  return true;
}

// narrow + K4a (monolithic level 0): f = narrow(scale r), x = M f; thread per block row
template <int B, typename V, typename X>
__global__ void __launch_bounds__(256) k_convert_M(int n, const double* __restrict__ r, double scale_v,
                                                   const double* scale_d, X* __restrict__ f, const V* __restrict__ M,
                                                   X* __restrict__ x) {
  const double scale = scale_d ? *scale_d : scale_v;
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const int64_t o = row * B;
  double fv[B];
#pragma unroll
  for (int c = 0; c < B; ++c) {
    const X t = to_out<X>(r[o + c] * scale);
    f[o + c] = t;
    fv[c] = (double)t;
  }
#pragma unroll
  for (int i = 0; i < B; ++i) {
    double m[B];
    load_b<B, false>(M + (o + i) * B, m);
    double t = m[0] * fv[0];
#pragma unroll
    for (int c = 1; c < B; ++c) t = fma(m[c], fv[c], t);
    x[o + i] = to_out<X>(t);
  }
}

bool launch_convert_M(int32_t n, int b, const double* r, double scale, void* f, int xt, const void* M, int mvt, void* x,
                      cudaStream_t s, const double* scale_dev) {
  if (n == 0) return true;
  ProfScope ps_(prof_name("convert_M", b, AMG_F64, xt),
                (double)n * b * (8.0 + 2.0 * dtype_size(xt)) + (double)n * b * b * dtype_size(mvt), s);
  dispatch_b(b, [&](auto Bc) {
    constexpr int B = decltype(Bc)::value;
    dispatch_t(mvt, [&](auto v) {
      using V = decltype(v);
      dispatch_t(xt, [&](auto xx) {
        using X = decltype(xx);
        k_convert_M<B, V, X><<<grid_for(n, 256), 256, 0, s>>>(n, r, scale, scale_dev, (X*)f, (const V*)M, (X*)x);
      });
    });
  });
  AMG_CK_LAUNCH();
  return true;
}

// BiCGStab's direction update p = r + beta (p - omega v) (k_bicg_p's expressions, device
// scalars) with the monolithic apply's narrowing + K4a of p in the same pass: p written, f =
// narrow(p), x = M f -- the values k_bicg_p + k_convert_M (scale 1) store, without p's re-read
template <int B, typename V, typename X>
__global__ void __launch_bounds__(256) k_bicg_p_convert_M(int n, const double* __restrict__ r,
                                                          const double* __restrict__ v, double* __restrict__ p,
                                                          const double* __restrict__ sc, X* __restrict__ f,
                                                          const V* __restrict__ M, X* __restrict__ x) {
  const bool first = sc[kBicgFirst] != 0.0;
  const double beta = (sc[kBicgRho] / sc[kBicgRhoOld]) * (sc[kBicgAlpha] / sc[kBicgOmega]);
  const double b2 = -beta * sc[kBicgOmega];
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const int64_t o = row * B;
  double fv[B];
#pragma unroll
  for (int c = 0; c < B; ++c) {
    const double pv = first ? r[o + c] : fma(1.0, r[o + c], fma(b2, v[o + c], beta * p[o + c]));
    p[o + c] = pv;
    const X t = to_out<X>(pv * 1.0);
    f[o + c] = t;
    fv[c] = (double)t;
  }
#pragma unroll
  for (int i = 0; i < B; ++i) {
    double m[B];
    load_b<B, false>(M + (o + i) * B, m);
    double t = m[0] * fv[0];
#pragma unroll
    for (int c = 1; c < B; ++c) t = fma(m[c], fv[c], t);
    x[o + i] = to_out<X>(t);
  }
}

bool launch_bicg_p_convert_M(int32_t n, int b, const double* r, const double* v, double* p, const double* sc, void* f,
                             int xt, const void* M, int mvt, void* x, cudaStream_t s) {
  if (n == 0) return true;
  ProfScope ps_(prof_name("bicg_p_convert_M", b, AMG_F64, xt),
                (double)n * b * (32.0 + 2.0 * dtype_size(xt)) + (double)n * b * b * dtype_size(mvt), s);
  dispatch_b(b, [&](auto Bc) {
    constexpr int B = decltype(Bc)::value;
    dispatch_t(mvt, [&](auto vv) {
      using V = decltype(vv);
      dispatch_t(xt, [&](auto xx) {
        using X = decltype(xx);
        k_bicg_p_convert_M<B, V, X><<<grid_for(n, 256), 256, 0, s>>>(n, r, v, p, sc, (X*)f, (const V*)M, (X*)x);
      });
    });
  });
  AMG_CK_LAUNCH();
  return true;
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

// One CTA per row (rows of 1.5-3 K unknowns: cfg 1 / cfg 5): 16-byte loads of the row and of f
// (rows 16-byte aligned: N * sizeof(V) % 16 == 0, else k_dense_gemv), fp64 partial sums
// combined in a fixed order (warp butterflies, then the warps' sums in warp order).  The
// warp-per-row kernel had ~10 warps per SM in flight and reached 1.5 TB/s.
template <typename V, typename X>
__global__ void __launch_bounds__(128) k_dense_gemv_cta(int N, const V* __restrict__ A, const X* __restrict__ f,
                                                        X* __restrict__ x) {
  constexpr int VW = 16 / sizeof(V);  // values per 16-byte load
  const int row = blockIdx.x;
  const V* a = A + (int64_t)row * N;
  double s = 0.0;
  const int nv = N / VW;
  // 4 loads of the row in flight per thread (the loop is otherwise one dependent load deep)
  constexpr int UN = 4;
  int q = threadIdx.x;
  for (; q + (UN - 1) * 128 < nv; q += UN * 128) {
    V av[UN][VW];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      if constexpr (std::is_same_v<V, float>) {
        const float4 t = __ldcs(reinterpret_cast<const float4*>(a) + q + u * 128);
        av[u][0] = t.x, av[u][1] = t.y, av[u][2] = t.z, av[u][3] = t.w;
      } else {
        const double2 t = __ldcs(reinterpret_cast<const double2*>(a) + q + u * 128);
        av[u][0] = t.x, av[u][1] = t.y;
      }
    }
#pragma unroll
    for (int u = 0; u < UN; ++u)
#pragma unroll
      for (int e = 0; e < VW; ++e) s = fma((double)av[u][e], (double)__ldg(f + (q + u * 128) * VW + e), s);
  }
  for (; q < nv; q += 128) {
    V av[VW];
    if constexpr (std::is_same_v<V, float>) {
      const float4 t = __ldcs(reinterpret_cast<const float4*>(a) + q);
      av[0] = t.x, av[1] = t.y, av[2] = t.z, av[3] = t.w;
    } else {
      const double2 t = __ldcs(reinterpret_cast<const double2*>(a) + q);
      av[0] = t.x, av[1] = t.y;
    }
#pragma unroll
    for (int e = 0; e < VW; ++e) s = fma((double)av[e], (double)__ldg(f + q * VW + e), s);
  }
  for (int j = nv * VW + threadIdx.x; j < N; j += 128) s = fma((double)a[j], (double)__ldg(f + j), s);
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
  __shared__ double ws[4];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) x[row] = to_out<X>(((ws[0] + ws[1]) + ws[2]) + ws[3]);
}

void launch_dense_gemv(int32_t N, const void* Ainv, int vt, const void* f, void* x, int xt,
                       cudaStream_t s) {
  if (N == 0) return;
  ProfScope ps_(prof_name("coarse_gemv", 1, vt, xt), (double)N * N * dtype_size(vt) + 2.0 * N * dtype_size(xt), s);
  const bool aligned = ((size_t)N * dtype_size(vt)) % 16 == 0 && ((uintptr_t)Ainv % 16) == 0;
  dispatch_t(vt, [&](auto v) {
    using V = decltype(v);
    dispatch_t(xt, [&](auto xx) {
      using X = decltype(xx);
      if (aligned)
        k_dense_gemv_cta<V, X><<<N, 128, 0, s>>>(N, (const V*)Ainv, (const X*)f, (X*)x);
      else
        k_dense_gemv<V, X><<<grid_for((int64_t)N * 32, 256), 256, 0, s>>>(N, (const V*)Ainv, (const X*)f, (X*)x);
    });
  });
  AMG_CK_LAUNCH();
}

void make_schur_views(const Mat& A, int nu, const void* Bv, const void* BTv, int vt, Mat& Bm, Mat& BTm,
                      cudaStream_t s, Arena* arena) {
  Bm = A;
  Bm.sell_ns = 0, Bm.sell_ptr = Bm.sell_col = Bm.sell_perm = Bm.sell_vptr = nullptr, Bm.sell_val = nullptr;
  Bm.b = 1;
  Bm.br = 1;
  Bm.bc = nu;
  Bm.val = const_cast<void*>(Bv);
  Bm.vt = vt;
  Bm.fast32 = false;  // fp64 accumulation of every product (as the direct kernels)
  BTm = Bm;
  BTm.br = nu;
  BTm.bc = 1;
  BTm.val = const_cast<void*>(BTv);
  // B on the lane kernel; B^T (3 x 1 blocks) on the interleaved copy when large enough (5.4
  // TB/s at cfg 5), else on the TMA-staged row-per-lane consumer (5.2 TB/s against 3.8-4.0
  // for the lane kernel)
  make_tma_plan(Bm, s, arena);
  make_tma_plan(BTm, s, arena, !env_int("AMG_NO_TMA_SCHUR", 0));
  if (env_set("AMG_SCHUR_B_VAR")) Bm.lane_var = env_int("AMG_SCHUR_B_VAR", Bm.lane_var);  // A/B switch (tools)
}

void launch_schur_p(const Mat& Bm, const void* mS, const void* rp, const void* us, void* p, int xt, cudaStream_t s) {
  const int n = Bm.n, vt = Bm.vt;
  if (n == 0) return;
  if (Bm.b == 1 && Bm.br == 0) {  // scalar B of the pressure-mask split (R21)
    ProfScope ps_(prof_name("schur_p", 1, vt, xt),
                  mat_bytes(Bm) + (double)n * dtype_size(vt) + (double)Bm.m * dtype_size(xt) + 2.0 * n * dtype_size(xt), s);
    dispatch_t(vt, [&](auto v) {
      using V = decltype(v);
      dispatch_t(xt, [&](auto xx) {
        using X = decltype(xx);
        launch_lane<1, 1, V, X>(Bm, (const X*)us, LEpiSchurP<V, X>{(const V*)mS, (const X*)rp, (X*)p}, s);
      });
    });
    AMG_CK_LAUNCH();
    return;
  }
  if (Bm.bc != 3) fail(AMG_EINVAL, "Schur split supports 3 velocity components");
  ProfScope ps_(prof_name("schur_p", 3, vt, xt),
                ((double)Bm.nnz * (4.0 + 3.0 * dtype_size(vt)) + 4.0 * (n + 1)) + (double)n * dtype_size(vt) + 5.0 * n * dtype_size(xt), s);
  dispatch_t(vt, [&](auto v) {
    using V = decltype(v);
    dispatch_t(xt, [&](auto xx) {
      using X = decltype(xx);
      if (Bm.tma_grid > 0)
        launch_tma_rows<1, 3, V, X, false>(Bm, (const X*)us, EpiSchurP<V, X>{(const V*)mS, (const X*)rp, (X*)p}, s);
      else
        launch_lane<1, 3, V, X>(Bm, (const X*)us, LEpiSchurP<V, X>{(const V*)mS, (const X*)rp, (X*)p}, s);
    });
  });
  AMG_CK_LAUNCH();
}

void launch_schur_u(const Mat& BTm, const void* ru, const void* p, void* ru2, int xt, cudaStream_t s) {
  const int n = BTm.n, vt = BTm.vt;
  if (n == 0) return;
  if (BTm.br != 3) fail(AMG_EINVAL, "Schur split supports 3 velocity components");
  ProfScope ps_(prof_name("schur_u", 3, vt, xt), ((double)BTm.nnz * (4.0 + 3.0 * dtype_size(vt)) + 4.0 * (n + 1)) + 7.0 * n * dtype_size(xt), s);
  dispatch_t(vt, [&](auto v) {
    using V = decltype(v);
    dispatch_t(xt, [&](auto xx) {
      using X = decltype(xx);
      if (BTm.tma_grid > 0)
        launch_tma_rows<3, 1, V, X, false>(BTm, (const X*)p, EpiSchurU<3, X>{(const X*)ru, (X*)ru2}, s);
      else
        launch_lane<3, 1, V, X>(BTm, (const X*)p, LEpiSchurU<X>{(const X*)ru, (X*)ru2}, s);
    });
  });
  AMG_CK_LAUNCH();
}

// ---- K9: split / join of the interleaved outer vector ----
template <typename X>
__global__ void k_split(int n, int b, int pc, const double* __restrict__ r, double scale_v, const double* scale_d,
                        X* __restrict__ ru, X* __restrict__ rp) {
  const double scale = scale_d ? *scale_d : scale_v;
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
__global__ void k_convert(int64_t N, const I* __restrict__ in, O* __restrict__ out, double scale_v, const double* scale_d) {
  const double scale = scale_d ? *scale_d : scale_v;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = to_out<O>((double)in[t] * scale);
}

// Hot shape (b = 4, pressure component 3, fp32 V-cycle vectors): thread per cell, one
// 32-byte read of the cell, the velocity triples staged in shared memory and written
// as float4 (coalesced), the pressure written directly.
__global__ void __launch_bounds__(256) k_split4(int n, const double* __restrict__ r, double scale_v,
                                                const double* scale_d, float* __restrict__ ru, float* __restrict__ rp) {
  const double scale = scale_d ? *scale_d : scale_v;
  __shared__ __align__(16) float su[3 * 256];
  const int64_t c0 = (int64_t)blockIdx.x * 256;
  const int64_t c = c0 + threadIdx.x;
  const int nc = (int)min((int64_t)256, (int64_t)n - c0);
  if (c < n) {
    const double2* q = reinterpret_cast<const double2*>(r + c * 4);
    const double2 a = __ldcs(q), b = __ldcs(q + 1);
    su[3 * threadIdx.x + 0] = (float)(a.x * scale);
    su[3 * threadIdx.x + 1] = (float)(a.y * scale);
    su[3 * threadIdx.x + 2] = (float)(b.x * scale);
    rp[c] = (float)(b.y * scale);
  }
  __syncthreads();
  float* dst = ru + c0 * 3;
  if (nc == 256) {  // 768 floats = 192 float4, 16-byte aligned (c0 * 12 bytes, c0 % 256 == 0)
    if (threadIdx.x < 192) reinterpret_cast<float4*>(dst)[threadIdx.x] = reinterpret_cast<const float4*>(su)[threadIdx.x];
  } else {
    for (int i = threadIdx.x; i < 3 * nc; i += 256) dst[i] = su[i];
  }
}

template <typename Z>
__global__ void __launch_bounds__(256) k_join4(int n, const float* __restrict__ u, const float* __restrict__ p,
                                               Z* __restrict__ z) {
  __shared__ __align__(16) float su[3 * 256];
  const int64_t c0 = (int64_t)blockIdx.x * 256;
  const int64_t c = c0 + threadIdx.x;
  const int nc = (int)min((int64_t)256, (int64_t)n - c0);
  const float* src = u + c0 * 3;
  if (nc == 256) {
    if (threadIdx.x < 192) reinterpret_cast<float4*>(su)[threadIdx.x] = __ldcs(reinterpret_cast<const float4*>(src) + threadIdx.x);
  } else {
    for (int i = threadIdx.x; i < 3 * nc; i += 256) su[i] = src[i];
  }
  __syncthreads();
  if (c < n) {
    const float pv = __ldcs(p + c);
    if constexpr (std::is_same_v<Z, float>) {
      reinterpret_cast<float4*>(z)[c] = make_float4(su[3 * threadIdx.x], su[3 * threadIdx.x + 1], su[3 * threadIdx.x + 2], pv);
    } else {
      double2* o = reinterpret_cast<double2*>(z + c * 4);
      o[0] = make_double2(su[3 * threadIdx.x], su[3 * threadIdx.x + 1]);
      o[1] = make_double2(su[3 * threadIdx.x + 2], pv);
    }
  }
}

// pressure-mask split / join (R21): ru[i] = narrow(scale r[uidx[i]]), rp[i] = narrow(scale r[pidx[i]]);
// z[uidx[i]] = u[i], z[pidx[i]] = p[i]
template <typename X>
__global__ void k_mask_split(int nu, int np, const int32_t* __restrict__ uidx, const int32_t* __restrict__ pidx,
                             const double* __restrict__ r, double scale_v, const double* scale_d, X* __restrict__ ru,
                             X* __restrict__ rp) {
  const double scale = scale_d ? *scale_d : scale_v;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nu) ru[t] = to_out<X>(r[uidx[t]] * scale);
  else if (t < (int64_t)nu + np) rp[t - nu] = to_out<X>(r[pidx[t - nu]] * scale);
}
template <typename X, typename Z>
__global__ void k_mask_join(int nu, int np, const int32_t* __restrict__ uidx, const int32_t* __restrict__ pidx,
                            const X* __restrict__ u, const X* __restrict__ p, Z* __restrict__ z) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nu) z[uidx[t]] = (Z)u[t];
  else if (t < (int64_t)nu + np) z[pidx[t - nu]] = (Z)p[t - nu];
}

void launch_mask_split(int32_t nu, int32_t np, const int32_t* uidx, const int32_t* pidx, const double* r,
                       double scale, void* ru, void* rp, int xt, cudaStream_t s, const double* scale_dev) {
  const int64_t N = (int64_t)nu + np;
  if (N == 0) return;
  ProfScope ps_(prof_name("split", 1, AMG_F64, xt), (double)N * (8.0 + 4.0 + dtype_size(xt)), s);
  dispatch_t(xt, [&](auto xx) {
    using X = decltype(xx);
    k_mask_split<X><<<grid_for(N, 256), 256, 0, s>>>(nu, np, uidx, pidx, r, scale, scale_dev, (X*)ru, (X*)rp);
  });
  AMG_CK_LAUNCH();
}

void launch_mask_join(int32_t nu, int32_t np, const int32_t* uidx, const int32_t* pidx, const void* u, const void* p,
                      int xt, void* z, int zt, cudaStream_t s) {
  const int64_t N = (int64_t)nu + np;
  if (N == 0) return;
  ProfScope ps_(prof_name("join", 1, zt, xt), (double)N * (4.0 + dtype_size(zt) + dtype_size(xt)), s);
  dispatch_t(xt, [&](auto xx) {
    using X = decltype(xx);
    dispatch_t(zt, [&](auto zz) {
      using Z = decltype(zz);
      k_mask_join<X, Z><<<grid_for(N, 256), 256, 0, s>>>(nu, np, uidx, pidx, (const X*)u, (const X*)p, (Z*)z);
    });
  });
  AMG_CK_LAUNCH();
}

void launch_split(int32_t n, int b, int pc, const double* r, double scale, void* ru, void* rp, int xt,
                  cudaStream_t s, const double* scale_dev) {
  if (n == 0) return;
  ProfScope ps_(prof_name("split", b, AMG_F64, xt), (double)n * b * (8.0 + dtype_size(xt)), s);
  if (b == 4 && pc == 3 && xt == AMG_F32) {
    k_split4<<<grid_for(n, 256), 256, 0, s>>>(n, r, scale, scale_dev, (float*)ru, (float*)rp);
    AMG_CK_LAUNCH();
    return;
  }
  dispatch_t(xt, [&](auto xx) {
    using X = decltype(xx);
    k_split<X><<<grid_for((int64_t)n * b, 256), 256, 0, s>>>(n, b, pc, r, scale, scale_dev, (X*)ru, (X*)rp);
  });
  AMG_CK_LAUNCH();
}

void launch_join(int32_t n, int b, int pc, const void* u, const void* p, int xt, void* z, int zt, cudaStream_t s) {
  if (n == 0) return;
  ProfScope ps_(prof_name("join", b, zt, xt), (double)n * b * (dtype_size(zt) + dtype_size(xt)), s);
  if (b == 4 && pc == 3 && xt == AMG_F32) {
    if (zt == AMG_F32) k_join4<float><<<grid_for(n, 256), 256, 0, s>>>(n, (const float*)u, (const float*)p, (float*)z);
    else k_join4<double><<<grid_for(n, 256), 256, 0, s>>>(n, (const float*)u, (const float*)p, (double*)z);
    AMG_CK_LAUNCH();
    return;
  }
  dispatch_t(xt, [&](auto xx) {
    using X = decltype(xx);
    dispatch_t(zt, [&](auto zz) {
      using Z = decltype(zz);
      k_join<X, Z><<<grid_for((int64_t)n * b, 256), 256, 0, s>>>(n, b, pc, (const X*)u, (const X*)p, (Z*)z);
    });
  });
  AMG_CK_LAUNCH();
}

void launch_convert(int64_t N, const void* in, int it, void* out, int ot, double scale, cudaStream_t s,
                    const double* scale_dev) {
  if (N == 0) return;
  ProfScope ps_(prof_name("convert", 1, ot, it), (double)N * (dtype_size(it) + dtype_size(ot)), s);
  unsigned g = grid_for(N, 256);
  if (g > 148u * 16u) g = 148u * 16u;
  dispatch_t(it, [&](auto ii) {
    using I = decltype(ii);
    dispatch_t(ot, [&](auto oo) {
      using O = decltype(oo);
      k_convert<I, O><<<g, 256, 0, s>>>(N, (const I*)in, (O*)out, scale, scale_dev);
    });
  });
  AMG_CK_LAUNCH();
}


bool has_solve_copy(const Mat& A) {
  return (A.lane_var == kLaneSellR && A.sell_vptr) || (A.lane_var == kLaneSell && A.sell_ptr);
}

void release_bsr_values(Mat& A, Arena& arena, cudaStream_t s) {
  if (!A.val || !has_solve_copy(A) || A.tma_grid > 0) return;
  AMG_CK(cudaStreamSynchronize(s));  // kernels still reading the values (the copy's fill) are done
  arena.release_one(A.val);
  A.val = nullptr;
}

// inverse of the column part of k_sell_fill / k_sellr_fill (C = 32 for the interleaved copy):
// slot (s, g) holds row s * C + g, or perm[slot] (sorted windows); its j-th step's column is
// the row's j-th BSR column
__global__ void k_sell_unfill_col(int n, int C, int ns, const int32_t* __restrict__ ptr,
                                  const int32_t* __restrict__ sptr, const int32_t* __restrict__ perm,
                                  const int32_t* __restrict__ scol, int32_t* __restrict__ col) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)ns * C) return;
  const int s = (int)(t / C), g = (int)(t % C);
  int64_t row = (int64_t)s * C + g;
  if (perm) row = perm[t] >= 0 ? perm[t] : n;
  if (row >= n) return;
  const int k0 = ptr[row], len = ptr[row + 1] - k0;
  for (int j = 0; j < len; ++j) col[k0 + j] = scol[((int64_t)sptr[s] + j) * C + g];
}

void release_bsr_cols(Mat& A, Arena& arena, cudaStream_t s) {
  if (!A.col || A.val || A.nnz == 0 || !has_solve_copy(A) || A.tma_grid > 0) return;
  AMG_CK(cudaStreamSynchronize(s));
  arena.release_one(A.col);
  A.col = nullptr;
}

void cols_from_copy(const Mat& A, int32_t* out, cudaStream_t s) {
  if (A.nnz == 0) return;
  if (!has_solve_copy(A)) fail(AMG_EINVAL, "cols_from_copy: no solve copy");
  const int C = A.lane_var == kLaneSellR ? 32 : 32 / A.b;
  k_sell_unfill_col<<<grid_for((int64_t)A.sell_ns * C, 256), 256, 0, s>>>(A.n, C, A.sell_ns, A.ptr, A.sell_ptr,
                                                                         A.sell_perm, A.sell_col, out);
  AMG_CK_LAUNCH();
}

void values_from_copy(const Mat& A, void* out, cudaStream_t s) {
  if (A.nnz == 0) return;
  if (!has_solve_copy(A)) fail(AMG_EINVAL, "values_from_copy: no solve copy");
  dispatch_t(A.vt, [&](auto v) {
    using V = decltype(v);
    if (A.lane_var == kLaneSellR) {
      const int E = A.rows_per_block() * A.cols_per_block();
      k_sellr_unfill<V><<<grid_for((int64_t)A.sell_ns * 32, 256), 256, 0, s>>>(
          A.n, E, A.sell_w, A.sell_ns, A.ptr, A.sell_vptr, A.sell_perm, (const V*)A.sell_val, (V*)out);
    } else {
      const int C = 32 / A.b;
      k_sell_unfill<V><<<grid_for((int64_t)A.sell_ns * C, 256), 256, 0, s>>>(
          A.n, A.b, C, A.sell_ns, A.ptr, A.sell_ptr, A.sell_perm, (const V*)A.sell_val, (V*)out);
    }
  });
  AMG_CK_LAUNCH();
}

}  // namespace amgb
