// dist.cu -- row-slab distributed solve.
//
// One rank per GPU owns a contiguous block-row range (z-slabs).  Setup is replicated:
// the ranks allgather the matrix, every rank builds the same global hierarchy with
// rank-local aggregation (strength edges across slabs dropped, so P and R
// never cross slabs), then keeps only its slab of every level.  The solve exchanges
// ghost values before every kernel that reads a distributed vector through A_l, B or
// B^T (grouped send/recv to the ranks owning the ghosts), allreduces every dot
// product, and replicates the coarsest level (allgather of the coarse right-hand side,
// dense inverse applied on every rank).
#include <nccl.h>

#include <algorithm>
#include <tuple>
#include <cstdlib>
#include <cstring>

#include "amg.h"
#include "comm.h"
#include "ops.h"
#include "prof.h"
#include "solver.h"

namespace amgb {
void set_last_error(const std::string& s);
int validate_bsr(const amg_bsr* A, bool square);
int check_params(const amg_params* p);
Mat view_of(const amg_bsr* A);
}  // namespace amgb

struct amg_comm {
  amgb::CommBase* c = nullptr;
};

namespace amgb {

namespace {

template <typename T>
__global__ void k_pack(int n, int b, const int32_t* __restrict__ idx, const T* __restrict__ x, T* __restrict__ buf) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n * b) return;
  const int64_t i = t / b;
  buf[t] = x[(int64_t)idx[i] * b + t % b];
}

__global__ void k_sqrt(double* d) { *d = sqrt(*d); }

__global__ void k_shift_ptr(int n, const int32_t* src, int32_t base_sub, int32_t add, int32_t* dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) dst[i] = src[i] - base_sub + add;
}

}  // namespace

void halo_exchange(Handle& h, const Halo& H, void* x, int dt, int b, cudaStream_t s) {
  if (!h.comm || H.peers.empty()) return;
  const size_t es = dtype_size(dt) * b;
  if (H.total_send > 0) {
    ProfScope ps_("halo_pack", (double)H.total_send * es * 2.0, s);
    if (dt == AMG_F32)
      k_pack<float><<<grid_for((int64_t)H.total_send * b, 256), 256, 0, s>>>(H.total_send, b, H.send_idx,
                                                                            (const float*)x, (float*)H.send_buf);
    else
      k_pack<double><<<grid_for((int64_t)H.total_send * b, 256), 256, 0, s>>>(H.total_send, b, H.send_idx,
                                                                             (const double*)x, (double*)H.send_buf);
    AMG_CK_LAUNCH();
  }
  char* xc = static_cast<char*>(x);
  h.comm->group_begin();
  for (size_t i = 0; i < H.peers.size(); ++i) {
    const int p = H.peers[i];
    if (H.send_cnt[i]) h.comm->send((char*)H.send_buf + (size_t)H.send_off[i] * es, (size_t)H.send_cnt[i] * es, p, s);
    if (H.recv_cnt[i]) h.comm->recv(xc + ((size_t)H.nloc + H.recv_off[i]) * es, (size_t)H.recv_cnt[i] * es, p, s);
  }
  h.comm->group_end(s);
}

void halo_overlapped(Handle& h, const Halo& H, const Mat& A, void* x, int dt, int b, cudaStream_t s,
                     const std::function<void(int, int)>& launch) {
  const bool off = env_set("AMG_NO_OVERLAP");  // A/B switch (tests)
  if (!h.comm || H.peers.empty()) {
    launch(0, A.n);
    return;
  }
  // the interleaved copy computes whole 32-row slices: round the interior inward
  int lo = H.int_lo, hi = H.int_hi;
  if (A.lane_var == kLaneSellR) lo = (lo + 31) / 32 * 32, hi = hi / 32 * 32;
  const bool sellr_ok = A.lane_var == kLaneSellR && hi > lo && sellr_range_ok(A, lo, hi);
  if (off || hi <= lo || (A.lane_var > kLaneCN4 && !sellr_ok) || A.tma_grid > 0 || !h.comm_s) {
    halo_exchange(h, H, x, dt, b, s);
    launch(0, A.n);
    return;
  }
  const size_t es = dtype_size(dt) * b;
  if (H.total_send > 0) {
    ProfScope ps_("halo_pack", (double)H.total_send * es * 2.0, s);
    if (dt == AMG_F32)
      k_pack<float><<<grid_for((int64_t)H.total_send * b, 256), 256, 0, s>>>(H.total_send, b, H.send_idx,
                                                                            (const float*)x, (float*)H.send_buf);
    else
      k_pack<double><<<grid_for((int64_t)H.total_send * b, 256), 256, 0, s>>>(H.total_send, b, H.send_idx,
                                                                             (const double*)x, (double*)H.send_buf);
    AMG_CK_LAUNCH();
  }
  AMG_CK(cudaEventRecord(h.ev_pack, s));
  AMG_CK(cudaStreamWaitEvent(h.comm_s, h.ev_pack, 0));
  char* xc = static_cast<char*>(x);
  h.comm->group_begin();
  for (size_t i = 0; i < H.peers.size(); ++i) {
    const int p = H.peers[i];
    if (H.send_cnt[i])
      h.comm->send((char*)H.send_buf + (size_t)H.send_off[i] * es, (size_t)H.send_cnt[i] * es, p, h.comm_s);
    if (H.recv_cnt[i])
      h.comm->recv(xc + ((size_t)H.nloc + H.recv_off[i]) * es, (size_t)H.recv_cnt[i] * es, p, h.comm_s);
  }
  h.comm->group_end(h.comm_s);
  AMG_CK(cudaEventRecord(h.ev_halo, h.comm_s));
  launch(lo, hi);  // interior rows: no ghost read
  AMG_CK(cudaStreamWaitEvent(s, h.ev_halo, 0));
  launch(0, lo);
  launch(hi, A.n);
}

void dist_allreduce(Handle& h, double* d, int n, cudaStream_t s) {
  if (h.comm) h.comm->allreduce_sum(d, n, s);
}

// every rank's slab of level l's right-hand side to every rank (levels >= rep_from replicated)
void replicated_allgather(Handle& h, size_t l, cudaStream_t s) {
  if (!h.comm || h.comm->nranks == 1) return;
  const bool coarsest = l == h.lv.size();
  const size_t es = dtype_size(h.xt) * (coarsest ? h.coarse.b : h.lv[l].A.b);
  char* f = static_cast<char*>(coarsest ? h.coarse.f : h.lv[l].f);
  const auto& bd = h.lbounds[l];
  const int me = h.comm->rank;
  h.comm->group_begin();
  for (int p = 0; p < h.comm->nranks; ++p) {
    if (p == me) continue;
    const int64_t cm = bd[me + 1] - bd[me], cp = bd[p + 1] - bd[p];
    if (cm) h.comm->send(f + bd[me] * es, cm * es, p, s);
    if (cp) h.comm->recv(f + bd[p] * es, cp * es, p, s);
  }
  h.comm->group_end(s);
}

void* level_f_slab(Handle& h, size_t l) {
  const bool coarsest = l == h.lv.size();
  char* f = static_cast<char*>(coarsest ? h.coarse.f : h.lv[l].f);
  // only the first replicated level is assembled from the ranks' slabs; past it every rank's
  // restriction computes the whole next level
  if (!h.comm || l != h.rep_from) return f;
  const int b = coarsest ? h.coarse.b : h.lv[l].A.b;
  return f + h.lbounds[l][h.comm->rank] * b * dtype_size(h.xt);
}

namespace {

// rows [r0, r1) of M: ptr rebased, columns kept, values copied (same dtype)
Mat slice_rows(Arena& ar, const Mat& M, int64_t r0, int64_t r1, cudaStream_t s) {
  std::vector<int32_t> pe(2);
  AMG_CK(cudaMemcpy(&pe[0], M.ptr + r0, sizeof(int32_t), cudaMemcpyDeviceToHost));
  AMG_CK(cudaMemcpy(&pe[1], M.ptr + r1, sizeof(int32_t), cudaMemcpyDeviceToHost));
  Mat L = M;
  L.n = (int32_t)(r1 - r0);
  L.nnz = pe[1] - pe[0];
  const size_t vb = (size_t)M.b * M.b * dtype_size(M.vt);
  L.ptr = ar.alloc_n<int32_t>(L.n + 1);
  L.col = ar.alloc_n<int32_t>(std::max<int64_t>(L.nnz, 1));
  L.val = ar.alloc(std::max<int64_t>(L.nnz, 1) * vb);
  k_shift_ptr<<<grid_for(L.n + 1, 256), 256, 0, s>>>(L.n, M.ptr + r0, pe[0], 0, L.ptr);
  AMG_CK_LAUNCH();
  if (L.nnz) {
    AMG_CK(cudaMemcpyAsync(L.col, M.col + pe[0], sizeof(int32_t) * L.nnz, cudaMemcpyDeviceToDevice, s));
    AMG_CK(cudaMemcpyAsync(L.val, (const char*)M.val + (size_t)pe[0] * vb, L.nnz * vb, cudaMemcpyDeviceToDevice, s));
  }
  AMG_CK(cudaStreamSynchronize(s));
  L.tma_grid = 0;
  return L;
}

// columns -= shift; every column must fall in [0, width) afterwards (slab-local P / R)
void remap_shift(Mat& M, int64_t shift, int64_t width) {
  std::vector<int32_t> c(M.nnz);
  if (M.nnz) AMG_CK(cudaMemcpy(c.data(), M.col, sizeof(int32_t) * M.nnz, cudaMemcpyDeviceToHost));
  for (auto& v : c) {
    v = (int32_t)(v - shift);
    if (v < 0 || v >= width) fail(AMG_EINVAL, "distributed setup: slab-local operator crosses a slab");
  }
  if (M.nnz) AMG_CK(cudaMemcpy(M.col, c.data(), sizeof(int32_t) * M.nnz, cudaMemcpyHostToDevice));
  M.m = (int32_t)width;
}

// distributed matrix: global columns -> [local | ghosts], ghost plan (both sides).  The local
// columns are [lo, lo + ncols) (ncols < 0: M.n, a square slab); bounds: the column owners.
void build_halo(Handle& h, Mat& M, int64_t lo, const std::vector<int64_t>& bounds, Halo& H, cudaStream_t s,
                int64_t ncols = -1) {
  CommBase* comm = h.comm;
  const int P = comm->nranks, me = comm->rank;
  const int32_t nl = (int32_t)(ncols < 0 ? M.n : ncols);
  const int64_t hi = lo + nl;
  std::vector<int32_t> c(M.nnz);
  if (M.nnz) AMG_CK(cudaMemcpy(c.data(), M.col, sizeof(int32_t) * M.nnz, cudaMemcpyDeviceToHost));
  std::vector<int32_t> ghosts;
  for (int32_t v : c)
    if (v < lo || v >= hi) ghosts.push_back(v);
  std::sort(ghosts.begin(), ghosts.end());
  ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
  for (auto& v : c) {
    if (v >= lo && v < hi) v = (int32_t)(v - lo);
    else v = (int32_t)(nl + (std::lower_bound(ghosts.begin(), ghosts.end(), v) - ghosts.begin()));
  }
  if (M.nnz) AMG_CK(cudaMemcpy(M.col, c.data(), sizeof(int32_t) * M.nnz, cudaMemcpyHostToDevice));
  H = Halo{};
  H.nloc = nl;
  H.nghost = (int)ghosts.size();
  {  // the longest run of rows without a ghost column (>= a quarter of the rows): overlap window
    std::vector<int32_t> hp((size_t)M.n + 1);
    AMG_CK(cudaMemcpy(hp.data(), M.ptr, sizeof(int32_t) * (M.n + 1), cudaMemcpyDeviceToHost));
    int32_t best_lo = 0, best_hi = 0, run_lo = 0;
    for (int32_t r = 0; r <= M.n; ++r) {
      bool ghost_row = r == M.n;
      if (r < M.n)
        for (int32_t k = hp[r]; k < hp[r + 1] && !ghost_row; ++k) ghost_row = c[k] >= nl;
      if (ghost_row) {
        if (r - run_lo > best_hi - best_lo) best_lo = run_lo, best_hi = r;
        run_lo = r + 1;
      }
    }
    if ((int64_t)(best_hi - best_lo) * 4 >= M.n && H.nghost > 0) H.int_lo = best_lo, H.int_hi = best_hi;
  }
  M.m = nl + H.nghost;
  // how many ghosts I need from every rank; everybody learns the full P x P matrix
  std::vector<int64_t> need(P, 0), all((size_t)P * P);
  for (int32_t g : ghosts) {
    int owner = (int)(std::upper_bound(bounds.begin(), bounds.end(), (int64_t)g) - bounds.begin()) - 1;
    if (owner < 0 || owner >= P || owner == me) fail(AMG_EINVAL, "distributed setup: bad ghost owner");
    need[owner]++;
  }
  comm->allgather_host(need.data(), P, all.data());
  int roff = 0, soff = 0;
  for (int p = 0; p < P; ++p) {
    const int rc = (int)all[(size_t)me * P + p], sc = (int)all[(size_t)p * P + me];
    if (rc == 0 && sc == 0) continue;
    H.peers.push_back(p);
    H.recv_cnt.push_back(rc);
    H.recv_off.push_back(roff);
    H.send_cnt.push_back(sc);
    H.send_off.push_back(soff);
    roff += rc;
    soff += sc;
  }
  H.total_send = soff;
  H.send_idx = h.arena.alloc_n<int32_t>(std::max(soff, 1));
  H.send_buf = h.arena.alloc((size_t)std::max(soff, 1) * 4 * sizeof(double));
  // send my ghost lists (global ids) to their owners; receive the lists I must serve
  int32_t* dg = h.arena.alloc_n<int32_t>(std::max<size_t>(ghosts.size(), 1));
  if (!ghosts.empty())
    AMG_CK(cudaMemcpy(dg, ghosts.data(), sizeof(int32_t) * ghosts.size(), cudaMemcpyHostToDevice));
  comm->group_begin();
  for (size_t i = 0; i < H.peers.size(); ++i) {
    if (H.recv_cnt[i]) comm->send(dg + H.recv_off[i], sizeof(int32_t) * H.recv_cnt[i], H.peers[i], s);
    if (H.send_cnt[i]) comm->recv(H.send_idx + H.send_off[i], sizeof(int32_t) * H.send_cnt[i], H.peers[i], s);
  }
  comm->group_end(s);
  AMG_CK(cudaStreamSynchronize(s));
  std::vector<int32_t> si(soff);
  if (soff) AMG_CK(cudaMemcpy(si.data(), H.send_idx, sizeof(int32_t) * soff, cudaMemcpyDeviceToHost));
  for (auto& v : si) {
    if (v < lo || v >= hi) fail(AMG_EINVAL, "distributed setup: ghost request outside the slab");
    v = (int32_t)(v - lo);
  }
  if (soff) AMG_CK(cudaMemcpy(H.send_idx, si.data(), sizeof(int32_t) * soff, cudaMemcpyHostToDevice));
}

// allgatherv of device byte ranges: rank r contributes bytes [off[r], off[r] + cnt[r]) of buf
void allgatherv_bytes(CommBase* comm, char* buf, const std::vector<int64_t>& off, const std::vector<int64_t>& cnt,
                      cudaStream_t s) {
  const int me = comm->rank;
  comm->group_begin();
  for (int p = 0; p < comm->nranks; ++p) {
    if (p == me) continue;
    if (cnt[me]) comm->send(buf + off[me], cnt[me], p, s);
    if (cnt[p]) comm->recv(buf + off[p], cnt[p], p, s);
  }
  comm->group_end(s);
  AMG_CK(cudaStreamSynchronize(s));
}

Handle* setup_dist_impl(const amg_bsr* A, int64_t row_begin, int64_t n_global, CommBase* comm, const amg_params* p,
                        cudaStream_t s, const uint8_t* pmask = nullptr) {
  const int P = comm->nranks, me = comm->rank;
  const int b = A->block_size;
  // 1. slabs and the global matrix on every rank (fp64)
  int64_t mine[3] = {A->n_block_rows, A->nnzb, row_begin};
  std::vector<int64_t> info((size_t)3 * P);
  comm->allgather_host(mine, 3, info.data());
  std::vector<int64_t> bounds(P + 1, 0), nnz_off(P + 1, 0);
  for (int r = 0; r < P; ++r) {
    if (info[3 * r + 2] != bounds[r]) fail(AMG_EINVAL, "amg_setup_dist: slabs must be contiguous in rank order");
    bounds[r + 1] = bounds[r] + info[3 * r];
    nnz_off[r + 1] = nnz_off[r] + info[3 * r + 1];
  }
  if (bounds[P] != n_global) fail(AMG_EDIM, "amg_setup_dist: slabs do not cover n_global_block_rows");
  if (nnz_off[P] >= (int64_t(1) << 31)) fail(AMG_EINDEX_OVERFLOW, "amg_setup_dist: global nnzb >= 2^31");
  Arena tmp;
  Mat G;
  G.n = (int32_t)n_global;
  G.m = (int32_t)n_global;
  G.b = b;
  G.nnz = nnz_off[P];
  G.vt = AMG_F64;
  G.ptr = tmp.alloc_n<int32_t>(n_global + 1);
  G.col = tmp.alloc_n<int32_t>(std::max<int64_t>(G.nnz, 1));
  G.val = tmp.alloc_n<double>(std::max<int64_t>(G.nnz, 1) * b * b);
  const Mat loc = view_of(A);
  k_shift_ptr<<<grid_for(loc.n + 1, 256), 256, 0, s>>>(loc.n, loc.ptr, 0, (int32_t)nnz_off[me], G.ptr + bounds[me]);
  AMG_CK_LAUNCH();
  if (loc.nnz) {
    AMG_CK(cudaMemcpyAsync(G.col + nnz_off[me], loc.col, sizeof(int32_t) * loc.nnz, cudaMemcpyDeviceToDevice, s));
    launch_convert(loc.nnz * b * b, loc.val, loc.vt, (double*)G.val + nnz_off[me] * b * b, AMG_F64, 1.0, s);
  }
  std::vector<int64_t> o(P), c(P);
  for (int r = 0; r < P; ++r) o[r] = bounds[r] * 4, c[r] = (bounds[r + 1] - bounds[r]) * 4;  // ptr[0..n) per slab
  allgatherv_bytes(comm, (char*)G.ptr, o, c, s);
  AMG_CK(cudaMemcpy(G.ptr + n_global, &nnz_off[P], sizeof(int32_t), cudaMemcpyHostToDevice));
  int32_t tot32 = (int32_t)nnz_off[P];
  AMG_CK(cudaMemcpy(G.ptr + n_global, &tot32, sizeof(int32_t), cudaMemcpyHostToDevice));
  for (int r = 0; r < P; ++r) o[r] = nnz_off[r] * 4, c[r] = (nnz_off[r + 1] - nnz_off[r]) * 4;
  allgatherv_bytes(comm, (char*)G.col, o, c, s);
  for (int r = 0; r < P; ++r) o[r] = nnz_off[r] * 8 * b * b, c[r] = (nnz_off[r + 1] - nnz_off[r]) * 8 * b * b;
  allgatherv_bytes(comm, (char*)G.val, o, c, s);

  // the global pressure mask (R27): every rank's scalar rows, in rank order
  uint8_t* gmask = nullptr;
  if (pmask) {
    gmask = tmp.alloc_n<uint8_t>(std::max<int64_t>(n_global * b, 1));
    if (loc.n) AMG_CK(cudaMemcpyAsync(gmask + bounds[me] * b, pmask, (size_t)loc.n * b, cudaMemcpyDeviceToDevice, s));
    for (int r = 0; r < P; ++r) o[r] = bounds[r] * b, c[r] = (bounds[r + 1] - bounds[r]) * b;
    allgatherv_bytes(comm, (char*)gmask, o, c, s);
  }

  // 2. the global hierarchy (identical on every rank), rank-local aggregation
  Handle* Gh = build_handle(G, p, bounds, s, /*workspace=*/false, gmask);
  tmp.release();
  if (Gh->amg_active && Gh->lv.empty() && P > 1) {
    delete Gh;
    fail(AMG_EINVAL, "amg_setup_dist: problem too small for a multilevel hierarchy (single level)");
  }

  // 3. this rank's slab of everything
  Handle* h = new Handle;
  try {
    h->p = Gh->p;
    h->vt = Gh->vt;
    h->xt = Gh->xt;
    h->n = (int32_t)(bounds[me + 1] - bounds[me]);
    h->b = b;
    h->schur = Gh->schur;
    h->pc = Gh->pc;
    h->nu = Gh->nu;
    h->amg_active = Gh->amg_active;
    h->bh = Gh->bh;
    h->comm = comm;
    h->row_lo = bounds[me];
    h->n_global_rows = n_global;
    h->lbounds = Gh->lbounds;
    // outer operator
    h->A = slice_rows(h->arena, Gh->A, bounds[me], bounds[me + 1], s);
    build_halo(*h, h->A, bounds[me], bounds, h->halo0, s);
    make_tma_plan(h->A, s, &h->arena);
    h->alg_bytes_spmv = (double)h->A.nnz * (4.0 + 8.0 * b * b) + 4.0 * (h->A.n + 1) + 16.0 * h->A.n * b;
    const size_t xs = dtype_size(h->xt);
    if (h->schur && !Gh->masked) {
      const int64_t k0 = 0;
      (void)k0;
      int32_t pe[2];
      AMG_CK(cudaMemcpy(&pe[0], Gh->A.ptr + bounds[me], 4, cudaMemcpyDeviceToHost));
      AMG_CK(cudaMemcpy(&pe[1], Gh->A.ptr + bounds[me + 1], 4, cudaMemcpyDeviceToHost));
      const size_t vs = dtype_size(h->vt) * h->nu;
      const int64_t nz = pe[1] - pe[0];
      h->Bv = h->arena.alloc(std::max<int64_t>(nz, 1) * vs);
      h->BTv = h->arena.alloc(std::max<int64_t>(nz, 1) * vs);
      h->mS = h->arena.alloc(std::max(h->n, 1) * dtype_size(h->vt));
      h->shat64 = h->arena.alloc_n<double>(std::max(h->n, 1));
      h->mS64 = h->arena.alloc_n<double>(std::max(h->n, 1));
      AMG_CK(cudaMemcpy(h->Bv, (char*)Gh->Bv + pe[0] * vs, nz * vs, cudaMemcpyDeviceToDevice));
      AMG_CK(cudaMemcpy(h->BTv, (char*)Gh->BTv + pe[0] * vs, nz * vs, cudaMemcpyDeviceToDevice));
      AMG_CK(cudaMemcpy(h->mS, (char*)Gh->mS + bounds[me] * dtype_size(h->vt), h->n * dtype_size(h->vt),
                        cudaMemcpyDeviceToDevice));
      AMG_CK(cudaMemcpy(h->shat64, Gh->shat64 + bounds[me], 8 * h->n, cudaMemcpyDeviceToDevice));
      AMG_CK(cudaMemcpy(h->mS64, Gh->mS64 + bounds[me], 8 * h->n, cudaMemcpyDeviceToDevice));
      make_schur_views(h->A, h->nu, h->Bv, h->BTv, h->vt, h->Bm, h->BTm, s, &h->arena);
    }
    if (Gh->masked) {  // general pressure mask (R27): this rank's unknowns of each class
      const auto &ub = Gh->ubounds, &pb = Gh->pbounds;
      if ((int)ub.size() != P + 1 || (int)pb.size() != P + 1) fail(AMG_EINVAL, "amg_setup_dist_pmask: class ranges");
      h->masked = true;
      h->ubounds = ub;
      h->pbounds = pb;
      h->nu_s = (int32_t)(ub[me + 1] - ub[me]);
      h->np_s = (int32_t)(pb[me + 1] - pb[me]);
      // index maps: class position -> local scalar unknown
      for (auto [dst, src, lo, cnt] : {std::tuple<int32_t**, const int32_t*, int64_t, int32_t>{&h->uidx, Gh->uidx, ub[me], h->nu_s},
                                       {&h->pidx, Gh->pidx, pb[me], h->np_s}}) {
        std::vector<int32_t> v(std::max(cnt, 1));
        if (cnt) AMG_CK(cudaMemcpy(v.data(), src + lo, 4 * (size_t)cnt, cudaMemcpyDeviceToHost));
        for (int32_t i = 0; i < cnt; ++i) v[i] -= (int32_t)(bounds[me] * b);
        *dst = h->arena.alloc_n<int32_t>(std::max(cnt, 1));
        AMG_CK(cudaMemcpy(*dst, v.data(), 4 * (size_t)std::max(cnt, 1), cudaMemcpyHostToDevice));
      }
      // scalar B (pressure rows x velocity columns) and B^T (velocity rows x pressure columns)
      h->Bm = slice_rows(h->arena, Gh->Bm, pb[me], pb[me + 1], s);
      build_halo(*h, h->Bm, ub[me], ub, h->haloBu, s, h->nu_s);
      h->BTm = slice_rows(h->arena, Gh->BTm, ub[me], ub[me + 1], s);
      build_halo(*h, h->BTm, pb[me], pb, h->haloBTp, s, h->np_s);
      h->Bm.fast32 = h->BTm.fast32 = false;
      make_tma_plan(h->Bm, s, &h->arena);
      make_tma_plan(h->BTm, s, &h->arena);
      const size_t vs = dtype_size(h->vt);
      h->mS = h->arena.alloc(std::max(h->np_s, 1) * vs);
      h->shat64 = h->arena.alloc_n<double>(std::max(h->np_s, 1));
      h->mS64 = h->arena.alloc_n<double>(std::max(h->np_s, 1));
      AMG_CK(cudaMemcpy(h->mS, (char*)Gh->mS + pb[me] * vs, h->np_s * vs, cudaMemcpyDeviceToDevice));
      AMG_CK(cudaMemcpy(h->shat64, Gh->shat64 + pb[me], 8 * (size_t)h->np_s, cudaMemcpyDeviceToDevice));
      AMG_CK(cudaMemcpy(h->mS64, Gh->mS64 + pb[me], 8 * (size_t)h->np_s, cudaMemcpyDeviceToDevice));
    }
    // hierarchy levels: levels 0 .. rep_from-1 as row slabs with halos; from rep_from on (the
    // first level with fewer than AMG_REPLICATE_ROWS block rows per rank, default 50,000;
    // SURVEY.md §8(e) mitigation 2) every rank holds the whole level and computes it
    // redundantly, so those levels exchange nothing but the one allgather of their
    // right-hand side.  Level 0 is always distributed.
    const size_t L = Gh->lv.size();
    h->lv.resize(L);
    const int64_t rep_rows = env_int("AMG_REPLICATE_ROWS", 50000);
    h->rep_from = L;
    for (size_t l = 1; l < L; ++l)
      if (Gh->lv[l].A.n < rep_rows * P) {
        h->rep_from = l;
        break;
      }
    for (size_t l = 0; l < L; ++l) {
      const Level& GL = Gh->lv[l];
      Level& LL = h->lv[l];
      const bool rep = l >= h->rep_from;
      const auto& bd = h->lbounds[l];
      const auto& bc = h->lbounds[l + 1];
      const int64_t r0 = rep ? 0 : bd[me], r1 = rep ? GL.A.n : bd[me + 1];
      const int64_t c0 = rep ? 0 : bc[me], c1 = rep ? GL.nc : bc[me + 1];
      LL.A = slice_rows(h->arena, GL.A, r0, r1, s);
      if (!rep) build_halo(*h, LL.A, bd[me], bd, LL.halo, s);
      LL.A.fast32 = GL.A.fast32;
      make_tma_plan(LL.A, s, &h->arena);
      LL.P = slice_rows(h->arena, GL.P, r0, r1, s);
      // slab-local coarse ids while the next level is distributed; global ids into a replicated one
      if (l + 1 < h->rep_from) remap_shift(LL.P, bc[me], bc[me + 1] - bc[me]);
      LL.P.fast32 = GL.P.fast32;
      make_tma_plan(LL.P, s, &h->arena);
      LL.R = slice_rows(h->arena, GL.R, c0, c1, s);
      if (!rep) remap_shift(LL.R, bd[me], bd[me + 1] - bd[me]);
      LL.R.fast32 = GL.R.fast32;
      make_tma_plan(LL.R, s, &h->arena);
      if (GL.Lf.ptr) {  // ILU(0) / ILUT: the slab's rows of the slab-local factors (R26)
        for (auto [F, GF] : {std::pair<Mat*, const Mat*>{&LL.Lf, &GL.Lf}, {&LL.Uf, &GL.Uf}}) {
          *F = slice_rows(h->arena, *GF, r0, r1, s);
          if (!rep) remap_shift(*F, bd[me], bd[me + 1] - bd[me]);
          F->fast32 = GF->fast32;
          make_tma_plan(*F, s, &h->arena);
        }
        for (void*& w : LL.w) w = h->arena.alloc(std::max<int64_t>((r1 - r0) * LL.A.b, 1) * xs);
      }
      const int bb = LL.A.b;
      const int64_t nl = LL.A.n;
      LL.M = h->arena.alloc(std::max<int64_t>(nl * bb * bb, 1) * dtype_size(h->vt));
      AMG_CK(cudaMemcpy(LL.M, (char*)GL.M + r0 * bb * bb * dtype_size(h->vt), nl * bb * bb * dtype_size(h->vt),
                        cudaMemcpyDeviceToDevice));
      LL.agg = h->arena.alloc_n<int32_t>(std::max<int64_t>(nl, 1));
      AMG_CK(cudaMemcpy(LL.agg, GL.agg + r0, 4 * nl, cudaMemcpyDeviceToDevice));
      LL.nc = (int32_t)(c1 - c0);
      // level 0 of a masked Schur hierarchy also receives B's velocity ghosts (R27)
      const int64_t ng = std::max<int64_t>(LL.halo.nghost, l == 0 && h->masked ? h->haloBu.nghost : 0);
      const int64_t nx = (int64_t)(nl + ng) * bb;
      LL.f = h->arena.alloc(std::max<int64_t>(nl * bb, 1) * xs);
      LL.r = h->arena.alloc(std::max<int64_t>(nl * bb, 1) * xs);
      LL.x = h->arena.alloc(std::max<int64_t>(nx, 1) * xs);
      LL.t = h->arena.alloc(std::max<int64_t>(nx, 1) * xs);
    }
    // coarsest level: replicated
    Coarse& C = h->coarse;
    const Coarse& GC = Gh->coarse;
    C.N = GC.N;
    C.n = GC.n;
    C.b = GC.b;
    if (C.N > 0) {
      C.inv = h->arena.alloc((size_t)C.N * C.N * dtype_size(h->vt));
      AMG_CK(cudaMemcpy(C.inv, GC.inv, (size_t)C.N * C.N * dtype_size(h->vt), cudaMemcpyDeviceToDevice));
    }
    C.A = GC.A;  // export only; points into Gh (cleared below)
    C.A.ptr = nullptr;
    C.A.nnz = 0;
    C.f = h->arena.alloc(std::max<int64_t>(C.N, 1) * xs);
    C.x = h->arena.alloc(std::max<int64_t>(C.N, 1) * xs);
    alloc_workspace(*h, s);
    h->alg_bytes_precond = precond_bytes(*h);
    h->setup_s = Gh->setup_s;
    AMG_CK(cudaStreamSynchronize(s));
  } catch (...) {
    h->comm = nullptr;
    delete h;
    delete Gh;
    throw;
  }
  delete Gh;
  return h;
}

}  // namespace
}  // namespace amgb

using namespace amgb;

#define AMG_GUARD_BEGIN try {
#define AMG_GUARD_END                  \
  }                                    \
  catch (const ::amgb::Error& e) {     \
    ::amgb::set_last_error(e.what);    \
    return e.code;                     \
  }                                    \
  catch (const std::bad_alloc&) {      \
    return AMG_ENOMEM;                 \
  }                                    \
  catch (...) {                        \
    return AMG_EINVAL;                 \
  }

extern "C" {

int amg_comm_unique_id(void* id128) {
  if (!id128) return AMG_EINVAL;
  ncclUniqueId id;
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  if (ncclGetUniqueId(&id) != ncclSuccess) return AMG_ENCCL;
  std::memcpy(id128, &id, sizeof(id));
  return AMG_OK;
}

int amg_comm_init(const void* id128, int32_t nranks, int32_t rank, struct amg_comm** out) {
  AMG_GUARD_BEGIN
  if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) return AMG_EINVAL;
  amg_comm* c = new amg_comm;
  try {
    c->c = make_nccl_comm(id128, nranks, rank);
  } catch (...) {
    delete c;
    throw;
  }
  *out = c;
  return AMG_OK;
  AMG_GUARD_END
}

int amg_local_group_create(int32_t nranks, void** group) {
  if (nranks < 1 || !group) return AMG_EINVAL;
  *group = new LocalGroup(nranks);
  return AMG_OK;
}

void amg_local_group_destroy(void* group) { delete static_cast<LocalGroup*>(group); }

int amg_comm_init_local(void* group, int32_t rank, struct amg_comm** out) {
  LocalGroup* g = static_cast<LocalGroup*>(group);
  if (!g || !out || rank < 0 || rank >= g->P) return AMG_EINVAL;
  amg_comm* c = new amg_comm;
  c->c = make_local_comm(g, rank);
  *out = c;
  return AMG_OK;
}

int amg_comm_init_host(const amg_host_comm_ops* ops, int32_t nranks, int32_t rank, int32_t flags,
                       struct amg_comm** out) {
  if (!ops || !out || nranks < 1 || rank < 0 || rank >= nranks || !ops->allreduce_sum || !ops->allgather_i64 ||
      !ops->exchange || !ops->barrier)
    return AMG_EINVAL;
  static_assert(sizeof(HostOps) == sizeof(amg_host_comm_ops), "HostOps mirrors amg_host_comm_ops");
  HostOps o;
  std::memcpy(&o, ops, sizeof(o));
  AMG_GUARD_BEGIN
  CommBase* cb = make_host_comm(o, nranks, rank, (flags & 1) != 0);
  amg_comm* c = new amg_comm;
  c->c = cb;
  *out = c;
  return AMG_OK;
  AMG_GUARD_END
}

void amg_comm_destroy(struct amg_comm* c) {
  if (!c) return;
  delete c->c;
  delete c;
}

int amg_setup_dist_pmask(const amg_bsr* A_local, const uint8_t* pmask_local, int64_t row_begin,
                         int64_t n_global_block_rows, struct amg_comm* c, const amg_params* p, void* stream,
                         struct amg_handle** out) {
  AMG_GUARD_BEGIN
  if (!c || !c->c || !out || !pmask_local || !p) return AMG_EINVAL;
  int rc = validate_bsr(A_local, false);
  if (rc != AMG_OK) return rc;
  rc = check_params(p);
  if (rc != AMG_OK) return rc;
  if (A_local->n_block_cols != n_global_block_rows || row_begin < 0) return AMG_EDIM;
  if (p->precond != AMG_PC_SCHUR || p->schur_shat == 2) return AMG_EINVAL;
  Handle* h = setup_dist_impl(A_local, row_begin, n_global_block_rows, c->c, p, (cudaStream_t)stream, pmask_local);
  *out = reinterpret_cast<amg_handle*>(h);
  return AMG_OK;
  AMG_GUARD_END
}

int amg_setup_dist(const amg_bsr* A_local, int64_t row_begin, int64_t n_global_block_rows, struct amg_comm* c,
                   const amg_params* p, void* stream, struct amg_handle** out) {
  AMG_GUARD_BEGIN
  if (!c || !c->c || !out) return AMG_EINVAL;
  int rc = validate_bsr(A_local, false);
  if (rc != AMG_OK) return rc;
  rc = check_params(p);
  if (rc != AMG_OK) return rc;
  if (A_local->n_block_cols != n_global_block_rows || row_begin < 0) return AMG_EDIM;
  Handle* h = setup_dist_impl(A_local, row_begin, n_global_block_rows, c->c, p, (cudaStream_t)stream);
  *out = reinterpret_cast<amg_handle*>(h);
  return AMG_OK;
  AMG_GUARD_END
}

}  // extern "C"
