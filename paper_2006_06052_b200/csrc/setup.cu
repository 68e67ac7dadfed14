// setup.cu -- GPU setup of the smoothed-aggregation hierarchy and the Schur split
// (off the hot path, timed separately).
//
// Compiled with --fmad=false: every fp64 product and sum rounds separately, in the
// order the oracle uses: Frobenius norms row-major, sums over
// ascending column / ascending k, no atomics in any numeric accumulation.  The
// strength graph, the aggregates and every sparsity pattern are therefore
// bit-identical to the oracle's, and so are the fp64 level values (up to the sign
// of zero).  Integer-only steps (counts, scans, transposes) may use atomics; every
// list they produce is sorted before use.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cmath>

#include "ops.h"
#include "solver.h"

namespace amgb {

namespace {

constexpr int kT = 256;
constexpr int32_t kInf = 0x7fffffff;

// ---------------------------------------------------------------- small helpers
template <int B>
__device__ __forceinline__ double fro2(const double* a) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < B * B; ++i) s = s + a[i] * a[i];
  return s;
}

// Gauss-Jordan with partial pivoting, first maximal |pivot|; singular if
// |pivot| <= 1e-14 ||X||_F (same steps as the oracle's block_inverse).
template <int B>
__device__ bool block_inverse(const double* x, double* inv) {
  double M[B * B], R[B * B];
#pragma unroll
  for (int i = 0; i < B * B; ++i) M[i] = x[i];
#pragma unroll
  for (int i = 0; i < B; ++i)
#pragma unroll
    for (int j = 0; j < B; ++j) R[i * B + j] = (i == j) ? 1.0 : 0.0;
  const double fn = sqrt(fro2<B>(x));
  for (int c = 0; c < B; ++c) {
    int p = c;
    for (int r = c + 1; r < B; ++r)
      if (fabs(M[r * B + c]) > fabs(M[p * B + c])) p = r;
    if (!(fabs(M[p * B + c]) > 1e-14 * fn)) return false;
    if (p != c)
      for (int j = 0; j < B; ++j) {
        double t = M[p * B + j]; M[p * B + j] = M[c * B + j]; M[c * B + j] = t;
        t = R[p * B + j]; R[p * B + j] = R[c * B + j]; R[c * B + j] = t;
      }
    const double d = M[c * B + c];
    for (int j = 0; j < B; ++j) {
      M[c * B + j] = M[c * B + j] / d;
      R[c * B + j] = R[c * B + j] / d;
    }
    for (int r = 0; r < B; ++r) {
      if (r == c) continue;
      const double f = M[r * B + c];
      for (int j = 0; j < B; ++j) {
        M[r * B + j] = M[r * B + j] - f * M[c * B + j];
        R[r * B + j] = R[r * B + j] - f * R[c * B + j];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < B * B; ++i) inv[i] = R[i];
  return true;
}

// c = a * b, each entry summed over m ascending starting from the first product
template <int B>
__device__ __forceinline__ void blk_mul(const double* a, const double* b, double* c) {
#pragma unroll
  for (int r = 0; r < B; ++r)
#pragma unroll
    for (int cc = 0; cc < B; ++cc) {
      double t = a[r * B] * b[cc];
#pragma unroll
      for (int m = 1; m < B; ++m) t = t + a[r * B + m] * b[m * B + cc];
      c[r * B + cc] = t;
    }
}

__device__ __forceinline__ int bsearch(const int32_t* a, int lo, int hi, int32_t key) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    int32_t v = a[mid];
    if (v == key) return mid;
    if (v < key) lo = mid + 1;
    else hi = mid;
  }
  return -1;
}

__device__ __forceinline__ void set_err(int* err, int code) { atomicCAS(err, 0, code); }

// ---------------------------------------------------------------- S2 strength
__global__ void k_find_diag(int n, const int32_t* ptr, const int32_t* col, int32_t* diag, int* err) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  int k = bsearch(col, ptr[I], ptr[I + 1], I);
  diag[I] = k;
  if (k < 0) set_err(err, AMG_EZERODIAG);
}

template <int B>
__global__ void k_diag_norm(int n, const double* val, const int32_t* diag, double* dn) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  dn[I] = sqrt(fro2<B>(val + (int64_t)diag[I] * B * B));
}

// strong(I,J): ||A_IJ||_F^2 > eps^2 ||A_II||_F ||A_JJ||_F, same slab
template <int B>
__global__ void k_strength(int n, const int32_t* ptr, const int32_t* col, const double* val, const double* dn,
                           double eps2, const int32_t* part, uint8_t* s) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  for (int k = ptr[I]; k < ptr[I + 1]; ++k) {
    int J = col[k];
    bool st = false;
    if (J != I && J < n && (!part || part[I] == part[J]))
      st = fro2<B>(val + (int64_t)k * B * B) > eps2 * dn[I] * dn[J];
    s[k] = st ? 1 : 0;
  }
}

// position of (J, I) for every stored (I, J); -1 if structurally absent
__global__ void k_tpos(int n, const int32_t* ptr, const int32_t* col, int32_t* tpos) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  for (int k = ptr[I]; k < ptr[I + 1]; ++k) {
    int J = col[k];
    tpos[k] = (J < n) ? bsearch(col, ptr[J], ptr[J + 1], I) : -1;
  }
}

// symmetric closure S u S^T restricted to A's pattern, plus a count of closure edges
// (J, I) whose position is absent from A's pattern ("extras")
__global__ void k_sym(int n, const int32_t* ptr, const int32_t* col, const uint8_t* s, const int32_t* tpos,
                      uint8_t* sym, int32_t* extra_cnt) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  for (int k = ptr[I]; k < ptr[I + 1]; ++k) {
    int t = tpos[k];
    sym[k] = (s[k] || (t >= 0 && s[t])) ? 1 : 0;
    if (s[k] && t < 0) atomicAdd(extra_cnt + col[k], 1);
  }
}

__global__ void k_adj_count(int n, const int32_t* ptr, const uint8_t* sym, const int32_t* extra_cnt, int32_t* deg) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  int d = extra_cnt[I];
  for (int k = ptr[I]; k < ptr[I + 1]; ++k) d += sym[k];
  deg[I] = d;
}

__global__ void k_adj_fill(int n, const int32_t* ptr, const int32_t* col, const uint8_t* sym, const int32_t* aptr,
                           int32_t* adj, int32_t* cursor) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  int o = aptr[I];
  for (int k = ptr[I]; k < ptr[I + 1]; ++k)
    if (sym[k]) adj[o++] = col[k];
  cursor[I] = o;
}

__global__ void k_adj_extras(int n, const int32_t* ptr, const int32_t* col, const uint8_t* s, const int32_t* tpos,
                             int32_t* adj, int32_t* cursor) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  for (int k = ptr[I]; k < ptr[I + 1]; ++k)
    if (s[k] && tpos[k] < 0) adj[atomicAdd(cursor + col[k], 1)] = I;
}

__global__ void k_sort_segments(int n, const int32_t* aptr, int32_t* a) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  for (int i = aptr[I] + 1; i < aptr[I + 1]; ++i) {
    int32_t v = a[i];
    int j = i - 1;
    while (j >= aptr[I] && a[j] > v) {
      a[j + 1] = a[j];
      --j;
    }
    a[j + 1] = v;
  }
}

// ---------------------------------------------------------------- S3 aggregation
// Lexicographically-first MIS of the distance-2 strength graph by parallel rounds
// (SURVEY.md C3): equals the oracle's sequential pass 1 roots.
enum : uint8_t { UND = 0, ROOT = 1, NOTR = 2 };

__global__ void k_mis_init(int n, const int32_t* aptr, uint8_t* st) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) st[v] = (aptr[v + 1] == aptr[v]) ? NOTR : UND;
}

__global__ void k_mis_1(int n, const int32_t* aptr, const int32_t* adj, const uint8_t* st, int32_t* m1, uint8_t* r1) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int32_t m = (st[v] == UND) ? v : kInf;
  uint8_t r = st[v] == ROOT;
  for (int k = aptr[v]; k < aptr[v + 1]; ++k) {
    int u = adj[k];
    uint8_t su = st[u];
    if (su == UND && u < m) m = u;
    r |= (su == ROOT);
  }
  m1[v] = m;
  r1[v] = r;
}

__global__ void k_mis_2(int n, const int32_t* aptr, const int32_t* adj, uint8_t* st, const int32_t* m1,
                        const uint8_t* r1, int* und) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n || st[v] != UND) return;
  int32_t m = m1[v];
  uint8_t r = r1[v];
  for (int k = aptr[v]; k < aptr[v + 1]; ++k) {
    int u = adj[k];
    int32_t mu = m1[u];
    if (mu < m) m = mu;
    r |= r1[u];
  }
  if (r) st[v] = NOTR;
  else if (m == v) st[v] = ROOT;
  else atomicAdd(und, 1);
}

__global__ void k_is_root(int n, const uint8_t* st, int32_t* flag) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) flag[v] = st[v] == ROOT;
}

// pass 1: roots and their (unique) adjacent members; pass 2: leftovers join the pass-1
// aggregate of their lowest-index strong neighbour assigned in pass 1
__global__ void k_pass1(int n, const int32_t* aptr, const int32_t* adj, const uint8_t* st, const int32_t* rid,
                        int32_t* agg1) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int a = -1;
  if (st[v] == ROOT) a = rid[v];
  else
    for (int k = aptr[v]; k < aptr[v + 1]; ++k)
      if (st[adj[k]] == ROOT) {
        a = rid[adj[k]];
        break;
      }
  agg1[v] = a;
}

__global__ void k_pass2(int n, const int32_t* aptr, const int32_t* adj, const int32_t* agg1, int32_t* agg) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int a = agg1[v];
  if (a < 0)
    for (int k = aptr[v]; k < aptr[v + 1]; ++k)
      if (agg1[adj[k]] >= 0) {
        a = agg1[adj[k]];
        break;
      }
  agg[v] = a;
}

// ---------------------------------------------------------------- S4/S5 prolongator
// D_I = A_II + sum of weak off-diagonal blocks (ascending column); D^-1
template <int B>
__global__ void k_filtered_diag(int n, const int32_t* ptr, const int32_t* col, const double* val,
                                const int32_t* diag, const uint8_t* sym, double* D, double* Dinv, int* err) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  double d[B * B];
  const double* a = val + (int64_t)diag[I] * B * B;
#pragma unroll
  for (int e = 0; e < B * B; ++e) d[e] = a[e];
  for (int k = ptr[I]; k < ptr[I + 1]; ++k) {
    if (k == diag[I] || sym[k]) continue;
    const double* w = val + (int64_t)k * B * B;
#pragma unroll
    for (int e = 0; e < B * B; ++e) d[e] = d[e] + w[e];
  }
#pragma unroll
  for (int e = 0; e < B * B; ++e) D[(int64_t)I * B * B + e] = d[e];
  if (!block_inverse<B>(d, Dinv + (int64_t)I * B * B)) set_err(err, AMG_ESINGULAR_BLOCK);
}

// candidate coarse columns of row I: agg(J) for J kept in A_F (diagonal or strong);
// sorted + unique in place in cand[ptr[I] ...]; count -> cnt[I]
__global__ void k_p_cand(int n, const int32_t* ptr, const int32_t* col, const int32_t* diag, const uint8_t* sym,
                         const int32_t* agg, int32_t* cand, int32_t* cnt) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  int o = ptr[I], m = 0;
  for (int k = ptr[I]; k < ptr[I + 1]; ++k) {
    if (!(k == diag[I] || sym[k])) continue;
    int a = agg[col[k]];
    if (a < 0) continue;
    int j = m - 1;  // insertion into the sorted prefix
    while (j >= 0 && cand[o + j] > a) {
      cand[o + j + 1] = cand[o + j];
      --j;
    }
    cand[o + j + 1] = a;
    ++m;
  }
  int u = 0;
  for (int i = 0; i < m; ++i)
    if (u == 0 || cand[o + u - 1] != cand[o + i]) cand[o + u++] = cand[o + i];
  cnt[I] = u;
}

// P_IC = P_tent,IC - omega * (D_I^-1 T_IC), T = A_F P_tent accumulated over ascending k
template <int B>
__global__ void k_p_fill(int n, const int32_t* ptr, const int32_t* col, const double* val, const int32_t* diag,
                         const uint8_t* sym, const int32_t* agg, const double* D, const double* Dinv,
                         const int32_t* cand, const int32_t* pptr, int32_t* pcol, double* pval, double omega) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  const int p0 = pptr[I], p1 = pptr[I + 1];
  for (int i = p0; i < p1; ++i) {
    pcol[i] = cand[ptr[I] + (i - p0)];
    for (int e = 0; e < B * B; ++e) pval[(int64_t)i * B * B + e] = 0.0;
  }
  for (int k = ptr[I]; k < ptr[I + 1]; ++k) {
    const bool isd = (k == diag[I]);
    if (!(isd || sym[k])) continue;
    int a = agg[col[k]];
    if (a < 0) continue;
    int pos = bsearch(pcol, p0, p1, a);
    const double* src = isd ? (D + (int64_t)I * B * B) : (val + (int64_t)k * B * B);
    double* t = pval + (int64_t)pos * B * B;
    for (int e = 0; e < B * B; ++e) t[e] = t[e] + src[e];
  }
  const double* di = Dinv + (int64_t)I * B * B;
  for (int i = p0; i < p1; ++i) {
    double* t = pval + (int64_t)i * B * B;
    double dt[B * B];
    blk_mul<B>(di, t, dt);
    const bool own = pcol[i] == agg[I];
    for (int r = 0; r < B; ++r)
      for (int c = 0; c < B; ++c) {
        double pt = (own && r == c) ? 1.0 : 0.0;
        t[r * B + c] = pt - omega * dt[r * B + c];
      }
  }
}

// plain aggregation (Listings V2-V4): P = P_tent, one identity block per aggregated row
__global__ void k_ptent_count(int n, const int32_t* agg, int32_t* cnt) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I < n) cnt[I] = agg[I] >= 0 ? 1 : 0;
}
template <int B>
__global__ void k_ptent_fill(int n, const int32_t* agg, const int32_t* pptr, int32_t* pcol, double* pval) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n || agg[I] < 0) return;
  const int i = pptr[I];
  pcol[i] = agg[I];
  for (int r = 0; r < B; ++r)
    for (int c = 0; c < B; ++c) pval[(int64_t)i * B * B + r * B + c] = (r == c) ? 1.0 : 0.0;
}
// over-interpolation (reading R19): A_c values times 1 / alpha
__global__ void k_scale_vals(int64_t m, double inv, double* v) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < m) v[e] = v[e] * inv;
}

// ---------------------------------------------------------------- S7 transpose
__global__ void k_count_cols(int64_t nnz, const int32_t* col, int32_t* cnt) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nnz) atomicAdd(cnt + col[k], 1);
}

template <int B>
__global__ void k_transpose_fill(int n, const int32_t* ptr, const int32_t* col, const double* val, int32_t* cursor,
                                 int32_t* tcol, double* tval) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  for (int k = ptr[I]; k < ptr[I + 1]; ++k) {
    int d = atomicAdd(cursor + col[k], 1);
    tcol[d] = I;
    const double* s = val + (int64_t)k * B * B;
    double* t = tval + (int64_t)d * B * B;
    for (int r = 0; r < B; ++r)
      for (int c = 0; c < B; ++c) t[c * B + r] = s[r * B + c];
  }
}

template <int B>
__global__ void k_sort_rows_blocks(int n, const int32_t* ptr, int32_t* col, double* val) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  for (int i = ptr[I] + 1; i < ptr[I + 1]; ++i) {
    int32_t key = col[i];
    double v[B * B];
    for (int e = 0; e < B * B; ++e) v[e] = val[(int64_t)i * B * B + e];
    int j = i - 1;
    while (j >= ptr[I] && col[j] > key) {
      col[j + 1] = col[j];
      for (int e = 0; e < B * B; ++e) val[(int64_t)(j + 1) * B * B + e] = val[(int64_t)j * B * B + e];
      --j;
    }
    col[j + 1] = key;
    for (int e = 0; e < B * B; ++e) val[(int64_t)(j + 1) * B * B + e] = v[e];
  }
}

// ---------------------------------------------------------------- S6 SpGEMM
// symbolic: k-way merge of the sorted B rows selected by A's row -> sorted unique cols
__global__ void k_spgemm_sym(int n, const int32_t* aptr, const int32_t* acol, const int32_t* bptr,
                             const int32_t* bcol, int32_t* heads, const int32_t* cptr, int32_t* ccol, int32_t* cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int a0 = aptr[i], a1 = aptr[i + 1];
  for (int e = a0; e < a1; ++e) heads[e] = bptr[acol[e]];
  int c = 0;
  int out = ccol ? cptr[i] : 0;
  while (true) {
    int32_t mn = kInf;
    for (int e = a0; e < a1; ++e) {
      int h = heads[e];
      if (h < bptr[acol[e] + 1]) {
        int32_t v = bcol[h];
        if (v < mn) mn = v;
      }
    }
    if (mn == kInf) break;
    if (ccol) ccol[out + c] = mn;
    ++c;
    for (int e = a0; e < a1; ++e) {
      int h = heads[e];
      if (h < bptr[acol[e] + 1] && bcol[h] == mn) heads[e] = h + 1;
    }
  }
  if (cnt) cnt[i] = c;
}

// numeric: C_ij = C_ij + A_ik B_kj over k ascending (A's row order), then B's row order
template <int B>
__global__ void k_spgemm_num(int n, const int32_t* aptr, const int32_t* acol, const double* aval,
                             const int32_t* bptr, const int32_t* bcol, const double* bval, const int32_t* cptr,
                             const int32_t* ccol, double* cval) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c0 = cptr[i], c1 = cptr[i + 1];
  for (int64_t e = (int64_t)c0 * B * B; e < (int64_t)c1 * B * B; ++e) cval[e] = 0.0;
  double tmp[B * B];
  for (int ka = aptr[i]; ka < aptr[i + 1]; ++ka) {
    const int k = acol[ka];
    const double* a = aval + (int64_t)ka * B * B;
    for (int kb = bptr[k]; kb < bptr[k + 1]; ++kb) {
      blk_mul<B>(a, bval + (int64_t)kb * B * B, tmp);
      int pos = bsearch(ccol, c0, c1, bcol[kb]);
      double* c = cval + (int64_t)pos * B * B;
#pragma unroll
      for (int e = 0; e < B * B; ++e) c[e] = c[e] + tmp[e];
    }
  }
}

// ---------------------------------------------------------------- S8 smoother
template <int B>
__global__ void k_smoother(int n, const int32_t* ptr, const double* val, const int32_t* diag, int spai0,
                           double omega_j, double* M, int* err) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  double inv[B * B];
  const double* a = val + (int64_t)diag[I] * B * B;
  if (!block_inverse<B>(a, inv)) {
    set_err(err, AMG_ESINGULAR_BLOCK);
    return;
  }
  double theta = omega_j;
  if (spai0) {
    double den = 0.0;
    for (int k = ptr[I]; k < ptr[I + 1]; ++k) den = den + fro2<B>(val + (int64_t)k * B * B);
    theta = fro2<B>(a) / den;
  }
  for (int e = 0; e < B * B; ++e) M[(int64_t)I * B * B + e] = theta * inv[e];
}

// ---------------------------------------------------------------- S8b block ILU(0)
// Row i of the IKJ factorisation on A's pattern (reading R20; the oracle's ilu0_factor, same
// operation order): for k < i ascending: a_ik <- a_ik D_k^-1, a_ij <- a_ij - a_ik a_kj for the
// later j of row i present in row k; then D_i^-1 = inverse(a_ii).  Rows of one dependency
// level run in parallel (their k < i rows are final).
template <int B>
__global__ void k_ilu_rows(int cnt, const int32_t* rows, const int32_t* ptr, const int32_t* col, double* a,
                           double* Dinv, int* err) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= cnt) return;
  const int i = rows[t];
  double tmp[B * B];
  int kd = -1;
  for (int kk = ptr[i]; kk < ptr[i + 1]; ++kk) {
    const int k = col[kk];
    if (k == i) kd = kk;
    if (k >= i) continue;
    double* aik = a + (int64_t)kk * B * B;
    blk_mul<B>(aik, Dinv + (int64_t)k * B * B, tmp);
    for (int e = 0; e < B * B; ++e) aik[e] = tmp[e];
    for (int jj = kk + 1; jj < ptr[i + 1]; ++jj) {
      const int kj = bsearch(col, ptr[k], ptr[k + 1], col[jj]);
      if (kj < 0) continue;
      blk_mul<B>(aik, a + (int64_t)kj * B * B, tmp);
      double* aij = a + (int64_t)jj * B * B;
      for (int e = 0; e < B * B; ++e) aij[e] = aij[e] - tmp[e];
    }
  }
  if (kd < 0) {
    set_err(err, AMG_EZERODIAG);
    return;
  }
  if (!block_inverse<B>(a + (int64_t)kd * B * B, Dinv + (int64_t)i * B * B)) set_err(err, AMG_ESINGULAR_BLOCK);
}

// ---------------------------------------------------------------- S8c block ILUT(tau, p)
// Row i of Saad's threshold IKJ factorisation on blocks (reading R25; the oracle's
// ilut_factor, same operation order, so patterns and fp64 values are bit-identical).
// Fill makes the dependency graph data-dependent, so rows are not level-scheduled: one warp
// per row, rows claimed in ascending order from a global counter, and a row waits for each
// row k it eliminates with (k < i) on k's completion flag (release / acquire at gpu scope).
// Every claimed row is held by a running warp and waits only on smaller rows, so the
// smallest unfinished row always progresses (no deadlock).  The working row w lives in
// shared memory as an unsorted list (original entries first, fill appended); entries are
// eliminated in ascending column order by a warp-wide min over the unprocessed ones.
// Kept entries are written to per-row slabs of capacity (row's A entries on that side) + p,
// compacted afterwards.
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int kIlutCap = 512;  // working-row entries per warp (error beyond)
template <int B>
struct IlutShape {
  static constexpr int BB = B * B;
  static constexpr int W = B == 4 ? 1 : 2;  // warps per block
  static constexpr size_t per_warp = (size_t)kIlutCap * (8 * BB + 8 + 4 + 1) + 8 * BB + 64;
  static constexpr size_t smem = per_warp * W;
};

template <int B>
__global__ void __launch_bounds__(32 * IlutShape<B>::W) k_ilut_rows(
    int n, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col, const double* __restrict__ val,
    double tau, int pfill, const int32_t* __restrict__ loff, const int32_t* __restrict__ uoff, int32_t* lcol,
    double* lval, int32_t* llen, int32_t* ucol, double* uval, int32_t* ulen, double* Dinv, int* done, int* counter,
    int* err) {
  constexpr int BB = B * B;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned char* base = smem_raw + (size_t)wid * IlutShape<B>::per_warp;
  double* wv = reinterpret_cast<double*>(base);                 // [cap][BB]
  double* nrm = wv + (size_t)kIlutCap * BB;                     // [cap] norms (phase 2)
  double* tl = nrm + kIlutCap;                                  // [BB] the current multiplier
  int32_t* wc = reinterpret_cast<int32_t*>(tl + BB);            // [cap] columns; -1 - col when dropped
  int* wlen = reinterpret_cast<int*>(wc + kIlutCap);           // list length
  uint8_t* kept = reinterpret_cast<uint8_t*>(wlen + 4);         // [cap] phase-2 decisions
  for (;;) {
    int i = 0;
    if (lane == 0) i = atomicAdd(counter, 1);
    i = __shfl_sync(kFull, i, 0);
    if (i >= n) return;
    const int r0 = ptr[i], len0 = ptr[i + 1] - r0;
    // a failed row (capacity, missing pivot, or another row's failure seen while waiting)
    // records the error and is still marked done, empty: no warp ever waits forever
    auto fail_row = [&](int code) {
      if (lane == 0) {
        if (code) set_err(err, code);
        llen[i] = 0, ulen[i] = 0;
      }
      __syncwarp();
      __threadfence();
      if (lane == 0) st_release(done + i, 1);
    };
    if (len0 > kIlutCap) {
      fail_row(AMG_EINVAL);
      continue;
    }
    for (int q = lane; q < len0; q += 32) {
      wc[q] = col[r0 + q];
      for (int e = 0; e < BB; ++e) wv[(size_t)q * BB + e] = val[(int64_t)(r0 + q) * BB + e];
    }
    if (lane == 0) *wlen = len0;
    double tau_i = 0.0;
    if (lane == 0) {
      double s2 = 0.0;
      for (int q = 0; q < len0; ++q) s2 = s2 + fro2<B>(val + (int64_t)(r0 + q) * BB);
      tau_i = tau * sqrt(s2);
    }
    tau_i = __shfl_sync(kFull, tau_i, 0);
    __syncwarp();
    int last = -1;
    bool overflow = false;
    int bad = 0;  // this row's error code (AMG_E*, negative), or 1: another row failed
    for (;;) {
      // next k: the smallest live column in (last, i)
      const int len = *wlen;
      int best = INT_MAX, bidx = -1;
      for (int q = lane; q < len; q += 32) {
        const int c = wc[q];
        if (c > last && c < i && c < best) best = c, bidx = q;
      }
      const int k = __reduce_min_sync(kFull, (unsigned)best);
      if (k == INT_MAX) break;
      const unsigned who = __ballot_sync(kFull, best == k);
      const int kq = __shfl_sync(kFull, bidx, __ffs(who) - 1);
      while (ld_acquire(done + k) == 0)
        if (*(volatile int*)err) break;
      if (__any_sync(kFull, *(volatile int*)err != 0)) {
        bad = 1;
        break;
      }
      // multiplier l = w_k D_k^-1 (lane e < BB: entry e, blk_mul's order)
      double le = 0.0;
      if (lane < BB) {
        const int r = lane / B, cc = lane - r * B;
        const double* a = wv + (size_t)kq * BB;
        const double* d = Dinv + (int64_t)k * BB;
        double t = a[r * B] * __ldcg(d + cc);
        for (int m = 1; m < B; ++m) t = t + a[r * B + m] * __ldcg(d + m * B + cc);
        le = t;
      }
      __syncwarp();
      if (lane < BB) tl[lane] = le;
      __syncwarp();
      double ln = 0.0;
      if (lane == 0) ln = sqrt(fro2<B>(tl));
      ln = __shfl_sync(kFull, ln, 0);
      last = k;
      if (ln < tau_i) {  // dropped: no update
        if (lane == 0) wc[kq] = -1 - k;
        __syncwarp();
        continue;
      }
      if (lane < BB) wv[(size_t)kq * BB + lane] = le;
      // w_j -= l U_kj for the stored U entries of row k (distinct j: one lane each)
      const int u0 = uoff[k], ul = __ldcg(ulen + k);
      for (int q = lane; q < ul; q += 32) {
        const int j = __ldcg(ucol + u0 + q);
        int idx = -1;
        for (int t = 0; t < len; ++t)
          if (wc[t] == j) {
            idx = t;
            break;
          }
        if (idx < 0) {
          idx = atomicAdd(wlen, 1);
          if (idx >= kIlutCap) {
            overflow = true;
            continue;
          }
          wc[idx] = j;
          for (int e = 0; e < BB; ++e) wv[(size_t)idx * BB + e] = 0.0;
        }
        const double* U = uval + (int64_t)(u0 + q) * BB;
        double* wj = wv + (size_t)idx * BB;
        for (int r = 0; r < B; ++r)
          for (int cc = 0; cc < B; ++cc) {
            double t = tl[r * B] * __ldcg(U + cc);
            for (int m = 1; m < B; ++m) t = t + tl[r * B + m] * __ldcg(U + m * B + cc);
            wj[r * B + cc] = wj[r * B + cc] - t;
          }
      }
      if (__any_sync(kFull, overflow)) {
        bad = AMG_EINVAL;
        break;
      }
      __syncwarp();
    }
    if (bad) {
      fail_row(bad == 1 ? 0 : bad);
      continue;
    }
    const int len = min(*wlen, kIlutCap);
    // pivot
    int dq = -1;
    for (int q = lane; q < len; q += 32)
      if (wc[q] == i) dq = q;
    const unsigned dm = __ballot_sync(kFull, dq >= 0);
    if (!dm) {
      fail_row(AMG_EZERODIAG);
      continue;
    }
    dq = __shfl_sync(kFull, dq, __ffs(dm) - 1);
    if (lane == 0 && !block_inverse<B>(wv + (size_t)dq * BB, Dinv + (int64_t)i * BB)) set_err(err, AMG_ESINGULAR_BLOCK);
    // norms; candidates: live, off-diagonal, ||w_j|| >= tau_i
    for (int q = lane; q < len; q += 32) {
      const int c = wc[q];
      nrm[q] = (c >= 0 && c != i) ? sqrt(fro2<B>(wv + (size_t)q * BB)) : -1.0;
      if (c >= 0 && c != i && nrm[q] < tau_i) nrm[q] = -1.0;
    }
    __syncwarp();
    // keep: original entries, and fill ranked < p by (norm desc, column asc) within its side
    int nl = 0, nu = 0;
    for (int q0 = 0; q0 < len; q0 += 32) {
      const int q = q0 + lane;
      bool keep = false;
      int c = -1;
      if (q < len && nrm[q] >= 0.0) {
        c = wc[q];
        keep = q < len0;
        if (!keep) {
          int rank = 0;
          for (int t = len0; t < len; ++t) {
            const int ct = wc[t];
            if (t == q || nrm[t] < 0.0 || ((ct < i) != (c < i))) continue;
            if (nrm[t] > nrm[q] || (nrm[t] == nrm[q] && ct < c)) ++rank;
          }
          keep = rank < pfill;
        }
      }
      if (q < len) kept[q] = keep;
      nl += __popc(__ballot_sync(kFull, keep && c < i));
      nu += __popc(__ballot_sync(kFull, keep && c > i));
    }
    __syncwarp();
    // positions: ascending column within each side
    for (int q = lane; q < len; q += 32) {
      if (!kept[q]) continue;
      const int c = wc[q];
      int pos = 0;
      for (int t = 0; t < len; ++t) {
        const int ct = wc[t];
        if (kept[t] && ((ct < i) == (c < i)) && ct < c) ++pos;
      }
      int32_t* oc = c < i ? lcol + loff[i] : ucol + uoff[i];
      double* ov = c < i ? lval + (int64_t)loff[i] * BB : uval + (int64_t)uoff[i] * BB;
      oc[pos] = c;
      for (int e = 0; e < BB; ++e) ov[(int64_t)pos * BB + e] = wv[(size_t)q * BB + e];
    }
    if (lane == 0) llen[i] = nl, ulen[i] = nu;
    __syncwarp();
    __threadfence();
    if (lane == 0) st_release(done + i, 1);
  }
}

__global__ void k_ilut_compact(int n, const int32_t* off, const int32_t* len, const int32_t* scol, const double* sval,
                               const int32_t* ptr, int32_t* col, double* val, int bb) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int q = 0; q < len[i]; ++q) {
    col[ptr[i] + q] = scol[off[i] + q];
    for (int e = 0; e < bb; ++e) val[(int64_t)(ptr[i] + q) * bb + e] = sval[(int64_t)(off[i] + q) * bb + e];
  }
}

__global__ void k_add_scalar(int n, int32_t* a, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] += v;
}

__global__ void k_tri_count(int n, const int32_t* ptr, const int32_t* col, int32_t* lc, int32_t* uc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int l = 0, u = 0;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) l += col[k] < i, u += col[k] > i;
  lc[i] = l;
  uc[i] = u;
}
template <int B>
__global__ void k_tri_fill(int n, const int32_t* ptr, const int32_t* col, const double* a, const int32_t* lp,
                           int32_t* lcol, double* lval, const int32_t* up, int32_t* ucol, double* uval) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int l = lp[i], u = up[i];
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    const int j = col[k];
    if (j == i) continue;
    const int o = j < i ? l++ : u++;
    int32_t* dc = j < i ? lcol : ucol;
    double* dv = j < i ? lval : uval;
    dc[o] = j;
    for (int e = 0; e < B * B; ++e) dv[(int64_t)o * B * B + e] = a[(int64_t)k * B * B + e];
  }
}

// ---------------------------------------------------------------- S9 Schur split
// A (b x b, fp64) -> A_u (nu x nu), B (row pc, vel cols), B^T (vel rows, col pc), C
__global__ void k_schur_split(int64_t nnz, int b, int pc, const double* val, double* au, double* bv, double* btv,
                              double* cv) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nnz) return;
  const int nu = b - 1;
  const double* a = val + k * b * b;
  for (int r = 0; r < nu; ++r) {
    int vr = r < pc ? r : r + 1;
    for (int c = 0; c < nu; ++c) {
      int vc = c < pc ? c : c + 1;
      au[k * nu * nu + r * nu + c] = a[vr * b + vc];
    }
    bv[k * nu + r] = a[pc * b + vr];
    btv[k * nu + r] = a[vr * b + pc];
  }
  cv[k] = a[pc * b + pc];
}

// Shat_ii = C_ii - sum_J sum_d B_iJ[d] (1/A_u,JJ[d][d]) B^T_Ji[d]  (Eq. 10, PAPER.md:541-543;
// mode 1) or C_ii (mode 0: S_hat = C); m_S,i = Shat_ii / sum_j Shat_ij^2 over C's pattern
// (SPAI0 of Shat)
__global__ void k_schur_shat(int n, int nu, int mode, const int32_t* ptr, const int32_t* col, const int32_t* diag,
                             const double* au, const double* bv, const double* btv, const double* cv, double* shat,
                             double* ms, int* err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double sum = 0.0;
  for (int k = ptr[i]; k < ptr[i + 1] && mode == 1; ++k) {
    int J = col[k];
    int kJJ = diag[J];
    int kJi = bsearch(col, ptr[J], ptr[J + 1], i);
    if (kJi < 0) continue;
    for (int d = 0; d < nu; ++d) {
      double dg = au[(int64_t)kJJ * nu * nu + d * nu + d];
      if (dg == 0.0) {
        set_err(err, AMG_EZERODIAG);
        return;
      }
      double t = bv[(int64_t)k * nu + d] * (1.0 / dg);
      sum = sum + t * btv[(int64_t)kJi * nu + d];
    }
  }
  const int kd = diag[i];
  double s = cv[kd] - sum;
  double den = 0.0;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    double v = (k == kd) ? s : cv[k];
    den = den + v * v;
  }
  if (den == 0.0) {
    set_err(err, AMG_EZERODIAG);
    return;
  }
  shat[i] = s;
  ms[i] = s / den;
}

// mode 2, the explicitly assembled S_hat = C - B diag(A_u)^-1 B^T (the PETSc variant,
// PAPER.md:558-561) on pattern(A A) (spgemm symbolic, sorted rows): sum_ij accumulated
// over k (row i's blocks ascending), then d; S_hat_ij = C_ij - sum_ij (C_ij = 0 off C's
// pattern); m_S,i = S_hat_ii / sum_j S_hat_ij^2 (j ascending).  Thread per pressure row.
__global__ void k_schur_shat_full(int n, int nu, const int32_t* ptr, const int32_t* col, const int32_t* diag,
                                  const double* au, const double* bv, const double* btv, const double* cv,
                                  const int32_t* sptr, const int32_t* scol, double* ssum, double* shat, double* ms,
                                  int* err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c0 = sptr[i], c1 = sptr[i + 1];
  for (int q = c0; q < c1; ++q) ssum[q] = 0.0;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    const int K = col[k], kKK = diag[K];
    for (int d = 0; d < nu; ++d) {
      const double dg = au[(int64_t)kKK * nu * nu + d * nu + d];
      if (dg == 0.0) {
        set_err(err, AMG_EZERODIAG);
        return;
      }
      const double t = bv[(int64_t)k * nu + d] * (1.0 / dg);
      for (int kk = ptr[K]; kk < ptr[K + 1]; ++kk) {
        const int q = bsearch(scol, c0, c1, col[kk]);
        ssum[q] = ssum[q] + t * btv[(int64_t)kk * nu + d];
      }
    }
  }
  double den = 0.0, sii = 0.0;
  int k = ptr[i];
  for (int q = c0; q < c1; ++q) {
    const int j = scol[q];
    while (k < ptr[i + 1] && col[k] < j) ++k;
    const double c = (k < ptr[i + 1] && col[k] == j) ? cv[k] : 0.0;
    const double v = c - ssum[q];
    if (j == i) sii = v;
    den = den + v * v;
  }
  if (den == 0.0) {
    set_err(err, AMG_EZERODIAG);
    return;
  }
  shat[i] = sii;
  ms[i] = sii / den;
}

// ---------------------------------------------------------------- S9b Schur split by a scalar mask
// (reading R21) on the scalar expansion As of A: class flags -> exclusive scans give each
// unknown its position in its class; rows split into A_u / B^T (u rows) and B / C (p rows),
// columns renumbered, order kept.
__global__ void k_mask_flags(int64_t N, const uint8_t* m, int32_t* iu, int32_t* ip) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= N) return;
  iu[q] = m[q] ? 0 : 1;
  ip[q] = m[q] ? 1 : 0;
}
__global__ void k_mask_index(int64_t N, const uint8_t* m, const int32_t* iu, const int32_t* ip, int32_t* uidx,
                             int32_t* pidx) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= N) return;
  if (m[q]) pidx[ip[q]] = (int32_t)q;
  else uidx[iu[q]] = (int32_t)q;
}
__global__ void k_mask_count(int64_t N, const int32_t* sp, const int32_t* sc, const uint8_t* m, const int32_t* iu,
                             const int32_t* ip, int32_t* cA, int32_t* cBT, int32_t* cB, int32_t* cC) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= N) return;
  int u = 0, p = 0;
  for (int k = sp[q]; k < sp[q + 1]; ++k) (m[sc[k]] ? p : u) += 1;
  if (m[q]) cB[ip[q]] = u, cC[ip[q]] = p;
  else cA[iu[q]] = u, cBT[iu[q]] = p;
}
__global__ void k_mask_fill(int64_t N, const int32_t* sp, const int32_t* sc, const double* sv, const uint8_t* m,
                            const int32_t* iu, const int32_t* ip, const int32_t* Ap, int32_t* Ac, double* Av,
                            const int32_t* BTp, int32_t* BTc, double* BTv, const int32_t* Bp, int32_t* Bc, double* Bv,
                            const int32_t* Cp, int32_t* Cc, double* Cv) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= N) return;
  const bool pr = m[q] != 0;
  const int r = pr ? ip[q] : iu[q];
  int o1 = pr ? Bp[r] : Ap[r], o2 = pr ? Cp[r] : BTp[r];
  int32_t* c1 = pr ? Bc : Ac;
  int32_t* c2 = pr ? Cc : BTc;
  double* v1 = pr ? Bv : Av;
  double* v2 = pr ? Cv : BTv;
  for (int k = sp[q]; k < sp[q + 1]; ++k) {
    const int j = sc[k];
    if (m[j]) c2[o2] = ip[j], v2[o2++] = sv[k];
    else c1[o1] = iu[j], v1[o1++] = sv[k];
  }
}
// Eq. 10 on the scalar split (mode 1) or S_hat = C (mode 0); m_S = SPAI0 (the oracle's order)
__global__ void k_schur_shat_scalar(int np, int mode, const int32_t* Bp, const int32_t* Bc, const double* Bv,
                                    const int32_t* Ap, const int32_t* Ac, const double* Av, const int32_t* BTp,
                                    const int32_t* BTc, const double* BTv, const int32_t* Cp, const int32_t* Cc,
                                    const double* Cv, double* shat, double* ms, int* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np) return;
  const int kd = bsearch(Cc, Cp[i], Cp[i + 1], i);
  if (kd < 0) {
    set_err(err, AMG_EZERODIAG);
    return;
  }
  double sum = 0.0;
  for (int k = Bp[i]; k < Bp[i + 1] && mode == 1; ++k) {
    const int J = Bc[k];
    const int kJJ = bsearch(Ac, Ap[J], Ap[J + 1], J);
    if (kJJ < 0) {
      set_err(err, AMG_EZERODIAG);
      return;
    }
    const int kJi = bsearch(BTc, BTp[J], BTp[J + 1], i);
    if (kJi < 0) continue;
    const double dg = Av[kJJ];
    if (dg == 0.0) {
      set_err(err, AMG_EZERODIAG);
      return;
    }
    const double t = Bv[k] * (1.0 / dg);
    sum = sum + t * BTv[kJi];
  }
  const double s = Cv[kd] - sum;
  double den = 0.0;
  for (int k = Cp[i]; k < Cp[i + 1]; ++k) {
    const double v = (k == kd) ? s : Cv[k];
    den = den + v * v;
  }
  if (den == 0.0) {
    set_err(err, AMG_EZERODIAG);
    return;
  }
  shat[i] = s;
  ms[i] = s / den;
}

// ---------------------------------------------------------------- S11 coarse inverse
template <int B>
__global__ void k_densify(int n, const int32_t* ptr, const int32_t* col, const double* val, double* W, int N) {
  int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= n) return;
  const int64_t ld = 2 * (int64_t)N;
  for (int k = ptr[I]; k < ptr[I + 1]; ++k)
    for (int r = 0; r < B; ++r)
      for (int c = 0; c < B; ++c) W[(int64_t)(I * B + r) * ld + (int64_t)col[k] * B + c] = val[(int64_t)k * B * B + r * B + c];
  for (int r = 0; r < B; ++r) W[(int64_t)(I * B + r) * ld + N + I * B + r] = 1.0;
}

// one block: pivot search (first max |W[r][c]|, r >= c), row swap, row scaling, multipliers
__global__ void k_gj_pivot(int N, int c, double* W, double* fcol, int* err) {
  __shared__ double sv[1024];
  __shared__ int si[1024];
  const int64_t ld = 2 * (int64_t)N;
  double best = -1.0;
  int bi = N;
  for (int r = c + threadIdx.x; r < N; r += blockDim.x) {
    double v = fabs(W[(int64_t)r * ld + c]);
    if (v > best) best = v, bi = r;
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      double v = sv[threadIdx.x + off];
      int i = si[threadIdx.x + off];
      if (v > sv[threadIdx.x] || (v == sv[threadIdx.x] && i < si[threadIdx.x])) sv[threadIdx.x] = v, si[threadIdx.x] = i;
    }
    __syncthreads();
  }
  const int p = si[0];
  if (!(sv[0] > 0.0)) {
    if (threadIdx.x == 0) set_err(err, AMG_ESINGULAR_BLOCK);
    return;
  }
  if (p != c)
    for (int64_t j = threadIdx.x; j < ld; j += blockDim.x) {
      double t = W[(int64_t)p * ld + j];
      W[(int64_t)p * ld + j] = W[(int64_t)c * ld + j];
      W[(int64_t)c * ld + j] = t;
    }
  __syncthreads();
  const double d = W[(int64_t)c * ld + c];
  __syncthreads();
  for (int64_t j = threadIdx.x; j < ld; j += blockDim.x) W[(int64_t)c * ld + j] = W[(int64_t)c * ld + j] / d;
  __syncthreads();
  for (int r = threadIdx.x; r < N; r += blockDim.x) fcol[r] = (r == c) ? 0.0 : W[(int64_t)r * ld + c];
}

__global__ void k_gj_elim(int N, int c, double* W, const double* fcol) {
  const int64_t ld = 2 * (int64_t)N;
  const int64_t w = ld - c;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)N * w) return;
  const int r = (int)(t / w);
  const int64_t j = c + t % w;
  const double f = fcol[r];
  if (f != 0.0) W[(int64_t)r * ld + j] = W[(int64_t)r * ld + j] - f * W[(int64_t)c * ld + j];
}

template <typename T>
__global__ void k_extract_inv(int N, const double* W, T* inv) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)N * N) return;
  int r = (int)(t / N), c = (int)(t % N);
  inv[t] = (T)W[(int64_t)r * 2 * N + N + c];
}

// ---------------------------------------------------------------- host helpers
template <typename F>
void dispatch_bs(int b, F&& f) {
  switch (b) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    default: fail(AMG_EINVAL, "block size must be 1..4");
  }
}

struct SetupCtx {
  cudaStream_t s;
  Arena tmp;     // freed at the end of setup
  int* err = nullptr;
  int* hcnt = nullptr;  // pinned
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
};

void check_err(SetupCtx& c, const char* where) {
  int e = 0;
  AMG_CK(cudaMemcpyAsync(&e, c.err, sizeof(int), cudaMemcpyDeviceToHost, c.s));
  AMG_CK(cudaStreamSynchronize(c.s));
  if (e != 0) fail(e, where);
}

// Scalar expansion of a BSR matrix (the V2 U-solver, reading R18): block (I, J) entry
// (r, c) -> scalar (b I + r, b J + c); exact zeros inside stored blocks dropped, the
// diagonal kept; rows stay sorted (J ascending, then c).  Thread per scalar row.
__global__ void k_expand_count(int n, int b, const int32_t* ptr, const int32_t* col, const double* val, int32_t* cnt) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= (int64_t)n * b) return;
  const int I = (int)(row / b), r = (int)(row % b);
  int32_t c0 = 0;
  for (int32_t k = ptr[I]; k < ptr[I + 1]; ++k)
    for (int c = 0; c < b; ++c)
      if (val[((int64_t)k * b + r) * b + c] != 0.0 || (int64_t)col[k] * b + c == row) ++c0;
  cnt[row] = c0;
}
__global__ void k_expand_fill(int n, int b, const int32_t* ptr, const int32_t* col, const double* val,
                              const int32_t* sptr, int32_t* scol, double* sval) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= (int64_t)n * b) return;
  const int I = (int)(row / b), r = (int)(row % b);
  int32_t o = sptr[row];
  for (int32_t k = ptr[I]; k < ptr[I + 1]; ++k)
    for (int c = 0; c < b; ++c) {
      const double v = val[((int64_t)k * b + r) * b + c];
      const int64_t j = (int64_t)col[k] * b + c;
      if (v != 0.0 || j == row) {
        scol[o] = (int32_t)j;
        sval[o] = v;
        ++o;
      }
    }
}

// in-place exclusive scan of cnt[0..n] (cnt[n] := 0 first); returns the total
int64_t scan(SetupCtx& c, int32_t* cnt, int n) {
  AMG_CK(cudaMemsetAsync(cnt + n, 0, sizeof(int32_t), c.s));
  size_t need = 0;
  AMG_CK(cub::DeviceScan::ExclusiveSum(nullptr, need, cnt, cnt, n + 1, c.s));
  if (need > c.cub_bytes) {
    c.cub_bytes = need * 2;
    c.cub_tmp = c.tmp.alloc(c.cub_bytes);
  }
  AMG_CK(cub::DeviceScan::ExclusiveSum(c.cub_tmp, need, cnt, cnt, n + 1, c.s));
  int32_t tot = 0;
  AMG_CK(cudaMemcpyAsync(&tot, cnt + n, sizeof(int32_t), cudaMemcpyDeviceToHost, c.s));
  AMG_CK(cudaStreamSynchronize(c.s));
  if (tot < 0) fail(AMG_EINDEX_OVERFLOW, "nnz overflow in setup");
  return tot;
}

// fp64 device matrix in the setup arena
Mat new_mat(Arena& a, int n, int m, int b, int64_t nnz) {
  Mat M;
  M.n = n, M.m = m, M.b = b, M.nnz = nnz, M.vt = AMG_F64;
  M.ptr = a.alloc_n<int32_t>(n + 1);
  M.col = a.alloc_n<int32_t>(std::max<int64_t>(nnz, 1));
  M.val = a.alloc_n<double>(std::max<int64_t>(nnz, 1) * b * b);
  return M;
}

Mat spgemm(SetupCtx& c, const Mat& A, const Mat& B) {
  const int n = A.n;
  int32_t* heads = c.tmp.alloc_n<int32_t>(std::max<int64_t>(A.nnz, 1));
  int32_t* cnt = c.tmp.alloc_n<int32_t>(n + 1);
  k_spgemm_sym<<<grid_for(n, kT), kT, 0, c.s>>>(n, A.ptr, A.col, B.ptr, B.col, heads, nullptr, nullptr, cnt);
  AMG_CK_LAUNCH();
  int64_t nnz = scan(c, cnt, n);
  Mat C;
  C.n = n, C.m = B.m, C.b = A.b, C.nnz = nnz, C.vt = AMG_F64;
  C.ptr = cnt;
  C.col = c.tmp.alloc_n<int32_t>(std::max<int64_t>(nnz, 1));
  C.val = c.tmp.alloc_n<double>(std::max<int64_t>(nnz, 1) * A.b * A.b);
  k_spgemm_sym<<<grid_for(n, kT), kT, 0, c.s>>>(n, A.ptr, A.col, B.ptr, B.col, heads, C.ptr, C.col, nullptr);
  AMG_CK_LAUNCH();
  dispatch_bs(A.b, [&](auto Bc) {
    constexpr int BB = decltype(Bc)::value;
    k_spgemm_num<BB><<<grid_for(n, kT), kT, 0, c.s>>>(n, A.ptr, A.col, (const double*)A.val, B.ptr, B.col,
                                                     (const double*)B.val, C.ptr, C.col, (double*)C.val);
  });
  AMG_CK_LAUNCH();
  return C;
}

Mat transpose(SetupCtx& c, const Mat& P) {
  Mat R;
  R.n = P.m, R.m = P.n, R.b = P.b, R.nnz = P.nnz, R.vt = AMG_F64;
  R.ptr = c.tmp.alloc_n<int32_t>(P.m + 1);
  AMG_CK(cudaMemsetAsync(R.ptr, 0, sizeof(int32_t) * (P.m + 1), c.s));
  if (P.nnz > 0) k_count_cols<<<grid_for(P.nnz, kT), kT, 0, c.s>>>(P.nnz, P.col, R.ptr);
  AMG_CK_LAUNCH();
  scan(c, R.ptr, P.m);
  int32_t* cursor = c.tmp.alloc_n<int32_t>(P.m + 1);
  AMG_CK(cudaMemcpyAsync(cursor, R.ptr, sizeof(int32_t) * (P.m + 1), cudaMemcpyDeviceToDevice, c.s));
  R.col = c.tmp.alloc_n<int32_t>(std::max<int64_t>(P.nnz, 1));
  R.val = c.tmp.alloc_n<double>(std::max<int64_t>(P.nnz, 1) * P.b * P.b);
  dispatch_bs(P.b, [&](auto Bc) {
    constexpr int BB = decltype(Bc)::value;
    k_transpose_fill<BB><<<grid_for(P.n, kT), kT, 0, c.s>>>(P.n, P.ptr, P.col, (const double*)P.val, cursor, R.col,
                                                            (double*)R.val);
    AMG_CK_LAUNCH();
    k_sort_rows_blocks<BB><<<grid_for(R.n, kT), kT, 0, c.s>>>(R.n, R.ptr, R.col, (double*)R.val);
  });
  AMG_CK_LAUNCH();
  return R;
}

// narrowed (or copied) solve copy of an fp64 setup matrix in the handle's arena
Mat solve_copy(Handle& h, const Mat& M64, cudaStream_t s) {
  Mat M = M64;
  M.vt = h.vt;
  M.ptr = h.arena.alloc_n<int32_t>(M64.n + 1);
  M.col = h.arena.alloc_n<int32_t>(std::max<int64_t>(M64.nnz, 1));
  M.val = h.arena.alloc(std::max<int64_t>(M64.nnz, 1) * M64.b * M64.b * dtype_size(h.vt));
  AMG_CK(cudaMemcpyAsync(M.ptr, M64.ptr, sizeof(int32_t) * (M64.n + 1), cudaMemcpyDeviceToDevice, s));
  if (M64.nnz > 0) {
    AMG_CK(cudaMemcpyAsync(M.col, M64.col, sizeof(int32_t) * M64.nnz, cudaMemcpyDeviceToDevice, s));
    launch_convert(M64.nnz * M64.b * M64.b, M64.val, AMG_F64, M.val, h.vt, 1.0, s);
  }
  M.fast32 = (h.vt == AMG_F32 && h.xt == AMG_F32);
  make_tma_plan(M, s, h.want_copies ? &h.arena : nullptr);
  return M;
}

}  // namespace

// Block ILU(0) of A (fp64): level schedule of the lower-triangular dependency graph on the
// host (level(i) = 1 + max level(k), k < i in row i), one launch per level, then the
// strictly lower / upper split.  D^-1 -> Dinv (n b^2).
void ilu0_factor(SetupCtx& c, const Mat& A, double* Dinv, Mat& Lo, Mat& Up) {
  const int n = A.n, b = A.b;
  cudaStream_t s = c.s;
  std::vector<int32_t> hp((size_t)n + 1), hc((size_t)std::max<int64_t>(A.nnz, 1));
  AMG_CK(cudaMemcpyAsync(hp.data(), A.ptr, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, s));
  if (A.nnz > 0) AMG_CK(cudaMemcpyAsync(hc.data(), A.col, sizeof(int32_t) * A.nnz, cudaMemcpyDeviceToHost, s));
  AMG_CK(cudaStreamSynchronize(s));
  std::vector<int32_t> lev(n, 0);
  int nlev = n > 0 ? 1 : 0;
  for (int i = 0; i < n; ++i) {
    int l = 0;
    for (int k = hp[i]; k < hp[i + 1]; ++k)
      if (hc[k] < i) l = std::max(l, lev[hc[k]] + 1);
    lev[i] = l;
    nlev = std::max(nlev, l + 1);
  }
  std::vector<int32_t> off(nlev + 1, 0), order(n);
  for (int i = 0; i < n; ++i) ++off[lev[i] + 1];
  for (int l = 0; l < nlev; ++l) off[l + 1] += off[l];
  std::vector<int32_t> cur(off.begin(), off.end() - 1);
  for (int i = 0; i < n; ++i) order[cur[lev[i]]++] = i;
  int32_t* dorder = c.tmp.alloc_n<int32_t>(std::max(n, 1));
  AMG_CK(cudaMemcpyAsync(dorder, order.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
  double* a = c.tmp.alloc_n<double>(std::max<int64_t>(A.nnz, 1) * b * b);
  AMG_CK(cudaMemcpyAsync(a, A.val, sizeof(double) * A.nnz * b * b, cudaMemcpyDeviceToDevice, s));
  dispatch_bs(b, [&](auto Bc) {
    constexpr int BB = decltype(Bc)::value;
    for (int l = 0; l < nlev; ++l) {
      const int cnt = off[l + 1] - off[l];
      k_ilu_rows<BB><<<grid_for(cnt, kT), kT, 0, s>>>(cnt, dorder + off[l], A.ptr, A.col, a, Dinv, c.err);
    }
    AMG_CK_LAUNCH();
  });
  check_err(c, "ILU(0) factorisation");
  int32_t* lc = c.tmp.alloc_n<int32_t>(n + 1);
  int32_t* uc = c.tmp.alloc_n<int32_t>(n + 1);
  k_tri_count<<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, A.col, lc, uc);
  AMG_CK_LAUNCH();
  const int64_t ln = scan(c, lc, n), un = scan(c, uc, n);
  Lo = new_mat(c.tmp, n, A.m, b, ln);
  Up = new_mat(c.tmp, n, A.m, b, un);
  AMG_CK(cudaMemcpyAsync(Lo.ptr, lc, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
  AMG_CK(cudaMemcpyAsync(Up.ptr, uc, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
  dispatch_bs(b, [&](auto Bc) {
    constexpr int BB = decltype(Bc)::value;
    k_tri_fill<BB><<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, A.col, a, Lo.ptr, Lo.col, (double*)Lo.val, Up.ptr,
                                                   Up.col, (double*)Up.val);
  });
  AMG_CK_LAUNCH();
  AMG_CK(cudaStreamSynchronize(s));
}

// A without the blocks that couple different slabs (part: slab of every block row)
__global__ void k_slab_count(int n, const int32_t* ptr, const int32_t* col, const int32_t* part, int32_t* cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = 0;
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) c += part[col[k]] == part[i];
  cnt[i] = c;
}
__global__ void k_slab_fill(int n, const int32_t* ptr, const int32_t* col, const double* val, const int32_t* part,
                            int bb, const int32_t* optr, int32_t* ocol, double* oval) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int o = optr[i];
  for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
    if (part[col[k]] != part[i]) continue;
    ocol[o] = col[k];
    for (int e = 0; e < bb; ++e) oval[(int64_t)o * bb + e] = val[(int64_t)k * bb + e];
    ++o;
  }
}
Mat slab_diagonal_blocks(SetupCtx& c, const Mat& A, const int32_t* part) {
  const int n = A.n;
  int32_t* cnt = c.tmp.alloc_n<int32_t>(n + 1);
  k_slab_count<<<grid_for(n, kT), kT, 0, c.s>>>(n, A.ptr, A.col, part, cnt);
  AMG_CK_LAUNCH();
  const int64_t nnz = scan(c, cnt, n);
  Mat F = new_mat(c.tmp, n, A.m, A.b, nnz);
  AMG_CK(cudaMemcpyAsync(F.ptr, cnt, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToDevice, c.s));
  k_slab_fill<<<grid_for(n, kT), kT, 0, c.s>>>(n, A.ptr, A.col, (const double*)A.val, part, A.b * A.b, F.ptr, F.col,
                                                (double*)F.val);
  AMG_CK_LAUNCH();
  return F;
}

// Block ILUT(tau, p) of A (fp64, reading R25): k_ilut_rows into per-row slabs, then
// compacted into L_s / U_s.  D^-1 -> Dinv (n b^2).
void ilut_factor(SetupCtx& c, const Mat& A, double tau, int pfill, double* Dinv, Mat& Lo, Mat& Up) {
  const int n = A.n, b = A.b;
  cudaStream_t s = c.s;
  int32_t* loff = c.tmp.alloc_n<int32_t>(n + 1);
  int32_t* uoff = c.tmp.alloc_n<int32_t>(n + 1);
  k_tri_count<<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, A.col, loff, uoff);
  AMG_CK_LAUNCH();
  k_add_scalar<<<grid_for(n, kT), kT, 0, s>>>(n, loff, pfill);
  k_add_scalar<<<grid_for(n, kT), kT, 0, s>>>(n, uoff, pfill);
  AMG_CK_LAUNCH();
  const int64_t lcap = scan(c, loff, n), ucap = scan(c, uoff, n);
  int32_t* scl = c.tmp.alloc_n<int32_t>(std::max<int64_t>(lcap, 1));
  int32_t* scu = c.tmp.alloc_n<int32_t>(std::max<int64_t>(ucap, 1));
  double* svl = c.tmp.alloc_n<double>(std::max<int64_t>(lcap, 1) * b * b);
  double* svu = c.tmp.alloc_n<double>(std::max<int64_t>(ucap, 1) * b * b);
  int32_t* llen = c.tmp.alloc_n<int32_t>(n + 1);
  int32_t* ulen = c.tmp.alloc_n<int32_t>(n + 1);
  int* flags = c.tmp.alloc_n<int>(n + 1);  // [n] done flags, [n] the row counter
  AMG_CK(cudaMemsetAsync(flags, 0, sizeof(int) * (n + 1), s));
  dispatch_bs(b, [&](auto Bc) {
    constexpr int BB = decltype(Bc)::value;
    using Sh = IlutShape<BB>;
    AMG_CK(cudaFuncSetAttribute(k_ilut_rows<BB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::smem));
    int per_sm = 0;
    AMG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ilut_rows<BB>, 32 * Sh::W, Sh::smem));
    const int grid = std::max(1, std::min(kSMs * std::max(per_sm, 1), (n + Sh::W - 1) / Sh::W));  // all resident
    k_ilut_rows<BB><<<grid, 32 * Sh::W, Sh::smem, s>>>(n, A.ptr, A.col, (const double*)A.val, tau, pfill, loff, uoff,
                                                       scl, svl, llen, scu, svu, ulen, Dinv, flags, flags + n, c.err);
  });
  AMG_CK_LAUNCH();
  check_err(c, "ILUT factorisation");
  int32_t* lc = c.tmp.alloc_n<int32_t>(n + 1);
  int32_t* uc = c.tmp.alloc_n<int32_t>(n + 1);
  AMG_CK(cudaMemcpyAsync(lc, llen, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
  AMG_CK(cudaMemcpyAsync(uc, ulen, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
  const int64_t ln = scan(c, lc, n), un = scan(c, uc, n);
  Lo = new_mat(c.tmp, n, A.m, b, ln);
  Up = new_mat(c.tmp, n, A.m, b, un);
  AMG_CK(cudaMemcpyAsync(Lo.ptr, lc, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
  AMG_CK(cudaMemcpyAsync(Up.ptr, uc, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
  k_ilut_compact<<<grid_for(n, kT), kT, 0, s>>>(n, loff, llen, scl, svl, Lo.ptr, Lo.col, (double*)Lo.val, b * b);
  k_ilut_compact<<<grid_for(n, kT), kT, 0, s>>>(n, uoff, ulen, scu, svu, Up.ptr, Up.col, (double*)Up.val, b * b);
  AMG_CK_LAUNCH();
  AMG_CK(cudaStreamSynchronize(s));
}

// ---------------------------------------------------------------- the setup driver
void setup_build(Handle& h, const Mat& A64, const std::vector<int64_t>& bounds0, cudaStream_t s) {
  SetupCtx c;
  c.s = s;
  c.err = c.tmp.alloc_n<int>(1);
  AMG_CK(cudaMemsetAsync(c.err, 0, sizeof(int), s));
  const amg_params& p = h.p;
  const int b = A64.b;

  // diagonal positions of the outer operator (needed by Schur and AMG alike)
  int32_t* diag0 = c.tmp.alloc_n<int32_t>(std::max(A64.n, 1));
  if (A64.n > 0) k_find_diag<<<grid_for(A64.n, kT), kT, 0, s>>>(A64.n, A64.ptr, A64.col, diag0, c.err);
  AMG_CK_LAUNCH();
  check_err(c, "diagonal");

  Mat Amg = A64;  // matrix the AMG hierarchy is built on
  if (h.schur && h.pmask_in) {  // general scalar pressure mask (R21)
    h.masked = true;
    const int64_t N = (int64_t)A64.n * b;
    if (N >= INT32_MAX) fail(AMG_EINDEX_OVERFLOW, "scalar expansion of A");
    int32_t* sp = c.tmp.alloc_n<int32_t>(N + 1);
    k_expand_count<<<grid_for(N, kT), kT, 0, s>>>(A64.n, b, A64.ptr, A64.col, (const double*)A64.val, sp);
    AMG_CK_LAUNCH();
    const int64_t snnz = scan(c, sp, (int)N);
    int32_t* sc = c.tmp.alloc_n<int32_t>(std::max<int64_t>(snnz, 1));
    double* sv = c.tmp.alloc_n<double>(std::max<int64_t>(snnz, 1));
    k_expand_fill<<<grid_for(N, kT), kT, 0, s>>>(A64.n, b, A64.ptr, A64.col, (const double*)A64.val, sp, sc, sv);
    int32_t* iu = c.tmp.alloc_n<int32_t>(N + 1);
    int32_t* ip = c.tmp.alloc_n<int32_t>(N + 1);
    k_mask_flags<<<grid_for(N, kT), kT, 0, s>>>(N, h.pmask_in, iu, ip);
    AMG_CK_LAUNCH();
    const int64_t nu = scan(c, iu, (int)N), np = scan(c, ip, (int)N);
    if (nu == 0 || np == 0) fail(AMG_EINVAL, "pressure mask selects no velocity or no pressure unknown");
    {  // each class's range per slab of block rows (several slabs: R27)
      h.ubounds.assign(bounds0.size(), 0);
      h.pbounds.assign(bounds0.size(), 0);
      for (size_t r = 0; r < bounds0.size(); ++r) {
        int32_t v[2];
        AMG_CK(cudaMemcpy(&v[0], iu + bounds0[r] * b, 4, cudaMemcpyDeviceToHost));
        AMG_CK(cudaMemcpy(&v[1], ip + bounds0[r] * b, 4, cudaMemcpyDeviceToHost));
        h.ubounds[r] = v[0];
        h.pbounds[r] = v[1];
      }
    }
    h.nu_s = (int32_t)nu;
    h.np_s = (int32_t)np;
    h.uidx = h.arena.alloc_n<int32_t>(nu);
    h.pidx = h.arena.alloc_n<int32_t>(np);
    k_mask_index<<<grid_for(N, kT), kT, 0, s>>>(N, h.pmask_in, iu, ip, h.uidx, h.pidx);
    int32_t* cA = c.tmp.alloc_n<int32_t>(nu + 1);
    int32_t* cBT = c.tmp.alloc_n<int32_t>(nu + 1);
    int32_t* cB = c.tmp.alloc_n<int32_t>(np + 1);
    int32_t* cC = c.tmp.alloc_n<int32_t>(np + 1);
    k_mask_count<<<grid_for(N, kT), kT, 0, s>>>(N, sp, sc, h.pmask_in, iu, ip, cA, cBT, cB, cC);
    AMG_CK_LAUNCH();
    const int64_t zA = scan(c, cA, (int)nu), zBT = scan(c, cBT, (int)nu), zB = scan(c, cB, (int)np),
                  zC = scan(c, cC, (int)np);
    auto mk = [&](int32_t* ptr, int n, int m, int64_t nnz) {
      Mat M;
      M.n = n, M.m = m, M.b = 1, M.nnz = nnz, M.vt = AMG_F64, M.ptr = ptr;
      M.col = c.tmp.alloc_n<int32_t>(std::max<int64_t>(nnz, 1));
      M.val = c.tmp.alloc_n<double>(std::max<int64_t>(nnz, 1));
      return M;
    };
    Mat Au = mk(cA, (int)nu, (int)nu, zA), BT = mk(cBT, (int)nu, (int)np, zBT), Bq = mk(cB, (int)np, (int)nu, zB),
        Cq = mk(cC, (int)np, (int)np, zC);
    k_mask_fill<<<grid_for(N, kT), kT, 0, s>>>(N, sp, sc, sv, h.pmask_in, iu, ip, Au.ptr, Au.col, (double*)Au.val,
                                                BT.ptr, BT.col, (double*)BT.val, Bq.ptr, Bq.col, (double*)Bq.val,
                                                Cq.ptr, Cq.col, (double*)Cq.val);
    AMG_CK_LAUNCH();
    h.shat64 = h.arena.alloc_n<double>(np);
    h.mS64 = h.arena.alloc_n<double>(np);
    k_schur_shat_scalar<<<grid_for(np, kT), kT, 0, s>>>(
        (int)np, p.schur_shat, Bq.ptr, Bq.col, (const double*)Bq.val, Au.ptr, Au.col, (const double*)Au.val, BT.ptr,
        BT.col, (const double*)BT.val, Cq.ptr, Cq.col, (const double*)Cq.val, h.shat64, h.mS64, c.err);
    AMG_CK_LAUNCH();
    check_err(c, "Schur complement approximation (pressure mask)");
    h.mS = h.arena.alloc(np * dtype_size(h.vt));
    launch_convert(np, h.mS64, AMG_F64, h.mS, h.vt, 1.0, s);
    h.Bm = solve_copy(h, Bq, s);
    h.BTm = solve_copy(h, BT, s);
    h.Bm.fast32 = h.BTm.fast32 = false;  // fp64 accumulation of every product (as the block Schur views)
    Amg = Au;
  } else if (h.schur) {
    if (b != 4) fail(AMG_EINVAL, "Schur pressure correction needs 4x4 blocks (u,v,w,p)");
    const int nu = b - 1;
    h.nu = nu;
    Mat Au = A64;
    Au.b = nu;
    Au.val = c.tmp.alloc_n<double>(std::max<int64_t>(A64.nnz, 1) * nu * nu);
    double* bv = c.tmp.alloc_n<double>(std::max<int64_t>(A64.nnz, 1) * nu);
    double* btv = c.tmp.alloc_n<double>(std::max<int64_t>(A64.nnz, 1) * nu);
    double* cv = c.tmp.alloc_n<double>(std::max<int64_t>(A64.nnz, 1));
    if (A64.nnz > 0)
      k_schur_split<<<grid_for(A64.nnz, kT), kT, 0, s>>>(A64.nnz, b, h.pc, (const double*)A64.val, (double*)Au.val,
                                                         bv, btv, cv);
    AMG_CK_LAUNCH();
    h.shat64 = h.arena.alloc_n<double>(std::max(A64.n, 1));
    h.mS64 = h.arena.alloc_n<double>(std::max(A64.n, 1));
    if (A64.n > 0 && p.schur_shat == 2) {
      int32_t* heads = c.tmp.alloc_n<int32_t>(std::max<int64_t>(A64.nnz, 1));
      int32_t* sptr = c.tmp.alloc_n<int32_t>(A64.n + 1);
      k_spgemm_sym<<<grid_for(A64.n, kT), kT, 0, s>>>(A64.n, A64.ptr, A64.col, A64.ptr, A64.col, heads, nullptr,
                                                       nullptr, sptr);
      AMG_CK_LAUNCH();
      const int64_t snnz = scan(c, sptr, A64.n);
      int32_t* scol = c.tmp.alloc_n<int32_t>(std::max<int64_t>(snnz, 1));
      double* ssum = c.tmp.alloc_n<double>(std::max<int64_t>(snnz, 1));
      k_spgemm_sym<<<grid_for(A64.n, kT), kT, 0, s>>>(A64.n, A64.ptr, A64.col, A64.ptr, A64.col, heads, sptr, scol,
                                                       nullptr);
      k_schur_shat_full<<<grid_for(A64.n, kT), kT, 0, s>>>(A64.n, nu, A64.ptr, A64.col, diag0, (const double*)Au.val,
                                                            bv, btv, cv, sptr, scol, ssum, h.shat64, h.mS64, c.err);
    } else if (A64.n > 0) {
      k_schur_shat<<<grid_for(A64.n, kT), kT, 0, s>>>(A64.n, nu, p.schur_shat, A64.ptr, A64.col, diag0,
                                                      (const double*)Au.val, bv, btv, cv, h.shat64, h.mS64, c.err);
    }
    AMG_CK_LAUNCH();
    check_err(c, "Schur complement approximation");
    h.Bv = h.arena.alloc(std::max<int64_t>(A64.nnz, 1) * nu * dtype_size(h.vt));
    h.BTv = h.arena.alloc(std::max<int64_t>(A64.nnz, 1) * nu * dtype_size(h.vt));
    h.mS = h.arena.alloc(std::max(A64.n, 1) * dtype_size(h.vt));
    launch_convert(A64.nnz * nu, bv, AMG_F64, h.Bv, h.vt, 1.0, s);
    launch_convert(A64.nnz * nu, btv, AMG_F64, h.BTv, h.vt, 1.0, s);
    launch_convert(A64.n, h.mS64, AMG_F64, h.mS, h.vt, 1.0, s);
    Amg = Au;
    if (p.schur_u_scalar) {  // V2: the U-solver hierarchy on the scalar expansion of A_u
      const int64_t ns = (int64_t)Au.n * nu;
      if (ns >= INT32_MAX) fail(AMG_EINDEX_OVERFLOW, "scalar expansion of A_u");
      int32_t* sptr = c.tmp.alloc_n<int32_t>(ns + 1);
      if (ns > 0)
        k_expand_count<<<grid_for(ns, kT), kT, 0, s>>>(Au.n, nu, Au.ptr, Au.col, (const double*)Au.val, sptr);
      AMG_CK_LAUNCH();
      const int64_t snnz = scan(c, sptr, (int)ns);
      Mat As;
      As.n = (int32_t)ns, As.m = (int32_t)((int64_t)Au.m * nu), As.b = 1, As.nnz = snnz, As.vt = AMG_F64;
      As.ptr = sptr;
      As.col = c.tmp.alloc_n<int32_t>(std::max<int64_t>(snnz, 1));
      As.val = c.tmp.alloc_n<double>(std::max<int64_t>(snnz, 1));
      if (ns > 0)
        k_expand_fill<<<grid_for(ns, kT), kT, 0, s>>>(Au.n, nu, Au.ptr, Au.col, (const double*)Au.val, As.ptr,
                                                       As.col, (double*)As.val);
      AMG_CK_LAUNCH();
      Amg = As;
    }
  }
  h.bh = Amg.b;

  // slab of every row (rank-local aggregation); a scalar U-solver
  // hierarchy has nu scalar rows per block row
  std::vector<int64_t> bounds = bounds0;
  if (h.schur && p.schur_u_scalar && !h.masked)
    for (int64_t& v : bounds) v *= h.nu;
  if (h.masked) bounds = h.ubounds.size() > 2 ? h.ubounds : std::vector<int64_t>{0, (int64_t)h.nu_s};
  const int nparts = (int)bounds.size() - 1;
  h.lbounds.clear();
  h.lbounds.push_back(bounds);

  Mat A = Amg;
  std::vector<Mat> lvA, lvP, lvR, lvL, lvU;
  std::vector<double*> lvM;
  std::vector<int32_t*> lvAgg;
  std::vector<int32_t> lvNc;
  while ((int64_t)A.n * A.b > p.coarse_enough && (int)lvA.size() < p.max_levels - 1) {
    const int n = A.n;
    const int64_t nnz = A.nnz;
    int32_t* diag = c.tmp.alloc_n<int32_t>(n);
    k_find_diag<<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, A.col, diag, c.err);
    AMG_CK_LAUNCH();
    check_err(c, "diagonal");
    double* dn = c.tmp.alloc_n<double>(n);
    uint8_t* st = c.tmp.alloc_n<uint8_t>(std::max<int64_t>(nnz, 1));
    uint8_t* sym = c.tmp.alloc_n<uint8_t>(std::max<int64_t>(nnz, 1));
    int32_t* tpos = c.tmp.alloc_n<int32_t>(std::max<int64_t>(nnz, 1));
    int32_t* extra = c.tmp.alloc_n<int32_t>(n + 1);
    int32_t* part = nullptr;
    if (nparts > 1) {
      std::vector<int32_t> hp(n);
      for (int r = 0; r < nparts; ++r)
        for (int64_t i = bounds[r]; i < bounds[r + 1]; ++i) hp[i] = r;
      part = c.tmp.alloc_n<int32_t>(n);
      AMG_CK(cudaMemcpyAsync(part, hp.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
      AMG_CK(cudaStreamSynchronize(s));
    }
    AMG_CK(cudaMemsetAsync(extra, 0, sizeof(int32_t) * (n + 1), s));
    double* D = c.tmp.alloc_n<double>((int64_t)n * A.b * A.b);
    double* Dinv = c.tmp.alloc_n<double>((int64_t)n * A.b * A.b);
    double* M = c.tmp.alloc_n<double>((int64_t)n * A.b * A.b);
    dispatch_bs(A.b, [&](auto Bc) {
      constexpr int BB = decltype(Bc)::value;
      k_diag_norm<BB><<<grid_for(n, kT), kT, 0, s>>>(n, (const double*)A.val, diag, dn);
      k_strength<BB><<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, A.col, (const double*)A.val, dn,
                                                     p.eps_strong * p.eps_strong, part, st);
    });
    AMG_CK_LAUNCH();
    k_tpos<<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, A.col, tpos);
    k_sym<<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, A.col, st, tpos, sym, extra);
    AMG_CK_LAUNCH();
    // adjacency (strength graph after closure)
    int32_t* aptr = c.tmp.alloc_n<int32_t>(n + 1);
    k_adj_count<<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, sym, extra, aptr);
    AMG_CK_LAUNCH();
    int64_t nadj = scan(c, aptr, n);
    int32_t* adj = c.tmp.alloc_n<int32_t>(std::max<int64_t>(nadj, 1));
    int32_t* cursor = c.tmp.alloc_n<int32_t>(n + 1);
    k_adj_fill<<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, A.col, sym, aptr, adj, cursor);
    k_adj_extras<<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, A.col, st, tpos, adj, cursor);
    k_sort_segments<<<grid_for(n, kT), kT, 0, s>>>(n, aptr, adj);
    AMG_CK_LAUNCH();

    // MIS-2 rounds
    uint8_t* state = c.tmp.alloc_n<uint8_t>(n);
    int32_t* m1 = c.tmp.alloc_n<int32_t>(n);
    uint8_t* r1 = c.tmp.alloc_n<uint8_t>(n);
    int* und = c.tmp.alloc_n<int>(1);
    k_mis_init<<<grid_for(n, kT), kT, 0, s>>>(n, aptr, state);
    AMG_CK_LAUNCH();
    for (int round = 0;; ++round) {
      AMG_CK(cudaMemsetAsync(und, 0, sizeof(int), s));
      k_mis_1<<<grid_for(n, kT), kT, 0, s>>>(n, aptr, adj, state, m1, r1);
      k_mis_2<<<grid_for(n, kT), kT, 0, s>>>(n, aptr, adj, state, m1, r1, und);
      AMG_CK_LAUNCH();
      if (round % 4 == 3 || round > 4 * n) {
        int hu = 0;
        AMG_CK(cudaMemcpyAsync(&hu, und, sizeof(int), cudaMemcpyDeviceToHost, s));
        AMG_CK(cudaStreamSynchronize(s));
        if (hu == 0) break;
        if (round > 4 * n) fail(AMG_EINVAL, "aggregation did not terminate");
      }
    }
    int32_t* rid = c.tmp.alloc_n<int32_t>(n + 1);
    k_is_root<<<grid_for(n, kT), kT, 0, s>>>(n, state, rid);
    AMG_CK_LAUNCH();
    const int64_t nc = scan(c, rid, n);
    // coarse slab bounds = number of roots before each slab boundary
    std::vector<int64_t> cb(nparts + 1, 0);
    if (nparts > 1) {
      std::vector<int32_t> hr(n + 1);
      AMG_CK(cudaMemcpyAsync(hr.data(), rid, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost, s));
      AMG_CK(cudaStreamSynchronize(s));
      for (int r = 0; r <= nparts; ++r) cb[r] = hr[bounds[r]];
    } else {
      cb[1] = nc;
    }
    if (nc == 0 || nc >= n) break;
    bounds = cb;
    h.lbounds.push_back(bounds);
    int32_t* agg1 = c.tmp.alloc_n<int32_t>(n);
    int32_t* agg = c.tmp.alloc_n<int32_t>(n);
    k_pass1<<<grid_for(n, kT), kT, 0, s>>>(n, aptr, adj, state, rid, agg1);
    k_pass2<<<grid_for(n, kT), kT, 0, s>>>(n, aptr, adj, agg1, agg);
    AMG_CK_LAUNCH();

    // smoothed prolongator (plain aggregation: the tentative one)
    const bool plain = p.coarsening == AMG_PLAIN_AGG;
    int32_t* cand = c.tmp.alloc_n<int32_t>(std::max<int64_t>(nnz, 1));
    int32_t* pcnt = c.tmp.alloc_n<int32_t>(n + 1);
    if (plain) k_ptent_count<<<grid_for(n, kT), kT, 0, s>>>(n, agg, pcnt);
    else k_p_cand<<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, A.col, diag, sym, agg, cand, pcnt);
    AMG_CK_LAUNCH();
    const int64_t pnnz = scan(c, pcnt, n);
    Mat P;
    P.n = n, P.m = (int32_t)nc, P.b = A.b, P.nnz = pnnz, P.vt = AMG_F64;
    P.ptr = pcnt;
    P.col = c.tmp.alloc_n<int32_t>(std::max<int64_t>(pnnz, 1));
    P.val = c.tmp.alloc_n<double>(std::max<int64_t>(pnnz, 1) * A.b * A.b);
    dispatch_bs(A.b, [&](auto Bc) {
      constexpr int BB = decltype(Bc)::value;
      if (plain) {
        k_ptent_fill<BB><<<grid_for(n, kT), kT, 0, s>>>(n, agg, P.ptr, P.col, (double*)P.val);
      } else {
        k_filtered_diag<BB><<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, A.col, (const double*)A.val, diag, sym, D,
                                                           Dinv, c.err);
        AMG_CK_LAUNCH();
        k_p_fill<BB><<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, A.col, (const double*)A.val, diag, sym, agg, D, Dinv,
                                                    cand, P.ptr, P.col, (double*)P.val, p.sa_omega);
      }
      AMG_CK_LAUNCH();
      if (p.smoother != AMG_ILU0 && p.smoother != AMG_ILUT)
        k_smoother<BB><<<grid_for(n, kT), kT, 0, s>>>(n, A.ptr, (const double*)A.val, diag,
                                                      p.smoother == AMG_SPAI0, p.jacobi_omega, M, c.err);
      AMG_CK_LAUNCH();
    });
    check_err(c, "prolongator / smoother");
    Mat Lo, Up;
    if (p.smoother == AMG_ILU0 || p.smoother == AMG_ILUT) {  // M <- D^-1
      // several slabs (reading R26): each slab's factors are those of its diagonal block
      const Mat F = part ? slab_diagonal_blocks(c, A, part) : A;
      if (p.smoother == AMG_ILU0) ilu0_factor(c, F, M, Lo, Up);
      else ilut_factor(c, F, p.ilut_tau, p.ilut_p, M, Lo, Up);
    }
    lvL.push_back(Lo);
    lvU.push_back(Up);
    Mat R = transpose(c, P);
    Mat AP = spgemm(c, A, P);
    Mat Ac = spgemm(c, R, AP);
    Ac.m = Ac.n;
    if (plain && p.over_interp != 1.0 && Ac.nnz > 0) {
      const int64_t m = Ac.nnz * Ac.b * Ac.b;
      k_scale_vals<<<grid_for(m, kT), kT, 0, s>>>(m, 1.0 / p.over_interp, (double*)Ac.val);
      AMG_CK_LAUNCH();
    }
    lvA.push_back(A);
    lvP.push_back(P);
    lvR.push_back(R);
    lvM.push_back(M);
    lvAgg.push_back(agg);
    lvNc.push_back((int32_t)nc);
    A = Ac;
  }

  // coarsest level: Gauss-Jordan explicit inverse (fp64), stored at hierarchy precision
  const int64_t N = (int64_t)A.n * A.b;
  if (N > 8192) fail(AMG_EINVAL, "coarsening stalled: coarsest level too large for a dense inverse");
  h.coarse.N = (int32_t)N;
  h.coarse.n = A.n;
  h.coarse.b = A.b;
  if (N > 0) {
    double* W = c.tmp.alloc_n<double>(N * 2 * N);
    double* fcol = c.tmp.alloc_n<double>(N);
    AMG_CK(cudaMemsetAsync(W, 0, sizeof(double) * N * 2 * N, s));
    dispatch_bs(A.b, [&](auto Bc) {
      constexpr int BB = decltype(Bc)::value;
      k_densify<BB><<<grid_for(A.n, kT), kT, 0, s>>>(A.n, A.ptr, A.col, (const double*)A.val, W, (int)N);
    });
    AMG_CK_LAUNCH();
    for (int col = 0; col < N; ++col) {
      k_gj_pivot<<<1, 1024, 0, s>>>((int)N, col, W, fcol, c.err);
      const int64_t work = N * (2 * N - col);
      k_gj_elim<<<grid_for(work, kT), kT, 0, s>>>((int)N, col, W, fcol);
    }
    AMG_CK_LAUNCH();
    check_err(c, "coarse inverse");
    h.coarse.inv = h.arena.alloc(N * N * dtype_size(h.vt));
    if (h.vt == AMG_F32)
      k_extract_inv<float><<<grid_for(N * N, kT), kT, 0, s>>>((int)N, W, (float*)h.coarse.inv);
    else
      k_extract_inv<double><<<grid_for(N * N, kT), kT, 0, s>>>((int)N, W, (double*)h.coarse.inv);
    AMG_CK_LAUNCH();
  }
  h.coarse.A = solve_copy(h, A, s);
  const size_t xs = dtype_size(h.xt);
  h.coarse.f = h.arena.alloc(std::max<int64_t>(N, 1) * xs);
  h.coarse.x = h.arena.alloc(std::max<int64_t>(N, 1) * xs);

  // solve copies of the levels (narrowed RNE when hier = F32), work vectors
  h.lv.resize(lvA.size());
  for (size_t l = 0; l < lvA.size(); ++l) {
    Level& L = h.lv[l];
    L.A = solve_copy(h, lvA[l], s);
    L.P = solve_copy(h, lvP[l], s);
    L.R = solve_copy(h, lvR[l], s);
    if (lvL[l].ptr) {  // AMG_ILU0: the factors and the sweep vectors
      L.Lf = solve_copy(h, lvL[l], s);
      L.Uf = solve_copy(h, lvU[l], s);
      const int64_t nbw = std::max<int64_t>((int64_t)lvA[l].n * lvA[l].b, 1);
      for (void*& w : L.w) w = h.arena.alloc(nbw * dtype_size(h.xt));
    }
    const int64_t nb = (int64_t)lvA[l].n * lvA[l].b;
    L.M = h.arena.alloc(std::max<int64_t>(nb * lvA[l].b, 1) * dtype_size(h.vt));
    launch_convert(nb * lvA[l].b, lvM[l], AMG_F64, L.M, h.vt, 1.0, s);
    L.agg = h.arena.alloc_n<int32_t>(std::max(lvA[l].n, 1));
    AMG_CK(cudaMemcpyAsync(L.agg, lvAgg[l], sizeof(int32_t) * lvA[l].n, cudaMemcpyDeviceToDevice, s));
    L.nc = lvNc[l];
    L.f = h.arena.alloc(std::max<int64_t>(nb, 1) * xs);
    L.x = h.arena.alloc(std::max<int64_t>(nb, 1) * xs);
    L.r = h.arena.alloc(std::max<int64_t>(nb, 1) * xs);
    L.t = h.arena.alloc(std::max<int64_t>(nb, 1) * xs);
  }
  AMG_CK(cudaStreamSynchronize(s));
}

}  // namespace amgb
