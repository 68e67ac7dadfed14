// oracle.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// Plain single-threaded fp64 CPU oracle of the solve phase of the paper's
// AMG-preconditioned Krylov solver for Stokes systems (arXiv 2006.06052).
// Every function cites the PAPER.md passage it follows, or the SURVEY.md §8(c)
// reading (C0..C12) taken where the paper is silent.  No blocking, fusion or
// reordering beyond what the cited definition states.  Built with
// -O2 -ffp-contract=off: every product and sum is rounded separately, in the
// order written.  Shares no code with the CUDA library.
//
// Parity-unpinned pieces (pinned only by invariants / small dense solves, see
// DESIGN.md): absolute iteration counts, level sizes of the large configs.

#include "oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <vector>

using std::vector;

struct orc_mat {
  int32_t n = 0, m = 0, b = 1;   // block rows, block cols, block size
  vector<int32_t> ptr, col;      // C0: CSR over blocks, sorted unique columns
  vector<double> val;            // nnz * b * b, row-major blocks
  int64_t nnz() const { return (int64_t)col.size(); }
  const double* blk(int64_t k) const { return val.data() + k * b * b; }
  double* blk(int64_t k) { return val.data() + k * b * b; }
};

static inline double f32r(double v) { return (double)(float)v; }  // RNE narrowing (C9)

// Timing instrumentation only (bench.py's reference arm): when orc_solve_timed is running,
// g_stamps[it] = seconds since the solve started, recorded as iteration `it` completes.
static thread_local double* g_stamps = nullptr;
static thread_local int32_t g_stamps_cap = 0;
static thread_local std::chrono::steady_clock::time_point g_t0;
static inline void stamp(int it) {
  if (g_stamps && it >= 0 && it < g_stamps_cap)
    g_stamps[it] = std::chrono::duration<double>(std::chrono::steady_clock::now() - g_t0).count();
}

extern "C" void orc_params_default(orc_params* p) {
  p->solver = ORC_GMRES;
  p->gmres_m = 30;
  p->precond = ORC_PC_AMG;
  p->maxiter = 1000;
  p->hier_f32 = 1;
  p->vec_f32 = 1;
  p->smoother = ORC_SPAI0;
  p->jacobi_omega = 2.0 / 3.0;
  p->sa_omega = 2.0 / 3.0;
  p->eps_strong = 1e-3;
  p->coarse_enough = 3000;
  p->max_levels = 20;
  p->npre = 1;
  p->npost = 1;
  p->schur_p_component = 3;
  p->nparts = 1;
  p->idrs_s = 5;
  p->idrs_seed = 1234;
  p->schur_u_scalar = 0;
  p->coarsening = ORC_SA;
  p->schur_shat = 1;
  p->over_interp = 1.5;
  p->ilu_sweeps = 2;
  p->ilut_tau = 1e-2;  // SPEC.md:443 (the paper gives none)
  p->ilut_p = 2;
  p->gmres_ortho = 0;  // CGS2; 1 = the two-pass Gram/Cholesky variant (R22)
}

// ---------------------------------------------------------------- C0 containers
extern "C" orc_mat* orc_mat_new(int32_t n_rows, int32_t n_cols, int32_t b, const int32_t* ptr,
                                const int32_t* col, const double* val) {
  if (n_rows < 0 || n_cols < 0 || b < 1 || b > 8) return nullptr;
  orc_mat* A = new orc_mat;
  A->n = n_rows;
  A->m = n_cols;
  A->b = b;
  A->ptr.assign(ptr, ptr + n_rows + 1);
  int64_t nnz = A->ptr[n_rows];
  A->col.assign(col, col + nnz);
  A->val.assign(val, val + nnz * b * b);
  return A;
}

extern "C" void orc_mat_free(orc_mat* A) { delete A; }

extern "C" void orc_mat_info(const orc_mat* A, int64_t* out) {
  out[0] = A->n;
  out[1] = A->m;
  out[2] = A->b;
  out[3] = A->nnz();
}

extern "C" void orc_mat_export(const orc_mat* A, int32_t* ptr, int32_t* col, double* val) {
  std::copy(A->ptr.begin(), A->ptr.end(), ptr);
  std::copy(A->col.begin(), A->col.end(), col);
  std::copy(A->val.begin(), A->val.end(), val);
}

// S1, PAPER.md:658-672 (§4 worked example): one block per non-empty b x b tile,
// absent scalars inside a stored tile are explicit zeros.
extern "C" orc_mat* orc_csr_to_bsr(int32_t n, int32_t m, int32_t b, const int32_t* ptr,
                                   const int32_t* col, const double* val) {
  if (b < 1 || n % b != 0 || m % b != 0) return nullptr;
  orc_mat* A = new orc_mat;
  A->n = n / b;
  A->m = m / b;
  A->b = b;
  A->ptr.assign(A->n + 1, 0);
  for (int32_t I = 0; I < A->n; ++I) {
    vector<int32_t> cols;
    for (int r = 0; r < b; ++r)
      for (int32_t k = ptr[I * b + r]; k < ptr[I * b + r + 1]; ++k) cols.push_back(col[k] / b);
    std::sort(cols.begin(), cols.end());
    cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
    size_t base = A->col.size();
    for (int32_t J : cols) A->col.push_back(J);
    A->val.resize(A->col.size() * b * b, 0.0);
    for (int r = 0; r < b; ++r)
      for (int32_t k = ptr[I * b + r]; k < ptr[I * b + r + 1]; ++k) {
        int32_t J = col[k] / b, c = col[k] % b;
        size_t pos = base + (std::lower_bound(cols.begin(), cols.end(), J) - cols.begin());
        A->val[pos * b * b + r * b + c] += val[k];
      }
    A->ptr[I + 1] = (int32_t)A->col.size();
  }
  return A;
}

// ---------------------------------------------------------------- C1 SpMV
// y_I = alpha * sum_{k in row I} A_k x_{col k} + beta * y_I ; beta == 0 overwrites.
// PAPER.md:284-312 (§2.3 backend spmv primitive); SURVEY.md §8(c) C1.
static void spmv(const orc_mat& A, double alpha, const double* x, double beta, double* y,
                 bool round_f32) {
  const int b = A.b;
  vector<double> acc(b);
  for (int32_t I = 0; I < A.n; ++I) {
    std::fill(acc.begin(), acc.end(), 0.0);
    for (int32_t k = A.ptr[I]; k < A.ptr[I + 1]; ++k) {
      const double* a = A.blk(k);
      const double* xj = x + (int64_t)A.col[k] * b;
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < b; ++c) acc[r] = acc[r] + a[r * b + c] * xj[c];
    }
    for (int r = 0; r < b; ++r) {
      double v = alpha * acc[r];
      if (beta != 0.0) v = v + beta * y[(int64_t)I * b + r];
      y[(int64_t)I * b + r] = round_f32 ? f32r(v) : v;
    }
  }
}

extern "C" int orc_spmv(const orc_mat* A, double alpha, const double* x, double beta, double* y) {
  spmv(*A, alpha, x, beta, y, false);
  return ORC_OK;
}

// r = f - A x (backend::residual)
static void residual(const orc_mat& A, const double* f, const double* x, double* out, bool rf) {
  const int b = A.b;
  vector<double> acc(b);
  for (int32_t I = 0; I < A.n; ++I) {
    std::fill(acc.begin(), acc.end(), 0.0);
    for (int32_t k = A.ptr[I]; k < A.ptr[I + 1]; ++k) {
      const double* a = A.blk(k);
      const double* xj = x + (int64_t)A.col[k] * b;
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < b; ++c) acc[r] = acc[r] + a[r * b + c] * xj[c];
    }
    for (int r = 0; r < b; ++r) {
      double v = f[(int64_t)I * b + r] - acc[r];
      out[(int64_t)I * b + r] = rf ? f32r(v) : v;
    }
  }
}

static double dot(const vector<double>& a, const vector<double>& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s = s + a[i] * b[i];
  return s;
}
static double nrm2(const vector<double>& a) { return std::sqrt(dot(a, a)); }
// a^T b with a's entries rounded to fp32 first (the fp32 shadow basis of reading R23)
static double dot_f32_basis(const vector<double>& a, const vector<double>& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s = s + f32r(a[i]) * b[i];
  return s;
}

// gmres_ortho = 3 (reading R28): the unit basis vector a scaled to unit rms (x sqrt(N)), rounded
// to IEEE binary16 (RNE, gradual underflow), scaled back
static double dot_f16_basis(const vector<double>& a, const vector<double>& b) {
  const double sq = std::sqrt((double)a.size());
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s = s + ((double)(_Float16)(a[i] * sq) / sq) * b[i];
  return s;
}

// ---------------------------------------------------------------- block helpers
// Frobenius norm squared, row-major order (C2 reading: Frobenius).
static double fro2(const double* a, int b) {
  double s = 0.0;
  for (int i = 0; i < b * b; ++i) s = s + a[i] * a[i];
  return s;
}

// b x b inverse by Gauss-Jordan with partial pivoting (first maximal |pivot|).
// A pivot below 1e-14 * ||X||_F is singular.
static int block_inverse(int b, const double* x, double* inv) {
  double M[64], R[64];
  for (int i = 0; i < b * b; ++i) M[i] = x[i];
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < b; ++j) R[i * b + j] = (i == j) ? 1.0 : 0.0;
  const double fn = std::sqrt(fro2(x, b));
  for (int c = 0; c < b; ++c) {
    int p = c;
    for (int r = c + 1; r < b; ++r)
      if (std::fabs(M[r * b + c]) > std::fabs(M[p * b + c])) p = r;
    if (!(std::fabs(M[p * b + c]) > 1e-14 * fn)) return ORC_ESINGULAR_BLOCK;
    if (p != c)
      for (int j = 0; j < b; ++j) {
        std::swap(M[p * b + j], M[c * b + j]);
        std::swap(R[p * b + j], R[c * b + j]);
      }
    const double d = M[c * b + c];
    for (int j = 0; j < b; ++j) {
      M[c * b + j] = M[c * b + j] / d;
      R[c * b + j] = R[c * b + j] / d;
    }
    for (int r = 0; r < b; ++r) {
      if (r == c) continue;
      const double f = M[r * b + c];
      for (int j = 0; j < b; ++j) {
        M[r * b + j] = M[r * b + j] - f * M[c * b + j];
        R[r * b + j] = R[r * b + j] - f * R[c * b + j];
      }
    }
  }
  for (int i = 0; i < b * b; ++i) inv[i] = R[i];
  return ORC_OK;
}

extern "C" int orc_block_inverse(int32_t b, const double* blk, double* inv) {
  return block_inverse(b, blk, inv);
}

// c = a * b for b x b blocks; each entry summed over m ascending from the first product.
static void blk_mul(int b, const double* a, const double* bb, double* c) {
  for (int r = 0; r < b; ++r)
    for (int cc = 0; cc < b; ++cc) {
      double t = a[r * b] * bb[cc];
      for (int m = 1; m < b; ++m) t = t + a[r * b + m] * bb[m * b + cc];
      c[r * b + cc] = t;
    }
}

static int64_t find_block(const orc_mat& A, int32_t I, int32_t J) {
  auto b0 = A.col.begin() + A.ptr[I], e0 = A.col.begin() + A.ptr[I + 1];
  auto it = std::lower_bound(b0, e0, J);
  if (it == e0 || *it != J) return -1;
  return it - A.col.begin();
}

// ---------------------------------------------------------------- C2 strength
// strong(I,J), I != J, block (I,J) present: ||A_IJ||_F^2 > eps^2 ||A_II||_F ||A_JJ||_F
// (PAPER.md:247-248, 257 eps_strong), dropped across slabs (C12),
// then symmetric closure S <- S u S^T.  Returns adjacency lists (sorted, unique).
static vector<int32_t> slab_bounds(int32_t n, int32_t nparts) {
  vector<int32_t> bd(nparts + 1);
  for (int32_t r = 0; r <= nparts; ++r) bd[r] = (int32_t)((int64_t)r * n / nparts);
  return bd;
}

static int strength(const orc_mat& A, double eps, const vector<int32_t>& part_of,
                    vector<vector<int32_t>>& adj) {
  const int b = A.b;
  vector<double> dn(A.n);
  for (int32_t I = 0; I < A.n; ++I) {
    int64_t k = find_block(A, I, I);
    if (k < 0) return ORC_EZERODIAG;
    dn[I] = std::sqrt(fro2(A.blk(k), b));
  }
  adj.assign(A.n, {});
  const double eps2 = eps * eps;
  for (int32_t I = 0; I < A.n; ++I)
    for (int32_t k = A.ptr[I]; k < A.ptr[I + 1]; ++k) {
      int32_t J = A.col[k];
      if (J == I || J >= A.n) continue;
      if (part_of[I] != part_of[J]) continue;
      if (fro2(A.blk(k), b) > eps2 * dn[I] * dn[J]) {
        adj[I].push_back(J);
        adj[J].push_back(I);  // symmetric closure
      }
    }
  for (auto& a : adj) {
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
  }
  return ORC_OK;
}

static vector<int32_t> part_of_rows(int32_t n, const vector<int32_t>& bd) {
  vector<int32_t> p(n);
  for (size_t r = 0; r + 1 < bd.size(); ++r)
    for (int32_t i = bd[r]; i < bd[r + 1]; ++i) p[i] = (int32_t)r;
  return p;
}

extern "C" int64_t orc_strength(const orc_mat* A, double eps, int32_t nparts, int32_t* ptr,
                                int32_t* col) {
  vector<vector<int32_t>> adj;
  auto bd = slab_bounds(A->n, nparts < 1 ? 1 : nparts);
  int rc = strength(*A, eps, part_of_rows(A->n, bd), adj);
  if (rc != ORC_OK) return rc;
  int64_t e = 0;
  for (int32_t I = 0; I < A->n; ++I) {
    if (ptr) ptr[I] = (int32_t)e;
    for (int32_t J : adj[I]) {
      if (col) col[e] = J;
      ++e;
    }
  }
  if (ptr) ptr[A->n] = (int32_t)e;
  return e;
}

// ---------------------------------------------------------------- C3 aggregation
// Pass 1 (SPEC.md:488 rule): for I ascending, if I is unassigned,
// not isolated and none of its strong neighbours is assigned, open a new
// aggregate with I and all its strong neighbours.  Pass 2: every still
// unassigned non-isolated node joins the pass-1 aggregate of its lowest-index
// strong neighbour assigned in pass 1.  Isolated nodes stay -1.
static int32_t aggregate(const vector<vector<int32_t>>& adj, vector<int32_t>& agg,
                         vector<int32_t>* roots) {
  const int32_t n = (int32_t)adj.size();
  agg.assign(n, -1);
  if (roots) roots->assign(n, 0);
  int32_t count = 0;
  for (int32_t I = 0; I < n; ++I) {
    if (agg[I] >= 0 || adj[I].empty()) continue;
    bool free_nb = true;
    for (int32_t J : adj[I])
      if (agg[J] >= 0) {
        free_nb = false;
        break;
      }
    if (!free_nb) continue;
    int32_t id = count++;
    agg[I] = id;
    if (roots) (*roots)[I] = 1;
    for (int32_t J : adj[I]) agg[J] = id;
  }
  vector<int32_t> pass1 = agg;
  for (int32_t I = 0; I < n; ++I) {
    if (pass1[I] >= 0 || adj[I].empty()) continue;
    for (int32_t J : adj[I])  // ascending: the first assigned one is the lowest index
      if (pass1[J] >= 0) {
        agg[I] = pass1[J];
        break;
      }
  }
  return count;
}

extern "C" int32_t orc_aggregate(const orc_mat* A, double eps, int32_t nparts, int32_t* agg) {
  vector<vector<int32_t>> adj;
  auto bd = slab_bounds(A->n, nparts < 1 ? 1 : nparts);
  int rc = strength(*A, eps, part_of_rows(A->n, bd), adj);
  if (rc != ORC_OK) return rc;
  vector<int32_t> a;
  int32_t nc = aggregate(adj, a, nullptr);
  std::copy(a.begin(), a.end(), agg);
  return nc;
}

extern "C" int32_t orc_roots(const orc_mat* A, double eps, int32_t nparts, int32_t* is_root) {
  vector<vector<int32_t>> adj;
  auto bd = slab_bounds(A->n, nparts < 1 ? 1 : nparts);
  int rc = strength(*A, eps, part_of_rows(A->n, bd), adj);
  if (rc != ORC_OK) return rc;
  vector<int32_t> a, r;
  int32_t nc = aggregate(adj, a, &r);
  std::copy(r.begin(), r.end(), is_root);
  return nc;
}

// ---------------------------------------------------------------- sparse products
// C = A * B (Gustavson), structural pattern sorted ascending, nothing dropped;
// every C_ij accumulated over k ascending from 0: C_ij = C_ij + (A_ik B_kj)
// (SURVEY.md C6 fixed-order reading).
static orc_mat spgemm(const orc_mat& A, const orc_mat& B) {
  const int b = A.b;
  orc_mat C;
  C.n = A.n;
  C.m = B.m;
  C.b = b;
  C.ptr.assign(A.n + 1, 0);
  vector<int64_t> pos(B.m, -1);
  vector<int32_t> cols;
  vector<double> tmp(b * b);
  for (int32_t i = 0; i < A.n; ++i) {
    cols.clear();
    for (int32_t ka = A.ptr[i]; ka < A.ptr[i + 1]; ++ka) {
      int32_t k = A.col[ka];
      for (int32_t kb = B.ptr[k]; kb < B.ptr[k + 1]; ++kb) {
        int32_t j = B.col[kb];
        if (pos[j] == -2) continue;
        pos[j] = -2;
        cols.push_back(j);
      }
    }
    std::sort(cols.begin(), cols.end());
    int64_t base = (int64_t)C.col.size();
    for (size_t t = 0; t < cols.size(); ++t) {
      pos[cols[t]] = base + (int64_t)t;
      C.col.push_back(cols[t]);
    }
    C.val.resize(C.col.size() * b * b, 0.0);
    for (int32_t ka = A.ptr[i]; ka < A.ptr[i + 1]; ++ka) {
      int32_t k = A.col[ka];
      for (int32_t kb = B.ptr[k]; kb < B.ptr[k + 1]; ++kb) {
        blk_mul(b, A.blk(ka), B.blk(kb), tmp.data());
        double* c = C.blk(pos[B.col[kb]]);
        for (int e = 0; e < b * b; ++e) c[e] = c[e] + tmp[e];
      }
    }
    for (int32_t j : cols) pos[j] = -1;
    C.ptr[i + 1] = (int32_t)C.col.size();
  }
  return C;
}

// R = P^T, each block transposed ("R = P^T")
static orc_mat transpose(const orc_mat& P) {
  const int b = P.b;
  orc_mat R;
  R.n = P.m;
  R.m = P.n;
  R.b = b;
  R.ptr.assign(P.m + 1, 0);
  for (int32_t c : P.col) R.ptr[c + 1]++;
  for (int32_t i = 0; i < P.m; ++i) R.ptr[i + 1] += R.ptr[i];
  R.col.resize(P.col.size());
  R.val.resize(P.val.size());
  vector<int32_t> fill(R.ptr.begin(), R.ptr.end() - 1);
  for (int32_t I = 0; I < P.n; ++I)  // ascending I: rows of R come out sorted
    for (int32_t k = P.ptr[I]; k < P.ptr[I + 1]; ++k) {
      int32_t c = P.col[k];
      int32_t d = fill[c]++;
      R.col[d] = I;
      const double* s = P.blk(k);
      double* t = R.blk(d);
      for (int r = 0; r < b; ++r)
        for (int cc = 0; cc < b; ++cc) t[cc * b + r] = s[r * b + cc];
    }
  return R;
}

// ---------------------------------------------------------------- C4/C5 prolongator
// P_tent(I, agg(I)) = I_b (C4).  A_F keeps the diagonal and strong blocks; every
// weak off-diagonal block is added (ascending column) into its row's diagonal
// (C5 lumping).  P = P_tent - omega * (D^-1 (A_F P_tent)), D_I = A_F,II,
// omega = sa_omega (C5 reading: 2/3).  PAPER.md:195, 209 (smoothed_aggregation).
static int smoothed_prolongator(const orc_mat& A, const vector<vector<int32_t>>& adj,
                                const vector<int32_t>& agg, int32_t nc, double omega,
                                orc_mat& P) {
  const int b = A.b, bb = b * b;
  // A_F
  orc_mat AF;
  AF.n = A.n;
  AF.m = A.m;
  AF.b = b;
  AF.ptr.assign(A.n + 1, 0);
  vector<double> Dinv((size_t)A.n * bb);
  for (int32_t I = 0; I < A.n; ++I) {
    int64_t kd = find_block(A, I, I);
    if (kd < 0) return ORC_EZERODIAG;
    vector<double> D(A.blk(kd), A.blk(kd) + bb);
    for (int32_t k = A.ptr[I]; k < A.ptr[I + 1]; ++k) {
      int32_t J = A.col[k];
      if (J == I) continue;
      bool strong = std::binary_search(adj[I].begin(), adj[I].end(), J);
      if (!strong)
        for (int e = 0; e < bb; ++e) D[e] = D[e] + A.blk(k)[e];
    }
    for (int32_t k = A.ptr[I]; k < A.ptr[I + 1]; ++k) {
      int32_t J = A.col[k];
      bool keep = (J == I) || std::binary_search(adj[I].begin(), adj[I].end(), J);
      if (!keep) continue;
      AF.col.push_back(J);
      const double* src = (J == I) ? D.data() : A.blk(k);
      AF.val.insert(AF.val.end(), src, src + bb);
    }
    AF.ptr[I + 1] = (int32_t)AF.col.size();
    int rc = block_inverse(b, D.data(), &Dinv[(size_t)I * bb]);
    if (rc != ORC_OK) return rc;
  }
  // P_tent
  orc_mat Pt;
  Pt.n = A.n;
  Pt.m = nc;
  Pt.b = b;
  Pt.ptr.assign(A.n + 1, 0);
  for (int32_t I = 0; I < A.n; ++I) {
    if (agg[I] >= 0) {
      Pt.col.push_back(agg[I]);
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < b; ++c) Pt.val.push_back(r == c ? 1.0 : 0.0);
    }
    Pt.ptr[I + 1] = (int32_t)Pt.col.size();
  }
  orc_mat T = spgemm(AF, Pt);  // pattern(A_F P_tent), contains pattern(P_tent)
  P = T;
  vector<double> dt(bb);
  for (int32_t I = 0; I < A.n; ++I)
    for (int32_t k = T.ptr[I]; k < T.ptr[I + 1]; ++k) {
      blk_mul(b, &Dinv[(size_t)I * bb], T.blk(k), dt.data());
      double* p = P.blk(k);
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < b; ++c) {
          double pt = (T.col[k] == agg[I] && r == c) ? 1.0 : 0.0;
          p[r * b + c] = pt - omega * dt[r * b + c];
        }
    }
  return ORC_OK;
}

// Plain aggregation (Listings V2-V4, "amgcl::coarsening::aggregation"): P = P_tent,
// one identity block per aggregated row at its aggregate (C4); isolated rows empty.
static orc_mat tentative_prolongator(const orc_mat& A, const vector<int32_t>& agg, int32_t nc) {
  const int b = A.b;
  orc_mat Pt;
  Pt.n = A.n;
  Pt.m = nc;
  Pt.b = b;
  Pt.ptr.assign(A.n + 1, 0);
  for (int32_t I = 0; I < A.n; ++I) {
    if (agg[I] >= 0) {
      Pt.col.push_back(agg[I]);
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < b; ++c) Pt.val.push_back(r == c ? 1.0 : 0.0);
    }
    Pt.ptr[I + 1] = (int32_t)Pt.col.size();
  }
  return Pt;
}

// ---------------------------------------------------------------- C8b ILU(0)
// Block ILU(0) on A's pattern (no fill; SURVEY.md §8(f) #3 -- the paper's U-solver
// smoother is ILU-type; Saad, Iterative Methods, Alg. 10.4 "IKJ"):
// for each row i ascending, for each k < i in row i ascending:
//   a_ik <- a_ik D_k^-1;  a_ij <- a_ij - a_ik a_kj for every later j of row i with (k,j) in A.
// Then D_i^-1 = inverse(a_ii) (error if singular).  L = I + strictly lower a_ik,
// U = D + strictly upper a_ij.  Reading R20.
static int ilu0_factor(const orc_mat& A, orc_mat& Lo, orc_mat& Up, vector<double>& Dinv) {
  const int b = A.b, bb = b * b;
  vector<double> a = A.val;
  Dinv.assign((size_t)A.n * bb, 0.0);
  vector<double> tmp(bb);
  for (int32_t i = 0; i < A.n; ++i) {
    int64_t kd = -1;
    for (int32_t kk = A.ptr[i]; kk < A.ptr[i + 1]; ++kk) {
      const int32_t k = A.col[kk];
      if (k == i) kd = kk;
      if (k >= i) continue;
      blk_mul(b, &a[(size_t)kk * bb], &Dinv[(size_t)k * bb], tmp.data());
      std::copy(tmp.begin(), tmp.end(), a.begin() + (size_t)kk * bb);
      for (int32_t jj = kk + 1; jj < A.ptr[i + 1]; ++jj) {
        const int64_t kj = find_block(A, k, A.col[jj]);
        if (kj < 0) continue;
        blk_mul(b, &a[(size_t)kk * bb], &a[(size_t)kj * bb], tmp.data());
        for (int e = 0; e < bb; ++e) a[(size_t)jj * bb + e] = a[(size_t)jj * bb + e] - tmp[e];
      }
    }
    if (kd < 0) return ORC_EZERODIAG;
    int rc = block_inverse(b, &a[(size_t)kd * bb], &Dinv[(size_t)i * bb]);
    if (rc != ORC_OK) return rc;
  }
  for (orc_mat* F : {&Lo, &Up}) {
    F->n = A.n;
    F->m = A.m;
    F->b = b;
    F->ptr.assign(A.n + 1, 0);
    F->col.clear();
    F->val.clear();
  }
  for (int32_t i = 0; i < A.n; ++i) {
    for (int32_t kk = A.ptr[i]; kk < A.ptr[i + 1]; ++kk) {
      const int32_t j = A.col[kk];
      if (j == i) continue;
      orc_mat& F = j < i ? Lo : Up;
      F.col.push_back(j);
      F.val.insert(F.val.end(), a.begin() + (size_t)kk * bb, a.begin() + (size_t)(kk + 1) * bb);
    }
    Lo.ptr[i + 1] = (int32_t)Lo.col.size();
    Up.ptr[i + 1] = (int32_t)Up.col.size();
  }
  return ORC_OK;
}

// ---------------------------------------------------------------- C8c ILUT(tau, p)
// Block ILUT -- the paper's U-solver smoother, "amgcl::relaxation::ilut" (Listing V2,
// PAPER.md:599; "AMG with ILU as a smoother has the best performance");
// the paper gives no (tau, p), SPEC.md:443 fixes the defaults tau = 1e-2, p = 2.  Saad's
// threshold IKJ factorisation (Iterative Methods, Alg. 10.6, ILUT) on blocks, reading R25:
//   w = row i of A;  tau_i = tau * ||row i of A||_2 (all its scalars)
//   for k < i in w, ascending (fill entries created on the way included):
//     w_k <- w_k D_k^-1;  if ||w_k||_F < tau_i: drop w_k (no update)
//     else w_j <- w_j - w_k U_kj for every stored U_kj of row k (new entries start at 0)
//   drop every w_j, j != i, with ||w_j||_F < tau_i;  of the surviving entries, L (j < i) and
//   U (j > i) each keep those on A's pattern and the p largest fill entries (||.||_F
//   descending, lower column first on ties);  D_i = w_i (error if singular).
// The factors are stored as ILU(0)'s are: L_s = the kept w_j, j < i; U_s = the kept w_j,
// j > i; Dinv = D_i^-1 -- applied by the same sweeps (R20).
static int ilut_factor(const orc_mat& A, double tau, int p, orc_mat& Lo, orc_mat& Up, vector<double>& Dinv) {
  const int b = A.b, bb = b * b;
  Dinv.assign((size_t)A.n * bb, 0.0);
  for (orc_mat* F : {&Lo, &Up}) {
    F->n = A.n;
    F->m = A.m;
    F->b = b;
    F->ptr.assign(A.n + 1, 0);
    F->col.clear();
    F->val.clear();
  }
  vector<double> tmp(bb);
  for (int32_t i = 0; i < A.n; ++i) {
    std::map<int32_t, vector<double>> w;
    double nrm2 = 0.0;
    for (int32_t kk = A.ptr[i]; kk < A.ptr[i + 1]; ++kk) {
      w[A.col[kk]] = vector<double>(A.blk(kk), A.blk(kk) + bb);
      nrm2 = nrm2 + fro2(A.blk(kk), b);
    }
    const double tau_i = tau * std::sqrt(nrm2);
    for (auto it = w.begin(); it != w.end() && it->first < i;) {
      const int32_t k = it->first;
      blk_mul(b, it->second.data(), &Dinv[(size_t)k * bb], tmp.data());
      if (std::sqrt(fro2(tmp.data(), b)) < tau_i) {
        it = w.erase(it);
        continue;
      }
      it->second = tmp;
      for (int32_t kj = Up.ptr[k]; kj < Up.ptr[k + 1]; ++kj) {
        auto jt = w.find(Up.col[kj]);
        if (jt == w.end()) jt = w.emplace(Up.col[kj], vector<double>(bb, 0.0)).first;
        blk_mul(b, it->second.data(), Up.blk(kj), tmp.data());
        for (int e = 0; e < bb; ++e) jt->second[e] = jt->second[e] - tmp[e];
      }
      ++it;
    }
    auto dt = w.find(i);
    if (dt == w.end()) return ORC_EZERODIAG;
    int rc = block_inverse(b, dt->second.data(), &Dinv[(size_t)i * bb]);
    if (rc != ORC_OK) return rc;
    for (int side = 0; side < 2; ++side) {  // 0: L (j < i), 1: U (j > i)
      vector<std::pair<double, int32_t>> fill;
      vector<int32_t> keep;
      for (auto& [j, v] : w) {
        if (j == i || (side == 0) != (j < i)) continue;
        const double nv = std::sqrt(fro2(v.data(), b));
        if (nv < tau_i) continue;
        if (find_block(A, i, j) >= 0) keep.push_back(j);
        else fill.push_back({nv, j});
      }
      std::sort(fill.begin(), fill.end(), [](const std::pair<double, int32_t>& x, const std::pair<double, int32_t>& y) {
        return x.first > y.first || (x.first == y.first && x.second < y.second);
      });
      for (size_t q = 0; q < fill.size() && (int)q < p; ++q) keep.push_back(fill[q].second);
      std::sort(keep.begin(), keep.end());
      orc_mat& F = side == 0 ? Lo : Up;
      for (int32_t j : keep) {
        F.col.push_back(j);
        F.val.insert(F.val.end(), w[j].begin(), w[j].end());
      }
      F.ptr[i + 1] = (int32_t)F.col.size();
    }
  }
  return ORC_OK;
}

// ---------------------------------------------------------------- C8 smoother
// SPAI0: M_I = theta_I A_II^-1, theta_I = ||A_II||_F^2 / sum_J ||A_IJ||_F^2
// (block generalisation of Broker-Grote SPAI(0)).
// Damped Jacobi: M_I = omega_J A_II^-1.
static int smoother_blocks(const orc_mat& A, int kind, double omega_j, vector<double>& M) {
  const int b = A.b, bb = b * b;
  M.assign((size_t)A.n * bb, 0.0);
  vector<double> inv(bb);
  for (int32_t I = 0; I < A.n; ++I) {
    int64_t kd = find_block(A, I, I);
    if (kd < 0) return ORC_EZERODIAG;
    int rc = block_inverse(b, A.blk(kd), inv.data());
    if (rc != ORC_OK) return rc;
    double theta = omega_j;
    if (kind == ORC_SPAI0) {
      double den = 0.0;
      for (int32_t k = A.ptr[I]; k < A.ptr[I + 1]; ++k) den = den + fro2(A.blk(k), b);
      theta = fro2(A.blk(kd), b) / den;
    }
    for (int e = 0; e < bb; ++e) M[(size_t)I * bb + e] = theta * inv[e];
  }
  return ORC_OK;
}

// ---------------------------------------------------------------- hierarchy
struct Level {
  orc_mat A, P, R;          // fp64 setup values
  vector<int32_t> agg;
  int32_t nc = 0;
  vector<double> M;         // fp64 setup values (ILU(0): the inverted pivot blocks D^-1)
  orc_mat L, U;             // ILU(0): strictly lower / strictly upper factor blocks
  orc_mat As, Ps, Rs, Ls, Us;  // solve copies (narrowed when hier_f32)
  vector<double> Ms;
};

struct Coarse {
  int32_t N = 0;
  vector<double> LU;        // dense N x N, row-major, partial pivoting
  vector<int32_t> piv;
};

struct orc_solver {
  orc_params p;
  orc_mat A;                // outer operator, fp64
  bool schur = false;
  int32_t bh = 0;           // block size of the AMG hierarchy
  vector<Level> lv;
  orc_mat Acoarse;          // coarsest matrix (fp64)
  Coarse coarse;
  // Schur split (C10) on A's block pattern
  orc_mat Au, Au_s;  // velocity block; its scalar expansion (schur_u_scalar)
  vector<double> Bv, BTv;   // nnz * 3 (row pc, cols vel) and (rows vel, col pc)
  vector<double> Shat_diag, mS;
  vector<double> Bs, BTs, mSs;
  vector<int32_t> vel;      // velocity component indices
  // general scalar pressure mask (R21): index maps and the scalar split of A
  bool masked = false;
  vector<int32_t> uidx, pidx;   // scalar unknowns of each class, ascending
  orc_mat Bm, BTm, Cm;          // B (p rows x u cols), B^T (u rows x p cols), C, b = 1
  orc_mat Bms, BTms;            // solve copies (narrowed when hier_f32)
};

static orc_mat narrowed(const orc_mat& A) {
  orc_mat B = A;
  for (double& v : B.val) v = f32r(v);
  return B;
}

// Dense LU with partial pivoting of the scalar expansion (C7).
static int coarse_factor(const orc_mat& A, Coarse& C) {
  const int b = A.b;
  const int32_t N = A.n * b;
  C.N = N;
  C.LU.assign((size_t)N * N, 0.0);
  C.piv.assign(N, 0);
  for (int32_t I = 0; I < A.n; ++I)
    for (int32_t k = A.ptr[I]; k < A.ptr[I + 1]; ++k)
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < b; ++c)
          C.LU[(size_t)(I * b + r) * N + (size_t)A.col[k] * b + c] = A.blk(k)[r * b + c];
  double* a = C.LU.data();
  for (int32_t c = 0; c < N; ++c) {
    int32_t p = c;
    for (int32_t r = c + 1; r < N; ++r)
      if (std::fabs(a[(size_t)r * N + c]) > std::fabs(a[(size_t)p * N + c])) p = r;
    if (a[(size_t)p * N + c] == 0.0) return ORC_ESINGULAR_BLOCK;
    C.piv[c] = p;
    if (p != c)
      for (int32_t j = 0; j < N; ++j) std::swap(a[(size_t)p * N + j], a[(size_t)c * N + j]);
    for (int32_t r = c + 1; r < N; ++r) {
      double l = a[(size_t)r * N + c] / a[(size_t)c * N + c];
      a[(size_t)r * N + c] = l;
      for (int32_t j = c + 1; j < N; ++j) a[(size_t)r * N + j] = a[(size_t)r * N + j] - l * a[(size_t)c * N + j];
    }
  }
  return ORC_OK;
}

static void coarse_solve(const Coarse& C, const double* f, double* x, bool rf) {
  const int32_t N = C.N;
  vector<double> y(f, f + N);
  for (int32_t c = 0; c < N; ++c) std::swap(y[c], y[C.piv[c]]);
  for (int32_t r = 0; r < N; ++r)
    for (int32_t j = 0; j < r; ++j) y[r] = y[r] - C.LU[(size_t)r * N + j] * y[j];
  for (int32_t r = N - 1; r >= 0; --r) {
    for (int32_t j = r + 1; j < N; ++j) y[r] = y[r] - C.LU[(size_t)r * N + j] * y[j];
    y[r] = y[r] / C.LU[(size_t)r * N + r];
  }
  for (int32_t i = 0; i < N; ++i) x[i] = rf ? f32r(y[i]) : y[i];
}

// A with the blocks coupling different slabs removed (bd: slab bounds over block rows)
static orc_mat slab_diagonal_blocks(const orc_mat& A, const vector<int32_t>& bd) {
  vector<int32_t> part = part_of_rows(A.n, bd);
  orc_mat F;
  F.n = A.n;
  F.m = A.m;
  F.b = A.b;
  F.ptr.assign(A.n + 1, 0);
  const int bb = A.b * A.b;
  for (int32_t i = 0; i < A.n; ++i) {
    for (int32_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k)
      if (part[A.col[k]] == part[i]) {
        F.col.push_back(A.col[k]);
        F.val.insert(F.val.end(), A.blk(k), A.blk(k) + bb);
      }
    F.ptr[i + 1] = (int32_t)F.col.size();
  }
  return F;
}

// C7: repeat C2-C6 while n_l * b > coarse_enough and l < max_levels - 1;
// stop if n_c == 0 or n_c >= n_l.  Coarsest: dense LU.
// unit: rows of A0 per partitioned row (the scalar U-solver of V2 has 3 scalar rows per cell
// and its slabs follow the cells' slabs, R18 / C12)
// bd0 (optional): explicit level-0 slab bounds (the pressure mask's velocity ranges, R27)
static int build_hierarchy(orc_solver& s, const orc_mat& A0, int unit = 1, const vector<int32_t>* bd0 = nullptr) {
  const orc_params& p = s.p;
  orc_mat A = A0;
  vector<int32_t> bd = slab_bounds(A.n / unit, p.nparts < 1 ? 1 : p.nparts);
  for (int32_t& v : bd) v *= unit;
  if (bd0) bd = *bd0;
  s.lv.clear();
  while ((int64_t)A.n * A.b > p.coarse_enough && (int32_t)s.lv.size() < p.max_levels - 1) {
    vector<vector<int32_t>> adj;
    int rc = strength(A, p.eps_strong, part_of_rows(A.n, bd), adj);
    if (rc != ORC_OK) return rc;
    Level L;
    vector<int32_t> roots;
    L.nc = aggregate(adj, L.agg, &roots);
    if (L.nc == 0 || L.nc >= A.n) break;
    if (p.coarsening == ORC_PLAIN)
      L.P = tentative_prolongator(A, L.agg, L.nc);
    else
      rc = smoothed_prolongator(A, adj, L.agg, L.nc, p.sa_omega, L.P);
    if (rc != ORC_OK) return rc;
    L.R = transpose(L.P);
    if (p.smoother == ORC_ILU0 || p.smoother == ORC_ILUT) {
      // multi-rank (reading R26): each slab's factors are those of its diagonal block --
      // the couplings between slabs are left out of the factorisation (block Jacobi across
      // ranks, the usual parallel ILU); the level's residuals still use the whole A
      const orc_mat Af = bd.size() > 2 ? slab_diagonal_blocks(A, bd) : orc_mat();
      const orc_mat& F = bd.size() > 2 ? Af : A;
      rc = p.smoother == ORC_ILU0 ? ilu0_factor(F, L.L, L.U, L.M) : ilut_factor(F, p.ilut_tau, p.ilut_p, L.L, L.U, L.M);
    }
    else
      rc = smoother_blocks(A, p.smoother, p.jacobi_omega, L.M);
    if (rc != ORC_OK) return rc;
    orc_mat AP = spgemm(A, L.P);
    orc_mat Ac = spgemm(L.R, AP);
    if (p.coarsening == ORC_PLAIN && p.over_interp != 1.0) {
      // over-interpolation (reading R19): the coarse correction scaled by alpha, i.e.
      // the Galerkin operator by 1 / alpha
      const double inv = 1.0 / p.over_interp;
      for (double& v : Ac.val) v = v * inv;
    }
    // coarse slab bounds: aggregates are numbered in ascending root order (C3, C12)
    vector<int32_t> nb(bd.size(), 0);
    for (size_t r = 1; r < bd.size(); ++r) {
      int32_t cnt = 0;
      for (int32_t i = 0; i < bd[r]; ++i) cnt += roots[i];
      nb[r] = cnt;
    }
    bd = nb;
    L.A = std::move(A);
    A = std::move(Ac);
    s.lv.push_back(std::move(L));
  }
  // coarsening stalled: dense coarse solve too large (reading R7: a coarsest
  // level above 8192 unknowns is an error on both sides)
  if ((int64_t)A.n * A.b > 8192) return ORC_EINVAL;
  s.Acoarse = A;
  int rc = coarse_factor(A, s.coarse);
  if (rc != ORC_OK) return rc;
  for (Level& L : s.lv) {
    L.As = p.hier_f32 ? narrowed(L.A) : L.A;
    L.Ps = p.hier_f32 ? narrowed(L.P) : L.P;
    L.Rs = p.hier_f32 ? narrowed(L.R) : L.R;
    L.Ls = p.hier_f32 ? narrowed(L.L) : L.L;
    L.Us = p.hier_f32 ? narrowed(L.U) : L.U;
    L.Ms = L.M;
    if (p.hier_f32)
      for (double& v : L.Ms) v = f32r(v);
  }
  return ORC_OK;
}

// ---------------------------------------------------------------- C9 V-cycle
// V(l, f): if l == L: return A_L^-1 f
//          x = M f;  r = f - A x;  xc = V(l+1, R r);  x = x + P xc;  x = x + M (f - A x)
// (npre = npost = 1 reading).  Every line computes in fp64 and
// rounds once when its vector is stored (vec_f32).
static void apply_M(const vector<double>& M, int b, int32_t n, const double* f, double* x, bool rf) {
  for (int32_t I = 0; I < n; ++I)
    for (int r = 0; r < b; ++r) {
      double t = 0.0;
      for (int c = 0; c < b; ++c) t = t + M[(size_t)I * b * b + r * b + c] * f[(int64_t)I * b + c];
      x[(int64_t)I * b + r] = rf ? f32r(t) : t;
    }
}

// x' = x + M (f - A x), every row from the old x (Jacobi-type)
static void smooth_step(const orc_mat& A, const vector<double>& M, const double* f,
                        vector<double>& x, bool rf) {
  const int b = A.b;
  vector<double> res((size_t)A.n * b), xn((size_t)A.n * b);
  residual(A, f, x.data(), res.data(), false);
  for (int32_t I = 0; I < A.n; ++I)
    for (int r = 0; r < b; ++r) {
      double t = 0.0;
      for (int c = 0; c < b; ++c) t = t + M[(size_t)I * b * b + r * b + c] * res[(int64_t)I * b + c];
      double v = x[(int64_t)I * b + r] + t;
      xn[(int64_t)I * b + r] = rf ? f32r(v) : v;
    }
  x.swap(xn);
}

// ILU(0) smoothing (R20): z = (LU)^-1 g with k = ilu_sweeps Jacobi sweeps per triangular
// solve (Anzt, Chow & Dongarra 2015): y_0 = g, y_m = g - L_s y_(m-1) (m = 1..k);
// z_0 = D^-1 y_k, z_m = D^-1 (y_k - U_s z_(m-1)) (m = 1..k); every sweep one stored vector.
// The last U sweep adds z_k into x (x0 == nullptr: from zero).  Exact once k reaches the
// depth of the factors' dependency graph.
static void ilu_into(const Level& L, int k, const double* g, const double* x0, double* xo, bool rf) {
  const int b = L.As.b, bb = b * b;
  const int32_t n = L.As.n;
  const size_t N = (size_t)n * b;
  vector<double> y(g, g + N), yn(N), z(N), zn(N), uz(N);
  for (int m = 1; m <= k; ++m) {
    residual(L.Ls, g, y.data(), yn.data(), rf);
    y.swap(yn);
  }
  apply_M(L.Ms, b, n, y.data(), z.data(), rf);
  for (int m = 1; m <= k; ++m) {
    residual(L.Us, y.data(), z.data(), uz.data(), false);  // y - U_s z, fp64 (fused in the sweep)
    const bool last = m == k;
    for (int32_t I = 0; I < n; ++I)
      for (int r = 0; r < b; ++r) {
        double t = 0.0;
        for (int c = 0; c < b; ++c) t = t + L.Ms[(size_t)I * bb + r * b + c] * uz[(size_t)I * b + c];
        const double v = (last && x0) ? x0[(size_t)I * b + r] + t : t;
        (last ? xo : zn.data())[(size_t)I * b + r] = rf ? f32r(v) : v;
      }
    if (!last) z.swap(zn);
  }
}

// x = S(f) from zero (K4a) and x <- x + S(f - A x) (K5) for the level's smoother
static void pre_smooth(const orc_solver& s, const Level& L, const double* f, double* x, bool rf) {
  if (s.p.smoother == ORC_ILU0 || s.p.smoother == ORC_ILUT) ilu_into(L, s.p.ilu_sweeps, f, nullptr, x, rf);
  else apply_M(L.Ms, L.As.b, L.As.n, f, x, rf);
}
static void post_smooth(const orc_solver& s, const Level& L, const double* f, vector<double>& x, bool rf) {
  if (s.p.smoother != ORC_ILU0 && s.p.smoother != ORC_ILUT) {
    smooth_step(L.As, L.Ms, f, x, rf);
    return;
  }
  vector<double> r(x.size());
  residual(L.As, f, x.data(), r.data(), rf);
  ilu_into(L, s.p.ilu_sweeps, r.data(), x.data(), x.data(), rf);
}

static void vcycle(const orc_solver& s, size_t l, const vector<double>& f, vector<double>& x) {
  const bool rf = s.p.vec_f32 != 0;
  if (l == s.lv.size()) {
    x.assign(f.size(), 0.0);
    coarse_solve(s.coarse, f.data(), x.data(), rf);
    return;
  }
  const Level& L = s.lv[l];
  const int b = L.As.b;
  const int32_t n = L.As.n;
  x.assign((size_t)n * b, 0.0);
  pre_smooth(s, L, f.data(), x.data(), rf);
  for (int k = 1; k < s.p.npre; ++k) post_smooth(s, L, f.data(), x, rf);
  vector<double> r((size_t)n * b);
  residual(L.As, f.data(), x.data(), r.data(), rf);
  vector<double> fc((size_t)L.nc * b), xc;
  spmv(L.Rs, 1.0, r.data(), 0.0, fc.data(), rf);
  vcycle(s, l + 1, fc, xc);
  spmv(L.Ps, 1.0, xc.data(), 1.0, x.data(), rf);
  for (int k = 0; k < s.p.npost; ++k) post_smooth(s, L, f.data(), x, rf);
}

// ---------------------------------------------------------------- C10 Schur
// Split by block component on A's block pattern: velocity = all components but
// pc, pressure = pc.  A_u (3x3), B (row pc x vel cols), B^T-part (vel rows x col
// pc), C (pc,pc).  Shat = C - diag(B diag(A_u)^-1 B^T) (Eq. 10, PAPER.md:541-543,
// adjust_p = 1 PAPER.md:622; diag(A_u) the scalar diagonal).  m_S = SPAI0(Shat):
// m_i = Shat_ii / sum_j Shat_ij^2.
// schur_shat = 2: the explicitly assembled S_hat = C - B diag(A_u)^-1 B^T (the PETSc
// variant), row i over the union of C's row and the rows of B^T reached
// through B's row; every sum_ij accumulated over k (row i's blocks ascending), then d,
// S_hat_ij = C_ij - sum_ij (C_ij = 0 off C's pattern), m_S,i = S_hat_ii / sum_j S_hat_ij^2
// (j ascending).  Same bars as Eq. 10 otherwise.
static int schur_shat_full(orc_solver& s, const orc_mat& A, const vector<double>& Cv) {
  const int bu = A.b - 1;
  const orc_mat& Au = s.Au;
  for (int32_t i = 0; i < A.n; ++i) {
    std::map<int32_t, double> sum, crow;
    for (int32_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) crow[A.col[k]] = Cv[k];
    if (crow.find(i) == crow.end()) return ORC_EZERODIAG;
    for (int32_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      const int32_t K = A.col[k];
      const int64_t kKK = find_block(A, K, K);
      if (kKK < 0) return ORC_EZERODIAG;
      for (int d = 0; d < bu; ++d) {
        const double diag = Au.val[kKK * bu * bu + d * bu + d];
        if (diag == 0.0) return ORC_EZERODIAG;
        const double t = s.Bv[k * bu + d] * (1.0 / diag);
        for (int32_t kk = A.ptr[K]; kk < A.ptr[K + 1]; ++kk) {
          double& acc = sum[A.col[kk]];  // value-initialised 0.0 on first use
          acc = acc + t * s.BTv[kk * bu + d];
        }
      }
    }
    double den = 0.0, sii = 0.0;
    for (const auto& e : sum) {  // pattern(B B^T) contains C's (diagonal blocks present)
      const auto c = crow.find(e.first);
      const double v = (c == crow.end() ? 0.0 : c->second) - e.second;
      if (e.first == i) sii = v;
      den = den + v * v;
    }
    if (den == 0.0) return ORC_EZERODIAG;
    s.Shat_diag[i] = sii;
    s.mS[i] = sii / den;
  }
  return ORC_OK;
}

static int schur_setup(orc_solver& s) {
  const orc_mat& A = s.A;
  const int b = A.b, pc = s.p.schur_p_component;
  if (pc < 0 || pc >= b || b < 2) return ORC_EINVAL;
  s.vel.clear();
  for (int c = 0; c < b; ++c)
    if (c != pc) s.vel.push_back(c);
  const int bu = b - 1;
  orc_mat& Au = s.Au;
  Au.n = A.n;
  Au.m = A.m;
  Au.b = bu;
  Au.ptr = A.ptr;
  Au.col = A.col;
  Au.val.assign((size_t)A.nnz() * bu * bu, 0.0);
  s.Bv.assign((size_t)A.nnz() * bu, 0.0);
  s.BTv.assign((size_t)A.nnz() * bu, 0.0);
  vector<double> Cv(A.nnz());
  for (int64_t k = 0; k < A.nnz(); ++k) {
    const double* a = A.blk(k);
    for (int r = 0; r < bu; ++r)
      for (int c = 0; c < bu; ++c) Au.val[k * bu * bu + r * bu + c] = a[s.vel[r] * b + s.vel[c]];
    for (int d = 0; d < bu; ++d) {
      s.Bv[k * bu + d] = a[pc * b + s.vel[d]];
      s.BTv[k * bu + d] = a[s.vel[d] * b + pc];
    }
    Cv[k] = a[pc * b + pc];
  }
  s.Shat_diag.assign(A.n, 0.0);
  s.mS.assign(A.n, 0.0);
  if (s.p.schur_shat == 2) {
    int rc = schur_shat_full(s, A, Cv);
    if (rc != ORC_OK) return rc;
  }
  for (int32_t i = 0; i < A.n && s.p.schur_shat != 2; ++i) {
    int64_t kd = find_block(A, i, i);
    if (kd < 0) return ORC_EZERODIAG;
    double sum = 0.0;
    if (s.p.schur_shat == 1)
    for (int32_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      int32_t J = A.col[k];
      int64_t kJJ = find_block(A, J, J), kJi = find_block(A, J, i);
      if (kJJ < 0) return ORC_EZERODIAG;
      if (kJi < 0) continue;  // structurally absent transpose entry contributes nothing
      for (int d = 0; d < bu; ++d) {
        double diag = Au.val[kJJ * bu * bu + d * bu + d];
        if (diag == 0.0) return ORC_EZERODIAG;
        double t = s.Bv[k * bu + d] * (1.0 / diag);
        sum = sum + t * s.BTv[kJi * bu + d];
      }
    }
    s.Shat_diag[i] = Cv[kd] - sum;
    double den = 0.0;
    for (int32_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      double v = (k == kd) ? s.Shat_diag[i] : Cv[k];
      den = den + v * v;
    }
    if (den == 0.0) return ORC_EZERODIAG;
    s.mS[i] = s.Shat_diag[i] / den;
  }
  s.Bs = s.Bv;
  s.BTs = s.BTv;
  s.mSs = s.mS;
  if (s.p.hier_f32) {
    for (double& v : s.Bs) v = f32r(v);
    for (double& v : s.BTs) v = f32r(v);
    for (double& v : s.mSs) v = f32r(v);
  }
  return ORC_OK;
}

// Scalar expansion of A_u for the V2 U-solver (Listing V2: the scalar builtin<double>
// backend; PAPER.md:660-672 shows the same matrix in both forms): block (I, J) entry
// (r, c) becomes scalar (bu I + r, bu J + c); entries that are exactly zero inside a
// stored block are not stored (the scalar CSR holds the structural non-zeros), the
// diagonal always is.  Rows stay sorted (J ascending, then c).  Reading R18.
static orc_mat scalar_expansion(const orc_mat& A) {
  const int b = A.b;
  orc_mat S;
  S.n = A.n * b;
  S.m = A.m * b;
  S.b = 1;
  S.ptr.assign((size_t)S.n + 1, 0);
  for (int32_t I = 0; I < A.n; ++I)
    for (int r = 0; r < b; ++r) {
      const int32_t row = I * b + r;
      for (int32_t k = A.ptr[I]; k < A.ptr[I + 1]; ++k)
        for (int c = 0; c < b; ++c) {
          const double v = A.blk(k)[r * b + c];
          const int32_t colj = A.col[k] * b + c;
          if (v != 0.0 || colj == row) {
            S.col.push_back(colj);
            S.val.push_back(v);
          }
        }
      S.ptr[row + 1] = (int32_t)S.col.size();
    }
  return S;
}

// Eq. 9a then 9b with one application each:
//   u* = V_u(r_u);  p = m_S o (r_p - B u*);  u = V_u(r_u - B^T p);  z = (u, p)
// ---------------------------------------------------------------- C10b Schur, scalar pmask
// Reading R21: the scalar expansion As of A (structural non-zeros, diagonal kept; R18) is
// split by the mask into A_u (u rows, u cols), B (p rows, u cols), B^T (u rows, p cols), C,
// each renumbered by the ascending position of its unknowns (rows stay sorted).  S_hat by
// Eq. 10 on the scalar diagonal of A_u (schur_shat 1) or C (0); m_S = SPAI0(S_hat).  With
// the mask "component pc of every b x b block" this is the V2 split term for term.
static int schur_setup_pmask(orc_solver& s, const vector<uint8_t>& pm) {
  const orc_mat As = scalar_expansion(s.A);
  const int32_t N = As.n;
  vector<int32_t> nid(N);
  s.uidx.clear();
  s.pidx.clear();
  for (int32_t q = 0; q < N; ++q) {
    vector<int32_t>& v = pm[q] ? s.pidx : s.uidx;
    nid[q] = (int32_t)v.size();
    v.push_back(q);
  }
  const int32_t nu = (int32_t)s.uidx.size(), np = (int32_t)s.pidx.size();
  if (nu == 0 || np == 0) return ORC_EINVAL;
  auto init = [](orc_mat& M, int32_t n, int32_t m) {
    M = orc_mat();
    M.n = n;
    M.m = m;
    M.b = 1;
    M.ptr.assign(n + 1, 0);
  };
  init(s.Au, nu, nu);
  init(s.BTm, nu, np);
  init(s.Bm, np, nu);
  init(s.Cm, np, np);
  for (int32_t q = 0; q < N; ++q) {
    const bool prow = pm[q] != 0;
    for (int32_t k = As.ptr[q]; k < As.ptr[q + 1]; ++k) {
      const int32_t j = As.col[k];
      const bool pcol = pm[j] != 0;
      orc_mat& M = prow ? (pcol ? s.Cm : s.Bm) : (pcol ? s.BTm : s.Au);
      M.col.push_back(nid[j]);
      M.val.push_back(As.val[k]);
    }
    orc_mat& M1 = prow ? s.Bm : s.Au;
    orc_mat& M2 = prow ? s.Cm : s.BTm;
    M1.ptr[nid[q] + 1] = (int32_t)M1.col.size();
    M2.ptr[nid[q] + 1] = (int32_t)M2.col.size();
  }
  s.Shat_diag.assign(np, 0.0);
  s.mS.assign(np, 0.0);
  for (int32_t i = 0; i < np; ++i) {
    const int64_t kd = find_block(s.Cm, i, i);
    if (kd < 0) return ORC_EZERODIAG;
    double sum = 0.0;
    if (s.p.schur_shat == 1)
      for (int32_t k = s.Bm.ptr[i]; k < s.Bm.ptr[i + 1]; ++k) {
        const int32_t J = s.Bm.col[k];
        const int64_t kJJ = find_block(s.Au, J, J), kJi = find_block(s.BTm, J, i);
        if (kJJ < 0) return ORC_EZERODIAG;
        if (kJi < 0) continue;
        const double diag = s.Au.val[kJJ];
        if (diag == 0.0) return ORC_EZERODIAG;
        const double t = s.Bm.val[k] * (1.0 / diag);
        sum = sum + t * s.BTm.val[kJi];
      }
    s.Shat_diag[i] = s.Cm.val[kd] - sum;
    double den = 0.0;
    for (int32_t k = s.Cm.ptr[i]; k < s.Cm.ptr[i + 1]; ++k) {
      const double v = (k == kd) ? s.Shat_diag[i] : s.Cm.val[k];
      den = den + v * v;
    }
    if (den == 0.0) return ORC_EZERODIAG;
    s.mS[i] = s.Shat_diag[i] / den;
  }
  s.Bms = s.p.hier_f32 ? narrowed(s.Bm) : s.Bm;
  s.BTms = s.p.hier_f32 ? narrowed(s.BTm) : s.BTm;
  s.mSs = s.mS;
  if (s.p.hier_f32)
    for (double& v : s.mSs) v = f32r(v);
  return ORC_OK;
}

// u* = V(r_u);  p = m_S o (r_p - B u*);  r_u' = r_u - B^T p;  u = V(r_u');  z = (u, p) by the maps
static void schur_apply_pmask(const orc_solver& s, const double* r, double* z) {
  const bool rf = s.p.vec_f32 != 0;
  const int32_t nu = (int32_t)s.uidx.size(), np = (int32_t)s.pidx.size();
  vector<double> ru(nu), rp(np);
  for (int32_t i = 0; i < nu; ++i) ru[i] = rf ? f32r(r[s.uidx[i]]) : r[s.uidx[i]];
  for (int32_t i = 0; i < np; ++i) rp[i] = rf ? f32r(r[s.pidx[i]]) : r[s.pidx[i]];
  vector<double> us, u, p(np), ru2(nu);
  vcycle(s, 0, ru, us);
  for (int32_t i = 0; i < np; ++i) {
    double acc = 0.0;
    for (int32_t k = s.Bms.ptr[i]; k < s.Bms.ptr[i + 1]; ++k) acc = acc + s.Bms.val[k] * us[s.Bms.col[k]];
    const double v = s.mSs[i] * (rp[i] - acc);
    p[i] = rf ? f32r(v) : v;
  }
  for (int32_t i = 0; i < nu; ++i) {
    double acc = 0.0;
    for (int32_t k = s.BTms.ptr[i]; k < s.BTms.ptr[i + 1]; ++k) acc = acc + s.BTms.val[k] * p[s.BTms.col[k]];
    const double v = ru[i] - acc;
    ru2[i] = rf ? f32r(v) : v;
  }
  vcycle(s, 0, ru2, u);
  for (int32_t i = 0; i < nu; ++i) z[s.uidx[i]] = u[i];
  for (int32_t i = 0; i < np; ++i) z[s.pidx[i]] = p[i];
}

static void schur_apply(const orc_solver& s, const double* r, double* z) {
  if (s.masked) {
    schur_apply_pmask(s, r, z);
    return;
  }
  const orc_mat& A = s.A;
  const int b = A.b, pc = s.p.schur_p_component, bu = b - 1;
  const bool rf = s.p.vec_f32 != 0;
  const int32_t n = A.n;
  vector<double> ru((size_t)n * bu), rp(n);
  for (int32_t I = 0; I < n; ++I) {
    for (int d = 0; d < bu; ++d) {
      double v = r[(int64_t)I * b + s.vel[d]];
      ru[(int64_t)I * bu + d] = rf ? f32r(v) : v;
    }
    double v = r[(int64_t)I * b + pc];
    rp[I] = rf ? f32r(v) : v;
  }
  vector<double> us, u;
  vcycle(s, 0, ru, us);
  vector<double> p(n);
  for (int32_t I = 0; I < n; ++I) {  // p = m_S o (r_p - B u*)
    double acc = 0.0;
    for (int32_t k = A.ptr[I]; k < A.ptr[I + 1]; ++k)
      for (int d = 0; d < bu; ++d) acc = acc + s.Bs[(size_t)k * bu + d] * us[(int64_t)A.col[k] * bu + d];
    double v = s.mSs[I] * (rp[I] - acc);
    p[I] = rf ? f32r(v) : v;
  }
  vector<double> ru2((size_t)n * bu);
  for (int32_t I = 0; I < n; ++I) {  // r_u' = r_u - B^T p
    for (int d = 0; d < bu; ++d) {
      double acc = 0.0;
      for (int32_t k = A.ptr[I]; k < A.ptr[I + 1]; ++k)
        acc = acc + s.BTs[(size_t)k * bu + d] * p[A.col[k]];
      double v = ru[(int64_t)I * bu + d] - acc;
      ru2[(int64_t)I * bu + d] = rf ? f32r(v) : v;
    }
  }
  vcycle(s, 0, ru2, u);
  for (int32_t I = 0; I < n; ++I) {
    for (int d = 0; d < bu; ++d) z[(int64_t)I * b + s.vel[d]] = u[(int64_t)I * bu + d];
    z[(int64_t)I * b + pc] = p[I];
  }
}

static void precond(const orc_solver& s, const double* r, double* z) {
  const int64_t N = (int64_t)s.A.n * s.A.b;
  if (s.p.precond == ORC_PC_NONE) {
    std::copy(r, r + N, z);
    return;
  }
  if (s.schur) {
    schur_apply(s, r, z);
    return;
  }
  // monolithic AMG: narrow once, V-cycle, widen exactly (C9 precision paragraph)
  vector<double> f(r, r + N), x;
  if (s.p.vec_f32)
    for (double& v : f) v = f32r(v);
  vcycle(s, 0, f, x);
  std::copy(x.begin(), x.end(), z);
}

extern "C" int orc_setup(const orc_mat* A, const orc_params* p, orc_solver** out) {
  if (!A || !p || !out || A->n != A->m) return ORC_EINVAL;
  if ((p->smoother == ORC_ILU0 || p->smoother == ORC_ILUT) && p->ilu_sweeps < 1) return ORC_EINVAL;
  if (p->smoother == ORC_ILUT && (!(p->ilut_tau >= 0.0) || p->ilut_p < 0)) return ORC_EINVAL;
  orc_solver* s = new orc_solver;
  s->p = *p;
  s->A = *A;
  int rc = ORC_OK;
  if (p->precond == ORC_PC_SCHUR) {
    s->schur = true;
    rc = schur_setup(*s);
    if (rc == ORC_OK && p->schur_u_scalar) s->Au_s = scalar_expansion(s->Au);
    if (rc == ORC_OK) rc = build_hierarchy(*s, p->schur_u_scalar ? s->Au_s : s->Au, p->schur_u_scalar ? s->Au.b : 1);
  } else if (p->precond == ORC_PC_AMG) {
    rc = build_hierarchy(*s, s->A);
  }
  if (rc != ORC_OK) {
    delete s;
    return rc;
  }
  *out = s;
  return ORC_OK;
}

extern "C" int orc_setup_pmask(const orc_mat* A, const uint8_t* pmask, const orc_params* p, orc_solver** out) {
  if (!A || !pmask || !p || !out || A->n != A->m || p->precond != ORC_PC_SCHUR) return ORC_EINVAL;
  if (p->schur_shat == 2 || ((p->smoother == ORC_ILU0 || p->smoother == ORC_ILUT) && p->ilu_sweeps < 1)) return ORC_EINVAL;
  if (p->smoother == ORC_ILUT && (!(p->ilut_tau >= 0.0) || p->ilut_p < 0)) return ORC_EINVAL;
  orc_solver* s = new orc_solver;
  s->p = *p;
  s->A = *A;
  s->schur = true;
  s->masked = true;
  vector<uint8_t> pm(pmask, pmask + (size_t)A->n * A->b);
  int rc = schur_setup_pmask(*s, pm);
  // P slabs of block rows (C12): the velocity unknowns of slab r, numbered in ascending scalar
  // order, are the range [bu[r], bu[r+1]) -- the U-solver hierarchy's level-0 slabs (R27)
  vector<int32_t> cb = slab_bounds(A->n, p->nparts < 1 ? 1 : p->nparts), bu(cb.size(), 0);
  for (size_t r = 1; r < cb.size(); ++r) {
    int32_t cnt = 0;
    for (int64_t q = 0; q < (int64_t)cb[r] * A->b; ++q) cnt += pm[q] ? 0 : 1;
    bu[r] = cnt;
  }
  if (rc == ORC_OK) rc = build_hierarchy(*s, s->Au, 1, &bu);
  if (rc != ORC_OK) {
    delete s;
    return rc;
  }
  *out = s;
  return ORC_OK;
}

extern "C" void orc_free(orc_solver* s) { delete s; }
extern "C" int32_t orc_levels(const orc_solver* s) {
  return s->p.precond == ORC_PC_NONE ? 0 : (int32_t)s->lv.size() + 1;
}

extern "C" const orc_mat* orc_level_mat(const orc_solver* s, int32_t level, int32_t which) {
  if (level < 0) return nullptr;
  if ((size_t)level == s->lv.size()) return which == 0 ? &s->Acoarse : nullptr;
  if ((size_t)level > s->lv.size()) return nullptr;
  const Level& L = s->lv[level];
  return which == 0 ? &L.A : which == 1 ? &L.P : which == 2 ? &L.R
       : which == 4 ? (L.L.n ? &L.L : nullptr) : which == 5 ? (L.U.n ? &L.U : nullptr) : nullptr;
}
extern "C" int orc_level_smooth(const orc_solver* s, int32_t level, const double* f, double* x) {
  if (level < 0 || (size_t)level >= s->lv.size()) return ORC_EINVAL;
  const Level& L = s->lv[level];
  pre_smooth(*s, L, f, x, s->p.vec_f32 != 0);
  return ORC_OK;
}
extern "C" const int32_t* orc_level_agg(const orc_solver* s, int32_t level) {
  if (level < 0 || (size_t)level >= s->lv.size()) return nullptr;
  return s->lv[level].agg.data();
}
extern "C" const double* orc_level_M(const orc_solver* s, int32_t level) {
  if (level < 0 || (size_t)level >= s->lv.size()) return nullptr;
  return s->lv[level].M.data();
}
extern "C" const orc_mat* orc_schur_Au(const orc_solver* s) { return s->schur ? &s->Au : nullptr; }
extern "C" const orc_mat* orc_schur_Au_amg(const orc_solver* s) {
  return s->schur ? (s->p.schur_u_scalar ? &s->Au_s : &s->Au) : nullptr;
}
extern "C" const double* orc_schur_Shat_diag(const orc_solver* s) {
  return s->schur ? s->Shat_diag.data() : nullptr;
}
extern "C" const double* orc_schur_mS(const orc_solver* s) { return s->schur ? s->mS.data() : nullptr; }
extern "C" int32_t orc_schur_np(const orc_solver* s) {
  return s->schur ? (s->masked ? (int32_t)s->pidx.size() : s->A.n) : 0;
}

extern "C" int orc_vcycle(const orc_solver* s, const double* f, double* x) {
  if (s->p.precond == ORC_PC_NONE) return ORC_EINVAL;
  const orc_mat& A0 = s->lv.empty() ? s->Acoarse : s->lv[0].A;
  vector<double> fv(f, f + (int64_t)A0.n * A0.b), xv;
  vcycle(*s, 0, fv, xv);
  std::copy(xv.begin(), xv.end(), x);
  return ORC_OK;
}

extern "C" int orc_precond(const orc_solver* s, const double* r, double* z) {
  precond(*s, r, z);
  return ORC_OK;
}

// ---------------------------------------------------------------- C11 Krylov
static bool is_fin(double v) { return std::isfinite(v); }

// PCG (cfg 1).  Stop on the recurrence ||r|| <= rtol ||b||, then verify the true
// residual; if it fails, continue from r = b - A x.
static int solve_cg(const orc_solver& s, const double* bp, double* xp, double rtol,
                    orc_report* rep, double* hist) {
  const int64_t N = (int64_t)s.A.n * s.A.b;
  vector<double> b(bp, bp + N), x(xp, xp + N), r(N), z(N), p(N), q(N);
  const double nb = nrm2(b);
  residual(s.A, b.data(), x.data(), r.data(), false);
  double nr = nrm2(r);
  if (hist) hist[0] = nr / nb;
  int it = 0;
  int status = ORC_NOT_CONVERGED;
  if (nr <= rtol * nb) status = ORC_OK;
  bool restart = true;
  double rho = 0.0;
  while (status != ORC_OK && it < s.p.maxiter) {
    if (restart) {
      precond(s, r.data(), z.data());
      p = z;
      rho = dot(r, z);
      restart = false;
    }
    spmv(s.A, 1.0, p.data(), 0.0, q.data(), false);
    double pq = dot(p, q);
    if (pq == 0.0 || !is_fin(pq)) {
      status = ORC_EBREAKDOWN;
      break;
    }
    double alpha = rho / pq;
    for (int64_t i = 0; i < N; ++i) x[i] = x[i] + alpha * p[i];
    for (int64_t i = 0; i < N; ++i) r[i] = r[i] - alpha * q[i];
    ++it;
    stamp(it);
    nr = nrm2(r);
    if (hist) hist[it] = nr / nb;
    if (nr <= rtol * nb) {
      residual(s.A, b.data(), x.data(), r.data(), false);
      if (nrm2(r) <= rtol * nb) {
        status = ORC_OK;
        break;
      }
      restart = true;
      continue;
    }
    precond(s, r.data(), z.data());
    double rho_new = dot(r, z);
    double beta = rho_new / rho;
    for (int64_t i = 0; i < N; ++i) p[i] = z[i] + beta * p[i];
    rho = rho_new;
  }
  std::copy(x.begin(), x.end(), xp);
  rep->iters = it;
  rep->restarts = 0;
  residual(s.A, b.data(), x.data(), r.data(), false);
  rep->relres_true = nrm2(r) / nb;
  rep->converged = status == ORC_OK;
  return status;
}

// Right-preconditioned BiCGStab (van der Vorst), shadow rhat = r0, half-step exit
// on ||s|| <= rtol ||b||; breakdown (|rho| <= 1e-30 ||b||^2, rhat.v = 0, t.t = 0,
// omega = 0 or non-finite) -> one restart, then ORC_EBREAKDOWN (C11).
static int solve_bicgstab(const orc_solver& s, const double* bp, double* xp, double rtol,
                          orc_report* rep, double* hist) {
  const int64_t N = (int64_t)s.A.n * s.A.b;
  vector<double> b(bp, bp + N), x(xp, xp + N), r(N), rh(N), p(N), ph(N), v(N), sv(N), sh(N), t(N);
  const double nb = nrm2(b);
  residual(s.A, b.data(), x.data(), r.data(), false);
  if (hist) hist[0] = nrm2(r) / nb;
  int it = 0, restarts = 0;
  int status = ORC_NOT_CONVERGED;
  if (nrm2(r) <= rtol * nb) status = ORC_OK;
  rh = r;
  bool first = true;
  double rho_old = 1.0, alpha = 1.0, omega = 1.0;
  auto do_restart = [&]() -> bool {
    if (restarts >= 1) return false;
    ++restarts;
    residual(s.A, b.data(), x.data(), r.data(), false);
    rh = r;
    first = true;
    return true;
  };
  auto verify = [&]() -> bool {  // true residual check
    residual(s.A, b.data(), x.data(), r.data(), false);
    if (nrm2(r) <= rtol * nb) return true;
    rh = r;
    first = true;
    return false;
  };
  while (status != ORC_OK && it < s.p.maxiter) {
    double rho = dot(rh, r);
    if (!(std::fabs(rho) > 1e-30 * nb * nb) || !is_fin(rho)) {
      if (do_restart()) continue;
      status = ORC_EBREAKDOWN;
      break;
    }
    if (first) {
      p = r;
      first = false;
    } else {
      double beta = (rho / rho_old) * (alpha / omega);
      for (int64_t i = 0; i < N; ++i) p[i] = r[i] + beta * (p[i] - omega * v[i]);
    }
    precond(s, p.data(), ph.data());
    spmv(s.A, 1.0, ph.data(), 0.0, v.data(), false);
    double rv = dot(rh, v);
    if (rv == 0.0 || !is_fin(rv)) {
      if (do_restart()) continue;
      status = ORC_EBREAKDOWN;
      break;
    }
    alpha = rho / rv;
    for (int64_t i = 0; i < N; ++i) sv[i] = r[i] - alpha * v[i];
    ++it;
    stamp(it);
    double ns = nrm2(sv);
    if (ns <= rtol * nb) {
      for (int64_t i = 0; i < N; ++i) x[i] = x[i] + alpha * ph[i];
      if (hist) hist[it] = ns / nb;
      if (verify()) {
        status = ORC_OK;
        break;
      }
      continue;
    }
    precond(s, sv.data(), sh.data());
    spmv(s.A, 1.0, sh.data(), 0.0, t.data(), false);
    double tt = dot(t, t);
    if (tt == 0.0 || !is_fin(tt)) {
      if (do_restart()) continue;
      status = ORC_EBREAKDOWN;
      break;
    }
    omega = dot(t, sv) / tt;
    for (int64_t i = 0; i < N; ++i) x[i] = x[i] + alpha * ph[i] + omega * sh[i];
    for (int64_t i = 0; i < N; ++i) r[i] = sv[i] - omega * t[i];
    rho_old = rho;
    double nr = nrm2(r);
    if (hist) hist[it] = nr / nb;
    if (omega == 0.0 || !is_fin(omega)) {
      if (do_restart()) continue;
      status = ORC_EBREAKDOWN;
      break;
    }
    if (nr <= rtol * nb && verify()) {
      status = ORC_OK;
      break;
    }
  }
  std::copy(x.begin(), x.end(), xp);
  rep->iters = it;
  rep->restarts = restarts;
  residual(s.A, b.data(), x.data(), r.data(), false);
  rep->relres_true = nrm2(r) / nb;
  rep->converged = status == ORC_OK;
  return status;
}

// Flexible right-preconditioned GMRES(m) (C11): z_j = M v_j, w = A z_j, CGS2 Arnoldi
// (two classical Gram-Schmidt passes, coefficients summed), Givens rotations, stop
// when |g_{j+1}| <= rtol ||b||, x += Z y, true residual recomputed at every cycle end.
// Listing 1 names GMRES; the flexible form is the C11 reading.
// If hist != NULL, hist[j] = true ||b - A x_j|| / ||b|| for every Arnoldi step j.
static int solve_gmres(const orc_solver& s, const double* bp, double* xp, double rtol,
                       orc_report* rep, double* hist) {
  const int64_t N = (int64_t)s.A.n * s.A.b;
  const int m = s.p.gmres_m;
  vector<double> b(bp, bp + N), x(xp, xp + N), r(N), w(N), tmpx(N), tmpr(N);
  vector<vector<double>> V(m + 1, vector<double>(N)), Z(m, vector<double>(N));
  vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m), h(m + 1), h2(m + 1);
  vector<double> Rg((size_t)(m + 1) * (m + 1), 0.0);  // gmres_ortho = 1: Cholesky factor of t^T t
  const double nb = nrm2(b);
  residual(s.A, b.data(), x.data(), r.data(), false);
  double beta = nrm2(r);
  if (hist) hist[0] = beta / nb;
  int it = 0, cycles = 0;
  int status = ORC_NOT_CONVERGED;
  if (beta <= rtol * nb) status = ORC_OK;
  while (status != ORC_OK && it < s.p.maxiter) {
    ++cycles;
    for (int64_t i = 0; i < N; ++i) V[0][i] = r[i] / beta;
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    std::fill(Rg.begin(), Rg.end(), 0.0);
    Rg[0] = 1.0;
    int j = 0;
    bool stop = false;
    for (; j < m && !stop; ++j) {
      precond(s, V[j].data(), Z[j].data());
      spmv(s.A, 1.0, Z[j].data(), 0.0, w.data(), false);
      double hn;
      if (s.p.gmres_ortho == 0) {  // CGS2 (C11)
        for (int i = 0; i <= j; ++i) h[i] = dot(V[i], w);
        for (int i = 0; i <= j; ++i)
          for (int64_t q = 0; q < N; ++q) w[q] = w[q] - h[i] * V[i][q];
        for (int i = 0; i <= j; ++i) h2[i] = dot(V[i], w);
        for (int i = 0; i <= j; ++i)
          for (int64_t q = 0; q < N; ++q) w[q] = w[q] - h2[i] * V[i][q];
        for (int i = 0; i <= j; ++i) h[i] = h[i] + h2[i];
        hn = nrm2(w);
        if (hn != 0.0)
          for (int64_t q = 0; q < N; ++q) V[j + 1][q] = w[q] / hn;
      } else {
        // two-pass Gram/Cholesky orthogonalisation (reading R22).  V holds t_i: once-
        // orthogonalised unit vectors, t = Q R with Q orthonormal and R the Cholesky factor
        // of G = t^T t.  p = t^T w; h = R^-T p (= Q^T w); w1 = w - t R^-1 h (= w - Q h);
        // q = t^T w1, ||w1||; t_{j+1} = w1 / ||w1||; R(:, j+1) = R^-T q / ||w1||,
        // R(j+1, j+1) = sqrt(1 - |R(0:j, j+1)|^2); H(:, j) = h + ||w1|| R(:, j+1).
        const int k = j + 1;
        vector<double> p(k), hv(k), cv(k), qv(k), h2v(k);
        // pass 1; gmres_ortho = 2 (reading R23): the dots read the basis rounded to fp32;
        // 3 (R28): rounded to fp16 at unit-rms scale
        for (int i = 0; i < k; ++i)
          p[i] = s.p.gmres_ortho == 2 ? dot_f32_basis(V[i], w)
                 : s.p.gmres_ortho == 3 ? dot_f16_basis(V[i], w) : dot(V[i], w);
        // project(pin): hout = R^-T pin, cv = R^-1 hout, w = w - t cv, qv = t^T w
        auto project = [&](const vector<double>& pin, vector<double>& hout) {
          for (int i = 0; i < k; ++i) {
            double t = pin[i];
            for (int l = 0; l < i; ++l) t = t - Rg[(size_t)l * (m + 1) + i] * hout[l];
            hout[i] = t / Rg[(size_t)i * (m + 1) + i];
          }
          for (int i = k - 1; i >= 0; --i) {
            double t = hout[i];
            for (int l = i + 1; l < k; ++l) t = t - Rg[(size_t)i * (m + 1) + l] * cv[l];
            cv[i] = t / Rg[(size_t)i * (m + 1) + i];
          }
          for (int i = 0; i < k; ++i)
            for (int64_t q = 0; q < N; ++q) w[q] = w[q] - cv[i] * V[i][q];
          for (int i = 0; i < k; ++i) qv[i] = dot(V[i], w);
        };
        project(p, hv);
        hn = 0.0;
        for (int pass = 0;; ++pass) {
          const double h0 = nrm2(w);
          hn = h0;
          if (h0 == 0.0) break;
          double ss = 0.0;
          for (int i = 0; i < k; ++i) {
            double t = qv[i] / h0;
            for (int l = 0; l < i; ++l) t = t - Rg[(size_t)l * (m + 1) + i] * Rg[(size_t)l * (m + 1) + k];
            Rg[(size_t)i * (m + 1) + k] = t / Rg[(size_t)i * (m + 1) + i];
            ss = ss + Rg[(size_t)i * (m + 1) + k] * Rg[(size_t)i * (m + 1) + k];
          }
          // reorthogonalisation safeguard: w still far from orthogonal to span(V)
          if (pass == 0 && (ss > 0.5 || !(1.0 - ss > 1e-8))) {
            project(qv, h2v);
            for (int i = 0; i < k; ++i) hv[i] = hv[i] + h2v[i];
            continue;
          }
          for (int64_t q = 0; q < N; ++q) V[j + 1][q] = w[q] / h0;
          Rg[(size_t)k * (m + 1) + k] = 1.0 - ss > 0.0 ? std::sqrt(1.0 - ss) : 0.0;
          for (int i = 0; i < k; ++i) hv[i] = hv[i] + h0 * Rg[(size_t)i * (m + 1) + k];
          hn = h0 * Rg[(size_t)k * (m + 1) + k];
          break;
        }
        for (int i = 0; i < k; ++i) h[i] = hv[i];
      }
      h[j + 1] = hn;
      for (int i = 0; i < j; ++i) {  // previous rotations
        double t = cs[i] * h[i] + sn[i] * h[i + 1];
        h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
        h[i] = t;
      }
      double rr = std::hypot(h[j], h[j + 1]);
      if (rr == 0.0 || !is_fin(rr)) {
        status = ORC_EBREAKDOWN;
        stop = true;
        break;
      }
      cs[j] = h[j] / rr;
      sn[j] = h[j + 1] / rr;
      h[j] = rr;
      h[j + 1] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = h[i];
      ++it;
      stamp(it);
      if (hist) {  // true residual of the current iterate x + Z y_j
        for (int i = j; i >= 0; --i) {
          double t = g[i];
          for (int k = i + 1; k <= j; ++k) t = t - H[(size_t)i * m + k] * y[k];
          y[i] = t / H[(size_t)i * m + i];
        }
        tmpx = x;
        for (int i = 0; i <= j; ++i)
          for (int64_t q = 0; q < N; ++q) tmpx[q] = tmpx[q] + y[i] * Z[i][q];
        residual(s.A, b.data(), tmpx.data(), tmpr.data(), false);
        hist[it] = nrm2(tmpr) / nb;
      }
      if (std::fabs(g[j + 1]) <= rtol * nb || it >= s.p.maxiter || hn == 0.0) stop = true;
    }
    if (status == ORC_EBREAKDOWN) break;
    int k = j;  // number of Arnoldi steps in this cycle
    for (int i = k - 1; i >= 0; --i) {
      double t = g[i];
      for (int c = i + 1; c < k; ++c) t = t - H[(size_t)i * m + c] * y[c];
      y[i] = t / H[(size_t)i * m + i];
    }
    for (int i = 0; i < k; ++i)
      for (int64_t q = 0; q < N; ++q) x[q] = x[q] + y[i] * Z[i][q];
    residual(s.A, b.data(), x.data(), r.data(), false);
    beta = nrm2(r);
    if (beta <= rtol * nb) status = ORC_OK;
  }
  std::copy(x.begin(), x.end(), xp);
  rep->iters = it;
  rep->restarts = cycles > 0 ? cycles - 1 : 0;
  residual(s.A, b.data(), x.data(), r.data(), false);
  rep->relres_true = nrm2(r) / nb;
  rep->converged = status == ORC_OK;
  return status;
}

// ---- IDR(s) (Table 1: the paper's outer solver for V1-V4, s = 5;
// "We use the IDR(s) solver [sonneveld2009idr]").  Reading R17: the
// bi-orthogonal IDR(s) of van Gijzen & Sonneveld (ACM TOMS 38(1) 5, 2011, "an elegant
// IDR(s) variant that efficiently exploits bi-orthogonality properties"), right
// preconditioned, omega by "maintaining the convergence" with kappa = 0.7,
// no residual smoothing.  Shadow space P: s vectors of N(0,1) draws of the
// counter RNG (below; stream 6, idx = (64 seed + s restarts + j) N + i), orthonormalised
// by modified Gram-Schmidt.  One iteration = one product with A (and one preconditioner
// application): s per IDR cycle plus the dimension-reduction step.  Stop on the
// recurrence ||r|| <= rtol ||b||, then verify the true residual; if it fails, restart
// the cycle from r = b - A x.  Breakdown (M_kk = 0, omega = 0, non-finite) -> one restart
// with a fresh shadow space, then ORC_EBREAKDOWN.
//
// Counter RNG (written out here, independently of gen/): SplitMix64
// finaliser mix, R(stream, idx) = mix(mix(SEED ^ (stream << 56)) ^ idx), SEED = 200606052,
// U01 = (R >> 11) 2^-53, N01 = sqrt(-2 ln(1 - U01(2 idx))) cos(2 pi U01(2 idx + 1)).
static uint64_t rng_mix(uint64_t z) {  // the SplitMix64 finaliser (no increment)
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static double rng_u01(uint64_t stream, uint64_t idx) {
  const uint64_t r = rng_mix(rng_mix(200606052ULL ^ (stream << 56)) ^ idx);
  return (double)(r >> 11) * (1.0 / 9007199254740992.0);
}
static double rng_n01(uint64_t stream, uint64_t idx) {
  const double u1 = 1.0 - rng_u01(stream, 2 * idx), u2 = rng_u01(stream, 2 * idx + 1);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
}

static void idrs_shadow(int64_t N, int sdim, uint64_t base, vector<vector<double>>& P) {
  P.assign(sdim, vector<double>(N));
  for (int j = 0; j < sdim; ++j) {
    for (int64_t i = 0; i < N; ++i) P[j][i] = rng_n01(6, (base + (uint64_t)j) * (uint64_t)N + (uint64_t)i);
    for (int l = 0; l < j; ++l) {  // modified Gram-Schmidt
      const double d = dot(P[l], P[j]);
      for (int64_t i = 0; i < N; ++i) P[j][i] = P[j][i] - d * P[l][i];
    }
    const double nr = nrm2(P[j]);
    for (int64_t i = 0; i < N; ++i) P[j][i] = P[j][i] / nr;
  }
}

static int solve_idrs(const orc_solver& s, const double* bp, double* xp, double rtol, orc_report* rep,
                      double* hist) {
  const int64_t N = (int64_t)s.A.n * s.A.b;
  const int sd = s.p.idrs_s;
  const double kappa = 0.7;
  vector<double> b(bp, bp + N), x(xp, xp + N), r(N), v(N), vh(N), t(N);
  const double nb = nrm2(b);
  residual(s.A, b.data(), x.data(), r.data(), false);
  double nr = nrm2(r);
  if (hist) hist[0] = nr / nb;
  int it = 0, restarts = 0, status = ORC_NOT_CONVERGED;
  if (nr <= rtol * nb) status = ORC_OK;
  vector<vector<double>> P, G(sd, vector<double>(N, 0.0)), U(sd, vector<double>(N, 0.0));
  vector<double> M((size_t)sd * sd, 0.0), f(sd), c(sd);
  uint64_t base = 64ULL * (uint64_t)s.p.idrs_seed;
  idrs_shadow(N, sd, base, P);
  auto reset = [&]() {
    for (int j = 0; j < sd; ++j) std::fill(G[j].begin(), G[j].end(), 0.0), std::fill(U[j].begin(), U[j].end(), 0.0);
    std::fill(M.begin(), M.end(), 0.0);
    for (int j = 0; j < sd; ++j) M[(size_t)j * sd + j] = 1.0;
  };
  reset();
  double om = 1.0;
  // true-residual check after the recurrence converged; false -> restart the cycle
  auto converged_true = [&]() -> bool {
    residual(s.A, b.data(), x.data(), r.data(), false);
    if (nrm2(r) <= rtol * nb) return true;
    reset();
    om = 1.0;
    return false;
  };
  auto breakdown = [&]() -> bool {  // true -> restarted, false -> give up
    if (restarts >= 1) return false;
    ++restarts;
    residual(s.A, b.data(), x.data(), r.data(), false);
    base += (uint64_t)sd;
    idrs_shadow(N, sd, base, P);
    reset();
    om = 1.0;
    return true;
  };
  while (status != ORC_OK && it < s.p.maxiter) {
    for (int i = 0; i < sd; ++i) f[i] = dot(P[i], r);
    bool restart_cycle = false;
    for (int k = 0; k < sd && status != ORC_OK && it < s.p.maxiter; ++k) {
      // lower-triangular solve M[k:s, k:s] c = f[k:s]
      for (int i = k; i < sd; ++i) {
        double a = f[i];
        for (int l = k; l < i; ++l) a = a - M[(size_t)i * sd + l] * c[l];
        c[i] = a / M[(size_t)i * sd + i];
      }
      for (int64_t q = 0; q < N; ++q) {
        double a = r[q];
        for (int i = k; i < sd; ++i) a = a - c[i] * G[i][q];
        v[q] = a;
      }
      precond(s, v.data(), vh.data());
      for (int64_t q = 0; q < N; ++q) {
        double a = om * vh[q];
        for (int i = k; i < sd; ++i) a = a + c[i] * U[i][q];
        U[k][q] = a;
      }
      spmv(s.A, 1.0, U[k].data(), 0.0, G[k].data(), false);
      for (int i = 0; i < k; ++i) {  // bi-orthogonalise G_k against P_0..P_{k-1}
        const double alpha = dot(P[i], G[k]) / M[(size_t)i * sd + i];
        for (int64_t q = 0; q < N; ++q) G[k][q] = G[k][q] - alpha * G[i][q];
        for (int64_t q = 0; q < N; ++q) U[k][q] = U[k][q] - alpha * U[i][q];
      }
      for (int i = k; i < sd; ++i) M[(size_t)i * sd + k] = dot(P[i], G[k]);
      const double mkk = M[(size_t)k * sd + k];
      if (mkk == 0.0 || !is_fin(mkk)) {
        if (breakdown()) {
          restart_cycle = true;
          break;
        }
        status = ORC_EBREAKDOWN;
        break;
      }
      const double beta = f[k] / mkk;
      for (int64_t q = 0; q < N; ++q) r[q] = r[q] - beta * G[k][q];
      for (int64_t q = 0; q < N; ++q) x[q] = x[q] + beta * U[k][q];
      ++it;
      stamp(it);
      nr = nrm2(r);
      if (hist) hist[it] = nr / nb;
      if (nr <= rtol * nb) {
        if (converged_true()) status = ORC_OK;
        restart_cycle = true;
        break;
      }
      for (int i = k + 1; i < sd; ++i) f[i] = f[i] - beta * M[(size_t)i * sd + k];
    }
    if (status == ORC_OK || status == ORC_EBREAKDOWN || restart_cycle || it >= s.p.maxiter) continue;
    // dimension reduction: v = M^-1 r, t = A v, omega ("maintaining the convergence")
    precond(s, r.data(), vh.data());
    spmv(s.A, 1.0, vh.data(), 0.0, t.data(), false);
    const double tr = dot(t, r), tt = dot(t, t), nt = std::sqrt(tt);
    om = tr / tt;
    const double rho = std::fabs(tr) / (nt * nr);
    if (rho < kappa) om = om * kappa / rho;
    if (om == 0.0 || !is_fin(om)) {
      if (breakdown()) continue;
      status = ORC_EBREAKDOWN;
      break;
    }
    for (int64_t q = 0; q < N; ++q) r[q] = r[q] - om * t[q];
    for (int64_t q = 0; q < N; ++q) x[q] = x[q] + om * vh[q];
    ++it;
    stamp(it);
    nr = nrm2(r);
    if (hist) hist[it] = nr / nb;
    if (nr <= rtol * nb && converged_true()) status = ORC_OK;
  }
  std::copy(x.begin(), x.end(), xp);
  rep->iters = it;
  rep->restarts = restarts;
  residual(s.A, b.data(), x.data(), r.data(), false);
  rep->relres_true = nrm2(r) / nb;
  rep->converged = status == ORC_OK;
  return status;
}

extern "C" int orc_idrs_shadow(int64_t n, int32_t sdim, int64_t base, double* out) {
  vector<vector<double>> P;
  idrs_shadow(n, sdim, (uint64_t)base, P);
  for (int j = 0; j < sdim; ++j) std::copy(P[j].begin(), P[j].end(), out + (int64_t)j * n);
  return ORC_OK;
}

extern "C" int orc_solve_timed(const orc_solver* s, const double* b, double* x, double rtol,
                               orc_report* rep, double* stamps, int32_t cap) {
  g_stamps = stamps;
  g_stamps_cap = cap;
  g_t0 = std::chrono::steady_clock::now();
  if (stamps && cap > 0) stamps[0] = 0.0;
  const int rc = orc_solve(s, b, x, rtol, rep, nullptr);
  g_stamps = nullptr;
  g_stamps_cap = 0;
  return rc;
}

extern "C" int orc_solve(const orc_solver* s, const double* b, double* x, double rtol,
                         orc_report* rep, double* history) {
  const int64_t N = (int64_t)s->A.n * s->A.b;
  rep->levels = orc_levels(s);
  double nb = 0.0;
  for (int64_t i = 0; i < N; ++i) nb = nb + b[i] * b[i];
  if (nb == 0.0) {  // ||b|| = 0 -> x = 0, converged, relres 0
    std::fill(x, x + N, 0.0);
    rep->iters = 0;
    rep->converged = 1;
    rep->restarts = 0;
    rep->relres_true = 0.0;
    return ORC_OK;
  }
  switch (s->p.solver) {
    case ORC_CG: return solve_cg(*s, b, x, rtol, rep, history);
    case ORC_BICGSTAB: return solve_bicgstab(*s, b, x, rtol, rep, history);
    case ORC_GMRES: return solve_gmres(*s, b, x, rtol, rep, history);
    case ORC_IDRS: return solve_idrs(*s, b, x, rtol, rep, history);
    default: return ORC_EINVAL;
  }
}
