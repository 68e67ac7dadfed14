/* gen.c -- seeded synthetic inputs (see gen.h).  Built with -O2 -ffp-contract=off
 * -fopenmp; every value is a pure function of (kind, n, global index), so the
 * OpenMP split never changes a bit of the output. */
#include "gen.h"

#include <math.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

uint64_t gen_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t gen_rand(uint64_t stream, uint64_t idx) {
  return gen_mix(gen_mix(GEN_SEED ^ (stream << 56)) ^ idx);
}

double gen_u01(uint64_t stream, uint64_t idx) {
  return (double)(gen_rand(stream, idx) >> 11) * (1.0 / 9007199254740992.0);
}

double gen_uni(uint64_t stream, uint64_t idx, double a, double b) {
  return a + (b - a) * gen_u01(stream, idx);
}

double gen_n01(uint64_t stream, uint64_t idx) {
  double u1 = 1.0 - gen_u01(stream, 2 * idx);
  double u2 = gen_u01(stream, 2 * idx + 1);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

int gen_block_size(int kind, int b_rand27) {
  switch (kind) {
    case GEN_POISSON3: return 3;
    case GEN_STOKES: return 4;
    case GEN_RAND27: return b_rand27;
    default: return -1;
  }
}

/* ---- stencil enumeration (ascending column order) ---------------------- */

/* 7-point: offsets in ascending global-index order: -z, -y, -x, 0, +x, +y, +z */
static const int d7_dir[7] = {2, 1, 0, -1, 0, 1, 2};
static const int d7_sgn[7] = {-1, -1, -1, 0, 1, 1, 1};

static int in_grid7(int n, int64_t i, int64_t j, int64_t k, int t) {
  int d = d7_dir[t], s = d7_sgn[t];
  if (d < 0) return 1;
  int64_t c = (d == 0) ? i : (d == 1) ? j : k;
  c += s;
  return c >= 0 && c < n;
}

static int64_t row_len(int kind, int n, int64_t I) {
  int64_t i = I % n, j = (I / n) % n, k = I / ((int64_t)n * n);
  int64_t cnt = 0;
  if (kind == GEN_RAND27) {
    for (int dk = -1; dk <= 1; ++dk)
      for (int dj = -1; dj <= 1; ++dj)
        for (int di = -1; di <= 1; ++di) {
          int64_t a = i + di, bb = j + dj, c = k + dk;
          if (a >= 0 && a < n && bb >= 0 && bb < n && c >= 0 && c < n) ++cnt;
        }
    return cnt;
  }
  for (int t = 0; t < 7; ++t) cnt += in_grid7(n, i, j, k, t);
  return cnt;
}

int64_t gen_nnzb(int kind, int n, int64_t row_begin, int64_t row_end) {
  int64_t tot = 0;
#pragma omp parallel for reduction(+ : tot) schedule(static)
  for (int64_t I = row_begin; I < row_end; ++I) tot += row_len(kind, n, I);
  return tot;
}

static void fill_row(int kind, int n, int b, int64_t I, int32_t* col, double* val) {
  const int64_t nn = (int64_t)n * n;
  int64_t i = I % n, j = (I / n) % n, k = I / nn;
  const int bb = b * b;
  int64_t e = 0; /* block counter within the row */
  if (kind == GEN_RAND27) {
    for (int dk = -1; dk <= 1; ++dk)
      for (int dj = -1; dj <= 1; ++dj)
        for (int di = -1; di <= 1; ++di) {
          int64_t a = i + di, b2 = j + dj, c = k + dk;
          if (!(a >= 0 && a < n && b2 >= 0 && b2 < n && c >= 0 && c < n)) continue;
          int slot = 9 * (dk + 1) + 3 * (dj + 1) + (di + 1);
          int64_t J = a + n * (b2 + (int64_t)n * c);
          col[e] = (int32_t)J;
          double* blk = val + e * bb;
          for (int q = 0; q < bb; ++q)
            blk[q] = gen_n01(3, (uint64_t)((27 * I + slot) * bb + q));
          if (J == I)
            for (int r = 0; r < b; ++r) blk[r * b + r] += 30.0;
          ++e;
        }
    return;
  }
  for (int t = 0; t < 7; ++t) {
    if (!in_grid7(n, i, j, k, t)) continue;
    int d = d7_dir[t], s = d7_sgn[t];
    int64_t off = (d < 0) ? 0 : (d == 0 ? 1 : (d == 1 ? n : nn));
    int64_t J = I + s * off;
    col[e] = (int32_t)J;
    double* blk = val + e * bb;
    memset(blk, 0, sizeof(double) * bb);
    if (kind == GEN_POISSON3) {
      if (d < 0) {
        /* A_II = 6 I3 + 0.1 G G^T, G[r][c] = N01(1, 9 I + 3 r + c) */
        double G[3][3];
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) G[r][c] = gen_n01(1, (uint64_t)(9 * I + 3 * r + c));
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) {
            double g = G[r][0] * G[c][0];
            g = g + G[r][1] * G[c][1];
            g = g + G[r][2] * G[c][2];
            blk[r * 3 + c] = (r == c ? 6.0 : 0.0) + 0.1 * g;
          }
      } else {
        for (int r = 0; r < 3; ++r) blk[r * 3 + r] = -1.0;
      }
    } else { /* GEN_STOKES, h = 1/n: 1/h^2 = n^2, 1/(2h) = n/2 (exact) */
      const double ih2 = (double)n * (double)n;
      const double i2h = 0.5 * (double)n;
      if (d < 0) {
        blk[0] = 6.0 * ih2; blk[5] = 6.0 * ih2; blk[10] = 6.0 * ih2; blk[15] = -6.0;
      } else {
        for (int r = 0; r < 3; ++r) blk[r * 4 + r] = -ih2;
        blk[d * 4 + 3] = -(double)s * i2h; /* B^T: gradient part */
        blk[3 * 4 + d] = (double)s * i2h;  /* B: central divergence */
        blk[15] = 1.0;                     /* C = -h^2 * (1/h^2)(6,-1) stencil off-diagonal */
      }
    }
    ++e;
  }
}

int gen_matrix(int kind, int n, int b, int64_t row_begin, int64_t row_end,
               int32_t* ptr, int32_t* col, double* val) {
  if (n <= 0 || row_begin < 0 || row_end < row_begin) return -1;
  if ((int64_t)n * n * n < row_end) return -1;
  if (kind == GEN_POISSON3 && b != 3) return -1;
  if (kind == GEN_STOKES && b != 4) return -1;
  if (kind == GEN_RAND27 && (b < 1 || b > 4)) return -1;
  const int64_t nr = row_end - row_begin;
  ptr[0] = 0;
  for (int64_t r = 0; r < nr; ++r) ptr[r + 1] = ptr[r] + (int32_t)row_len(kind, n, row_begin + r);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < nr; ++r)
    fill_row(kind, n, b, row_begin + r, col + ptr[r], val + (int64_t)ptr[r] * b * b);
  return 0;
}

int gen_rhs(int rhs_kind, int n, int b, int64_t row_begin, int64_t row_end, double* out) {
  if (n <= 0 || row_end < row_begin) return -1;
  const int64_t nn = (int64_t)n * n;
  const double h = 1.0 / (double)n;
  const int64_t nr = row_end - row_begin;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < nr; ++r) {
    int64_t I = row_begin + r;
    int64_t i = I % n, j = (I / n) % n, k = I / nn;
    for (int c = 0; c < b; ++c) {
      uint64_t q = (uint64_t)(I * b + c);
      double v = 0.0;
      switch (rhs_kind) {
        case GEN_RHS_UNIFORM: v = gen_uni(2, q, -1.0, 1.0); break;
        case GEN_X_UNIFORM: v = gen_uni(4, q, -1.0, 1.0); break;
        case GEN_RHS_LID:
          v = (c == 0 && k == n - 1) ? (double)n * (double)n : 0.0;
          break;
        case GEN_RHS_FORCE_NOISE: {
          double x = ((double)i + 0.5) * h, y = ((double)j + 0.5) * h;
          double f = (c == 0) ? sin(M_PI * x) : (c == 1) ? cos(M_PI * y) : 0.0;
          v = f + 0.01 * gen_n01(5, q);
          break;
        }
        case GEN_RHS_LID_NOISE:
          v = ((c == 0 && k == n - 1) ? (double)n * (double)n : 0.0) + 0.01 * gen_n01(5, q);
          break;
        default: v = 0.0;
      }
      out[r * b + c] = v;
    }
  }
  return 0;
}
