/*
 * tileinv_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference tileinv numeric path, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER.  It
 * is never linked into, loaded by, or called from the product path
 * (paper_2504_19171_b200/), which fails loudly without its CUDA library.
 *
 * Parity is pinned: tests/test_oracle.py checks this file against the
 * reference itself (oracle/_ref, built from /root/reference/proj/src by
 * oracle/Makefile) and against the reference's own known-answer tests.
 *
 * Each routine follows the reference file:line named in its comment; tiles
 * are b x b row-major doubles exactly like proj/include/tileinv/kernels.hpp:14-22.
 * The symbolic half (fill, closure, column work lists) is restated in
 * oracle/oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- SplitMix64, proj/src/matgen.cpp:17-29 ------------------------------ */
static uint64_t sm_next(uint64_t* s) {
  *s += 0x9e3779b97f4a7c15ull;
  uint64_t z = *s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static double sm_unit(uint64_t* s) { return (double)(sm_next(s) >> 11) * 0x1.0p-53; }

/* generate_arrowhead (proj/src/matgen.cpp:59-120), pass 1: mask[ti*N+tj] = 1
 * for every tile that receives an entry (draw order r asc, c asc; a band slot
 * draws acceptance then value, an arrow entry draws only the value). */
void orc_generate_mask(long n, long w, long t, double density, uint64_t seed, int b, int N,
                       unsigned char* mask) {
  uint64_t st = seed;
  for (long r = 0; r < n; ++r) {
    long c0 = r < n - t ? (r - w > 0 ? r - w : 0) : 0;
    for (long c = c0; c < r; ++c) {
      if (r < n - t && !(sm_unit(&st) < density)) continue;
      sm_next(&st);
      mask[(size_t)(r / b) * N + (c / b)] = 1;
    }
  }
  for (int i = 0; i < N; ++i) mask[(size_t)i * N + i] = 1;
}

static long slot_of(const long* cs, const int* rows, int i, int j);

/* pass 2: values into the CSC tile payload; diagonal = |row| sum + 1 in draw
 * order (matgen.cpp:76-77, 98-102), padding diagonal 1 (matgen.cpp:103-106). */
void orc_generate_fill(long n, long w, long t, double density, uint64_t seed, int b, int N,
                       const long* cs, const int* rows, double* pay) {
  const size_t bb = (size_t)b * b;
  uint64_t st = seed;
  double* rowsum = (double*)calloc((size_t)n, sizeof(double));
  memset(pay, 0, sizeof(double) * bb * (size_t)cs[N]);
  for (long r = 0; r < n; ++r) {
    long c0 = r < n - t ? (r - w > 0 ? r - w : 0) : 0;
    for (long c = c0; c < r; ++c) {
      if (r < n - t && !(sm_unit(&st) < density)) continue;
      double v = 2.0 * sm_unit(&st) - 1.0;
      long s = slot_of(cs, rows, (int)(r / b), (int)(c / b));
      pay[(size_t)s * bb + (size_t)(r % b) * b + (c % b)] = v;
      rowsum[r] += fabs(v);
      rowsum[c] += fabs(v);
    }
  }
  for (long r = 0; r < (long)N * b; ++r) {
    long s = cs[r / b];
    pay[(size_t)s * bb + (size_t)(r % b) * b + (r % b)] = r < n ? rowsum[r] + 1.0 : 1.0;
  }
  free(rowsum);
}

/* ---- tile kernels, proj/src/kernels.cpp ---------------------------------- */
#define AT(p, r, c) (p)[(size_t)(r) * b + (c)]

/* potrf_tile, kernels.cpp:48-69 (Crout, lower read).  Returns -1 or the
 * failing in-tile pivot. */
static int potrf(int b, const double* a, double* l) {
  memset(l, 0, sizeof(double) * (size_t)b * b);
  for (int j = 0; j < b; ++j) {
    double s = AT(a, j, j);
    for (int k = 0; k < j; ++k) s -= AT(l, j, k) * AT(l, j, k);
    if (!(s > 0.0) || !isfinite(s)) return j;
    double d = sqrt(s);
    AT(l, j, j) = d;
    for (int i = j + 1; i < b; ++i) {
      double x = AT(a, i, j);
      for (int k = 0; k < j; ++k) x -= AT(l, i, k) * AT(l, j, k);
      AT(l, i, j) = x / d;
    }
  }
  return -1;
}

/* trsm_tile(kRight, kTrans) with lower L: X L^T = B, kernels.cpp:144-150
 * (effective upper: column substitution, ascending j). */
static void trsm_right_trans(int b, const double* L, double* B) {
  double* x = (double*)malloc(sizeof(double) * (size_t)b * b);
  for (int j = 0; j < b; ++j)
    for (int i = 0; i < b; ++i) {
      double s = AT(B, i, j);
      for (int k = 0; k < j; ++k) s -= AT(x, i, k) * AT(L, j, k);
      AT(x, i, j) = s / AT(L, j, j);
    }
  memcpy(B, x, sizeof(double) * (size_t)b * b);
  free(x);
}

/* syrk_tile, kernels.cpp:156-176: C -= A A^T lower, then mirrored. */
static void syrk(int b, double* C, const double* A) {
  for (int i = 0; i < b; ++i)
    for (int k = 0; k < b; ++k) {
      double aik = AT(A, i, k);
      for (int j = 0; j <= i; ++j) AT(C, i, j) -= aik * AT(A, j, k);
    }
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < i; ++j) AT(C, j, i) = AT(C, i, j);
}

/* gemm_tile with alpha = -1, kernels.cpp:178-208: C -= op(A) op(B), i-k-j. */
static void gemm_minus(int b, double* C, const double* A, int ta, const double* B, int tb) {
  for (int i = 0; i < b; ++i)
    for (int k = 0; k < b; ++k) {
      double aik = ta ? AT(A, k, i) : AT(A, i, k);
      for (int j = 0; j < b; ++j) AT(C, i, j) -= aik * (tb ? AT(B, j, k) : AT(B, k, j));
    }
}

/* trtri_tile on transpose_tile(L) (upper), kernels.cpp:71-100 + :38-46. */
static void trtri_upper_of_lower(int b, const double* L, double* U) {
  memset(U, 0, sizeof(double) * (size_t)b * b);
  for (int j = 0; j < b; ++j) {
    AT(U, j, j) = 1.0 / AT(L, j, j);
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int k = i + 1; k <= j; ++k) s += AT(L, k, i) * AT(U, k, j); /* t[i][k] = L[k][i] */
      AT(U, i, j) = -s / AT(L, i, i);
    }
  }
}

/* trmm_tile(kRight, kTrans) with upper U: B <- B U^T, kernels.cpp:210-246. */
static void trmm_right_trans_upper(int b, double* B, const double* U) {
  double* out = (double*)malloc(sizeof(double) * (size_t)b * b);
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < b; ++j) {
      double s = 0.0;
      for (int k = j; k < b; ++k) s += AT(B, i, k) * AT(U, j, k);
      AT(out, i, j) = s;
    }
  memcpy(B, out, sizeof(double) * (size_t)b * b);
  free(out);
}

/* lauum_tile on upper U, kernels.cpp:248-266: U U^T mirrored. */
static void lauum_upper(int b, const double* U, double* C) {
  for (int i = 0; i < b; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = 0.0;
      for (int k = i; k < b; ++k) s += AT(U, i, k) * AT(U, j, k);
      AT(C, i, j) = s;
    }
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < i; ++j) AT(C, j, i) = AT(C, i, j);
}

/* ---- drivers --------------------------------------------------------------
 * Patterns are passed as CSC over tile columns: col_start[N+1], rows[T]
 * ascending within each column (the reference's neighbors(j), layout.hpp:57),
 * payload[T][b][b] in the same slot order. */
static long slot_of(const long* cs, const int* rows, int i, int j) {
  long lo = cs[j], hi = cs[j + 1];
  while (lo < hi) {
    long mid = (lo + hi) / 2;
    if (rows[mid] < i) lo = mid + 1;
    else hi = mid;
  }
  return (lo < cs[j + 1] && rows[lo] == i) ? lo : -1;
}

/* factorize, cholesky.cpp:62-192, serial task order of symbolic_cholesky
 * (cholesky.cpp:17-49): per column POTRF, TRSMs, then SYRK/GEMM for
 * b' ascending, a >= b'.  In place over the FILLED pattern payload.  Returns
 * -1 or the global pivot j*b + p of the first non-SPD pivot (cholesky.cpp:98-104). */
long orc_factorize(int N, int b, const long* cs, const int* rows, double* pay) {
  const size_t bb = (size_t)b * b;
  double* tmp = (double*)malloc(sizeof(double) * bb);
  for (int j = 0; j < N; ++j) {
    double* d = pay + (size_t)cs[j] * bb;
    int p = potrf(b, d, tmp);
    if (p >= 0) {
      free(tmp);
      return (long)j * b + p;
    }
    memcpy(d, tmp, sizeof(double) * bb);
    for (long s = cs[j] + 1; s < cs[j + 1]; ++s) trsm_right_trans(b, d, pay + (size_t)s * bb);
    for (long sb = cs[j] + 1; sb < cs[j + 1]; ++sb)
      for (long sa = sb; sa < cs[j + 1]; ++sa) {
        int a_row = rows[sa], b_row = rows[sb];
        long ts = slot_of(cs, rows, a_row, b_row);
        if (ts < 0) {
          free(tmp);
          return -2; /* pattern not closed under fill */
        }
        if (sa == sb) syrk(b, pay + (size_t)ts * bb, pay + (size_t)sa * bb);
        else gemm_minus(b, pay + (size_t)ts * bb, pay + (size_t)sa * bb, 0, pay + (size_t)sb * bb, 1);
      }
  }
  free(tmp);
  return -1;
}

/* 2 * sum_{r < n} log L_rr (not a reference API). */
double orc_logdet(int N, int b, long n, const long* cs, const double* pay) {
  const size_t bb = (size_t)b * b;
  double s = 0.0;
  for (long r = 0; r < n; ++r) {
    const double* d = pay + (size_t)cs[r / b] * bb;
    s += log(d[(size_t)(r % b) * b + (r % b)]);
  }
  return 2.0 * s;
}

/* phase 1 in place, selinv.cpp:195-223: U_i = trtri(L_ii^T), W_ki = L_ki U_i^T. */
void orc_phase1(int N, int b, const long* cs, double* pay) {
  const size_t bb = (size_t)b * b;
  double* u = (double*)malloc(sizeof(double) * bb);
  for (int i = N - 1; i >= 0; --i) {
    double* d = pay + (size_t)cs[i] * bb;
    trtri_upper_of_lower(b, d, u);
    for (long s = cs[i] + 1; s < cs[i + 1]; ++s) trmm_right_trans_upper(b, pay + (size_t)s * bb, u);
    memcpy(d, u, sizeof(double) * bb);
  }
  free(u);
}

/* phase 2, selinv.cpp:239-345, serial order: columns descending, off-diagonal
 * rows as given (descending), k ascending, then the diagonal.  `work` lists,
 * per closure column in sweep order: col, has_diag, n_off, then n_off rows. */
int orc_phase2(int N, int b, const long* fcs, const int* frows, const double* p1, const long* ccs,
               const int* crows, double* sigma, const int* work, long work_len) {
  const size_t bb = (size_t)b * b;
  (void)N;
  memset(sigma, 0, sizeof(double) * bb * (size_t)ccs[N]);
  long w = 0;
  while (w < work_len) {
    int i = work[w], diag = work[w + 1], noff = work[w + 2];
    const int* off = work + w + 3;
    w += 3 + noff;
    for (int q = 0; q < noff; ++q) {
      int j = off[q];
      double* tgt = sigma + (size_t)slot_of(ccs, crows, j, i) * bb;
      for (long s = fcs[i]; s < fcs[i + 1]; ++s) {
        int k = frows[s];
        if (k <= i) continue;
        long ms = slot_of(ccs, crows, j > k ? j : k, j < k ? j : k);
        if (ms < 0) return 1;
        gemm_minus(b, tgt, sigma + (size_t)ms * bb, k > j, p1 + (size_t)s * bb, 0);
      }
    }
    if (diag) {
      double* tgt = sigma + (size_t)slot_of(ccs, crows, i, i) * bb;
      lauum_upper(b, p1 + (size_t)fcs[i] * bb, tgt);
      for (long s = fcs[i]; s < fcs[i + 1]; ++s) {
        int k = frows[s];
        if (k <= i) continue;
        long os = slot_of(ccs, crows, k, i);
        if (os < 0) return 1;
        gemm_minus(b, tgt, p1 + (size_t)s * bb, 1, sigma + (size_t)os * bb, 0);
      }
      for (int r = 0; r < b; ++r)
        for (int c = r + 1; c < b; ++c) AT(tgt, r, c) = AT(tgt, c, r);
    }
  }
  return 0;
}
