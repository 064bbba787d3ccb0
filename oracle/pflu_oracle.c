/*
 * pflu_oracle.c -- CPU restatement of the reference LU-with-partial-pivoting hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200 kernels and
 * the CPU baseline of bench.py; the product path (paper_1804_07017_b200/, libpflu.so)
 * never links, loads or calls it.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it.
 *
 * It restates, op for op, the arithmetic of the reference package `panelforge`:
 *   orc_lu_unb     <- pkg/src/panelforge/_jit.py:154-187   (lu_unb_run: strict '>' argmax so
 *                     ties go to the smallest row, swap across the panel width, scale by
 *                     DIVISION, rank-1 update as separate multiply then subtract)
 *   orc_laswp      <- _jit.py:141-151                      (ascending LAPACK ipiv swaps)
 *   orc_trsm_llnu  <- _jit.py:104-113                      (right-looking unit-lower solve,
 *                     pivot rows ascending)
 *   orc_gemm_sub   <- _jit.py:54-80 + factor.py:282-285    (C += A*(-B): per element the
 *                     accumulator is seeded from C and updated with p ascending, multiply then
 *                     add; a*(-b) == -(a*b) exactly, so this is c - a*b)
 *   orc_getrf      <- factor.py:382-412 (dmf_mtb) with the step body of factor.py:235-285;
 *                     dmf_la (factor.py:455-515) is bitwise identical.
 *
 * Storage here is ROW-MAJOR (element (i,j) at a[i*lda+j]); the reference stores column-major
 * but its per-element operation sequence does not depend on the layout.  Pivots are 0-based
 * global row indices (reference pivots - 1).  Built with -ffp-contract=off so that no
 * multiply/subtract pair is fused: the results are bitwise equal to the reference (pinned by
 * tests/test_oracle.py against tests/golden/, generated from the reference itself).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <omp.h>

#define IDX(i, j, ld) ((int64_t)(i) * (ld) + (j))

static int g_threads = 0;
void orc_set_threads(int t) { g_threads = t; }
static int nthreads(void) { return g_threads > 0 ? g_threads : omp_get_max_threads(); }

/* Unblocked right-looking LU on an m x w panel (row-major, leading dim lda).  Processes the
 * first `steps` columns (steps <= min(m, w); pass -1 for all).  piv[j] = 0-based panel-local
 * pivot row.  Returns 0 or 1 + first column whose pivot was exactly zero (left as is). */
int64_t orc_lu_unb(double *a, int64_t m, int64_t w, int64_t lda, int64_t *piv, int64_t steps) {
  int64_t kmax = m < w ? m : w;
  if (steps >= 0 && steps < kmax) kmax = steps;
  int64_t info = 0;
  int nt = nthreads();
  for (int64_t j = 0; j < kmax; ++j) {
    int64_t pbest = j;
    double vbest = fabs(a[IDX(j, j, lda)]);
    for (int64_t i = j + 1; i < m; ++i) {
      double v = fabs(a[IDX(i, j, lda)]);
      if (v > vbest) { vbest = v; pbest = i; }
    }
    piv[j] = pbest;
    if (vbest == 0.0) {
      if (info == 0) info = j + 1;
      continue;
    }
    if (pbest != j) {
      double *r1 = a + IDX(j, 0, lda), *r2 = a + IDX(pbest, 0, lda);
      for (int64_t c = 0; c < w; ++c) { double t = r1[c]; r1[c] = r2[c]; r2[c] = t; }
    }
    const double pivot = a[IDX(j, j, lda)];
    const double *u = a + IDX(j, 0, lda);
    int64_t rows = m - j - 1;
#pragma omp parallel for num_threads(nt) schedule(static) if (rows * (w - j) > 32768)
    for (int64_t i = j + 1; i < m; ++i) {
      double *ri = a + IDX(i, 0, lda);
      double l = ri[j] / pivot;
      ri[j] = l;
      for (int64_t c = j + 1; c < w; ++c) {
        double t = l * u[c];
        ri[c] = ri[c] - t;
      }
    }
  }
  return info;
}

/* Rows k1..k2-1 swapped with piv[k] (0-based global rows), ascending k, on columns [c0, c1). */
void orc_laswp(double *a, int64_t lda, int64_t c0, int64_t c1, const int64_t *piv, int64_t k1, int64_t k2) {
  for (int64_t k = k1; k < k2; ++k) {
    int64_t p = piv[k];
    if (p == k) continue;
    double *r1 = a + IDX(k, 0, lda), *r2 = a + IDX(p, 0, lda);
    for (int64_t c = c0; c < c1; ++c) { double t = r1[c]; r1[c] = r2[c]; r2[c] = t; }
  }
}

/* X (bsz x ncols) <- unit_lower(L)^-1 X; element (r, j) takes its updates for i ascending. */
void orc_trsm_llnu(const double *l, int64_t ldl, int64_t bsz, double *x, int64_t ldx, int64_t ncols) {
  int nt = nthreads();
#pragma omp parallel for num_threads(nt) schedule(static) if (bsz * ncols > 65536)
  for (int64_t j0 = 0; j0 < ncols; j0 += 64) {
    int64_t j1 = j0 + 64 < ncols ? j0 + 64 : ncols;
    for (int64_t i = 0; i < bsz; ++i) {
      const double *xi = x + IDX(i, 0, ldx);
      for (int64_t r = i + 1; r < bsz; ++r) {
        double lri = l[IDX(r, i, ldl)];
        double *xr = x + IDX(r, 0, ldx);
        for (int64_t j = j0; j < j1; ++j) {
          double t = lri * xi[j];
          xr[j] = xr[j] - t;
        }
      }
    }
  }
}

/* C (m x n) <- C - A (m x k) * B (k x n), per element p ascending, multiply then subtract. */
void orc_gemm_sub(double *c, int64_t ldc, const double *a, int64_t lda, const double *b, int64_t ldb,
                  int64_t m, int64_t n, int64_t k) {
  if (m <= 0 || n <= 0 || k <= 0) return;
  int nt = nthreads();
  const int64_t JB = 512, IB = 16;
  int64_t nib = (m + IB - 1) / IB, njb = (n + JB - 1) / JB;
#pragma omp parallel for collapse(2) num_threads(nt) schedule(dynamic, 1) if (m * n * k > 1000000)
  for (int64_t jb = 0; jb < njb; ++jb) {
    for (int64_t ib = 0; ib < nib; ++ib) {
      int64_t j0 = jb * JB, j1 = j0 + JB < n ? j0 + JB : n;
      int64_t i0 = ib * IB, i1 = i0 + IB < m ? i0 + IB : m;
      int64_t i = i0;
      for (; i + 4 <= i1; i += 4) {
        double *c0 = c + IDX(i, 0, ldc), *c1 = c0 + ldc, *c2 = c1 + ldc, *c3 = c2 + ldc;
        const double *a0 = a + IDX(i, 0, lda), *a1 = a0 + lda, *a2 = a1 + lda, *a3 = a2 + lda;
        for (int64_t p = 0; p < k; ++p) {
          const double *bp = b + IDX(p, 0, ldb);
          const double x0 = a0[p], x1 = a1[p], x2 = a2[p], x3 = a3[p];
          for (int64_t j = j0; j < j1; ++j) {
            double bv = bp[j];
            double t0 = x0 * bv, t1 = x1 * bv, t2 = x2 * bv, t3 = x3 * bv;
            c0[j] = c0[j] - t0; c1[j] = c1[j] - t1; c2[j] = c2[j] - t2; c3[j] = c3[j] - t3;
          }
        }
      }
      for (; i < i1; ++i) {
        double *ci = c + IDX(i, 0, ldc);
        const double *ai = a + IDX(i, 0, lda);
        for (int64_t p = 0; p < k; ++p) {
          const double *bp = b + IDX(p, 0, ldb);
          const double x = ai[p];
          for (int64_t j = j0; j < j1; ++j) { double t = x * bp[j]; ci[j] = ci[j] - t; }
        }
      }
    }
  }
}

/* Blocked right-looking LUpp (dmf_mtb order, factor.py:382-412): for each panel k: panel
 * factorization (lu_unb on rows col0.., panel width), left swaps on [0, col0), right swaps +
 * trsm + gemm on [col0+bw, n).  m >= n >= 1 (caller validates).  piv: 0-based global rows. */
int64_t orc_getrf_steps(double *a, int64_t m, int64_t n, int64_t lda, int64_t b, int64_t *piv, int64_t nsteps) {
  int64_t info = 0;
  int64_t step = 0;
  for (int64_t col0 = 0; col0 < n && (nsteps < 0 || step < nsteps); col0 += b, ++step) {
    int64_t bw = n - col0 < b ? n - col0 : b;
    double *panel = a + IDX(col0, col0, lda);
    int64_t pinfo = orc_lu_unb(panel, m - col0, bw, lda, piv + col0, -1);
    if (pinfo && !info) info = col0 + pinfo;
    int64_t kk = (m - col0) < bw ? (m - col0) : bw;
    for (int64_t j = 0; j < kk; ++j) piv[col0 + j] += col0;
    orc_laswp(a, lda, 0, col0, piv, col0, col0 + kk);                 /* left swaps */
    int64_t lo = col0 + bw;
    if (lo < n) {
      orc_laswp(a, lda, lo, n, piv, col0, col0 + kk);                /* right swaps */
      orc_trsm_llnu(a + IDX(col0, col0, lda), lda, bw, a + IDX(col0, lo, lda), lda, n - lo);
      if (col0 + bw < m)
        orc_gemm_sub(a + IDX(col0 + bw, lo, lda), lda, a + IDX(col0 + bw, col0, lda), lda,
                     a + IDX(col0, lo, lda), lda, m - col0 - bw, n - lo, bw);
    }
  }
  return info;
}

int64_t orc_getrf(double *a, int64_t m, int64_t n, int64_t lda, int64_t b, int64_t *piv) {
  return orc_getrf_steps(a, m, n, lda, b, piv, -1);
}

/* First `steps` elimination steps of the unblocked algorithm on the full m x n matrix
 * (full-width swaps).  Rows 0..steps-1 of the result and piv[0..steps) are FINAL values of
 * the complete factorization (later steps only touch rows >= steps), so this pins a prefix
 * of a factorization too large to run completely on the host (C4/C5). */
int64_t orc_lu_prefix(double *a, int64_t m, int64_t n, int64_t lda, int64_t *piv, int64_t steps) {
  return orc_lu_unb(a, m, n, lda, piv, steps);
}
