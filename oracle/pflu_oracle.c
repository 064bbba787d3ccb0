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
 *   orc_getrf_steps_top2 <- the same, instrumented: per column the winner's and the runner-up's
 *                     magnitudes of _jit.py:162-170's search (tie classification, north_star);
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
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define IDX(i, j, ld) ((int64_t)(i) * (ld) + (j))

static int g_threads = 0;
void orc_set_threads(int t) { g_threads = t; }
static int nthreads(void) { return g_threads > 0 ? g_threads : omp_get_max_threads(); }

/* Unblocked right-looking LU on an m x w panel (row-major, leading dim lda).  Processes the
 * first `steps` columns (steps <= min(m, w); pass -1 for all).  piv[j] = 0-based panel-local
 * pivot row.  Returns 0 or 1 + first column whose pivot was exactly zero (left as is). */
/* top2 (optional, 4 doubles per column): the tie classifier's record of column j's search --
 * |winner|, the largest |candidate| among the OTHER rows (-1 if none), that runner-up's panel-local
 * row (the smallest such row, as the strict '>' scan would take it), and the number of candidates
 * within 1e-12 relative of the winner (the winner included).  North_star allows a pivot mismatch only
 * where the top two magnitudes tie within 1e-12 relative. */
static int64_t lu_unb_impl(double *a, int64_t m, int64_t w, int64_t lda, int64_t *piv, int64_t steps,
                           double *top2) {
  int64_t kmax = m < w ? m : w;
  if (steps >= 0 && steps < kmax) kmax = steps;
  int64_t info = 0;
  int nt = nthreads();
  for (int64_t j = 0; j < kmax; ++j) {
    int64_t pbest = j, p2 = -1;
    double vbest = fabs(a[IDX(j, j, lda)]), v2 = -1.0;
    for (int64_t i = j + 1; i < m; ++i) {
      double v = fabs(a[IDX(i, j, lda)]);
      if (v > vbest) { v2 = vbest; p2 = pbest; vbest = v; pbest = i; }
      else if (top2 && v > v2) { v2 = v; p2 = i; }
    }
    if (top2) {
      int64_t nt = 0;
      const double lim = vbest * (1.0 - 1e-12);
      for (int64_t i = j; i < m; ++i) nt += fabs(a[IDX(i, j, lda)]) >= lim;
      top2[4 * j] = vbest; top2[4 * j + 1] = v2; top2[4 * j + 2] = (double)p2; top2[4 * j + 3] = (double)nt;
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

int64_t orc_lu_unb(double *a, int64_t m, int64_t w, int64_t lda, int64_t *piv, int64_t steps) {
  return lu_unb_impl(a, m, w, lda, piv, steps, NULL);
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
/* top2: NULL, or 4 doubles per column (see lu_unb_impl; the runner-up row made global). */
int64_t orc_getrf_steps_top2(double *a, int64_t m, int64_t n, int64_t lda, int64_t b, int64_t *piv,
                             int64_t nsteps, double *top2) {
  int64_t info = 0;
  int64_t step = 0;
  for (int64_t col0 = 0; col0 < n && (nsteps < 0 || step < nsteps); col0 += b, ++step) {
    int64_t bw = n - col0 < b ? n - col0 : b;
    double *panel = a + IDX(col0, col0, lda);
    int64_t pinfo = lu_unb_impl(panel, m - col0, bw, lda, piv + col0, -1, top2 ? top2 + 4 * col0 : NULL);
    if (pinfo && !info) info = col0 + pinfo;
    int64_t kk = (m - col0) < bw ? (m - col0) : bw;
    for (int64_t j = 0; j < kk; ++j) {
      piv[col0 + j] += col0;
      if (top2 && top2[4 * (col0 + j) + 2] >= 0.0) top2[4 * (col0 + j) + 2] += (double)col0;
    }
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

int64_t orc_getrf_steps(double *a, int64_t m, int64_t n, int64_t lda, int64_t b, int64_t *piv, int64_t nsteps) {
  return orc_getrf_steps_top2(a, m, n, lda, b, piv, nsteps, NULL);
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

/* ==========================================================================================
 * Householder QR (Kind.QR), SURVEY.md §8(f) row 4.  Same storage conventions (row-major).
 *   orc_qr_unb    <- _jit.py:190-218 (qr_unb_run: beta opposite in sign to the leading entry,
 *                    tau = (beta - alpha) / beta, v scaled by 1 / (alpha - beta), each reflector
 *                    applied to the panel's later columns as s = a_jc + sum v_i a_ic (i
 *                    ascending), s *= tau, a -= s v).  Pinned bitwise to the reference.
 *   orc_larft     <- factor.py:174-189 (larft_forward_columnwise: T[j,j] = tau_j,
 *                    T[:j,j] = -tau_j T[:j,:j] (V[:,:j]^T v_j)).  The reference evaluates the two
 *                    products with numpy/BLAS, so this loop order matches it only to rounding.
 *   orc_apply_block_reflector <- factor.py:192-205 + kernels.py:249-270 + _jit.py:54-80 and
 *                    the trmm_upper_run loop (W = 0 + V^T C p ascending; W = T^T W zero-seeded,
 *                    l ascending; C += V (-W) p ascending, multiply then add).
 *   orc_geqrf     <- dmf_mtb (factor.py:382-412) with kind=Kind.QR: per panel qr_unb + larft,
 *                    then the block reflector on the columns to the right.
 */
/* The panel is staged column-major (the reference's own F-order layout) so the column loops are
 * contiguous; the arithmetic is op for op _jit.qr_unb_run. */
void orc_qr_unb(double *a0, int64_t m, int64_t w, int64_t lda0, double *tau) {
  double *a = (double *)malloc((size_t)(m * w) * sizeof(double));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < w; ++j) a[j * m + i] = a0[IDX(i, j, lda0)];
#define A_(i, j) a[(int64_t)(j) * m + (i)]
  for (int64_t j = 0; j < w; ++j) {
    const double alpha = A_(j, j);
    double sq = 0.0;
    for (int64_t i = j + 1; i < m; ++i) { double v = A_(i, j); double t = v * v; sq = sq + t; }
    if (sq == 0.0) { tau[j] = 0.0; continue; }
    double aa = alpha * alpha;
    const double norm = sqrt(aa + sq);
    const double beta = alpha >= 0.0 ? -norm : norm;
    tau[j] = (beta - alpha) / beta;
    const double scale = 1.0 / (alpha - beta);
    for (int64_t i = j + 1; i < m; ++i) A_(i, j) *= scale;
    A_(j, j) = beta;
    for (int64_t c = j + 1; c < w; ++c) {
      double s = A_(j, c);
      for (int64_t i = j + 1; i < m; ++i) { double t = A_(i, j) * A_(i, c); s = s + t; }
      s = s * tau[j];
      A_(j, c) -= s;
      for (int64_t i = j + 1; i < m; ++i) { double t = s * A_(i, j); A_(i, c) -= t; }
    }
  }
#undef A_
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < w; ++j) a0[IDX(i, j, lda0)] = a[j * m + i];
  free(a);
}

/* v(i, j) of the stored reflectors: unit diagonal, zero above, the panel below. */
static inline double vref(const double *v, int64_t ldv, int64_t i, int64_t j) {
  return i > j ? v[IDX(i, j, ldv)] : (i == j ? 1.0 : 0.0);
}

/* T (k x k row-major, upper) from the reflectors stored in the m x k panel v and tau (V staged
 * column-major so the products V[:, :j]^T v_j run down contiguous columns). */
void orc_larft(const double *v, int64_t m, int64_t k, int64_t ldv, const double *tau, double *t) {
  for (int64_t i = 0; i < k * k; ++i) t[i] = 0.0;
  double *wv = (double *)calloc((size_t)(k > 0 ? k : 1), sizeof(double));
  double *vc = (double *)malloc((size_t)(m * (k > 0 ? k : 1)) * sizeof(double));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < k; ++j) vc[j * m + i] = vref(v, ldv, i, j);
  for (int64_t j = 0; j < k; ++j) {
    t[IDX(j, j, k)] = tau[j];
    if (!j) continue;
    for (int64_t l = 0; l < j; ++l) {
      double s = 0.0;
      const double *x = vc + l * m, *y = vc + j * m;
      for (int64_t i = 0; i < m; ++i) { double p = x[i] * y[i]; s = s + p; }
      wv[l] = s;
    }
    for (int64_t i = 0; i < j; ++i) {
      double s = 0.0;
      for (int64_t l = i; l < j; ++l) { double p = t[IDX(i, l, k)] * wv[l]; s = s + p; }
      t[IDX(i, j, k)] = -tau[j] * s;
    }
  }
  free(vc);
  free(wv);
}

/* c (m x nc) <- (I - V T V^T)^T c = c - V (T^T (V^T c)).  Column blocks of c in parallel; inside a
 * block the loops run row by row (cache friendly) but every element still sees its reference
 * operation sequence (p ascending for W and C, l ascending for Z, multiply then add). */
void orc_apply_block_reflector(const double *v, int64_t m, int64_t k, int64_t ldv, const double *t,
                               double *c, int64_t nc, int64_t ldc) {
  if (m <= 0 || nc <= 0 || k <= 0) return;
  const int64_t JB = 64;
  const int64_t nblk = (nc + JB - 1) / JB;
  int nt = nthreads();
#pragma omp parallel num_threads(nt) if (m * nc * k > 1000000)
  {
    double *w = (double *)malloc((size_t)(k * JB) * sizeof(double));
    double *z = (double *)malloc((size_t)(k * JB) * sizeof(double));
    double *vr = (double *)malloc((size_t)k * sizeof(double));
#pragma omp for schedule(dynamic, 1)
    for (int64_t jb = 0; jb < nblk; ++jb) {
      const int64_t j0 = jb * JB, jw = nc - j0 < JB ? nc - j0 : JB;
      for (int64_t i = 0; i < k * JB; ++i) { w[i] = 0.0; z[i] = 0.0; }
      for (int64_t p = 0; p < m; ++p) {                 /* W = 0 + V^T C, p ascending */
        for (int64_t r = 0; r < k; ++r) vr[r] = vref(v, ldv, p, r);
        const double *cp = c + IDX(p, j0, ldc);
        for (int64_t r = 0; r < k; ++r) {
          const double x = vr[r];
          double *wr = w + r * JB;
          for (int64_t jj = 0; jj < jw; ++jj) { double q = x * cp[jj]; wr[jj] = wr[jj] + q; }
        }
      }
      for (int64_t l = 0; l < k; ++l)                  /* Z = T^T W, zero-seeded, l ascending */
        for (int64_t i = l; i < k; ++i) {
          const double tv = t[IDX(l, i, k)];
          for (int64_t jj = 0; jj < jw; ++jj) { double q = tv * w[l * JB + jj]; z[i * JB + jj] = z[i * JB + jj] + q; }
        }
      for (int64_t i = 0; i < k * JB; ++i) z[i] = -z[i];
      for (int64_t i = 0; i < m; ++i) {                 /* C += V (-Z), p ascending */
        double *ci = c + IDX(i, j0, ldc);
        for (int64_t p = 0; p < k; ++p) {
          const double x = vref(v, ldv, i, p);
          const double *zp = z + p * JB;
          for (int64_t jj = 0; jj < jw; ++jj) { double q = x * zp[jj]; ci[jj] = ci[jj] + q; }
        }
      }
    }
    free(w);
    free(z);
    free(vr);
  }
}

/* Blocked Householder QR, dmf_mtb order.  m >= n >= 1.  tau: double[n]. */
void orc_geqrf_steps(double *a, int64_t m, int64_t n, int64_t lda, int64_t b, double *tau, int64_t nsteps) {
  int64_t step = 0;
  for (int64_t col0 = 0; col0 < n && (nsteps < 0 || step < nsteps); col0 += b, ++step) {
    const int64_t bw = n - col0 < b ? n - col0 : b;
    double *panel = a + IDX(col0, col0, lda);
    orc_qr_unb(panel, m - col0, bw, lda, tau + col0);
    const int64_t lo = col0 + bw;
    if (lo < n) {
      double *t = (double *)malloc((size_t)(bw * bw) * sizeof(double));
      orc_larft(panel, m - col0, bw, lda, tau + col0, t);
      orc_apply_block_reflector(panel, m - col0, bw, lda, t, a + IDX(col0, lo, lda), n - lo, lda);
      free(t);
    }
  }
}

void orc_geqrf(double *a, int64_t m, int64_t n, int64_t lda, int64_t b, double *tau) {
  orc_geqrf_steps(a, m, n, lda, b, tau, -1);
}
