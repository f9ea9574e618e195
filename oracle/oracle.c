/*
 * oracle.c — CPU restatement of the reference's solve phase.  TEST
 * INFRASTRUCTURE ONLY (see oracle.h): the checker for the GPU path and the
 * timed CPU baseline; never linked into the product.
 *
 * Threading: the row-, block- and chunk-parallel loops below (OpenMP) change
 * no arithmetic.  Every output value is produced by exactly one thread with
 * the same operands in the same order as the sequential loop it replaces
 * (per-row SpMV sums, per-DOF sums over ascending blocks / ascending rows of
 * R, per-chunk dot trees); only ORC_SEQ dots stay sequential.  So the result
 * is bit-identical for every thread count (tests/test_oracle.py checks 1 vs
 * many threads), and the many-thread run is the CPU baseline "with all the
 * host threads it can use".
 */
#define _POSIX_C_SOURCE 199309L
#include "oracle.h"

#include <limits.h>
#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

void orc_set_threads(int n) { omp_set_num_threads(n > 0 ? n : omp_get_num_procs()); }
int orc_get_threads(void) { return omp_get_max_threads(); }

/* [lo, hi) slice t of T of the index range [0, n). */
static void slice_of(int64_t n, int t, int T, int64_t *lo, int64_t *hi) {
  *lo = n * t / T;
  *hi = n * (t + 1) / T;
}

/* ---------------------------------------------------------- reductions -- */

/* One chunk of 256 values: 8 warps x (32-lane xor butterfly), then
 * ((w0+w1)+(w2+w3))+((w4+w5)+(w6+w7)).  Mirrors csrc/reduce.cuh. */
static double tree256(const double *v) {
  double w[8];
  for (int g = 0; g < 8; ++g) {
    double lane[32];
    memcpy(lane, v + 32 * g, sizeof(lane));
    for (int off = 16; off >= 1; off >>= 1) {
      double nxt[32];
      for (int l = 0; l < 32; ++l) nxt[l] = lane[l] + lane[l ^ off];
      memcpy(lane, nxt, sizeof(lane));
    }
    w[g] = lane[0];
  }
  return ((w[0] + w[1]) + (w[2] + w[3])) + ((w[4] + w[5]) + (w[6] + w[7]));
}

/* Second pass over the chunk partials: lane t sums P[t], P[t+256], ... from
 * 0.0 in ascending order, then tree256 over the 256 lane sums. */
static double finish_partials(int64_t nc, const double *P) {
  double acc[256];
  for (int t = 0; t < 256; ++t) {
    double a = 0.0;
    for (int64_t k = t; k < nc; k += 256) a = a + P[k];
    acc[t] = a;
  }
  return tree256(acc);
}

double orc_dot(int mode, int64_t n, const double *a, const double *b) {
  if (mode == ORC_SEQ) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s = s + a[i] * b[i];
    return s;
  }
  const int64_t nc = (n + 255) / 256;
  double *P = (double *)malloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1));
#pragma omp parallel for schedule(static) if (nc > 64)
  for (int64_t c = 0; c < nc; ++c) {
    double v[256];
    for (int t = 0; t < 256; ++t) {
      const int64_t i = 256 * c + t;
      v[t] = i < n ? a[i] * b[i] : 0.0;
    }
    P[c] = tree256(v);
  }
  const double s = finish_partials(nc, P);
  free(P);
  return s;
}

/* ------------------------------------------------------------- sparse --- */

void orc_spmv(const ig_csr *A, const double *x, double *y, int resid) {
#pragma omp parallel for schedule(static, 256) if (A->n_rows > 4096)
  for (int32_t i = 0; i < A->n_rows; ++i) {
    double acc = 0.0;
    for (int32_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k) acc = acc + A->val[k] * x[A->col_idx[k]];
    y[i] = resid ? y[i] - acc : acc;
  }
}

void orc_spmv_t(const ig_csr *A, const double *x, double *y) {
  /* y[f] = sum over rows c ascending (then k ascending) of A(c,f) x[c].  Each
   * thread owns a contiguous range of f and walks the rows whose column
   * span meets it, so every y[f] is summed in the sequential order. */
  const int32_t nr = A->n_rows, ncol = A->n_cols;
  int32_t *cmin = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nr > 0 ? nr : 1));
  int32_t *cmax = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nr > 0 ? nr : 1));
#pragma omp parallel for schedule(static) if (nr > 4096)
  for (int32_t c = 0; c < nr; ++c) {
    int32_t lo = INT_MAX, hi = -1;
    for (int32_t k = A->row_ptr[c]; k < A->row_ptr[c + 1]; ++k) {
      const int32_t f = A->col_idx[k];
      lo = f < lo ? f : lo;
      hi = f > hi ? f : hi;
    }
    cmin[c] = lo;
    cmax[c] = hi;
  }
#pragma omp parallel if (nr > 4096)
  {
    int64_t f0, f1;
    slice_of(ncol, omp_get_thread_num(), omp_get_num_threads(), &f0, &f1);
    for (int64_t j = f0; j < f1; ++j) y[j] = 0.0;
    for (int32_t c = 0; c < nr; ++c) {
      if (cmax[c] < f0 || cmin[c] >= f1) continue;
      const double xc = x[c];
      for (int32_t k = A->row_ptr[c]; k < A->row_ptr[c + 1]; ++k) {
        const int32_t f = A->col_idx[k];
        if (f >= f0 && f < f1) y[f] = y[f] + A->val[k] * xc;
      }
    }
  }
  free(cmin);
  free(cmax);
}

/* --------------------------------------------------------- block solves -- */

/* Eigen LLT::solve (smoothers.cpp:180): forward substitution with L (column
 * oriented), then backward substitution with L^T in row-dot form
 * y_i = (y_i - sum_{k>i} L(k,i) y_k) / L(i,i).  Eigen's panel/SIMD order is
 * not observable here, so the dot order is DEFINED as descending k (the
 * order in which the y_k become available), which the device reproduces
 * exactly.  ld = leading dimension of the column-major factor. */
static void tri_solve(int s, int ld, const double *L, double *y) {
  for (int j = 0; j < s; ++j) {
    const double yj = y[j] / L[(size_t)j * ld + j];
    y[j] = yj;
    for (int i = j + 1; i < s; ++i) y[i] = y[i] - L[(size_t)j * ld + i] * yj;
  }
  for (int i = s - 1; i >= 0; --i) {
    double acc = 0.0;
    for (int k = s - 1; k > i; --k) acc = acc + L[(size_t)i * ld + k] * y[k]; /* L(k,i) */
    y[i] = (y[i] - acc) / L[(size_t)i * ld + i];
  }
}
static void llt_solve(int s, const double *L, double *y) { tri_solve(s, s, L, y); }

void orc_as_apply(const ig_level *lv, int32_t n, const double *r, double *x) {
  /* x[d] = gamma * (0 + sum over blocks b ascending of (L_b^-T L_b^-1 P_b^T r)_d).
   * Phase 1 solves every block into Y (block-parallel); phase 2 gives each
   * thread a DOF range and adds the block results in ascending block order,
   * exactly the sequential accumulation. */
  const ig_blocks *B = &lv->blocks;
  const int32_t nb = B->n_blocks;
  const int64_t tot = nb > 0 ? B->blk_ptr[nb] : 0;
  double *Y = (double *)malloc(sizeof(double) * (size_t)(tot > 0 ? tot : 1));
  int32_t *bmin = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nb > 0 ? nb : 1));
  int32_t *bmax = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nb > 0 ? nb : 1));
#pragma omp parallel for schedule(dynamic, 512) if (nb > 2048)
  for (int32_t b = 0; b < nb; ++b) {
    const int32_t o = B->blk_ptr[b];
    const int s = B->blk_ptr[b + 1] - o;
    int32_t lo = INT_MAX, hi = -1;
    for (int i = 0; i < s; ++i) {
      const int32_t d = B->blk_dofs[o + i];
      Y[o + i] = r[d];
      lo = d < lo ? d : lo;
      hi = d > hi ? d : hi;
    }
    llt_solve(s, B->fac + B->fac_ptr[b], Y + o);
    bmin[b] = lo;
    bmax[b] = hi;
  }
#pragma omp parallel if (nb > 2048)
  {
    int64_t d0, d1;
    slice_of(n, omp_get_thread_num(), omp_get_num_threads(), &d0, &d1);
    for (int64_t i = d0; i < d1; ++i) x[i] = 0.0;
    for (int32_t b = 0; b < nb; ++b) {
      if (bmax[b] < d0 || bmin[b] >= d1) continue;
      const int32_t o = B->blk_ptr[b];
      const int s = B->blk_ptr[b + 1] - o;
      for (int i = 0; i < s; ++i) {
        const int32_t d = B->blk_dofs[o + i];
        if (d >= d0 && d < d1) x[d] = x[d] + Y[o + i];
      }
    }
    for (int64_t i = d0; i < d1; ++i) x[i] = lv->gamma * x[i];
  }
  free(Y);
  free(bmin);
  free(bmax);
}

/* Colored multiplicative sweep (smoothers.cpp:186-208).  The residual `cur`
 * is frozen within a colour; same-colour blocks touch disjoint DOFs; the
 * residual update `cur -= A * delta` runs after every colour but the last,
 * as a full Eigen RowMajor product (per-row ascending sum) subtracted from
 * cur.  Colours without blocks are skipped (`if (!any) continue`). */
void orc_ms_apply(const ig_level *lv, int32_t n, const double *r, double *x, int dir) {
  const ig_blocks *B = &lv->blocks;
  const int C = B->n_colors;
  double *cur = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double *delta = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  const int par = n > 4096;
#pragma omp parallel for schedule(static) if (par)
  for (int32_t i = 0; i < n; ++i) {
    x[i] = 0.0;
    cur[i] = r[i];
  }
  for (int step = 0; step < C; ++step) {
    const int col = dir == 0 ? C - 1 - step : step;
    int any = 0;
#pragma omp parallel for schedule(static) if (par)
    for (int32_t i = 0; i < n; ++i) delta[i] = 0.0;
    /* Same-colour blocks touch disjoint DOFs: block-parallel, each delta[d]
     * written by one block as 0 + y. */
#pragma omp parallel for schedule(dynamic, 512) reduction(| : any) if (par)
    for (int32_t b = 0; b < B->n_blocks; ++b) {
      if (B->color_of[b] != col) continue;
      double y[1024];
      const int32_t o = B->blk_ptr[b];
      const int s = B->blk_ptr[b + 1] - o;
      for (int i = 0; i < s; ++i) y[i] = cur[B->blk_dofs[o + i]];
      llt_solve(s, B->fac + B->fac_ptr[b], y);
      for (int i = 0; i < s; ++i) {
        const int32_t d = B->blk_dofs[o + i];
        delta[d] = delta[d] + y[i];
      }
      any = 1;
    }
    if (!any) continue;
#pragma omp parallel for schedule(static) if (par)
    for (int32_t i = 0; i < n; ++i) x[i] = x[i] + delta[i];
    if (step + 1 < C) orc_spmv(&lv->A, delta, cur, 1); /* cur -= A * delta */
  }
#pragma omp parallel for schedule(static) if (par)
  for (int32_t i = 0; i < n; ++i) x[i] = lv->gamma * x[i];
  free(cur);
  free(delta);
}

void orc_smoother_apply(const ig_level *lv, int32_t n, const double *r, double *x, int dir) {
  if (lv->smoother_kind == IG_SMOOTHER_MULTIPLICATIVE_SCHWARZ)
    orc_ms_apply(lv, n, r, x, dir);
  else
    orc_as_apply(lv, n, r, x); /* additive: both directions agree (smoothers.cpp:174-184) */
}

void orc_coarse_solve(const ig_coarse *co, const double *r, double *x) {
  const int n = co->n, rk = co->rank;
  double *y = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  double *perm = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (int k = 0; k < n; ++k) perm[k] = r[co->piv[k] - 1];
  for (int k = 0; k < rk; ++k) y[k] = perm[k];
  /* L11 = topLeftCorner(rank, rank) of the n x n factor (multigrid.cpp:82-84). */
  tri_solve(rk, n, co->L, y);
  for (int k = 0; k < n; ++k) x[co->piv[k] - 1] = y[k];
  free(y);
  free(perm);
}

/* -------------------------------------------------------------- V-cycle -- */

int orc_vcycle_at(const ig_level *levels, int32_t n_levels, const ig_coarse *co, int32_t l,
                  const double *r, double *x) {
  if (l < 0 || l >= n_levels) return IG_INVALID_ARGUMENT;
  if (l == 0) {
    orc_coarse_solve(co, r, x);
    return IG_OK;
  }
  const ig_level *lv = &levels[l];
  const int32_t n = lv->A.n_rows, nc = lv->R.n_rows;
  double *res = (double *)malloc(sizeof(double) * (size_t)n);
  double *tmp = (double *)malloc(sizeof(double) * (size_t)n);
  double *rc = (double *)malloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1));
  double *xc = (double *)malloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1));

  orc_smoother_apply(lv, n, r, x, 0);                 /* x = S(r, Forward)        */
  memcpy(res, r, sizeof(double) * (size_t)n);
  orc_spmv(&lv->A, x, res, 1);                        /* res = r - A x            */
  orc_spmv(&lv->R, res, rc, 0);                       /* R res                    */
  orc_vcycle_at(levels, n_levels, co, l - 1, rc, xc); /* coarse_x                 */
  orc_spmv_t(&lv->R, xc, tmp);                        /* correction = R^T coarse_x */
#pragma omp parallel for schedule(static) if (n > 4096)
  for (int32_t i = 0; i < n; ++i) x[i] = x[i] + tmp[i];
  orc_spmv(&lv->A, tmp, res, 1);                      /* res -= A correction      */
  orc_smoother_apply(lv, n, res, tmp, 1);             /* S(res, Reverse)          */
#pragma omp parallel for schedule(static) if (n > 4096)
  for (int32_t i = 0; i < n; ++i) x[i] = x[i] + tmp[i];
  free(res);
  free(tmp);
  free(rc);
  free(xc);
  return IG_OK;
}

/* ------------------------------------------------------------------ PCG -- */

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int orc_pcg(const ig_level *levels, int32_t n_levels, const ig_coarse *co, int mode,
            const double *b, double tol, int32_t maxit, double *x, double *residuals,
            int32_t *iterations, double *seconds) {
  const ig_csr *A = &levels[n_levels - 1].A;
  const int32_t n = A->n_rows;
  if (A->n_rows != A->n_cols) return IG_INVALID_ARGUMENT;
  const double t0 = now_s();
  *iterations = 0;
  for (int32_t i = 0; i < n; ++i) x[i] = 0.0;
  const double bnorm = sqrt(orc_dot(mode, n, b, b));
  if (bnorm == 0.0) {
    residuals[0] = 0.0;
    *seconds = now_s() - t0;
    return IG_OK;
  }
  residuals[0] = 1.0;
  if (1.0 <= tol) {
    *seconds = now_s() - t0;
    return IG_OK;
  }
  double *r = (double *)malloc(sizeof(double) * (size_t)n);
  double *z = (double *)malloc(sizeof(double) * (size_t)n);
  double *p = (double *)malloc(sizeof(double) * (size_t)n);
  double *ap = (double *)malloc(sizeof(double) * (size_t)n);
  memcpy(r, b, sizeof(double) * (size_t)n);
  orc_vcycle_at(levels, n_levels, co, n_levels - 1, r, z);
  memcpy(p, z, sizeof(double) * (size_t)n);
  double rz = orc_dot(mode, n, r, z);
  int status = IG_NOT_CONVERGED;
  for (int32_t k = 0; k < maxit; ++k) {
    orc_spmv(A, p, ap, 0);
    const double pap = orc_dot(mode, n, p, ap);
    if (pap <= 0.0) {
      status = IG_BREAKDOWN;
      break;
    }
    const double alpha = rz / pap;
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int32_t i = 0; i < n; ++i) {
      x[i] = x[i] + alpha * p[i];
      r[i] = r[i] - alpha * ap[i];
    }
    *iterations = k + 1;
    const double rel = sqrt(orc_dot(mode, n, r, r)) / bnorm;
    residuals[k + 1] = rel;
    if (rel <= tol) {
      status = IG_OK;
      break;
    }
    orc_vcycle_at(levels, n_levels, co, n_levels - 1, r, z);
    const double rz_next = orc_dot(mode, n, r, z);
    const double beta = rz_next / rz;
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int32_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rz = rz_next;
  }
  *seconds = now_s() - t0;
  free(r);
  free(z);
  free(p);
  free(ap);
  return status;
}

/* ----------------------------------------------------------- Richardson -- */

/* richardson (solvers.cpp:73-120).  Status 0 converged, 1 NotConverged,
 * 6 Diverged (10 consecutive growths). */
int orc_richardson(const ig_level *levels, int32_t n_levels, const ig_coarse *co, int mode,
                   const double *b, double tol, int32_t maxit, double *x, double *residuals,
                   int32_t *iterations, double *seconds) {
  const ig_csr *A = &levels[n_levels - 1].A;
  const int32_t n = A->n_rows;
  if (A->n_rows != A->n_cols) return IG_INVALID_ARGUMENT;
  const double t0 = now_s();
  for (int32_t i = 0; i < n; ++i) x[i] = 0.0;
  *iterations = 0;
  const double bnorm = sqrt(orc_dot(mode, n, b, b));
  if (bnorm == 0.0) {
    residuals[0] = 0.0;
    *seconds = now_s() - t0;
    return IG_OK;
  }
  double *r = (double *)malloc(sizeof(double) * (size_t)n);
  double *dx = (double *)malloc(sizeof(double) * (size_t)n);
  memcpy(r, b, sizeof(double) * (size_t)n);
  int growth = 0, status = IG_NOT_CONVERGED;
  for (int32_t k = 0; k <= maxit; ++k) {
    const double rel = sqrt(orc_dot(mode, n, r, r)) / bnorm;
    residuals[k] = rel;
    if (k > 0 && rel > residuals[k - 1])
      ++growth;
    else
      growth = 0;
    if (rel <= tol) {
      *iterations = k;
      status = IG_OK;
      break;
    }
    if (growth >= 10) {
      *iterations = k;
      status = 6; /* Diverged */
      break;
    }
    if (k == maxit) {
      *iterations = maxit;
      break;
    }
    orc_vcycle_at(levels, n_levels, co, n_levels - 1, r, dx);
#pragma omp parallel for schedule(static) if (n > 4096)
    for (int32_t i = 0; i < n; ++i) x[i] = x[i] + dx[i];
    orc_spmv(A, dx, r, 1); /* r -= A dx */
  }
  *seconds = now_s() - t0;
  free(r);
  free(dx);
  return status;
}
