/*
 * oracle.h — CPU restatement of the reference's solve phase.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker for the GPU path
 * (tests/, __graft_entry__.smoke()) and the timed CPU baseline in bench.py's
 * cpu_baseline / --impl reference legs.  Nothing in the product
 * (paper_1903_10977_b200/) links, loads or calls it.
 *
 * It consumes exactly the payload that crosses the drop-in boundary
 * (include/ig_gpu.h: ig_level[], ig_coarse) and restates (OpenMP-parallel
 * over rows / blocks / chunks with every value summed in the sequential
 * order, so bit-identical for any thread count; see oracle.c):
 *   pcg              proj/src/solvers.cpp:17-71
 *   richardson       proj/src/solvers.cpp:73-120
 *   vcycle_at        proj/src/multigrid.cpp:90-108
 *   coarse_solve     proj/src/multigrid.cpp:77-88
 *   Smoother::apply  proj/src/smoothers.cpp:169-184 (additive Schwarz),
 *                    :186-208 (colored multiplicative Schwarz sweep)
 *   LLT::solve       Eigen (forward column-oriented with L, backward row-dot with L^T)
 *   SpMV             Eigen RowMajor sparse*dense: per-row ascending sum
 *
 * Parity pinning: the reference cannot be built as shipped (Eigen/LAPACKE
 * absent), but its own hot-path sources (solvers.cpp,
 * multigrid.cpp, smoothers.cpp) compile unmodified against the Eigen / LAPACKE
 * stand-in of oracle/ref_shim into oracle/_ref/libimmergrid_ref.so (`make ref`,
 * ref_glue.cpp).  tests/test_reference_pin.py holds this restatement to that
 * library BIT FOR BIT in ORC_SEQ mode (pcg, richardson, vcycle_at, both
 * sweeps, coarse_solve, on C1-C5 at full size through the committed records
 * of tests/golden/reference_solves.json), and tests/test_oracle.py to the
 * reference's known-answer tests.  Not observable in any build here: Eigen's
 * internal kernel orders (SIMD dot, blocked triangular solves, blocked
 * dpstrf); tests/test_noise_floor.py bounds their effect.
 *
 * Reductions (dot, norm): ORC_SEQ sums in ascending index order (the natural
 * reading of Eigen's redux); ORC_GPU_ORDER sums in the documented chunked tree
 * the device kernels use (chunks of 256: 32-lane xor butterfly, pairwise over
 * 8 warps; partials strided over 256 lanes, then the same tree).  Everything
 * else is identical in both modes.  Compiled with -ffp-contract=off.
 */
#ifndef IG_ORACLE_H
#define IG_ORACLE_H

#include <stdint.h>

#include "../include/ig_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_SEQ = 0, ORC_GPU_ORDER = 1 };

/* Thread count for the parallel loops (n <= 0: all processors). */
void orc_set_threads(int n);
int orc_get_threads(void);

/* Canonical dot product (mode as above). */
double orc_dot(int mode, int64_t n, const double *a, const double *b);
/* y = A x (resid == 0) or y = r - A x (resid == 1, r passed in y). */
void orc_spmv(const ig_csr *A, const double *x, double *y, int resid);
/* y = A^T x for a CSR A (accumulation over ascending row index of A). */
void orc_spmv_t(const ig_csr *A, const double *x, double *y);
/* Smoother::apply for additive Schwarz: x = gamma * sum_b P_b L_b^-T L_b^-1 P_b^T r. */
void orc_as_apply(const ig_level *lv, int32_t n, const double *r, double *x);
/* Smoother::apply for multiplicative Schwarz (colored sweep): dir 0 =
 * Forward (colours descending), 1 = Reverse (ascending). */
void orc_ms_apply(const ig_level *lv, int32_t n, const double *r, double *x, int dir);
/* The level's smoother (additive or multiplicative by smoother_kind). */
void orc_smoother_apply(const ig_level *lv, int32_t n, const double *r, double *x, int dir);
void orc_coarse_solve(const ig_coarse *co, const double *r, double *x);
/* MgHierarchy::vcycle_at(l, r). Returns 0, or 3 on bad arguments. */
int orc_vcycle_at(const ig_level *levels, int32_t n_levels, const ig_coarse *co,
                  int32_t l, const double *r, double *x);
/* pcg(A = levels[n_levels-1].A, b, V-cycle, tol, maxit).  Status codes as
 * ig_status.  residuals: maxit+1. */
int orc_pcg(const ig_level *levels, int32_t n_levels, const ig_coarse *co,
            int mode, const double *b, double tol, int32_t maxit, double *x,
            double *residuals, int32_t *iterations, double *seconds);

/* richardson(A = levels[n_levels-1].A, b, V-cycle, tol, maxit)
 * (solvers.cpp:73-120).  Returns 0, 1 (NotConverged) or 6 (Diverged). */
int orc_richardson(const ig_level *levels, int32_t n_levels, const ig_coarse *co, int mode,
                   const double *b, double tol, int32_t maxit, double *x, double *residuals,
                   int32_t *iterations, double *seconds);

#ifdef __cplusplus
}
#endif
#endif
