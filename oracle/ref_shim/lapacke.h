/* LAPACKE stand-in, TEST INFRASTRUCTURE ONLY (see Eigen/Core in this
 * directory): the one routine multigrid.cpp calls.  Defined in
 * oracle/ref_glue.cpp as the unblocked dpstf2 'L' (LAPACK's dpstrf runs it for
 * n <= NB), the same restatement as host/hierarchy.cpp pstrf_lower. */
#ifndef IG_REF_SHIM_LAPACKE_H
#define IG_REF_SHIM_LAPACKE_H
typedef int lapack_int;
#define LAPACK_ROW_MAJOR 101
#define LAPACK_COL_MAJOR 102
#ifdef __cplusplus
extern "C" {
#endif
lapack_int LAPACKE_dpstrf(int matrix_layout, char uplo, lapack_int n, double *a, lapack_int lda, lapack_int *piv,
                          lapack_int *rank, double tol);
#ifdef __cplusplus
}
#endif
#endif
