/*
 * ig_gpu.h — C-ABI of the B200 solve phase (PCG + geometric-multigrid V-cycle
 * with additive-Schwarz smoothing), the drop-in boundary for the reference's
 * CPU solve in /root/reference/proj.
 *
 * Every array argument is a plain pointer + size; no C++ or torch types cross
 * this boundary.  Unless a function name ends in `_device`, vector arguments
 * are HOST pointers and the call is synchronous.  `_device` variants take
 * device pointers and are asynchronous on the handle's CUDA stream
 * (ig_hier_stream).
 *
 * Interfaces replaced (reference file:line):
 *   ig_csr            SpMat = Eigen::SparseMatrix<double,RowMajor> compressed
 *                     (proj/include/immergrid/common.hpp:16): int32 outer/inner
 *                     indices, ascending inner indices per row.
 *   ig_blocks         BlockLayout (post-filter) + std::vector<Eigen::LLT<MatX>>
 *                     (proj/include/immergrid/smoothers.hpp:24-27, :70-75)
 *   ig_level          MgLevel {A, R, smoother}  (multigrid.hpp:21-26)
 *   ig_coarse         MgHierarchy::{coarse_chol_, coarse_piv_, rank_}
 *                     (multigrid.hpp:70-73; built at multigrid.cpp:57-73)
 *   ig_hier_create    the upload half of MgHierarchy::build (multigrid.cpp:12-75)
 *   ig_vcycle         MgHierarchy::apply (multigrid.hpp:52)
 *   ig_vcycle_at      MgHierarchy::vcycle_at (multigrid.hpp:49, multigrid.cpp:90-108)
 *   ig_coarse_solve   MgHierarchy::coarse_solve (multigrid.cpp:77-88)
 *   ig_smoother_apply Smoother::apply, additive Schwarz (smoothers.cpp:169-184)
 *   ig_pcg            pcg(A, b, precond, tol, maxit) with precond = the hierarchy
 *                     (solvers.hpp:51-53, solvers.cpp:17-71)
 *   ig_level_spmv     the Eigen RowMajor SpMVs at solvers.cpp:45,
 *                     multigrid.cpp:99,101,102,104 (debug / parity entry point)
 *
 * Status codes mirror the reference's exception types (solvers.hpp:25-47);
 * exceptions never cross the ABI.  The C++ wrapper in
 * include/immergrid_gpu/solve.hpp and the Python mirror in
 * paper_1903_10977_b200/__init__.py re-throw them.
 */
#ifndef IG_GPU_H
#define IG_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum ig_status {
  IG_OK = 0,                /* converged / success                           */
  IG_NOT_CONVERGED = 1,     /* NotConverged{report, x}  (solvers.cpp:67-70)  */
  IG_BREAKDOWN = 2,         /* Breakdown{report}        (solvers.cpp:47-50)  */
  IG_INVALID_ARGUMENT = 3,  /* std::invalid_argument    (solvers.cpp:20-21)  */
  IG_CUDA_ERROR = 4,        /* device failure (no reference counterpart)     */
  IG_UNSUPPORTED = 5,       /* smoother kind not implemented on the device   */
  IG_DIVERGED = 6           /* Diverged{report}         (solvers.cpp:108-112)*/
};

/* SmootherKind order of proj/include/immergrid/smoothers.hpp:15. */
enum ig_smoother_kind {
  IG_SMOOTHER_JACOBI = 0,
  IG_SMOOTHER_GAUSS_SEIDEL = 1,
  IG_SMOOTHER_ADDITIVE_SCHWARZ = 2,
  IG_SMOOTHER_MULTIPLICATIVE_SCHWARZ = 3
};

/* CSR == Eigen RowMajor compressed storage. */
typedef struct {
  int32_t n_rows, n_cols;
  int64_t nnz;
  const int32_t *row_ptr; /* n_rows+1 */
  const int32_t *col_idx; /* nnz, ascending within a row */
  const double *val;      /* nnz */
} ig_csr;

/* Post-filter Schwarz layout.  Block b owns blk_dofs[blk_ptr[b]..blk_ptr[b+1])
 * (ascending DOFs) and its lower Cholesky factor L_b, s_b x s_b column-major,
 * at fac[fac_ptr[b] .. fac_ptr[b] + s_b*s_b) (upper triangle ignored).
 * Blocks are in ascending owner order (smoothers.cpp:56-66). */
typedef struct {
  int32_t n_blocks;
  const int32_t *blk_ptr;  /* n_blocks+1 */
  const int32_t *blk_dofs; /* blk_ptr[n_blocks] */
  const int64_t *fac_ptr;  /* n_blocks+1 */
  const double *fac;
  /* Multiplicative sweeps only (ColorClasses, smoothers.hpp:35-42): greedy
   * colour of each block (pre-filter supports), colours 0..n_colors-1.  Same-
   * colour blocks have disjoint DOFs.  NULL / 0 for additive Schwarz. */
  int32_t n_colors;
  const int32_t *color_of; /* n_blocks */
} ig_blocks;

/* One level.  levels[0] is the coarsest (A only; R empty, no smoother),
 * levels[n_levels-1] the finest.  R of level l restricts level-l vectors to
 * level l-1 (n_rows = n_{l-1}, n_cols = n_l), as MgLevel::R. */
typedef struct {
  ig_csr A;
  ig_csr R;
  int32_t smoother_kind; /* ig_smoother_kind: ADDITIVE_ or MULTIPLICATIVE_SCHWARZ on the device */
  double gamma;          /* damping, already resolved (smoothers.cpp:234-239) */
  ig_blocks blocks;
} ig_level;

/* Coarsest-level pivoted Cholesky (LAPACK dpstrf('L') output). */
typedef struct {
  int32_t n, rank;
  const double *L;    /* n x n column-major; first `rank` columns are L11 */
  const int32_t *piv; /* n, 1-based (dpstrf) */
} ig_coarse;

/* Finest-level assembly payload (the reference's assemble(),
 * proj/src/assembly.cpp:36-183, after the element loop): element matrices
 * and load vectors in tables, the uniform space's element cells, physical
 * supports and anchor numbering.  ig_assemble runs the global assembly (the
 * setFromTriplets summation, :164-176) and the symmetrisation (:177-180). */
typedef struct {
  int32_t dim, p, family;  /* family 1: B-spline (first anchor = cell), 0: Lagrange (p * cell) */
  int32_t n, n_elements, n_tables;
  int32_t nf[3];                                /* untrimmed functions per axis */
  const int32_t *el_ix, *el_iy, *el_iz;         /* element cells (el_iz NULL in 2D) */
  const int32_t *el_table;                      /* element -> table */
  const double *K;                              /* n_tables x nloc x nloc, row-major */
  const double *F;                              /* n_tables x nloc */
  const int64_t *anchors;                       /* DOF -> untrimmed linear anchor */
  const int64_t *supp_ptr;                      /* n + 1 */
  const int32_t *supp_el;                       /* physical support, elements ascending */
  const int32_t *kept;                          /* untrimmed -> DOF or -1 */
} ig_assembly;

/* Cut-element quadrature of the 3D uniform B-spline case on the device (the
 * element integration of the reference's assemble(), proj/src/assembly.cpp
 * :55-160, for elements classified Cut; this repository's 3D extension of
 * recurse_cut, proj/src/quadrature.cpp:255-300: octree bisection to `depth`,
 * Kuhn 6-tetrahedra per cut leaf clipped against psi >= 0 with bisection edge
 * roots, collapsed Gauss rules, interface penalty).  igh_cut3_payload fills it
 * from a host-built case; ig_cut_quadrature3 returns the same element
 * matrices as the host, bit for bit. */
typedef struct {
  int32_t p;                /* degree: q = p + 1 local functions per axis, nl = q^3 */
  int32_t n_cut;            /* cut elements */
  const double *lo;         /* n_cut x 3: lower corner of each cut element (physical) */
  const int32_t *cls;       /* n_cut x 3: extraction class per axis */
  int32_t n_cls[3];
  const double *ext[3];     /* per axis: n_cls[d] x q x q, column-major E(i, k) */
  double h[3];              /* cell size */
  double beta, f;           /* penalty (already resolved), body force */
  int32_t depth, classify_depth;
  double edge_tol;
  int32_t prog_len;         /* level-set program: postfix, op codes 0 const(v), 1 linear(c0 c1 c2 d dim), */
  const double *prog;       /* 2 ball(c0 c1 c2 r dim), 3 box(lo0 lo1 lo2 hi0 hi1 hi2 dim), 4 min, 5 max, 6 neg */
  const double *gauss_tet;  /* 2 nodes, then 2 weights on [0,1] (tetrahedra, 2 x 2 x 2 points) */
  const double *gauss_tri;  /* 3 nodes, then 3 weights on [0,1] (interface triangles, 3 x 3 points) */
  const double *gauss_box;  /* q nodes, then q weights on [-1,1] (inside sub-boxes, tensor moments) */
  const int32_t *table;     /* n_cut: the element's table index in igh_assembly_payload (K, F) */
} ig_cut3;

/* The reference's 2D cut-cell quadrature on the device (proj/src/
 * quadrature.cpp:128-372 recurse_cut / leaf_polygons / refine_chords /
 * fan_triangulate / interface_segments / side_rule, and the element loop of
 * assemble(), proj/src/assembly.cpp:55-162) for every individually integrated
 * element of a uniform 2D case: cut elements and elements on the embedding-box
 * boundary.  igh_cut2_payload fills it; ig_cut_quadrature2 returns the host's
 * element matrices bit for bit. */
typedef struct {
  int32_t p;               /* degree: q = p + 1, nl = q^2 */
  int32_t n_elem;
  const double *lo, *hi;   /* n_elem x 2: the element cell (physical) */
  const int32_t *cls;      /* n_elem x 2: extraction class per axis */
  const int32_t *cut;      /* n_elem: 1 = cut element (recurse_cut + interface), 0 = tensor rule */
  const int32_t *sides;    /* n_elem: bit k = box side k of the element carries the Dirichlet penalty */
  int32_t n_cls[2];
  const double *ext[2];    /* per axis: n_cls[d] x q x q, column-major */
  double beta, f;
  int32_t depth, classify_depth, gauss_order;
  double edge_tol;
  int32_t prog_len;
  const double *prog;      /* level-set program (ig_cut3) */
  const double *gauss_q;   /* gauss_order nodes, then weights, on [-1,1] */
  const double *gauss_q1;  /* gauss_order + 1 nodes, then weights (collapsed triangle rule, q > 3) */
  const int32_t *table;    /* n_elem: table index in igh_assembly_payload */
} ig_cut2;

/* THB (truncated hierarchical B-spline) element integration and global
 * assembly on the device (the host's assemble_g, host/thb.cpp: the reference's
 * assemble() over a hierarchical mesh, proj/src/assembly.cpp:36-183).  Every
 * element is integrated individually (its truncated functions: `erow_ptr`
 * rows of `E`, Bernstein coefficients x fastest) with the 2D quadrature of
 * ig_cut2; rows are gathered per DOF over its support in ascending element
 * order (setFromTriplets), exact zeros dropped, then A = 0.5 (A + A^T). */
typedef struct {
  int32_t p, n, n_elem;
  const double *lo, *hi;      /* n_elem x 2: element cells at their levels */
  const int32_t *cut;         /* n_elem */
  const int32_t *sides;       /* n_elem: box-side bit mask (at the element's level) */
  const int32_t *erow_ptr;    /* n_elem + 1: the element's functions */
  const int32_t *anchors;     /* erow_ptr[n_elem]: their global DOFs, in row order */
  const double *E;            /* erow_ptr[n_elem] x (p+1)^2 */
  const int64_t *supp_ptr;    /* n + 1 */
  const int32_t *supp_el;     /* elements of each DOF's support, ascending */
  const int32_t *supp_li;     /* the DOF's row in that element */
  double beta, f;
  int32_t depth, classify_depth, gauss_order;
  double edge_tol;
  int32_t prog_len;
  const double *prog;
  const double *gauss_q, *gauss_q1;
} ig_thb_asm;

typedef struct ig_hier ig_hier;

/* Device-side sizes and algorithmic byte counts. */
typedef struct {
  int32_t n_levels;
  int32_t n[16];           /* DOFs per level, [0] coarsest */
  int64_t nnz_A[16];
  int64_t nnz_R[16];
  int32_t n_blocks[16];
  int32_t n_multi_blocks[16]; /* blocks with s_b > 1 */
  int64_t sum_s[16];          /* sum of block sizes */
  int64_t sum_s2[16];         /* sum of s_b^2 (stored factor entries) */
  int64_t sell_slots_A[16];   /* padded SELL-32 slots of A (>= nnz_A) */
  int64_t bytes_vcycle;       /* algorithmic bytes of one V-cycle */
  int64_t bytes_pcg_iter;     /* algorithmic bytes of one PCG iteration */
  int64_t bytes_spmv_finest;  /* algorithmic bytes of one finest y = A x */
  int64_t device_bytes;       /* device memory held by the handle */
  int32_t kernels_vcycle;     /* kernel launches per V-cycle */
  int32_t kernels_pcg_iter;   /* kernel launches per PCG iteration */
  /* Row-dictionary SELL (kernels.cuh): matrix entries whose value / column
   * is actually read from HBM, per level, and the bytes one finest SpMV must
   * move with that layout (vs. the CSR-minimal bytes_spmv_finest). */
  int64_t explicit_vals_A[16];
  int64_t explicit_cols_A[16];
  int64_t bytes_spmv_finest_layout;
  int64_t bytes_vcycle_layout;
  int32_t coarse_n;           /* coarsest level size and accepted pivots      */
  int32_t coarse_rank;        /* (MgHierarchy::coarse_rank, multigrid.hpp:60) */
} ig_info;

/* Upload a hierarchy (copied; the host arrays may be freed afterwards).
 * Returns IG_INVALID_ARGUMENT on inconsistent sizes. */
int ig_hier_create(const ig_level *levels, int32_t n_levels,
                   const ig_coarse *coarse, ig_hier **out);
void ig_hier_destroy(ig_hier *h);
int ig_hier_info(const ig_hier *h, ig_info *out);
/* cudaStream_t of the handle (as void*). */
void *ig_hier_stream(ig_hier *h);

/* --- reference-shaped entry points (host buffers, synchronous) --------- */
int ig_vcycle(ig_hier *h, const double *r, double *x);
int ig_vcycle_at(ig_hier *h, int32_t level, const double *r, double *x);
int ig_coarse_solve(ig_hier *h, const double *r, double *x);
int ig_smoother_apply(ig_hier *h, int32_t level, const double *r, double *x);
/* Smoother::apply(r, dir) (smoothers.hpp:70-73): dir 0 Forward, 1 Reverse
 * (multiplicative sweeps: colours descending / ascending). */
int ig_smoother_apply_dir(ig_hier *h, int32_t level, const double *r, double *x, int32_t dir);
/* Smoother::apply_symmetric (smoothers.cpp:211-214):
 * x1 = S(r, Forward); x = x1 + S(r - A x1, Reverse). */
int ig_smoother_apply_symmetric(ig_hier *h, int32_t level, const double *r, double *x);
/* mode 0: y = A x; 1: y = r - A x (r passed in y); 2: y = R x; 3: y = R^T x */
int ig_level_spmv(ig_hier *h, int32_t level, const double *x, double *y,
                  int32_t mode);

/* PCG on A = levels[n_levels-1].A preconditioned by one V-cycle.
 * residuals must hold maxit+1 doubles; *iterations and the residual prefix
 * follow ConvergenceReport (solvers.hpp:16-23).  x is written on IG_OK and on
 * IG_NOT_CONVERGED (the partial iterate).  seconds = device time of the solve
 * (CUDA events), host copies excluded. */
int ig_pcg(ig_hier *h, const double *b, double tol, int32_t maxit, double *x,
           double *residuals, int32_t *iterations, double *seconds);

/* --- device-resident variants (async on ig_hier_stream) -----------------
 * Device vectors must be 16-byte aligned (the kernels read x with 16-byte
 * vector loads; cudaMalloc / torch allocations are); an unaligned pointer,
 * e.g. a torch slice t[1:], returns IG_INVALID_ARGUMENT. */
int ig_vcycle_device(ig_hier *h, const double *d_r, double *d_x);
/* vcycle_at(level, r) (multigrid.hpp:49) on device buffers of that level's size. */
int ig_vcycle_at_device(ig_hier *h, int32_t level, const double *d_r, double *d_x);
/* ig_level_spmv on device buffers (modes as ig_level_spmv); used to time the
 * dominant kernel in isolation. */
int ig_level_spmv_device(ig_hier *h, int32_t level, const double *d_x,
                         double *d_y, int32_t mode);
/* Launches the whole solve (CUDA graph with a device-side WHILE loop); no
 * host synchronisation.  Read the outcome with ig_pcg_result. */
int ig_pcg_device(ig_hier *h, const double *d_b, double tol, int32_t maxit,
                  double *d_x);
/* Synchronises the stream and returns the status of the last
 * ig_pcg_device; residuals (maxit+1, may be NULL), iterations. */
int ig_pcg_result(ig_hier *h, double *residuals, int32_t *iterations);

/* richardson(A = finest A, b, V-cycle, tol, maxit) — solvers.hpp:55-59,
 * solvers.cpp:73-120: x <- x + M^{-1}(b - A x) from x = 0; residuals has
 * room for maxit+1 entries.  IG_OK, IG_NOT_CONVERGED (x = last iterate) or
 * IG_DIVERGED (residual grew 10 steps in a row). */
int ig_richardson(ig_hier *h, const double *b, double tol, int32_t maxit, double *x,
                  double *residuals, int32_t *iterations, double *seconds);

/* Host-only (no device work): slice statistics of the pattern-SELL layout the
 * library would build for `a` (out: >= 32 entries; see csrc/ig_gpu.cu). */
int ig_debug_psell_stats(const ig_csr *a, int64_t *out, int32_t n_out);
/* Host-only: y = A x through that layout, interpreted on the CPU with the
 * kernels' index arithmetic and summation order, every index bounds-checked
 * (a layout validation for the tests: each row exactly once, no load outside
 * its array; the result equals the serial CSR row sums bit for bit). */
int ig_debug_psell_apply(const ig_csr *a, const double *x, double *y);
/* Debug: run one V-cycle with direct launches and an event after every step
 * (smoother, residual, restriction, prolongation, coarse solve); writes the
 * elapsed ms per step, its level and a label (label_len bytes each). */
int ig_debug_vcycle_timeline(ig_hier *h, const double *d_r, double *d_x,
                             int32_t max_steps, float *ms, int32_t *levels,
                             char *labels, int32_t label_len, int32_t *count);

/* --- the step before the path: global assembly -- */
/* A = 0.5 (K + K^T) and b from the element tables on the device, bit-identical
 * to the host assembly (each entry sums its element contributions in
 * ascending element order, exact zeros dropped, as setFromTriplets does;
 * assembly.cpp:164-180).  A_out: library-owned host CSR (ig_csr_free);
 * b_out: n doubles.  seconds (may be NULL): [0] wall, [1] device time. */
int ig_assemble(const ig_assembly *a, ig_csr *A_out, double *b_out, double *seconds);

/* --- composed spectral operators ---------------- */
/* Columns j0 .. j0+count-1 of a composed operator on the finest level, the
 * LinOps proj/src/runner.cpp:84-122 hands to dense_spectrum
 * (proj/src/spectral.cpp:28-50 materialises them column by column from unit
 * vectors): IG_OP_A = A e_j; IG_OP_VCYCLE = MgHierarchy::apply(A e_j)
 * ("vcycle"); IG_OP_SMOOTHER_SYMMETRIC = Smoother::apply_symmetric(A e_j) of
 * the finest smoother ("as2" / "ms2").  out: n x count, column-major, host. */
#define IG_OP_A 0
#define IG_OP_VCYCLE 1
#define IG_OP_SMOOTHER_SYMMETRIC 2
int ig_operator_columns(ig_hier *h, int32_t kind, int32_t j0, int32_t count, double *out);

/* --- device-side hierarchy setup ---------------- */
/* Galerkin coarse operators on the device: starting from A_fine (the finest
 * level's A), A_{l-1} = R_l (A_l R_l^T) for l = n_levels-1 .. 1, exactly the
 * products of MgHierarchy::build (proj/src/multigrid.cpp:37-41,
 * `r * (down.back().A * rt)`), bit-identical to Eigen's sparse-product
 * summation order (each entry summed over the inner index ascending, first
 * product assigned).  R[l] (l >= 1) is the restriction of level l (rows
 * n_{l-1}, cols n_l), as ig_level.R; R[0] is ignored.  A_out[l] for
 * l = 0 .. n_levels-2 receives the coarse operators in host arrays owned by
 * the library (release each with ig_csr_free).  seconds (may be NULL) gets
 * 2 doubles: [0] wall time of the call (uploads and downloads included),
 * [1] device time of the transposes and products (CUDA events).
 * IG_UNSUPPORTED if a product row has more than 768 distinct columns. */
int ig_galerkin_hierarchy(const ig_csr *A_fine, const ig_csr *R, int32_t n_levels, ig_csr *A_out,
                          double *seconds);
void ig_csr_free(ig_csr *m);
/* Batched Schwarz block factorisation on the device (factorize_blocks of
 * make_smoother, proj/src/smoothers.cpp:131-162): for each pre-filter block
 * (blk_ptr / blk_dofs: blocks in owner order, DOFs ascending) gather A_b from
 * A, drop the DOF with the largest |component| of the lowest eigenvector
 * while lambda_min < filter_ratio * max diag (no filtering when
 * filter_ratio <= 0), then the lower Cholesky factor (Eigen::LLT).  Output:
 * the post-filter layout in `out` (host arrays owned by the library; release
 * with ig_blocks_free; n_colors = 0), bit-identical to the host factorisation.
 * *filtered_dofs (may be NULL) = DOFs removed.  seconds (may be NULL): [0]
 * wall time, [1] device time.  IG_INVALID_ARGUMENT if a block loses every DOF
 * (the reference's std::runtime_error). */
int ig_factorize_blocks(const ig_csr *A, int32_t n_blocks, const int32_t *blk_ptr, const int32_t *blk_dofs,
                        double filter_ratio, ig_blocks *out, int64_t *filtered_dofs, double *seconds);
void ig_blocks_free(ig_blocks *b);
/* Coarsest-level pivoted Cholesky on the device (LAPACK dpstf2, UPLO 'L', as
 * MgHierarchy::build calls dpstrf, proj/src/multigrid.cpp:57-73): a is n x n
 * column-major (host buffer, factored in place), piv 1-based, *rank the
 * accepted pivots; bit-identical to the host restatement igh_pstrf. */
int ig_pstrf(int32_t n, double *a, int32_t *piv, double tol, int32_t *rank);
/* MgHierarchy::build's algebraic half on the device (multigrid.cpp:12-75 from
 * the fine matrix on): the Galerkin chain (ig_galerkin_hierarchy), every
 * level's block factorisation (ig_factorize_blocks) and the coarsest pivoted
 * Cholesky (ig_pstrf, tol 1e-14 max diag), then ig_hier_create.  Inputs: the
 * finest A, R[l] (l >= 1, as ig_level.R), prefilter[l] (l >= 1: the
 * pre-filter layouts of select_blocks in blk_ptr / blk_dofs, fac ignored;
 * n_colors / color_of for multiplicative sweeps), gamma[l] (resolved damping),
 * the smoother kind and filter ratio of every level.  The result is the same
 * handle the host-built payload gives (bit-identical operators, factors and
 * solves).  seconds (may be NULL): [0] wall time, [1] device time of the
 * Galerkin / factorisation / pstrf kernels, [2] of which ig_hier_create. */
int ig_hier_build(const ig_csr *A_fine, const ig_csr *R, const ig_blocks *prefilter, const double *gamma,
                  int32_t smoother_kind, double filter_ratio, int32_t n_levels, ig_hier **out,
                  double *seconds);

/* Element matrices of the cut elements on the device: K (n_cut x nl x nl,
 * row-major, symmetric), F (n_cut x nl), vol (n_cut: integrated volume
 * fraction, may be NULL); bit-identical to the host's element tables.
 * seconds (may be NULL): device time.  IG_UNSUPPORTED for level sets without
 * a device program or p > 2 (shared-memory basis tables). */
int ig_cut_quadrature3(const ig_cut3 *in, double *K, double *F, double *vol, double *seconds);
/* 2D: K (n_elem x nl x nl), F (n_elem x nl), vol (volume-rule weight sums, may
 * be NULL), bit-identical to the host.  p <= 4. */
int ig_cut_quadrature2(const ig_cut2 *in, double *K, double *F, double *vol, double *seconds);
/* THB: A_out (host CSR, free with ig_csr_free) and b_out (n doubles),
 * bit-identical to the host assembly.  seconds (may be NULL): [0] wall,
 * [1] device time.  Elements with more than 64 functions: IG_UNSUPPORTED. */
int ig_assemble_thb(const ig_thb_asm *in, ig_csr *A_out, double *b_out, double *seconds);

/* Thread-local message for the last non-OK status. */
const char *ig_last_error(void);

/* Options.  ig_set_option sets the process-wide DEFAULTS; ig_hier_create
 * snapshots them into the new handle (later ig_set_option calls do not
 * affect existing handles, so handles with different options coexist and
 * run concurrently).  ig_hier_set_option changes the runtime options of one
 * handle: IG_OPT_USE_GRAPH, IG_OPT_PDL, IG_OPT_RED_CTAS (layout options only
 * act at creation and are rejected there with IG_INVALID_ARGUMENT). */
#define IG_OPT_USE_GRAPH 1 /* 1 (default): CUDA-graph PCG loop; 0: host loop */
#define IG_OPT_ROW_DICT 2  /* 1 (default): row-dictionary SELL; 0: plain SELL */
#define IG_OPT_SMALL_ROWS 4   /* matrices with <= this many rows use the 8-lanes-per-row SpMV */
#define IG_OPT_PSELL 7        /* 1 (default): pattern SELL for matrices above IG_OPT_SMALL_ROWS rows */
#define IG_OPT_PDL 9          /* 1 (default): programmatic dependent launch for every kernel; 0: plain stream order */
#define IG_OPT_RED_CTAS 13    /* CTAs per SM of the canonical-reduction kernels (default 8) */
#define IG_OPT_PSELL_CTAS 15  /* pattern-SELL SpMV occupancy cap, CTAs per SM (0 = registers decide) */
#define IG_OPT_L2_ROWS 18       /* levels below the finest with <= this many DOFs in an L2-persisting arena (default 300000; 0 = off) */
#define IG_OPT_PSELL_LINES2 27    /* 1 (default): pattern-SELL slices covering two x-lines (shared column runs) */
#define IG_OPT_PSELL_MULTI 34     /* 1 (default): pattern-SELL slices packing row pairs of up to four short runs (FAST2M) */
#define IG_OPT_PSELL_ROWS4 36     /* 1 (default): two-line pattern-SELL slices with four rows of each line per lane (FAST8) */
#define IG_OPT_PSELL_EDGE_ROWS 37 /* pattern-SELL slices over an edge-compacted copy of x (FASTE: the x-line end rows) for square matrices with at least this many rows (default 100000; 0 = off) */
#define IG_OPT_PSELL_ROWS4_ROWS 38 /* ... only for matrices with at least this many rows (default 1000000) */
#define IG_OPT_PSELL_ORDER 39      /* pattern-SELL slice launch order: 1 (default) by class, GENERAL spread through the two-line slices, then multi-piece, rest; 2: GENERAL first; 0: row order */
#define IG_OPT_PSELL_AB 35        /* 1 (default): pattern-SELL slices of row pairs sharing one column list (FASTAB, prolongations) */
#define IG_OPT_PSELL_CTAB 23     /* 1 (default): FAST2 value sequences of the pattern SELL from a constant-bank table */
#define IG_OPT_GAL_SHORT 21      /* 1 (default): device Galerkin uses the prefetching SpGEMM when B rows have <= 32 entries */
#define IG_OPT_L2_MB 19          /* size of that arena in MiB (default 48) */
#define IG_OPT_COMPLEX4_ROWS 28  /* additive smoother: four lanes per multi-block DOF up to this many DOFs (default 100000) */
#define IG_OPT_PSELL_PAIRS_ROWS 32 /* pattern-SELL pair / two-line slices only for matrices with at least this many rows (default 100000) */
#define IG_OPT_FAST_BLOCKS 33     /* tolerance mode: additive-Schwarz block solves as explicit-inverse matvecs (not bit-identical; default 0) */
#define IG_OPT_FAST_COARSE 30     /* tolerance mode: coarse solve as an explicit-inverse GEMV (not bit-identical; default 0) */
#define IG_OPT_ONE_STREAM_ROWS 29 /* additive smoother without fork / join up to this many DOFs (default 40000) */
int ig_set_option(int32_t option, int64_t value);
int ig_hier_set_option(ig_hier *h, int32_t option, int64_t value);

/* pcg(A, b, precond) / richardson (solvers.hpp:51-59) multiply by the A they
 * are given; the device solve multiplies by the finest A of the hierarchy.
 * IG_OK when `a` is that operator -- the same arrays passed to ig_hier_create
 * (or ig_hier_build), or a copy with identical sizes, row pointers, columns and
 * value bits (content hash) -- else IG_INVALID_ARGUMENT.  The drop-in
 * surfaces (immergrid_gpu::pcg, Python pcg) call it before solving. */
int ig_hier_matches(ig_hier *h, const ig_csr *a);

#ifdef __cplusplus
}
#endif
#endif /* IG_GPU_H */
