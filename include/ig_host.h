/*
 * ig_host.h — C-ABI of the host-side setup (CPU, C++/OpenMP): builds the
 * algebraic multigrid hierarchy that ig_hier_create (ig_gpu.h) uploads.
 *
 * Replaces, for the solve-phase drop-in, the reference's setup chain
 *   build_case            proj/src/runner.cpp:523-532  (trim, build_space, assemble)
 *   MgHierarchy::build    proj/src/multigrid.cpp:12-75 (coarsen, R, Galerkin,
 *                         make_smoother per level, dpstrf on the coarsest)
 *   make_smoother         proj/src/smoothers.cpp:216-241
 * and writes/reads the same payload as a versioned binary file (.igh).
 */
#ifndef IG_HOST_H
#define IG_HOST_H

#include <stdint.h>

#include "ig_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t dim;             /* 2 or 3                                          */
  const char *geometry;    /* level-set expression (config.hpp:21-31 + 3D)    */
  double origin[3];
  double extent[3];
  int32_t resolution[3];   /* background cells per axis (finest level)        */
  int32_t family;          /* 0 Lagrange (2D), 1 B-spline, 2 THB (2D)         */
  int32_t degree;          /* 1..4                                            */
  int32_t levels;          /* total MG levels, >= 1                           */
  int32_t quad_depth;      /* cut-cell bisection depth (QuadratureConfig)     */
  int32_t gauss_order;     /* 0 = p+1 (config.cpp:647-650)                    */
  int32_t classify_depth;  /* lattice depth for trimming                      */
  double edge_tol;
  double body_force;       /* f (constant)                                    */
  double beta;             /* penalty; 0 = 2/h (assembly.cpp:7-10)            */
  int32_t dirichlet_box_sides; /* penalty also on embedding-box sides (2D)    */
  int32_t smoother_kind;   /* ig_smoother_kind                                */
  double gamma;            /* 0 = automatic (smoothers.cpp:234-239)           */
  double filter_ratio;     /* block eigen-filter ratio (default 1e-16)        */
  int32_t threads;         /* host threads for setup; 0 = all                 */
  /* THB (family 2, 2D) local refinement of the finest mesh, applied in order:
   * refine-by-box passes (mesh.cpp:51-56), then refine_passes passes of
   * "elements of the current finest level within refine_dist of the circle
   * (cx, cy, r)" (configs[4]; HierarchicalMesh::refine, mesh.cpp:35-49). */
  int32_t n_refine_boxes;
  const double *refine_boxes; /* 4 per box: x0, y0, x1, y1 */
  int32_t refine_passes;
  double refine_circle[3];
  double refine_dist;
} igh_config;

typedef struct igh_case igh_case;

typedef struct {
  int32_t n_levels;
  int32_t n[16];          /* DOFs per level, [0] coarsest */
  int64_t nnz[16];
  int32_t max_nk[16];
  int64_t filtered_dofs[16];
  int32_t coarse_rank;
  int64_t cut_elements;   /* finest level */
  double eta;             /* min volume fraction, finest level */
  double seconds_assemble;
  double seconds_mg_setup;
} igh_info;

void igh_config_default(igh_config *cfg);
int igh_build(const igh_config *cfg, igh_case **out);
/* The geometric half of igh_build only -- the host part of the device setup
 * pipeline: trimmed spaces of every level, the
 * restrictions R, the pre-filter Schwarz layouts (+ colours), the damping,
 * the Inside-class element tables and the element -> table map.  The cut /
 * box-side elements are NOT integrated (their tables stay zero: the device
 * computes them, ig_cut_quadrature2/3), nothing is assembled (A of every
 * level is an n x n pattern without entries, the rhs zeros), no Galerkin
 * product, block factorisation or pivoted Cholesky is formed (ig_assemble +
 * ig_hier_build do that on the device).  The payload functions
 * (igh_cut2/3_payload, igh_thb_payload, igh_assembly_payload,
 * igh_prefilter_blocks) and igh_levels (R, gamma, colours) work on such a
 * case; igh_write and igh_support_fraction do not. */
int igh_build_geometry(const igh_config *cfg, igh_case **out);
/* Pointers stay owned by the case (valid until igh_destroy). */
int igh_levels(const igh_case *c, const ig_level **levels, int32_t *n_levels,
               const ig_coarse **coarse);
const double *igh_rhs(const igh_case *c, int32_t *n);
/* Finest-level assembly payload for ig_assemble (uniform B-spline / Lagrange
 * cases; owned by the case). */
int igh_assembly_payload(const igh_case *c, ig_assembly *out);
/* Pre-filter Schwarz layout of level >= 1 (select_blocks output, the input of
 * factorize_blocks, smoothers.cpp:131-162): blocks in owner order, DOFs
 * ascending.  Owned by the case; built cases only (not igh_read). */
int igh_prefilter_blocks(const igh_case *c, int32_t level, int32_t *n_blocks,
                         const int32_t **blk_ptr, const int32_t **blk_dofs);
int igh_get_info(const igh_case *c, igh_info *out);
/* Finest level, per DOF: physical volume of the DOF's support divided by the
 * volume of its untrimmed support cells (1 = support entirely inside the
 * domain; sliver DOFs near a cut boundary -> 0).  out: n doubles.  Built
 * uniform (B-spline / Lagrange) cases only; THB and .igh-read cases return
 * IG_UNSUPPORTED.  Used by the parity tests to exclude sliver DOFs (whose
 * coefficients reach 1e19 on C4) from per-DOF error checks. */
int igh_support_fraction(const igh_case *c, double *out);
/* Cut-element quadrature payload of a built 3D uniform B-spline case
 * (ig_cut3, ig_gpu.h): the finest level's cut elements, their extraction
 * classes, the level-set program and the quadrature rules.  Owned by the case.
 * IG_UNSUPPORTED for 2D, THB, file-read cases or level sets without a device
 * program. */
int igh_cut3_payload(igh_case *c, ig_cut3 *out);
/* 2D uniform (B-spline / Lagrange) case: every individually integrated
 * element (cut, or with embedding-box sides) for ig_cut_quadrature2. */
int igh_cut2_payload(igh_case *c, ig_cut2 *out);
/* THB case (family 2): the finest level's elements, truncated extraction
 * rows, supports and quadrature data for ig_assemble_thb. */
int igh_thb_payload(igh_case *c, ig_thb_asm *out);
/* Kept anchors of level l as untrimmed tensor indices (ax, ay, az) -> n x 3. */
int igh_anchors(const igh_case *c, int32_t level, int32_t *out_xyz);
int igh_write(const igh_case *c, const char *path);
int igh_read(const char *path, igh_case **out);
void igh_destroy(igh_case *c);
const char *igh_last_error(void);

/* Standalone pieces (tests): LAPACK dpstrf('L') restatement on an n x n
 * column-major matrix (overwritten); returns rank, piv 1-based. */
int32_t igh_pstrf(int32_t n, double *a, int32_t *piv, double tol);
/* min volume fraction of a 2D/3D case without building the hierarchy. */
int igh_eta(const igh_config *cfg, double *eta, int64_t *cut_elements, int32_t *n_dofs);

#ifdef __cplusplus
}
#endif
#endif /* IG_HOST_H */
