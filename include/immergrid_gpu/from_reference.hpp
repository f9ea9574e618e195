// immergrid_gpu/from_reference.hpp — hand a built reference hierarchy
// (immergrid::MgHierarchy, /root/reference/proj/include/immergrid/multigrid.hpp)
// to the device solve WITHOUT modifying the reference.
//
// Everything the device needs is public in the reference: the per-level
// operators (MgLevel::A, ::R), each level's Smoother (kind(), gamma(),
// partition(): post-filter blocks, their Eigen::LLT factors and the colours)
// and coarse_rank().  The coarse factor itself is private (coarse_chol_,
// coarse_piv_), so it is recomputed here from level(0).A with exactly the call
// MgHierarchy::build makes (multigrid.cpp:57-73): dense column-major copy,
// tol = 1e-14 * max diag, pivoted Cholesky 'L'.  With
// IMMERGRID_GPU_COARSE_LAPACKE defined that call is LAPACKE_dpstrf itself (the
// same library and input as the reference, so the same factor); otherwise the
// device restatement ig_pstrf (unblocked dpstf2 order; its distance from the
// blocked LAPACK factor is bounded in tests/test_noise_floor.py).  The rank
// must equal the reference's coarse_rank().
//
// Usage inside the reference's tree (runner.cpp:219-235):
//
//   #include "immergrid_gpu/from_reference.hpp"
//   const auto mg  = immergrid::MgHierarchy::build(space, A, levels, smoother_cfg);
//   const auto gpu = immergrid_gpu::from_reference(mg);         // upload once
//   auto [x, rep]  = immergrid_gpu::pcg(immergrid_gpu::ig_from_eigen(A), b, gpu, tol, maxit);
//
// Compiled in CI against a minimal Eigen / immergrid API shim
// (tests/shim/, tests/test_reference_adapter.py) and run on the GPU against
// the direct boundary path (bit-identical solve).
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "immergrid/multigrid.hpp"
#include "immergrid_gpu/solve.hpp"

#ifdef IMMERGRID_GPU_COARSE_LAPACKE
#include <lapacke.h>
#endif

namespace immergrid_gpu {

inline MgHierarchy from_reference(const immergrid::MgHierarchy& h) {
  const int L = h.levels();
  std::vector<ig_level> lv(static_cast<size_t>(L));
  std::vector<std::vector<int32_t>> ptr(L), dofs(L), color(L);
  std::vector<std::vector<int64_t>> fptr(L);
  std::vector<std::vector<double>> fac(L);
  for (int l = 0; l < L; ++l) {
    const immergrid::MgLevel& m = h.level(l);
    lv[l] = ig_level{};
    lv[l].A = ig_from_eigen(m.A);  // compressed after build
    if (l > 0) lv[l].R = ig_from_eigen(m.R);
    if (!m.smoother) continue;  // level 0: the coarse solve
    const immergrid::Smoother& s = *m.smoother;
    int32_t kind;
    if (s.kind() == immergrid::SmootherKind::AdditiveSchwarz)
      kind = IG_SMOOTHER_ADDITIVE_SCHWARZ;
    else if (s.kind() == immergrid::SmootherKind::MultiplicativeSchwarz)
      kind = IG_SMOOTHER_MULTIPLICATIVE_SCHWARZ;
    else
      throw std::invalid_argument("from_reference: Jacobi / Gauss-Seidel smoothers do not run on the device");
    const immergrid::SchwarzPartition& part = s.partition();
    const auto& blocks = part.layout.blocks;
    ptr[l].push_back(0);
    fptr[l].push_back(0);
    for (size_t b = 0; b < blocks.size(); ++b) {
      dofs[l].insert(dofs[l].end(), blocks[b].begin(), blocks[b].end());
      ptr[l].push_back(static_cast<int32_t>(dofs[l].size()));
      const auto& LL = part.factor[b].matrixLLT();  // lower triangle = L, column-major
      fac[l].insert(fac[l].end(), LL.data(), LL.data() + LL.rows() * LL.cols());
      fptr[l].push_back(static_cast<int64_t>(fac[l].size()));
    }
    const bool mult = kind == IG_SMOOTHER_MULTIPLICATIVE_SCHWARZ;
    if (mult) color[l].assign(part.colors.color_of.begin(), part.colors.color_of.end());
    lv[l].smoother_kind = kind;
    lv[l].gamma = s.gamma();
    lv[l].blocks.n_blocks = static_cast<int32_t>(blocks.size());
    lv[l].blocks.blk_ptr = ptr[l].data();
    lv[l].blocks.blk_dofs = dofs[l].data();
    lv[l].blocks.fac_ptr = fptr[l].data();
    lv[l].blocks.fac = fac[l].data();
    lv[l].blocks.n_colors = mult ? part.colors.num_colors : 0;
    lv[l].blocks.color_of = mult ? color[l].data() : nullptr;
  }
  // Coarse factor as MgHierarchy::build computes it (multigrid.cpp:57-73).
  const ig_csr a1 = lv[0].A;
  const int32_t n = a1.n_rows;
  std::vector<double> a(static_cast<size_t>(n) * n, 0.0);
  for (int32_t i = 0; i < n; ++i)
    for (int32_t k = a1.row_ptr[i]; k < a1.row_ptr[i + 1]; ++k)
      a[static_cast<size_t>(a1.col_idx[k]) * n + i] = a1.val[k];
  double max_diag = 0.0;
  for (int32_t i = 0; i < n; ++i) max_diag = std::max(max_diag, a[static_cast<size_t>(i) * n + i]);
  std::vector<int32_t> piv(static_cast<size_t>(std::max(n, 1)), 0);
  int32_t rank = 0;
  const double tol = 1e-14 * max_diag;
#ifdef IMMERGRID_GPU_COARSE_LAPACKE
  lapack_int lrank = 0;
  if (LAPACKE_dpstrf(LAPACK_COL_MAJOR, 'L', n, a.data(), std::max(n, 1), piv.data(), &lrank, tol) < 0)
    throw std::runtime_error("from_reference: coarse factorization failed");
  rank = static_cast<int32_t>(lrank);
#else
  check(ig_pstrf(n, a.data(), piv.data(), tol, &rank), "from_reference: coarse factor");
#endif
  if (rank != h.coarse_rank())
    throw std::runtime_error("from_reference: coarse rank differs from the reference's coarse_rank()");
  const ig_coarse co{n, rank, a.data(), piv.data()};
  return MgHierarchy(lv.data(), L, co);  // ig_hier_create copies; the host arrays may go
}

}  // namespace immergrid_gpu
