// ref_glue.cpp -- C entry points over the REFERENCE'S OWN hot-path code.
// TEST INFRASTRUCTURE ONLY (like everything under oracle/).
//
// oracle/Makefile `ref` compiles /root/reference/proj/src/{solvers,multigrid,
// smoothers}.cpp unmodified, from where they lie, against the Eigen / LAPACKE
// stand-in in oracle/ref_shim/ (Eigen and LAPACKE are absent from this image),
// and links them with this file into oracle/_ref/libimmergrid_ref.so.  The
// functions below hand a hierarchy payload (include/ig_gpu.h structs, the same
// ones the oracle and the device take) to the reference's classes and run the
// reference's pcg / richardson / vcycle_at / Smoother::apply / coarse_solve /
// factorize_blocks.  tests/test_reference_pin.py holds oracle/oracle.c to
// those outputs bit for bit (sequential-order mode).
//
// The payload enters an immergrid::MgHierarchy through its private members
// (the class has no public constructor; MgHierarchy::build needs the meshing
// half of the reference, which is not compiled here): this translation unit
// alone sees them as public.  The reference's sources are compiled as they are.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <Eigen/Cholesky>
#include <Eigen/Core>
#include <Eigen/Dense>
#include <Eigen/SparseCore>
#include <lapacke.h>

#define private public
#include "immergrid/multigrid.hpp"
#undef private
#include "immergrid/mesh.hpp"
#include "immergrid/solvers.hpp"

#include "ig_gpu.h"

namespace ig = immergrid;

// ---- link-time stand-ins for the meshing half (only MgHierarchy::build
// ---- references them; it is never called here).
namespace immergrid {
HierarchicalMesh coarsen(const HierarchicalMesh&) { throw std::logic_error("ref_glue: coarsen is not part of the pinned path"); }
std::shared_ptr<const TrimmedMesh> trim(const HierarchicalMesh&, const LevelSet&, int) {
  throw std::logic_error("ref_glue: trim is not part of the pinned path");
}
FunctionSpace build_space(std::shared_ptr<const TrimmedMesh>, Family, int, int) {
  throw std::logic_error("ref_glue: build_space is not part of the pinned path");
}
SpMat restriction_matrix(const FunctionSpace&, const FunctionSpace&) {
  throw std::logic_error("ref_glue: restriction_matrix is not part of the pinned path");
}
}  // namespace immergrid

// LAPACK dpstf2, UPLO = 'L' (what dpstrf runs for n <= NB); reference-BLAS
// operation order.  Same restatement as host/hierarchy.cpp pstrf_lower.
extern "C" lapack_int LAPACKE_dpstrf(int layout, char uplo, lapack_int n, double* a, lapack_int lda, lapack_int* piv,
                                     lapack_int* rank, double tol) {
  if (layout != LAPACK_COL_MAJOR || (uplo != 'L' && uplo != 'l')) return -1;
  auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(j) * lda + i]; };
  for (int i = 0; i < n; ++i) piv[i] = i + 1;
  *rank = 0;
  if (n == 0) return 0;
  int pvt = 0;
  double ajj = A(0, 0);
  for (int i = 1; i < n; ++i)
    if (A(i, i) > ajj) {
      pvt = i;
      ajj = A(pvt, pvt);
    }
  if (ajj <= 0.0 || std::isnan(ajj)) return 1;
  const double dstop = tol >= 0.0 ? tol : n * 2.220446049250313e-16 * ajj;
  std::vector<double> work(2 * static_cast<size_t>(n), 0.0);
  for (int j = 0; j < n; ++j) {
    for (int i = j; i < n; ++i) {
      if (j > 0) work[i] = work[i] + A(i, j - 1) * A(i, j - 1);
      work[n + i] = A(i, i) - work[i];
    }
    if (j > 0) {
      pvt = j;
      for (int i = j + 1; i < n; ++i)
        if (work[n + i] > work[n + pvt]) pvt = i;
      ajj = work[n + pvt];
      if (ajj <= dstop || std::isnan(ajj)) {
        A(j, j) = ajj;
        *rank = j;
        return 1;
      }
    }
    if (j != pvt) {
      A(pvt, pvt) = A(j, j);
      for (int k = 0; k < j; ++k) std::swap(A(j, k), A(pvt, k));
      for (int k = pvt + 1; k < n; ++k) std::swap(A(k, j), A(k, pvt));
      for (int k = 0; k < pvt - j - 1; ++k) std::swap(A(j + 1 + k, j), A(pvt, j + 1 + k));
      std::swap(work[j], work[pvt]);
      std::swap(piv[j], piv[pvt]);
    }
    ajj = std::sqrt(ajj);
    A(j, j) = ajj;
    if (j < n - 1) {
      for (int k = 0; k < j; ++k) {
        const double t = -A(j, k);
        for (int i = j + 1; i < n; ++i) A(i, j) = A(i, j) + t * A(i, k);
      }
      const double r = 1.0 / ajj;
      for (int i = j + 1; i < n; ++i) A(i, j) *= r;
    }
  }
  *rank = n;
  return 0;
}

namespace {

ig::SpMat to_spmat(const ig_csr& m) {
  if (m.n_rows == 0 && m.n_cols == 0) return ig::SpMat{};
  std::vector<int> outer(m.row_ptr, m.row_ptr + m.n_rows + 1);
  std::vector<int> inner(m.col_idx, m.col_idx + m.nnz);
  std::vector<double> val(m.val, m.val + m.nnz);
  return ig::SpMat(m.n_rows, m.n_cols, std::move(outer), std::move(inner), std::move(val));
}
ig::VecX to_vec(const double* p, int64_t n) {
  ig::VecX v(n);
  for (int64_t i = 0; i < n; ++i) v[i] = p[i];
  return v;
}
void from_vec(const ig::VecX& v, double* p) {
  for (Eigen::Index i = 0; i < v.size(); ++i) p[i] = v[i];
}

struct RefHier {
  ig::MgHierarchy h;
};

ig::SmootherKind kind_of(int k) {
  switch (k) {
    case IG_SMOOTHER_JACOBI: return ig::SmootherKind::Jacobi;
    case IG_SMOOTHER_GAUSS_SEIDEL: return ig::SmootherKind::GaussSeidel;
    case IG_SMOOTHER_MULTIPLICATIVE_SCHWARZ: return ig::SmootherKind::MultiplicativeSchwarz;
    default: return ig::SmootherKind::AdditiveSchwarz;
  }
}

template <class F>
int guarded(F f) {
  try {
    return f();
  } catch (const std::invalid_argument&) {
    return IG_INVALID_ARGUMENT;
  } catch (const std::exception&) {
    return IG_UNSUPPORTED;
  }
}

int report_out(const ig::ConvergenceReport& rep, double* residuals, int32_t* iterations, int32_t* n_res) {
  for (size_t i = 0; i < rep.residuals.size(); ++i) residuals[i] = rep.residuals[i];
  *iterations = rep.iterations;
  *n_res = static_cast<int32_t>(rep.residuals.size());
  return 0;
}

}  // namespace

extern "C" {

// The payload as the reference's MgHierarchy: levels_[l] = {space (unused by
// the solve), A, R, Smoother(A, kind, {post-filter layout, colours, LLT of the
// gathered block (factorize_blocks with the filter off, smoothers.cpp:131-162)},
// gamma)}; coarse_chol_ / coarse_piv_ / rank_ from the payload's dpstrf output.
void* ref_hier_create(const ig_level* levels, int32_t n_levels, const ig_coarse* co) {
  try {
    auto out = std::make_unique<RefHier>();
    ig::MgHierarchy& h = out->h;
    h.levels_.reserve(n_levels);
    for (int l = 0; l < n_levels; ++l)
      h.levels_.push_back(ig::MgLevel{nullptr, to_spmat(levels[l].A), l > 0 ? to_spmat(levels[l].R) : ig::SpMat{}, nullptr});
    for (int l = 1; l < n_levels; ++l) {
      const ig_blocks& B = levels[l].blocks;
      ig::SchwarzPartition part;
      part.layout.blocks.resize(B.n_blocks);
      part.layout.owners.resize(B.n_blocks);
      for (int b = 0; b < B.n_blocks; ++b) {
        part.layout.blocks[b].assign(B.blk_dofs + B.blk_ptr[b], B.blk_dofs + B.blk_ptr[b + 1]);
        part.layout.owners[b] = b;  // owner order == block order; apply never reads owners
      }
      if (B.color_of != nullptr) {
        part.colors.color_of.assign(B.color_of, B.color_of + B.n_blocks);
        part.colors.num_colors = B.n_colors;
      }
      part.factor = ig::factorize_blocks(h.levels_[l].A, part.layout, 0.0);
      h.levels_[l].smoother = std::make_unique<ig::Smoother>(h.levels_[l].A, kind_of(levels[l].smoother_kind),
                                                             std::move(part), levels[l].gamma);
    }
    h.coarse_chol_.resize(co->n, co->n);
    std::memcpy(h.coarse_chol_.data(), co->L, sizeof(double) * static_cast<size_t>(co->n) * co->n);
    h.coarse_piv_.assign(co->piv, co->piv + co->n);
    h.rank_ = co->rank;
    return out.release();
  } catch (const std::exception&) {
    return nullptr;
  }
}
void ref_hier_free(void* p) { delete static_cast<RefHier*>(p); }
int32_t ref_coarse_rank(void* p) { return static_cast<RefHier*>(p)->h.coarse_rank(); }

// The LLT factor the reference holds for block b of level l (s x s, column-major).
int32_t ref_block_factor(void* p, int32_t l, int32_t b, double* out) {
  const auto& f = static_cast<RefHier*>(p)->h.level(l).smoother->partition().factor.at(b).matrixLLT();
  std::memcpy(out, f.data(), sizeof(double) * static_cast<size_t>(f.rows()) * f.cols());
  return static_cast<int32_t>(f.rows());
}

int32_t ref_vcycle_at(void* p, int32_t l, const double* r, int64_t n, double* x) {
  return guarded([&] {
    from_vec(static_cast<RefHier*>(p)->h.vcycle_at(l, to_vec(r, n)), x);
    return 0;
  });
}
int32_t ref_coarse_solve(void* p, const double* r, int64_t n, double* x) {
  return guarded([&] {
    from_vec(static_cast<RefHier*>(p)->h.coarse_solve(to_vec(r, n)), x);
    return 0;
  });
}
int32_t ref_smoother_apply(void* p, int32_t l, const double* r, int64_t n, double* x, int32_t dir) {
  return guarded([&] {
    const auto& s = *static_cast<RefHier*>(p)->h.level(l).smoother;
    from_vec(s.apply(to_vec(r, n), dir == 0 ? ig::SweepDir::Forward : ig::SweepDir::Reverse), x);
    return 0;
  });
}
int32_t ref_smoother_apply_symmetric(void* p, int32_t l, const double* r, int64_t n, double* x) {
  return guarded([&] {
    from_vec(static_cast<RefHier*>(p)->h.level(l).smoother->apply_symmetric(to_vec(r, n)), x);
    return 0;
  });
}

// pcg(A, b, precond = h.apply, tol, maxit) (solvers.cpp:17-71).  Status as
// ig_status: Breakdown / NotConverged are the reference's exceptions.
int32_t ref_pcg(void* p, const double* b, int64_t n, double tol, int32_t maxit, double* x, double* residuals,
                int32_t* iterations, int32_t* n_res) {
  return guarded([&] {
    const ig::MgHierarchy& h = static_cast<RefHier*>(p)->h;
    const ig::SpMat& A = h.level(h.levels() - 1).A;
    const ig::Preconditioner M = [&h](const ig::VecX& r) { return h.apply(r); };
    try {
      auto [sol, rep] = ig::pcg(A, to_vec(b, n), M, tol, maxit);
      from_vec(sol, x);
      report_out(rep, residuals, iterations, n_res);
      return static_cast<int>(rep.converged ? IG_OK : IG_NOT_CONVERGED);
    } catch (const ig::Breakdown& e) {
      report_out(e.report, residuals, iterations, n_res);
      return static_cast<int>(IG_BREAKDOWN);
    } catch (const ig::NotConverged& e) {
      from_vec(e.x, x);
      report_out(e.report, residuals, iterations, n_res);
      return static_cast<int>(IG_NOT_CONVERGED);
    }
  });
}
int32_t ref_richardson(void* p, const double* b, int64_t n, double tol, int32_t maxit, double* x, double* residuals,
                       int32_t* iterations, int32_t* n_res) {
  return guarded([&] {
    const ig::MgHierarchy& h = static_cast<RefHier*>(p)->h;
    const ig::SpMat& A = h.level(h.levels() - 1).A;
    const ig::Preconditioner M = [&h](const ig::VecX& r) { return h.apply(r); };
    try {
      auto [sol, rep] = ig::richardson(A, to_vec(b, n), M, tol, maxit);
      from_vec(sol, x);
      report_out(rep, residuals, iterations, n_res);
      return static_cast<int>(rep.converged ? IG_OK : IG_NOT_CONVERGED);
    } catch (const ig::Diverged& e) {
      report_out(e.report, residuals, iterations, n_res);
      return static_cast<int>(IG_DIVERGED);
    } catch (const ig::NotConverged& e) {
      from_vec(e.x, x);
      report_out(e.report, residuals, iterations, n_res);
      return static_cast<int>(IG_NOT_CONVERGED);
    }
  });
}

// factorize_blocks(A, layout, filter_ratio) (smoothers.cpp:131-162) on a
// pre-filter layout: post-filter member lists and factors.  out_ptr nb+1,
// out_dofs / fac sized for the pre-filter layout.  Returns 0, or 7 for
// EmptyBlockAfterFilter.
int32_t ref_factorize_blocks(const ig_csr* A, int32_t nb, const int32_t* ptr, const int32_t* dofs, double filter_ratio,
                             int32_t* out_ptr, int32_t* out_dofs, int64_t* fac_ptr, double* fac) {
  return guarded([&] {
    const ig::SpMat a = to_spmat(*A);
    ig::BlockLayout L;
    L.blocks.resize(nb);
    L.owners.resize(nb);
    for (int b = 0; b < nb; ++b) {
      L.blocks[b].assign(dofs + ptr[b], dofs + ptr[b + 1]);
      L.owners[b] = b;
    }
    std::vector<Eigen::LLT<ig::MatX>> f;
    try {
      f = ig::factorize_blocks(a, L, filter_ratio);
    } catch (const ig::EmptyBlockAfterFilter&) {
      return 7;
    }
    out_ptr[0] = 0;
    fac_ptr[0] = 0;
    for (int b = 0; b < nb; ++b) {
      const int s = static_cast<int>(L.blocks[b].size());
      std::copy(L.blocks[b].begin(), L.blocks[b].end(), out_dofs + out_ptr[b]);
      out_ptr[b + 1] = out_ptr[b] + s;
      std::memcpy(fac + fac_ptr[b], f[b].matrixLLT().data(), sizeof(double) * static_cast<size_t>(s) * s);
      fac_ptr[b + 1] = fac_ptr[b] + static_cast<int64_t>(s) * s;
    }
    return 0;
  });
}

// The coarsest factorisation exactly as MgHierarchy::build states it
// (multigrid.cpp:57-73): dense copy, max diagonal, tol = 1e-14 max_diag, dpstrf.
int32_t ref_coarse_factor(const ig_csr* A, double* L, int32_t* piv) {
  const ig::SpMat a1 = to_spmat(*A);
  const int n = static_cast<int>(a1.rows());
  ig::MatX chol = ig::MatX(a1);
  double max_diag = 0.0;
  for (int i = 0; i < n; ++i) max_diag = std::max(max_diag, chol(i, i));
  std::vector<int> pv(std::max(n, 1), 0);
  lapack_int rank = 0;
  const double tol = 1e-14 * max_diag;
  const lapack_int info = LAPACKE_dpstrf(LAPACK_COL_MAJOR, 'L', n, chol.data(), std::max(n, 1), pv.data(), &rank, tol);
  if (info < 0) return -1;
  std::memcpy(L, chol.data(), sizeof(double) * static_cast<size_t>(n) * n);
  for (int i = 0; i < n; ++i) piv[i] = pv[i];
  return rank;
}

}  // extern "C"
