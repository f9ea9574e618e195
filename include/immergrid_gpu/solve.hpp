// immergrid_gpu/solve.hpp — header-only C++ surface over the C-ABI
// (include/ig_gpu.h) that restores the reference's solver / preconditioner
// interface (/root/reference/proj/include/immergrid/solvers.hpp,
// multigrid.hpp): same names, argument meaning and exceptions, so a caller of
// the reference's CPU solve can switch to the device path by changing the
// namespace.  Vectors are std::vector<double> (Eigen is optional: with
// <Eigen/SparseCore> available, ig_from_eigen() views an Eigen RowMajor
// SpMat as an ig_csr without copying).
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../ig_gpu.h"

namespace immergrid_gpu {

using Vec = std::vector<double>;

// solvers.hpp:16-23
struct ConvergenceReport {
  std::vector<double> residuals;
  int iterations = 0;
  bool converged = false;
  double seconds = 0.0;
};

// solvers.hpp:25-31
struct Breakdown : std::runtime_error {
  Breakdown(std::string what, ConvergenceReport r) : std::runtime_error(std::move(what)), report(std::move(r)) {}
  ConvergenceReport report;
};

// solvers.hpp:33-41
struct NotConverged : std::runtime_error {
  NotConverged(std::string what, ConvergenceReport r, Vec last)
      : std::runtime_error(std::move(what)), report(std::move(r)), x(std::move(last)) {}
  ConvergenceReport report;
  Vec x;
};

// solvers.hpp:42-48.
struct Diverged : std::runtime_error {
  Diverged(const std::string& what, ConvergenceReport r) : std::runtime_error(what), report(std::move(r)) {}
  ConvergenceReport report;
};

struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int status, const char* what) {
  if (status == IG_OK) return;
  const std::string msg = std::string(what) + ": " + ig_last_error();
  if (status == IG_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw DeviceError(msg);
}

// MgHierarchy (multigrid.hpp:34-74) on the device.  Built from the boundary
// payload (levels[0] = coarsest), immutable afterwards; calls on one object
// serialise inside the library (multigrid.hpp:31-33 reentrancy contract).
class MgHierarchy {
 public:
  MgHierarchy(const ig_level* levels, int n_levels, const ig_coarse& coarse) : n_levels_(n_levels) {
    ig_hier* h = nullptr;
    check(ig_hier_create(levels, n_levels, &coarse, &h), "MgHierarchy");
    h_.reset(h);
    for (int l = 0; l < n_levels; ++l) n_.push_back(levels[l].A.n_rows);
    rank_ = coarse.rank;
  }
  int levels() const { return n_levels_; }
  int coarse_rank() const { return rank_; }
  Vec vcycle_at(int l, const Vec& r) const {
    if (l < 0 || l >= n_levels_) throw std::invalid_argument("vcycle_at: level out of range");
    if (static_cast<int>(r.size()) != n_[l]) throw std::invalid_argument("vcycle_at: residual size mismatch");
    Vec x(r.size());
    check(ig_vcycle_at(h_.get(), l, r.data(), x.data()), "vcycle_at");
    return x;
  }
  Vec apply(const Vec& r) const { return vcycle_at(n_levels_ - 1, r); }
  Vec operator()(const Vec& r) const { return apply(r); }
  Vec coarse_solve(const Vec& r) const { return vcycle_at(0, r); }
  ig_hier* handle() const { return h_.get(); }
  int n(int l) const { return n_[l]; }

  // MgHierarchy::build's algebraic half on the device (ig_hier_build): the
  // Galerkin chain, block factorisations and coarse pstrf from the finest A,
  // the restrictions R[1..L-1] and the pre-filter block layouts
  // prefilter[1..L-1] (fac ignored); gamma[l] resolved per level.
  static MgHierarchy build_on_device(const ig_csr& a_fine, const ig_csr* R, const ig_blocks* prefilter,
                                     const double* gamma, int smoother_kind, double filter_ratio, int n_levels,
                                     double* seconds = nullptr) {
    ig_hier* h = nullptr;
    check(ig_hier_build(&a_fine, R, prefilter, gamma, smoother_kind, filter_ratio, n_levels, &h, seconds),
          "MgHierarchy::build_on_device");
    MgHierarchy m;
    m.h_.reset(h);
    m.n_levels_ = n_levels;
    ig_info info{};
    check(ig_hier_info(h, &info), "MgHierarchy::build_on_device");
    for (int l = 0; l < n_levels; ++l) m.n_.push_back(info.n[l]);
    m.rank_ = info.coarse_rank;  // the device pstrf's accepted pivots
    return m;
  }

  // Dense columns j0.. of the composed operator (IG_OP_A / IG_OP_VCYCLE /
  // IG_OP_SMOOTHER_SYMMETRIC) for dense_spectrum (runner.cpp:84-122),
  // column-major n x count.
  Vec operator_columns(int kind, int j0, int count) const {
    Vec out(static_cast<size_t>(n_[n_levels_ - 1]) * count);
    check(ig_operator_columns(h_.get(), kind, j0, count, out.data()), "operator_columns");
    return out;
  }

 private:
  MgHierarchy() = default;
  struct Del {
    void operator()(ig_hier* h) const { ig_hier_destroy(h); }
  };
  std::unique_ptr<ig_hier, Del> h_;
  int n_levels_ = 0, rank_ = 0;
  std::vector<int> n_;
};

enum class SweepDir { Forward, Reverse };  // smoothers.hpp:14

// Smoother of one level (smoothers.hpp:67-85) as held by the device
// hierarchy: apply(r, dir) and apply_symmetric(r).  A view: the hierarchy must
// outlive it (as the reference's Smoother references its level's A).
class Smoother {
 public:
  Smoother(const MgHierarchy& h, int level) : h_(&h), level_(level) {
    if (level < 1 || level >= h.levels())
      throw std::invalid_argument("Smoother: levels 1..levels()-1 carry a smoother (level 0 is the coarse solve)");
  }
  Vec apply(const Vec& r, SweepDir dir = SweepDir::Forward) const {
    size_check(r);
    Vec x(r.size());
    check(ig_smoother_apply_dir(h_->handle(), level_, r.data(), x.data(), dir == SweepDir::Forward ? 0 : 1),
          "Smoother::apply");
    return x;
  }
  // Symmetric double iteration (M^-1 + M^-T - M^-T A M^-1) r (smoothers.cpp:211-214).
  Vec apply_symmetric(const Vec& r) const {
    size_check(r);
    Vec x(r.size());
    check(ig_smoother_apply_symmetric(h_->handle(), level_, r.data(), x.data()), "Smoother::apply_symmetric");
    return x;
  }
  int level() const { return level_; }

 private:
  void size_check(const Vec& r) const {
    if (static_cast<int>(r.size()) != h_->n(level_)) throw std::invalid_argument("Smoother: size mismatch");
  }
  const MgHierarchy* h_;
  int level_;
};

// One-based wrapper (multigrid.hpp:73-75).
inline Vec vcycle(const MgHierarchy& h, int ell, const Vec& r) { return h.vcycle_at(ell - 1, r); }

// pcg(A, b, precond, tol, maxit) (solvers.hpp:51-53) with precond = the device
// hierarchy built on A (the reference passes the same fine matrix to build and
// pcg, runner.cpp:219,233); the whole iteration runs on the device and
// multiplies by the hierarchy's finest A, so `a` must be that operator (the
// same arrays or an identical copy: ig_hier_matches), else invalid_argument.
inline std::pair<Vec, ConvergenceReport> pcg(const ig_csr& a, const Vec& b, const MgHierarchy& precond,
                                             double tol = 1e-10, int maxit = 1000) {
  const int n = precond.n(precond.levels() - 1);
  if (a.n_rows != a.n_cols || a.n_rows != static_cast<int>(b.size()) || n != a.n_rows)
    throw std::invalid_argument("pcg: dimension mismatch");
  check(ig_hier_matches(precond.handle(), &a), "pcg");
  Vec x(b.size()), res(static_cast<size_t>(maxit) + 1);
  int32_t it = 0;
  double sec = 0.0;
  const int st = ig_pcg(precond.handle(), b.data(), tol, maxit, x.data(), res.data(), &it, &sec);
  ConvergenceReport rep;
  rep.residuals.assign(res.begin(), res.begin() + it + 1);
  rep.iterations = it;
  rep.converged = st == IG_OK;
  rep.seconds = sec;
  if (st == IG_OK) return {std::move(x), std::move(rep)};
  if (st == IG_NOT_CONVERGED) throw NotConverged(ig_last_error(), std::move(rep), std::move(x));
  if (st == IG_BREAKDOWN) throw Breakdown(ig_last_error(), std::move(rep));
  check(st, "pcg");
  return {};
}

// richardson (solvers.hpp:55-59, solvers.cpp:73-120), M = one device V-cycle.
inline std::pair<Vec, ConvergenceReport> richardson(const ig_csr& a, const Vec& b, const MgHierarchy& precond,
                                                    double tol = 1e-10, int maxit = 1000) {
  const int n = precond.n(precond.levels() - 1);
  if (a.n_rows != a.n_cols || a.n_rows != static_cast<int>(b.size()) || n != a.n_rows)
    throw std::invalid_argument("richardson: dimension mismatch");
  check(ig_hier_matches(precond.handle(), &a), "richardson");
  Vec x(b.size()), res(static_cast<size_t>(maxit) + 1);
  int32_t it = 0;
  double sec = 0.0;
  const int st = ig_richardson(precond.handle(), b.data(), tol, maxit, x.data(), res.data(), &it, &sec);
  ConvergenceReport rep;
  rep.residuals.assign(res.begin(), res.begin() + it + 1);
  rep.iterations = it;
  rep.converged = st == IG_OK;
  rep.seconds = sec;
  if (st == IG_OK) return {std::move(x), std::move(rep)};
  if (st == IG_NOT_CONVERGED) throw NotConverged(ig_last_error(), std::move(rep), std::move(x));
  if (st == IG_DIVERGED) throw Diverged(ig_last_error(), std::move(rep));
  check(st, "richardson");
  return {};
}

#if defined(__has_include)
#if __has_include(<Eigen/SparseCore>)
#include <Eigen/SparseCore>
// View an Eigen RowMajor SpMat (immergrid::SpMat, common.hpp:16) as ig_csr;
// the matrix must be compressed (makeCompressed()) and outlive the view.
template <typename SpMatT>
inline ig_csr ig_from_eigen(const SpMatT& m) {
  static_assert(SpMatT::IsRowMajor, "ig_from_eigen: RowMajor SpMat required");
  ig_csr c;
  c.n_rows = static_cast<int32_t>(m.rows());
  c.n_cols = static_cast<int32_t>(m.cols());
  c.nnz = static_cast<int64_t>(m.nonZeros());
  c.row_ptr = m.outerIndexPtr();
  c.col_idx = m.innerIndexPtr();
  c.val = m.valuePtr();
  return c;
}
#endif
#endif

}  // namespace immergrid_gpu
