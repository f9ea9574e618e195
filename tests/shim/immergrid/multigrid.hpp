// Minimal shim of the reference's public hierarchy API (TEST INFRASTRUCTURE):
// the declarations include/immergrid_gpu/from_reference.hpp uses, with the
// names, types and member layout of /root/reference/proj/include/immergrid/
// common.hpp:13-16, smoothers.hpp:14-85 and multigrid.hpp:18-62.  The
// private state the reference keeps (coarse factor, level storage) is public
// here so tests/reference_adapter_check.cpp can fill a hierarchy from the
// boundary payload.
#pragma once
#include <memory>
#include <vector>

#include <Eigen/Cholesky>
#include <Eigen/SparseCore>

namespace immergrid {
using VecX = Eigen::VectorXd;
using MatX = Eigen::MatrixXd;
using SpMat = Eigen::SparseMatrix<double, Eigen::RowMajor>;

enum class SmootherKind { Jacobi, GaussSeidel, AdditiveSchwarz, MultiplicativeSchwarz };
enum class SweepDir { Forward, Reverse };

struct BlockLayout {
  std::vector<int> owners;
  std::vector<std::vector<int>> blocks;
};
struct ColorClasses {
  std::vector<int> color_of;
  int num_colors = 0;
};
struct SchwarzPartition {
  BlockLayout layout;
  ColorClasses colors;
  std::vector<Eigen::LLT<MatX>> factor;
  int max_nk = 0;
};

class Smoother {
 public:
  Smoother(const SpMat& A, SmootherKind kind, SchwarzPartition part, double gamma)
      : A_(&A), kind_(kind), part_(std::move(part)), gamma_(gamma) {}
  SmootherKind kind() const { return kind_; }
  double gamma() const { return gamma_; }
  const SchwarzPartition& partition() const { return part_; }

 private:
  const SpMat* A_;
  SmootherKind kind_;
  SchwarzPartition part_;
  double gamma_ = 1.0;
};

struct FunctionSpace;
struct MgLevel {
  std::shared_ptr<const FunctionSpace> space;
  SpMat A;
  SpMat R;
  std::unique_ptr<Smoother> smoother;
};

class MgHierarchy {
 public:
  int levels() const { return static_cast<int>(levels_.size()); }
  const MgLevel& level(int l) const { return levels_.at(l); }
  int coarse_rank() const { return rank_; }

  // shim-only (private in the reference)
  std::vector<MgLevel> levels_;
  int rank_ = 0;
};
}  // namespace immergrid
