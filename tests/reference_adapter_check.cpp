// TEST INFRASTRUCTURE: runs include/immergrid_gpu/from_reference.hpp against
// the reference-API shim (tests/shim/).  Reads a hierarchy payload (.igh,
// libig_host.so), fills an immergrid::MgHierarchy the way
// MgHierarchy::build leaves it (per-level A and R, Smoother with its
// post-filter blocks / LLT factors / colours, coarse_rank), uploads it with
// from_reference() and checks that
//   * the solve is bit-identical to the direct boundary path
//     (immergrid_gpu::MgHierarchy(levels, n, coarse) on the same payload);
//   * pcg accepts an identical copy of A and rejects a modified one
//     (ig_hier_matches).
// Prints "adapter ok ..." and exits 0.
//
//   reference_adapter_check <case.igh>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "ig_host.h"
#include "immergrid_gpu/from_reference.hpp"

namespace {

immergrid::SpMat copy_of(const ig_csr& m) {
  std::vector<int> outer(m.row_ptr, m.row_ptr + m.n_rows + 1);
  std::vector<int> inner(m.col_idx, m.col_idx + m.nnz);
  std::vector<double> val(m.val, m.val + m.nnz);
  return immergrid::SpMat(m.n_rows, m.n_cols, std::move(outer), std::move(inner), std::move(val));
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s case.igh\n", argv[0]);
    return 2;
  }
  igh_case* c = nullptr;
  if (igh_read(argv[1], &c) != IG_OK) {
    std::fprintf(stderr, "igh_read: %s\n", igh_last_error());
    return 2;
  }
  const ig_level* lv = nullptr;
  const ig_coarse* co = nullptr;
  int32_t nl = 0, n = 0;
  igh_levels(c, &lv, &nl, &co);
  const double* bp = igh_rhs(c, &n);
  const immergrid_gpu::Vec b(bp, bp + n);

  // The reference's hierarchy, as MgHierarchy::build leaves it.
  immergrid::MgHierarchy ref;
  ref.levels_.resize(static_cast<size_t>(nl));
  for (int l = 0; l < nl; ++l) {
    immergrid::MgLevel& m = ref.levels_[l];
    m.A = copy_of(lv[l].A);
    if (l == 0) continue;
    m.R = copy_of(lv[l].R);
    const ig_blocks& B = lv[l].blocks;
    immergrid::SchwarzPartition part;
    for (int32_t k = 0; k < B.n_blocks; ++k) {
      const int32_t o = B.blk_ptr[k], s = B.blk_ptr[k + 1] - o;
      part.layout.owners.push_back(B.blk_dofs[o]);
      part.layout.blocks.emplace_back(B.blk_dofs + o, B.blk_dofs + o + s);
      immergrid::MatX L(s, s);
      std::memcpy(L.data(), B.fac + B.fac_ptr[k], sizeof(double) * s * s);
      part.factor.emplace_back(std::move(L));
    }
    const bool mult = lv[l].smoother_kind == IG_SMOOTHER_MULTIPLICATIVE_SCHWARZ;
    if (mult) {
      part.colors.num_colors = B.n_colors;
      part.colors.color_of.assign(B.color_of, B.color_of + B.n_blocks);
    }
    m.smoother = std::make_unique<immergrid::Smoother>(
        m.A, mult ? immergrid::SmootherKind::MultiplicativeSchwarz : immergrid::SmootherKind::AdditiveSchwarz,
        std::move(part), lv[l].gamma);
  }
  ref.rank_ = co->rank;

  try {
    const immergrid_gpu::MgHierarchy gpu = immergrid_gpu::from_reference(ref);
    const immergrid_gpu::MgHierarchy direct(lv, nl, *co);
    const ig_csr A = immergrid_gpu::ig_from_eigen(ref.level(nl - 1).A);  // the reference's A (a copy of the payload's)
    auto [x, rep] = immergrid_gpu::pcg(A, b, gpu, 1e-8, 1000);
    auto [xd, repd] = immergrid_gpu::pcg(lv[nl - 1].A, b, direct, 1e-8, 1000);
    if (rep.iterations != repd.iterations || std::memcmp(x.data(), xd.data(), sizeof(double) * x.size()) != 0 ||
        rep.residuals != repd.residuals) {
      std::fprintf(stderr, "adapter solve differs from the direct path (%d vs %d iterations)\n", rep.iterations,
                   repd.iterations);
      return 1;
    }
    // A modified operator must be rejected (the device multiplies by its own A).
    std::vector<double> v(A.val, A.val + A.nnz);
    v[v.size() / 2] *= 1.0 + 1e-12;
    ig_csr bad = A;
    bad.val = v.data();
    bool rejected = false;
    try {
      immergrid_gpu::pcg(bad, b, gpu, 1e-8, 1000);
    } catch (const std::invalid_argument&) {
      rejected = true;
    }
    if (!rejected) {
      std::fprintf(stderr, "pcg accepted an operator that differs from the hierarchy's A\n");
      return 1;
    }
    std::printf("adapter ok n=%d levels=%d iterations=%d coarse_rank=%d (bit-identical to the direct path)\n", n,
                nl, rep.iterations, gpu.coarse_rank());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
  igh_destroy(c);
  return 0;
}
