// Restriction matrices, Schwarz block setup, coarse pivoted Cholesky and the
// multigrid hierarchy build, plus the ig_host.h C-ABI.
//   restriction_matrix   proj/src/basis.cpp:376-432 (Lagrange :395-415, B-spline :416-432)
//   select_blocks        proj/src/smoothers.cpp:20-67
//   max_blocks_per_element proj/src/smoothers.cpp:82-97,124-129
//   factorize_blocks     proj/src/smoothers.cpp:131-162
//   make_smoother gamma  proj/src/smoothers.cpp:216-241
//   MgHierarchy::build   proj/src/multigrid.cpp:12-75
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>

#include "../../include/ig_host.h"
#include "host.hpp"
#include "thb.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace igh {

// ------------------------------------------------------------ restriction --

namespace {
double lagrange_coarse_at_fine_node(int p, int a, int coarse_cells, int f) {
  const double sraw = static_cast<double>(f) / (2 * p);
  const int ex = std::min(coarse_cells - 1, static_cast<int>(sraw + 1e-9));
  const int iloc = a - p * ex;
  if (iloc < 0 || iloc > p) return 0.0;
  const double u = sraw - ex;
  double v = 1.0;
  for (int j = 0; j <= p; ++j) {
    if (j == iloc) continue;
    v *= (u - static_cast<double>(j) / p) / (static_cast<double>(iloc - j) / p);
  }
  return v;
}
}  // namespace

Csr restriction_matrix(const Space& fine, const Space& coarse) {
  if (fine.family != coarse.family || fine.p != coarse.p || fine.grid.dim != coarse.grid.dim)
    throw SetupError("restriction_matrix: space families/degrees differ");
  const int dim = fine.grid.dim, p = fine.p;
  for (int d = 0; d < dim; ++d)
    if (fine.grid.res[d] != 2 * coarse.grid.res[d])
      throw SetupError("restriction_matrix: coarse mesh is not the derefinement of fine");
  Csr R;
  R.nr = coarse.n();
  R.nc = fine.n();
  R.ptr.assign(static_cast<size_t>(R.nr) + 1, 0);
  std::vector<std::vector<std::pair<int32_t, double>>> rows(static_cast<size_t>(R.nr));

  if (fine.family == Family::Bspline) {
    Mat T[3];
    for (int d = 0; d < dim; ++d) T[d] = spline::dyadic_refine_matrix(coarse.grid.res[d], p);
    // Nonzero column ranges of each two-scale row.
    std::vector<std::pair<int, int>> cr[3];
    for (int d = 0; d < dim; ++d) {
      cr[d].resize(T[d].r);
      for (int i = 0; i < T[d].r; ++i) {
        int lo = -1, hi = -2;
        for (int j = 0; j < T[d].c; ++j)
          if (T[d](i, j) != 0.0) {
            if (lo < 0) lo = j;
            hi = j;
          }
        cr[d][i] = {lo, hi};
      }
    }
#pragma omp parallel for schedule(dynamic, 256)
    for (int ca = 0; ca < coarse.n(); ++ca) {
      const int64_t u = coarse.anchors[ca];
      const int ax = static_cast<int>(u % coarse.nf[0]);
      const int ay = static_cast<int>((u / coarse.nf[0]) % coarse.nf[1]);
      const int az = static_cast<int>(u / (static_cast<int64_t>(coarse.nf[0]) * coarse.nf[1]));
      auto& row = rows[ca];
      const int zl = dim == 3 ? cr[2][az].first : 0, zh = dim == 3 ? cr[2][az].second : 0;
      for (int fz = zl; fz <= zh; ++fz) {
        const double tz = dim == 3 ? T[2](az, fz) : 1.0;
        if (tz == 0.0) continue;
        for (int fy = cr[1][ay].first; fy <= cr[1][ay].second; ++fy) {
          const double ty = T[1](ay, fy);
          if (ty == 0.0) continue;
          for (int fx = cr[0][ax].first; fx <= cr[0][ax].second; ++fx) {
            const double tx = T[0](ax, fx);
            if (tx == 0.0) continue;
            const int32_t fk = fine.kept[fine.untrimmed(fx, fy, fz)];
            if (fk >= 0) row.push_back({fk, dim == 3 ? tx * ty * tz : tx * ty});
          }
        }
      }
    }
  } else {
    const int ccx = coarse.grid.res[0], ccy = coarse.grid.res[1];
    for (int ca = 0; ca < coarse.n(); ++ca) {
      const int64_t u = coarse.anchors[ca];
      const int ax = static_cast<int>(u % coarse.nf[0]);
      const int ay = static_cast<int>(u / coarse.nf[0]);
      int exlo, exhi, eylo, eyhi;
      anchor_cells(Family::Lagrange, ax, p, ccx, exlo, exhi);
      anchor_cells(Family::Lagrange, ay, p, ccy, eylo, eyhi);
      for (int fy = eylo * 2 * p; fy <= (eyhi + 1) * 2 * p; ++fy) {
        const double ly = lagrange_coarse_at_fine_node(p, ay, ccy, fy);
        if (ly == 0.0) continue;
        for (int fx = exlo * 2 * p; fx <= (exhi + 1) * 2 * p; ++fx) {
          const double lx = lagrange_coarse_at_fine_node(p, ax, ccx, fx);
          if (lx == 0.0) continue;
          const int32_t fk = fine.kept[fine.untrimmed(fx, fy, 0)];
          if (fk >= 0) rows[ca].push_back({fk, lx * ly});
        }
      }
      std::sort(rows[ca].begin(), rows[ca].end(),
                [](const auto& a, const auto& b) { return a.first < b.first; });
    }
  }
  for (int ca = 0; ca < R.nr; ++ca) R.ptr[ca + 1] = R.ptr[ca] + static_cast<int32_t>(rows[ca].size());
  R.col.resize(R.ptr.back());
  R.val.resize(R.ptr.back());
  for (int ca = 0; ca < R.nr; ++ca) {
    int32_t o = R.ptr[ca];
    for (const auto& [c, v] : rows[ca]) {
      R.col[o] = c;
      R.val[o++] = v;
    }
  }
  return R;
}

// ---------------------------------------------------------------- blocks ---

namespace {

// Active-cell counts over axis-aligned cell boxes in O(1) (3D prefix sums).
struct CellCounter {
  int nx, ny, nz;
  std::vector<int32_t> P;  // (nx+1)(ny+1)(nz+1)
  explicit CellCounter(const Space& s) {
    nx = s.grid.res[0];
    ny = s.grid.res[1];
    nz = s.grid.dim == 3 ? s.grid.res[2] : 1;
    P.assign(static_cast<size_t>(nx + 1) * (ny + 1) * (nz + 1), 0);
    for (int x = 0; x < nx; ++x)
      for (int y = 0; y < ny; ++y)
        for (int z = 0; z < nz; ++z)
          P[idx(x + 1, y + 1, z + 1)] = (s.cell_to_el[s.grid.cell_linear(x, y, z)] >= 0) +
                                        P[idx(x, y + 1, z + 1)] + P[idx(x + 1, y, z + 1)] +
                                        P[idx(x + 1, y + 1, z)] - P[idx(x, y, z + 1)] -
                                        P[idx(x, y + 1, z)] - P[idx(x + 1, y, z)] + P[idx(x, y, z)];
  }
  size_t idx(int x, int y, int z) const { return (static_cast<size_t>(x) * (ny + 1) + y) * (nz + 1) + z; }
  // inclusive cell box [l, h]
  int count(const int* l, const int* h) const {
    if (l[0] > h[0] || l[1] > h[1] || l[2] > h[2]) return 0;
    const int x0 = l[0], y0 = l[1], z0 = l[2], x1 = h[0] + 1, y1 = h[1] + 1, z1 = h[2] + 1;
    return P[idx(x1, y1, z1)] - P[idx(x0, y1, z1)] - P[idx(x1, y0, z1)] - P[idx(x1, y1, z0)] +
           P[idx(x0, y0, z1)] + P[idx(x0, y1, z0)] + P[idx(x1, y0, z0)] - P[idx(x0, y0, z0)];
  }
};

void anchor_xyz(const Space& s, int a, int* xyz) {
  const int64_t u = s.anchors[a];
  xyz[0] = static_cast<int>(u % s.nf[0]);
  xyz[1] = static_cast<int>((u / s.nf[0]) % s.nf[1]);
  xyz[2] = static_cast<int>(u / (static_cast<int64_t>(s.nf[0]) * s.nf[1]));
}

void anchor_box(const Space& s, const int* xyz, int* lo, int* hi) {
  for (int d = 0; d < 3; ++d) {
    if (d < s.grid.dim) {
      anchor_cells(s.family, xyz[d], s.p, s.grid.res[d], lo[d], hi[d]);
    } else {
      lo[d] = hi[d] = 0;
    }
  }
}

}  // namespace

Blocks select_blocks(const Space& s, int threads) {
  // Encapsulating-support blocks: members of owner j are the DOFs k whose
  // physical support is contained in j's (smoothers.cpp:20-43).  Supports are
  // the active cells of a tensor box of cells, so supp(k) ⊆ supp(j) iff
  // count(box k) == count(box k ∩ box j); any such k overlaps j, hence lies in
  // the +-W anchor window and is one of the reference's candidates.
  const int n = s.n(), p = s.p, dim = s.grid.dim;
  const CellCounter cc(s);
  const int W = s.family == Family::Bspline ? p : 2 * p;
  std::vector<uint8_t> is_owner(static_cast<size_t>(n), 1);
  if (s.family == Family::Lagrange)
    for (int a = 0; a < n; ++a) {
      int xyz[3];
      anchor_xyz(s, a, xyz);
      is_owner[a] = (xyz[0] % p == 0 && xyz[1] % p == 0);  // nodal owners only
    }
  std::vector<std::vector<int32_t>> mem(static_cast<size_t>(n));
#pragma omp parallel for schedule(dynamic, 1024) num_threads(threads)
  for (int j = 0; j < n; ++j) {
    if (!is_owner[j]) continue;
    int jx[3], jl[3], jh[3];
    anchor_xyz(s, j, jx);
    anchor_box(s, jx, jl, jh);
    const int zr = dim == 3 ? W : 0;
    for (int dz = -zr; dz <= zr; ++dz)
      for (int dy = -W; dy <= W; ++dy)
        for (int dx = -W; dx <= W; ++dx) {
          const int kx[3] = {jx[0] + dx, jx[1] + dy, jx[2] + dz};
          if (kx[0] < 0 || kx[1] < 0 || kx[2] < 0 || kx[0] >= s.nf[0] || kx[1] >= s.nf[1] ||
              kx[2] >= s.nf[2])
            continue;
          const int32_t k = s.kept[s.untrimmed(kx[0], kx[1], kx[2])];
          if (k < 0) continue;
          int kl[3], kh[3], il[3], ih[3];
          anchor_box(s, kx, kl, kh);
          for (int d = 0; d < 3; ++d) {
            il[d] = std::max(kl[d], jl[d]);
            ih[d] = std::min(kh[d], jh[d]);
          }
          const int ck = cc.count(kl, kh);
          if (ck > 0 && cc.count(il, ih) == ck) mem[j].push_back(k);
        }
  }
  Blocks B;
  std::vector<uint8_t> covered(static_cast<size_t>(n), 0);
  for (int j = 0; j < n; ++j)
    for (int32_t k : mem[j]) covered[k] = 1;
  // Owner order with safety-net singletons merged in (stable sort by owner).
  for (int j = 0; j < n; ++j) {
    if (is_owner[j]) {
      B.owners.push_back(j);
      B.dofs.insert(B.dofs.end(), mem[j].begin(), mem[j].end());
      B.ptr.push_back(static_cast<int32_t>(B.dofs.size()));
    }
    if (!covered[j] && !is_owner[j]) {
      B.owners.push_back(j);
      B.dofs.push_back(j);
      B.ptr.push_back(static_cast<int32_t>(B.dofs.size()));
    }
  }
  return B;
}

int max_blocks_per_element(const Blocks& b, const Space& s) {
  // N_K = number of blocks having a member supported on K (smoothers.cpp:82-97).
  const int ne = static_cast<int>(s.el_ix.size());
  std::vector<int32_t> cnt(static_cast<size_t>(ne), 0), mark(static_cast<size_t>(ne), -1);
  const int nb = static_cast<int>(b.owners.size());
  for (int k = 0; k < nb; ++k)
    for (int32_t q = b.ptr[k]; q < b.ptr[k + 1]; ++q) {
      const int a = b.dofs[q];
      for (int64_t t = s.supp_ptr[a]; t < s.supp_ptr[a + 1]; ++t) {
        const int e = s.supp_el[t];
        if (mark[e] != k) {
          mark[e] = k;
          ++cnt[e];
        }
      }
    }
  int mx = 0;
  for (int e = 0; e < ne; ++e) mx = std::max(mx, cnt[e]);
  return mx;
}

namespace {

// Cyclic Jacobi eigen-decomposition of a symmetric s x s matrix (col-major);
// returns eigenvalues ascending and the eigenvector of the smallest one.
void sym_eig_min(const std::vector<double>& A0, int s, double& lmin, std::vector<double>& v0,
                 double& maxdiag) {
  std::vector<double> A = A0, V(static_cast<size_t>(s) * s, 0.0);
  for (int i = 0; i < s; ++i) V[i * s + i] = 1.0;
  maxdiag = -INFINITY;
  for (int i = 0; i < s; ++i) maxdiag = std::max(maxdiag, A0[i * s + i]);
  auto a = [&](int i, int j) -> double& { return A[static_cast<size_t>(j) * s + i]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) {
        const double x = a(i, j) * a(i, j);
        tot += x;
        if (i != j) off += x;
      }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int pp = 0; pp < s - 1; ++pp)
      for (int q = pp + 1; q < s; ++q) {
        const double apq = a(pp, q);
        if (apq == 0.0) continue;
        const double theta = (a(q, q) - a(pp, pp)) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < s; ++k) {
          const double akp = a(k, pp), akq = a(k, q);
          a(k, pp) = c * akp - sn * akq;
          a(k, q) = sn * akp + c * akq;
        }
        for (int k = 0; k < s; ++k) {
          const double apk = a(pp, k), aqk = a(q, k);
          a(pp, k) = c * apk - sn * aqk;
          a(q, k) = sn * apk + c * aqk;
        }
        for (int k = 0; k < s; ++k) {
          const double vkp = V[pp * s + k], vkq = V[q * s + k];
          V[pp * s + k] = c * vkp - sn * vkq;
          V[q * s + k] = sn * vkp + c * vkq;
        }
      }
  }
  int imin = 0;
  for (int i = 1; i < s; ++i)
    if (a(i, i) < a(imin, imin)) imin = i;
  lmin = a(imin, imin);
  v0.assign(V.begin() + static_cast<size_t>(imin) * s, V.begin() + static_cast<size_t>(imin + 1) * s);
}

// Eigen::LLT unblocked in-place lower factorisation (size < 32 path).
void llt_lower(std::vector<double>& m, int n) {
  auto at = [&](int i, int j) -> double& { return m[static_cast<size_t>(j) * n + i]; };
  for (int k = 0; k < n; ++k) {
    double x = at(k, k);
    double sq = 0.0;
    for (int j = 0; j < k; ++j) sq += at(k, j) * at(k, j);
    x -= sq;
    if (x <= 0.0) return;  // NumericalIssue: rest left as is (Eigen returns early)
    x = std::sqrt(x);
    at(k, k) = x;
    for (int i = k + 1; i < n; ++i) {
      double acc = 0.0;
      for (int j = 0; j < k; ++j) acc += at(i, j) * at(k, j);
      at(i, k) = (at(i, k) - acc) / x;
    }
  }
  for (int j = 1; j < n; ++j)
    for (int i = 0; i < j; ++i) at(i, j) = 0.0;  // upper triangle unused
}

}  // namespace

void factorize_blocks(const Csr& A, Blocks& b, double filter_ratio, int threads) {
  const int nb = static_cast<int>(b.owners.size());
  std::vector<std::vector<int32_t>> dofs(static_cast<size_t>(nb));
  std::vector<std::vector<double>> fac(static_cast<size_t>(nb));
  std::vector<int> errs(static_cast<size_t>(nb), 0);
#pragma omp parallel for schedule(dynamic, 1024) num_threads(threads)
  for (int k = 0; k < nb; ++k) {
    std::vector<int32_t>& d = dofs[k];
    d.assign(b.dofs.begin() + b.ptr[k], b.dofs.begin() + b.ptr[k + 1]);
    std::vector<double> Ab;
    auto gather = [&] {
      const int s = static_cast<int>(d.size());
      Ab.assign(static_cast<size_t>(s) * s, 0.0);
      for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j) Ab[static_cast<size_t>(j) * s + i] = A.coeff(d[i], d[j]);
    };
    gather();
    if (filter_ratio > 0.0 && d.size() > 1) {
      while (true) {
        if (d.empty()) {
          errs[k] = 1;
          break;
        }
        const int s = static_cast<int>(d.size());
        double lmin, maxdiag;
        std::vector<double> v0;
        if (s == 1) {
          lmin = Ab[0];
          maxdiag = Ab[0];
          v0.assign(1, 1.0);
        } else {
          sym_eig_min(Ab, s, lmin, v0, maxdiag);
        }
        if (lmin >= filter_ratio * maxdiag) break;
        int worst = 0;
        for (int i = 1; i < s; ++i)
          if (std::fabs(v0[i]) > std::fabs(v0[worst])) worst = i;
        d.erase(d.begin() + worst);
        gather();
      }
    } else if (filter_ratio > 0.0 && d.size() == 1 && !(Ab[0] >= filter_ratio * Ab[0])) {
      // 1x1: lambda = a; a < ratio*a only for a < 0 (or NaN): drop -> empty.
      errs[k] = 1;
    }
    if (d.empty()) errs[k] = 1;
    if (errs[k]) continue;
    llt_lower(Ab, static_cast<int>(d.size()));
    fac[k] = std::move(Ab);
  }
  for (int k = 0; k < nb; ++k)
    if (errs[k]) throw SetupError("factorize_blocks: all DOFs filtered from a block");
  Blocks out;
  out.owners = b.owners;
  out.max_nk = b.max_nk;
  out.color = std::move(b.color);  // colours stay with the pre-filter block indices
  out.n_colors = b.n_colors;
  out.ptr.reserve(static_cast<size_t>(nb) + 1);
  out.fptr.reserve(static_cast<size_t>(nb) + 1);
  int64_t filtered = 0;
  for (int k = 0; k < nb; ++k) {
    filtered += (b.ptr[k + 1] - b.ptr[k]) - static_cast<int64_t>(dofs[k].size());
    out.dofs.insert(out.dofs.end(), dofs[k].begin(), dofs[k].end());
    out.ptr.push_back(static_cast<int32_t>(out.dofs.size()));
    out.fac.insert(out.fac.end(), fac[k].begin(), fac[k].end());
    out.fptr.push_back(static_cast<int64_t>(out.fac.size()));
  }
  out.filtered_dofs = filtered;
  b = std::move(out);
}

int pstrf_lower(int n, double* a, int32_t* piv, double tol) {
  // LAPACK dpstf2, UPLO = 'L' (the unblocked kernel dpstrf runs for n <= NB).
  auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(j) * n + i]; };
  for (int i = 0; i < n; ++i) piv[i] = i + 1;
  if (n == 0) return 0;
  int pvt = 0;
  double ajj = A(0, 0);
  for (int i = 1; i < n; ++i)
    if (A(i, i) > ajj) {
      pvt = i;
      ajj = A(pvt, pvt);
    }
  if (ajj <= 0.0 || std::isnan(ajj)) return 0;
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
        if (work[n + i] > work[n + pvt]) pvt = i;  // MAXLOC: first maximum
      ajj = work[n + pvt];
      if (ajj <= dstop || std::isnan(ajj)) {
        A(j, j) = ajj;
        return j;
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
      // DGEMV('N', n-j-1, j, -1, A(j+1,0), lda, A(j,0), lda, 1, A(j+1,j), 1):
      // reference BLAS column order: y += (-x_k) * A(:,k) for k ascending.
      for (int k = 0; k < j; ++k) {
        const double t = -A(j, k);
        for (int i = j + 1; i < n; ++i) A(i, j) = A(i, j) + t * A(i, k);
      }
      const double r = 1.0 / ajj;  // DSCAL by ONE / AJJ
      for (int i = j + 1; i < n; ++i) A(i, j) *= r;
    }
  }
  return n;
}

}  // namespace igh

// ============================================================== C-ABI ======

using namespace igh;

struct igh_case {
  igh_config cfg{};
  std::string geometry;
  std::vector<std::unique_ptr<Space>> spaces;  // [0] = coarsest (empty when read from file)
  std::vector<std::unique_ptr<GSpace>> gspaces;  // THB levels
  std::vector<Csr> A, R;
  std::vector<Blocks> B;
  // Pre-filter Schwarz layouts (block pointers, DOFs) as select_blocks made
  // them: the input of factorize_blocks, kept for the device factorisation.
  std::vector<std::vector<int32_t>> pre_ptr, pre_dofs;
  // Finest-level element tables (device assembly payload; uniform spaces).
  std::vector<double> tabK, tabF;
  std::vector<int32_t> el_table;
  int32_t n_tables = 0;
  // Finest level: physical support volume / untrimmed support cell volume per DOF.
  std::vector<double> supp_frac;
  // Cut-element quadrature payload (igh_cut3_payload), built on demand.
  std::vector<double> cut_lo, cut_ext[3], cut_prog, g_tet, g_tri, g_box;
  std::vector<int32_t> cut_cls, cut_table;
  std::vector<double> c2_lo, c2_hi, c2_ext[2], c2_gq, c2_gq1;
  std::vector<int32_t> c2_cls, c2_cut, c2_sides, c2_table;
  std::vector<double> t_lo, t_hi, t_E;
  std::vector<int32_t> t_cut, t_sides, t_rptr, t_anchors, t_sel, t_sli;
  std::vector<int64_t> t_sptr;
  std::vector<double> gamma;
  std::vector<int32_t> kind;
  std::vector<double> coarseL;
  std::vector<int32_t> piv;
  int32_t rank = 0;
  std::vector<double> b;
  std::vector<ig_level> lv;
  ig_coarse co{};
  igh_info info{};
  std::vector<std::vector<int32_t>> xyz;  // per level anchors (ax,ay,az)
  bool geometric = false;  // igh_build_geometry: no operators, factors or rhs
  void wire();
};

namespace {
thread_local std::string g_err;
int fail(const std::string& m, int code = IG_INVALID_ARGUMENT) {
  g_err = m;
  return code;
}
double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
ig_csr view(const Csr& m) {
  ig_csr c;
  c.n_rows = m.nr;
  c.n_cols = m.nc;
  c.nnz = m.nnz();
  c.row_ptr = m.ptr.data();
  c.col_idx = m.col.data();
  c.val = m.val.data();
  return c;
}
int resolve_threads(int t) {
#ifdef _OPENMP
  return t > 0 ? t : omp_get_max_threads();
#else
  (void)t;
  return 1;
#endif
}
}  // namespace

void igh_case::wire() {
  const int L = static_cast<int>(A.size());
  lv.assign(L, ig_level{});
  for (int l = 0; l < L; ++l) {
    lv[l].A = view(A[l]);
    lv[l].R = view(R[l]);
    lv[l].smoother_kind = kind[l];
    lv[l].gamma = gamma[l];
    ig_blocks& bb = lv[l].blocks;
    bb.n_blocks = static_cast<int32_t>(B[l].owners.size());
    bb.blk_ptr = B[l].ptr.data();
    bb.blk_dofs = B[l].dofs.data();
    bb.fac_ptr = B[l].fptr.data();
    bb.fac = B[l].fac.data();
    bb.n_colors = B[l].n_colors;
    bb.color_of = B[l].color.empty() ? nullptr : B[l].color.data();
  }
  co.n = (A.empty() || geometric) ? 0 : A[0].nr;
  co.rank = rank;
  co.L = coarseL.data();
  co.piv = piv.data();
  info.n_levels = L;
  for (int l = 0; l < L && l < 16; ++l) {
    info.n[l] = A[l].nr;
    info.nnz[l] = A[l].nnz();
    info.max_nk[l] = B[l].max_nk;
    info.filtered_dofs[l] = B[l].filtered_dofs;
  }
  info.coarse_rank = rank;
}

extern "C" {

const char* igh_last_error(void) { return g_err.c_str(); }

void igh_config_default(igh_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->dim = 2;
  c->geometry = "constant(1)";
  c->origin[0] = c->origin[1] = c->origin[2] = 0.0;
  c->extent[0] = c->extent[1] = c->extent[2] = 1.0;
  c->resolution[0] = c->resolution[1] = c->resolution[2] = 16;
  c->family = 1;
  c->degree = 2;
  c->levels = 2;
  c->quad_depth = 3;
  c->gauss_order = 0;
  c->classify_depth = 2;
  c->edge_tol = 1e-12;
  c->body_force = 1.0;
  c->beta = 0.0;
  c->dirichlet_box_sides = 1;
  c->smoother_kind = IG_SMOOTHER_ADDITIVE_SCHWARZ;
  c->gamma = 0.0;
  c->filter_ratio = 1e-16;
  c->threads = 0;
}

}  // extern "C"

namespace {
// igh_build (numeric) and igh_build_geometry (numeric = false: spaces,
// restrictions, pre-filter block layouts, colours, damping and the element
// tables of the Inside classes; no cut-element integration, no assembly, no
// Galerkin products, no factorisations -- the device pipeline computes those).
int build_impl(const igh_config* cfg, igh_case** out, bool numeric) {
  if (!cfg || !out) return fail("igh_build: null argument");
  *out = nullptr;
  try {
    auto c = std::make_unique<igh_case>();
    c->cfg = *cfg;
    c->geometry = cfg->geometry ? cfg->geometry : "constant(1)";
    c->cfg.geometry = nullptr;
    const int threads = resolve_threads(cfg->threads);
    const int dim = cfg->dim;
    if (dim != 2 && dim != 3) return fail("igh_build: dim must be 2 or 3");
    if (cfg->levels < 1) return fail("build: levels must be >= 1");
    if (cfg->levels > 16) return fail("build: at most 16 levels");
    if (cfg->smoother_kind != IG_SMOOTHER_ADDITIVE_SCHWARZ &&
        cfg->smoother_kind != IG_SMOOTHER_MULTIPLICATIVE_SCHWARZ)
      return fail("igh_build: only Schwarz smoothers are set up on the host", IG_UNSUPPORTED);
    Grid g;
    g.dim = dim;
    for (int d = 0; d < 3; ++d) {
      g.origin[d] = cfg->origin[d];
      g.extent[d] = cfg->extent[d];
      g.res[d] = d < dim ? cfg->resolution[d] : 1;
    }
    const LevelSet ls = parse_levelset(c->geometry);
    const bool thb = cfg->family == 2;
    if (thb && dim != 2) return fail("igh_build: THB is 2D only");
    const Family fam = cfg->family == 0 ? Family::Lagrange : Family::Bspline;
    QuadConfig qc;
    qc.depth = cfg->quad_depth;
    qc.gauss_order = cfg->gauss_order > 0 ? cfg->gauss_order : cfg->degree + 1;
    qc.classify_depth = cfg->classify_depth;
    qc.edge_tol = cfg->edge_tol;
    ProblemConfig prob;
    prob.body_force = cfg->body_force;
    prob.beta = cfg->beta;
    prob.dirichlet_box_sides = cfg->dirichlet_box_sides != 0;

    const double t0 = now();
    const int L = cfg->levels;
    std::vector<Csr> Adown, Rdown;
    Assembled as;
    double t1 = 0.0;
    std::vector<std::unique_ptr<Space>> down;
    std::vector<std::unique_ptr<GSpace>> gdown;
    double t_gal = 0.0, t_fac = 0.0;
    auto empty_op = [](int32_t n) {  // geometric half: an n x n operator without entries
      Csr m;
      m.nr = m.nc = n;
      m.ptr.assign(static_cast<size_t>(n) + 1, 0);
      return m;
    };
    auto galerkin = [&](Csr r) {  // A_c = R (A R^T) (multigrid.cpp:39-41)
      if (!numeric) {
        Adown.push_back(empty_op(r.nr));
        Rdown.push_back(std::move(r));
        return;
      }
      const double tg = now();
      struct Acc { double& t; double t0; ~Acc() { t += now() - t0; } } acc_{t_gal, tg};
      const Csr rt = transpose(r);
      Csr ap = spgemm(Adown.back(), rt, threads);
      Adown.push_back(spgemm(r, ap, threads));
      Rdown.push_back(std::move(r));
    };
    if (thb) {
      HMesh mesh = HMesh::uniform(g);
      for (int k = 0; k < cfg->n_refine_boxes; ++k) mesh.refine_by_box(cfg->refine_boxes + 4 * k);
      for (int k = 0; k < cfg->refine_passes; ++k)
        mesh.refine_near_circle(cfg->refine_circle[0], cfg->refine_circle[1], cfg->refine_circle[2], cfg->refine_dist);
      gdown.push_back(build_thb(mesh, ls, cfg->degree, cfg->classify_depth, threads));
      if (numeric) {
        as = assemble_g(*gdown[0], prob, qc, threads);
      } else {
        as.A = empty_op(gdown[0]->n());
        as.b.assign(static_cast<size_t>(gdown[0]->n()), 0.0);
      }
      t1 = now();
      Adown.push_back(std::move(as.A));
      for (int l = 1; l < L; ++l) {
        const HMesh& fm = gdown.back()->mesh;
        if (fm.g.res[0] % 2 != 0 || fm.g.res[1] % 2 != 0)
          return fail("mesh does not support " + std::to_string(L - 1) + " coarsenings");
        gdown.push_back(build_thb(coarsen(fm), ls, cfg->degree, cfg->classify_depth, threads));
        galerkin(restriction_thb(*gdown[l - 1], *gdown[l], threads));
      }
    } else {
      down.push_back(build_space(g, ls, fam, cfg->degree, cfg->classify_depth, threads));
      as = assemble(*down[0], prob, qc, threads, numeric);
      c->tabK = std::move(as.tabK);
      c->tabF = std::move(as.tabF);
      c->el_table = std::move(as.el_table);
      c->n_tables = as.n_tables;
      t1 = now();
      Adown.push_back(std::move(as.A));
      for (int l = 1; l < L; ++l) {
        Grid cg = down.back()->grid;
        for (int d = 0; d < dim; ++d) {
          if (cg.res[d] % 2 != 0)
            return fail("mesh does not support " + std::to_string(L - 1) + " coarsenings");
          cg.res[d] /= 2;
        }
        down.push_back(build_space(cg, ls, fam, cfg->degree, cfg->classify_depth, threads));
        galerkin(restriction_matrix(*down[l - 1], *down[l]));
      }
    }
    Rdown.push_back(Csr{});  // coarsest: empty R
    // Reverse: [0] = coarsest (multigrid.cpp:47-50).
    for (int l = L - 1; l >= 0; --l) {
      if (thb)
        c->gspaces.push_back(std::move(gdown[l]));
      else
        c->spaces.push_back(std::move(down[l]));
      c->A.push_back(std::move(Adown[l]));
      c->R.push_back(std::move(Rdown[l]));
    }
    c->R[0].nr = 0;
    c->R[0].nc = 0;
    // R on level l maps level l -> l-1: rows n_{l-1}, cols n_l (already so).
    c->B.resize(L);
    c->gamma.assign(L, 0.0);
    c->kind.assign(L, cfg->smoother_kind);
    for (int l = 1; l < L; ++l) {
      Blocks b;
      if (thb) {
        b = select_blocks_g(*c->gspaces[l]);
        b.max_nk = max_blocks_per_element_g(b, *c->gspaces[l]);
      } else {
        b = select_blocks(*c->spaces[l], threads);
        b.max_nk = max_blocks_per_element(b, *c->spaces[l]);
      }
      // Colours of the pre-filter layout (make_smoother: color_blocks runs
      // before factorize_blocks, smoothers.cpp:228-232).
      if (cfg->smoother_kind == IG_SMOOTHER_MULTIPLICATIVE_SCHWARZ) {
        if (thb) {
          const GSpace& gs = *c->gspaces[l];
          color_blocks(b, static_cast<int>(gs.el.size()), [&](int d, auto&& f) {
            for (int e : gs.supp[d]) f(e);
          });
        } else {
          const Space& sp = *c->spaces[l];
          color_blocks(b, static_cast<int>(sp.el_ix.size()), [&](int d, auto&& f) {
            for (int64_t t = sp.supp_ptr[d]; t < sp.supp_ptr[d + 1]; ++t) f(sp.supp_el[t]);
          });
        }
      }
      if (c->pre_ptr.size() < static_cast<size_t>(L)) {
        c->pre_ptr.resize(L);
        c->pre_dofs.resize(L);
      }
      c->pre_ptr[l] = b.ptr;
      c->pre_dofs[l] = b.dofs;
      const double tf = now();
      if (numeric) factorize_blocks(c->A[l], b, cfg->filter_ratio, threads);
      t_fac += now() - tf;
      double gm = cfg->gamma;
      if (gm <= 0.0) {
        const bool damped = cfg->smoother_kind == IG_SMOOTHER_ADDITIVE_SCHWARZ;
        gm = damped ? 1.0 / std::max(1, b.max_nk) : 1.0;
      }
      c->gamma[l] = gm;
      c->B[l] = std::move(b);
    }
    // Coarsest pivoted Cholesky (multigrid.cpp:57-73).
    const Csr& a1 = c->A[0];
    const int n0 = numeric ? a1.nr : 0;
    c->coarseL.assign(static_cast<size_t>(n0) * n0, 0.0);
    for (int i = 0; i < n0; ++i)
      for (int32_t k = a1.ptr[i]; k < a1.ptr[i + 1]; ++k)
        c->coarseL[static_cast<size_t>(a1.col[k]) * n0 + i] = a1.val[k];
    double max_diag = 0.0;
    for (int i = 0; i < n0; ++i) max_diag = std::max(max_diag, c->coarseL[static_cast<size_t>(i) * n0 + i]);
    c->piv.assign(std::max(n0, 1), 0);
    c->rank = pstrf_lower(n0, c->coarseL.data(), c->piv.data(), 1e-14 * max_diag);
    const double t2 = now();
    c->b = std::move(as.b);
    if (numeric && !thb && !as.el_vol.empty()) {
      const Space& s = *c->spaces.back();
      const int dim = s.grid.dim;
      c->supp_frac.assign(static_cast<size_t>(s.n()), 0.0);
      for (int a = 0; a < s.n(); ++a) {
        int32_t ax[3];
        anchor_xyz(s, a, ax);
        double cells = 1.0;
        for (int d = 0; d < dim; ++d) {
          int lo, hi;
          anchor_cells(s.family, ax[d], s.p, s.grid.res[d], lo, hi);
          cells *= hi - lo + 1;
        }
        double v = 0.0;
        for (int64_t k = s.supp_ptr[a]; k < s.supp_ptr[a + 1]; ++k) v += as.el_vol[s.supp_el[k]];
        c->supp_frac[a] = v / cells;
      }
    }
    c->xyz.resize(L);
    for (int l = 0; l < L; ++l) {
      if (thb) {  // (ax, ay, hierarchy level)
        const GSpace& s = *c->gspaces[l];
        c->xyz[l].resize(static_cast<size_t>(s.n()) * 3);
        for (int a = 0; a < s.n(); ++a) {
          c->xyz[l][3 * a] = s.anchors[a][1];
          c->xyz[l][3 * a + 1] = s.anchors[a][2];
          c->xyz[l][3 * a + 2] = s.anchors[a][0];
        }
        continue;
      }
      const Space& s = *c->spaces[l];
      c->xyz[l].resize(static_cast<size_t>(s.n()) * 3);
      for (int a = 0; a < s.n(); ++a) anchor_xyz(s, a, &c->xyz[l][static_cast<size_t>(a) * 3]);
    }
    c->geometric = !numeric;
    c->wire();
    c->info.cut_elements = as.cut_elements;
    c->info.eta = as.eta;
    c->info.seconds_assemble = t1 - t0;
    c->info.seconds_mg_setup = t2 - t1;
    if (std::getenv("IG_TIMING"))
      std::fprintf(stderr, "igh_build: assemble %.3f s, mg setup %.3f s (galerkin %.3f, block factorization %.3f)\n",
                   t1 - t0, t2 - t1, t_gal, t_fac);
    *out = c.release();
    return IG_OK;
  } catch (const std::exception& e) {
    return fail(e.what());
  }
}
}  // namespace

extern "C" {

int igh_build(const igh_config* cfg, igh_case** out) { return build_impl(cfg, out, true); }
int igh_build_geometry(const igh_config* cfg, igh_case** out) { return build_impl(cfg, out, false); }

int igh_cut3_payload(igh_case* c, ig_cut3* out) {
  if (!c || !out) return fail("igh_cut3_payload: null argument");
  if (c->spaces.empty() || c->el_table.empty() || c->cfg.dim != 3 || c->cfg.family != 1)
    return fail("igh_cut3_payload: built 3D uniform B-spline cases only", IG_UNSUPPORTED);
  try {
    const Space& s = *c->spaces.back();
    const int q = s.p + 1;
    if (c->cut_prog.empty() && !s.ls.program(c->cut_prog))
      return fail("igh_cut3_payload: the level set has no device program (star / affine)", IG_UNSUPPORTED);
    const int ncls = static_cast<int>(s.ext[0].size() * s.ext[1].size() * s.ext[2].size());
    if (c->cut_table.empty()) {
      const int ne = static_cast<int>(s.el_ix.size());
      for (int e = 0; e < ne; ++e) {
        if (c->el_table[e] < ncls) continue;  // Inside class tables; the rest are the cut elements
        double lo[3], hi[3];
        s.grid.cell_box(s.el_ix[e], s.el_iy[e], s.el_iz[e], lo, hi);
        c->cut_lo.insert(c->cut_lo.end(), lo, lo + 3);
        c->cut_cls.push_back(s.ext_cls[0][s.el_ix[e]]);
        c->cut_cls.push_back(s.ext_cls[1][s.el_iy[e]]);
        c->cut_cls.push_back(s.ext_cls[2][s.el_iz[e]]);
        c->cut_table.push_back(c->el_table[e]);
      }
      for (int d = 0; d < 3; ++d) {
        c->cut_ext[d].clear();
        for (const Mat& m : s.ext[d]) c->cut_ext[d].insert(c->cut_ext[d].end(), m.a.begin(), m.a.end());
      }
      auto rule01 = [](int n, std::vector<double>& out01) {  // assembly.cpp gauss01
        std::vector<double> nd, wt;
        gauss_legendre(n, nd, wt);
        out01.clear();
        for (int i = 0; i < n; ++i) out01.push_back(0.5 * (nd[i] + 1.0));
        for (int i = 0; i < n; ++i) out01.push_back(0.5 * wt[i]);
      };
      rule01(2, c->g_tet);
      rule01(3, c->g_tri);
      std::vector<double> nd, wt;
      gauss_legendre(q, nd, wt);
      c->g_box = nd;
      c->g_box.insert(c->g_box.end(), wt.begin(), wt.end());
    }
    *out = ig_cut3{};
    out->p = s.p;
    out->n_cut = static_cast<int32_t>(c->cut_table.size());
    out->lo = c->cut_lo.data();
    out->cls = c->cut_cls.data();
    for (int d = 0; d < 3; ++d) {
      out->n_cls[d] = static_cast<int32_t>(s.ext[d].size());
      out->ext[d] = c->cut_ext[d].data();
      out->h[d] = s.grid.h(d);
    }
    double hmin = s.grid.h(0);
    for (int d = 1; d < 3; ++d) hmin = std::min(hmin, s.grid.h(d));
    out->beta = c->cfg.beta > 0.0 ? c->cfg.beta : 2.0 / hmin;  // default_penalty (assembly.cpp:7-10)
    out->f = c->cfg.body_force;
    out->depth = c->cfg.quad_depth;
    out->classify_depth = c->cfg.classify_depth;
    out->edge_tol = c->cfg.edge_tol;
    out->prog_len = static_cast<int32_t>(c->cut_prog.size());
    out->prog = c->cut_prog.data();
    out->gauss_tet = c->g_tet.data();
    out->gauss_tri = c->g_tri.data();
    out->gauss_box = c->g_box.data();
    out->table = c->cut_table.data();
    return IG_OK;
  } catch (const std::exception& e) {
    return fail(e.what());
  }
}

int igh_cut2_payload(igh_case* c, ig_cut2* out) {
  if (!c || !out) return fail("igh_cut2_payload: null argument");
  if (c->spaces.empty() || c->el_table.empty() || c->cfg.dim != 2)
    return fail("igh_cut2_payload: built 2D uniform cases only", IG_UNSUPPORTED);
  try {
    const Space& s = *c->spaces.back();
    if (c->cut_prog.empty() && !s.ls.program(c->cut_prog))
      return fail("igh_cut2_payload: the level set has no device program (star / affine)", IG_UNSUPPORTED);
    const int ncls = static_cast<int>(s.ext[0].size() * s.ext[1].size());
    const int go = c->cfg.gauss_order > 0 ? c->cfg.gauss_order : c->cfg.degree + 1;
    if (c->c2_table.empty()) {
      const int ne = static_cast<int>(s.el_ix.size());
      for (int e = 0; e < ne; ++e) {
        if (c->el_table[e] < ncls) continue;
        double lo[3], hi[3];
        s.grid.cell_box(s.el_ix[e], s.el_iy[e], 0, lo, hi);
        c->c2_lo.insert(c->c2_lo.end(), lo, lo + 2);
        c->c2_hi.insert(c->c2_hi.end(), hi, hi + 2);
        c->c2_cls.push_back(s.ext_cls[0][s.el_ix[e]]);
        c->c2_cls.push_back(s.ext_cls[1][s.el_iy[e]]);
        c->c2_cut.push_back(s.el_tag[e] == kCut ? 1 : 0);
        int mask = 0;  // box_sides (assembly.cpp:24-33): 0 bottom, 1 right, 2 top, 3 left
        if (c->cfg.dirichlet_box_sides) {
          if (s.el_iy[e] == 0) mask |= 1;
          if (s.el_ix[e] == s.grid.res[0] - 1) mask |= 2;
          if (s.el_iy[e] == s.grid.res[1] - 1) mask |= 4;
          if (s.el_ix[e] == 0) mask |= 8;
        }
        c->c2_sides.push_back(mask);
        c->c2_table.push_back(c->el_table[e]);
      }
      for (int d = 0; d < 2; ++d) {
        c->c2_ext[d].clear();
        for (const Mat& m : s.ext[d]) c->c2_ext[d].insert(c->c2_ext[d].end(), m.a.begin(), m.a.end());
      }
      std::vector<double> nd, wt;
      gauss_legendre(go, nd, wt);
      c->c2_gq = nd;
      c->c2_gq.insert(c->c2_gq.end(), wt.begin(), wt.end());
      gauss_legendre(go + 1, nd, wt);
      c->c2_gq1 = nd;
      c->c2_gq1.insert(c->c2_gq1.end(), wt.begin(), wt.end());
    }
    *out = ig_cut2{};
    out->p = s.p;
    out->n_elem = static_cast<int32_t>(c->c2_table.size());
    out->lo = c->c2_lo.data();
    out->hi = c->c2_hi.data();
    out->cls = c->c2_cls.data();
    out->cut = c->c2_cut.data();
    out->sides = c->c2_sides.data();
    for (int d = 0; d < 2; ++d) {
      out->n_cls[d] = static_cast<int32_t>(s.ext[d].size());
      out->ext[d] = c->c2_ext[d].data();
    }
    const double hmin = std::min(s.grid.h(0), s.grid.h(1));
    out->beta = c->cfg.beta > 0.0 ? c->cfg.beta : 2.0 / hmin;
    out->f = c->cfg.body_force;
    out->depth = c->cfg.quad_depth;
    out->classify_depth = c->cfg.classify_depth;
    out->gauss_order = go;
    out->edge_tol = c->cfg.edge_tol;
    out->prog_len = static_cast<int32_t>(c->cut_prog.size());
    out->prog = c->cut_prog.data();
    out->gauss_q = c->c2_gq.data();
    out->gauss_q1 = c->c2_gq1.data();
    out->table = c->c2_table.data();
    return IG_OK;
  } catch (const std::exception& e) {
    return fail(e.what());
  }
}

int igh_thb_payload(igh_case* c, ig_thb_asm* out) {
  if (!c || !out) return fail("igh_thb_payload: null argument");
  if (c->gspaces.empty()) return fail("igh_thb_payload: built THB cases only", IG_UNSUPPORTED);
  try {
    const GSpace& s = *c->gspaces.back();
    if (c->cut_prog.empty() && !s.ls.program(c->cut_prog))
      return fail("igh_thb_payload: the level set has no device program (star / affine)", IG_UNSUPPORTED);
    const HMesh& mesh = s.mesh;
    const int go = c->cfg.gauss_order > 0 ? c->cfg.gauss_order : c->cfg.degree + 1;
    if (c->t_rptr.empty()) {
      const int ne = static_cast<int>(s.el.size());
      c->t_rptr.assign(1, 0);
      for (int e = 0; e < ne; ++e) {
        const GSpace::El& el = s.el[e];
        double lo[2], hi[2];
        mesh.cell_box(el.l, el.ix, el.iy, lo, hi);
        c->t_lo.insert(c->t_lo.end(), lo, lo + 2);
        c->t_hi.insert(c->t_hi.end(), hi, hi + 2);
        c->t_cut.push_back(el.tag == kCut ? 1 : 0);
        int mask = 0;
        if (c->cfg.dirichlet_box_sides) {
          const int cx = mesh.cells_x(el.l), cy = mesh.cells_y(el.l);
          if (el.iy == 0) mask |= 1;
          if (el.ix == cx - 1) mask |= 2;
          if (el.iy == cy - 1) mask |= 4;
          if (el.ix == 0) mask |= 8;
        }
        c->t_sides.push_back(mask);
        c->t_anchors.insert(c->t_anchors.end(), el.anchors.begin(), el.anchors.end());
        c->t_E.insert(c->t_E.end(), el.E.begin(), el.E.end());
        c->t_rptr.push_back(static_cast<int32_t>(c->t_anchors.size()));
      }
      const int n = s.n();
      c->t_sptr.assign(1, 0);
      for (int a = 0; a < n; ++a) {
        for (int e : s.supp[a]) {
          const GSpace::El& el = s.el[e];
          const int li = static_cast<int>(std::find(el.anchors.begin(), el.anchors.end(), a) - el.anchors.begin());
          c->t_sel.push_back(e);
          c->t_sli.push_back(li);
        }
        c->t_sptr.push_back(static_cast<int64_t>(c->t_sel.size()));
      }
      std::vector<double> nd, wt;
      gauss_legendre(go, nd, wt);
      c->c2_gq = nd;
      c->c2_gq.insert(c->c2_gq.end(), wt.begin(), wt.end());
      gauss_legendre(go + 1, nd, wt);
      c->c2_gq1 = nd;
      c->c2_gq1.insert(c->c2_gq1.end(), wt.begin(), wt.end());
    }
    *out = ig_thb_asm{};
    out->p = s.p;
    out->n = s.n();
    out->n_elem = static_cast<int32_t>(s.el.size());
    out->lo = c->t_lo.data();
    out->hi = c->t_hi.data();
    out->cut = c->t_cut.data();
    out->sides = c->t_sides.data();
    out->erow_ptr = c->t_rptr.data();
    out->anchors = c->t_anchors.data();
    out->E = c->t_E.data();
    out->supp_ptr = c->t_sptr.data();
    out->supp_el = c->t_sel.data();
    out->supp_li = c->t_sli.data();
    const int M = mesh.max_level();
    const double hmin = std::min(mesh.g.extent[0] / mesh.cells_x(M), mesh.g.extent[1] / mesh.cells_y(M));
    out->beta = c->cfg.beta > 0.0 ? c->cfg.beta : 2.0 / hmin;
    out->f = c->cfg.body_force;
    out->depth = c->cfg.quad_depth;
    out->classify_depth = c->cfg.classify_depth;
    out->gauss_order = go;
    out->edge_tol = c->cfg.edge_tol;
    out->prog_len = static_cast<int32_t>(c->cut_prog.size());
    out->prog = c->cut_prog.data();
    out->gauss_q = c->c2_gq.data();
    out->gauss_q1 = c->c2_gq1.data();
    return IG_OK;
  } catch (const std::exception& e) {
    return fail(e.what());
  }
}

int igh_support_fraction(const igh_case* c, double* out) {
  if (!c || !out) return fail("igh_support_fraction: null argument");
  if (c->supp_frac.empty())
    return fail("igh_support_fraction: only built uniform (B-spline / Lagrange) cases carry support fractions",
                IG_UNSUPPORTED);
  std::copy(c->supp_frac.begin(), c->supp_frac.end(), out);
  return IG_OK;
}

int igh_prefilter_blocks(const igh_case* c, int32_t level, int32_t* n_blocks, const int32_t** blk_ptr,
                         const int32_t** blk_dofs) {
  if (!c || !n_blocks || !blk_ptr || !blk_dofs) return fail("igh_prefilter_blocks: null argument");
  if (level < 1 || static_cast<size_t>(level) >= c->pre_ptr.size() || c->pre_ptr[level].empty())
    return fail("igh_prefilter_blocks: no pre-filter layout for this level (levels 1.., built cases only)");
  *n_blocks = static_cast<int32_t>(c->pre_ptr[level].size()) - 1;
  *blk_ptr = c->pre_ptr[level].data();
  *blk_dofs = c->pre_dofs[level].data();
  return IG_OK;
}

int igh_assembly_payload(const igh_case* c, ig_assembly* out) {
  if (!c || !out) return fail("igh_assembly_payload: null argument");
  if (c->spaces.empty() || c->el_table.empty())
    return fail("igh_assembly_payload: only built uniform (B-spline / Lagrange) cases carry the element tables");
  const Space& s = *c->spaces.back();
  *out = ig_assembly{};
  out->dim = s.grid.dim;
  out->p = s.p;
  out->family = s.family == Family::Bspline ? 1 : 0;
  out->n = s.n();
  out->n_elements = static_cast<int32_t>(s.el_ix.size());
  out->n_tables = c->n_tables;
  for (int d = 0; d < 3; ++d) out->nf[d] = s.nf[d];
  out->el_ix = s.el_ix.data();
  out->el_iy = s.el_iy.data();
  out->el_iz = s.grid.dim == 3 ? s.el_iz.data() : nullptr;
  out->el_table = c->el_table.data();
  out->K = c->tabK.data();
  out->F = c->tabF.data();
  out->anchors = s.anchors.data();
  out->supp_ptr = s.supp_ptr.data();
  out->supp_el = s.supp_el.data();
  out->kept = s.kept.data();
  return IG_OK;
}

int igh_levels(const igh_case* c, const ig_level** levels, int32_t* n_levels, const ig_coarse** coarse) {
  if (!c) return fail("igh_levels: null case");
  if (levels) *levels = c->lv.data();
  if (n_levels) *n_levels = static_cast<int32_t>(c->lv.size());
  if (coarse) *coarse = &c->co;
  return IG_OK;
}

const double* igh_rhs(const igh_case* c, int32_t* n) {
  if (!c) return nullptr;
  if (n) *n = static_cast<int32_t>(c->b.size());
  return c->b.data();
}

int igh_get_info(const igh_case* c, igh_info* out) {
  if (!c || !out) return fail("igh_get_info: null argument");
  *out = c->info;
  return IG_OK;
}

int igh_anchors(const igh_case* c, int32_t level, int32_t* out_xyz) {
  if (!c || level < 0 || level >= static_cast<int32_t>(c->xyz.size())) return fail("igh_anchors: bad level");
  std::memcpy(out_xyz, c->xyz[level].data(), c->xyz[level].size() * sizeof(int32_t));
  return IG_OK;
}

void igh_destroy(igh_case* c) { delete c; }

int32_t igh_pstrf(int32_t n, double* a, int32_t* piv, double tol) { return pstrf_lower(n, a, piv, tol); }

int igh_eta(const igh_config* cfg, double* eta, int64_t* cut, int32_t* n_dofs) {
  try {
    const int threads = resolve_threads(cfg->threads);
    Grid g;
    g.dim = cfg->dim;
    for (int d = 0; d < 3; ++d) {
      g.origin[d] = cfg->origin[d];
      g.extent[d] = cfg->extent[d];
      g.res[d] = d < cfg->dim ? cfg->resolution[d] : 1;
    }
    const LevelSet ls = parse_levelset(cfg->geometry ? cfg->geometry : "constant(1)");
    if (cfg->family == 2) {  // THB: DOF count of the trimmed hierarchical space
      HMesh mesh = HMesh::uniform(g);
      for (int k = 0; k < cfg->n_refine_boxes; ++k) mesh.refine_by_box(cfg->refine_boxes + 4 * k);
      for (int k = 0; k < cfg->refine_passes; ++k)
        mesh.refine_near_circle(cfg->refine_circle[0], cfg->refine_circle[1], cfg->refine_circle[2], cfg->refine_dist);
      auto gs = build_thb(mesh, ls, cfg->degree, cfg->classify_depth, threads);
      int64_t nc = 0;
      for (const auto& e : gs->el) nc += e.tag == kCut;
      if (eta) *eta = -1.0;  // not computed for THB here
      if (cut) *cut = nc;
      if (n_dofs) *n_dofs = gs->n();
      return IG_OK;
    }
    auto s = build_space(g, ls, cfg->family == 0 ? Family::Lagrange : Family::Bspline, cfg->degree,
                         cfg->classify_depth, threads);
    QuadConfig qc;
    qc.depth = cfg->quad_depth;
    qc.gauss_order = cfg->gauss_order > 0 ? cfg->gauss_order : cfg->degree + 1;
    qc.classify_depth = cfg->classify_depth;
    qc.edge_tol = cfg->edge_tol;
    double e = 1.0;
    int64_t nc = 0;
    for (size_t k = 0; k < s->el_ix.size(); ++k) {
      if (s->el_tag[k] != kCut) continue;
      ++nc;
      double lo[3], hi[3];
      g.cell_box(s->el_ix[k], s->el_iy[k], s->el_iz[k], lo, hi);
      if (g.dim != 2) continue;
      const QuadRule2 vr = volume_rule2(ls, lo, hi, kCut, qc);
      double tw = 0.0;
      for (double w : vr.w) tw += w;
      e = std::min(e, tw / ((hi[0] - lo[0]) * (hi[1] - lo[1])));
    }
    if (eta) *eta = e;
    if (cut) *cut = nc;
    if (n_dofs) *n_dofs = s->n();
    return IG_OK;
  } catch (const std::exception& ex) {
    return fail(ex.what());
  }
}

}  // extern "C"

// ---- .igh file: little-endian binary, version 2 (v1 = no block colours) ----
namespace {
template <typename T>
void wr(std::ofstream& f, const T* p, size_t n) {
  f.write(reinterpret_cast<const char*>(p), static_cast<std::streamsize>(n * sizeof(T)));
}
template <typename T>
void wv(std::ofstream& f, const std::vector<T>& v) {
  const uint64_t n = v.size();
  wr(f, &n, 1);
  wr(f, v.data(), v.size());
}
template <typename T>
void rd(std::ifstream& f, T* p, size_t n) {
  f.read(reinterpret_cast<char*>(p), static_cast<std::streamsize>(n * sizeof(T)));
  if (!f) throw SetupError("igh_read: truncated file");
}
template <typename T>
void rv(std::ifstream& f, std::vector<T>& v) {
  uint64_t n = 0;
  rd(f, &n, 1);
  if (n > (1ull << 36)) throw SetupError("igh_read: corrupt length");
  v.resize(n);
  rd(f, v.data(), n);
}
void wcsr(std::ofstream& f, const Csr& m) {
  wr(f, &m.nr, 1);
  wr(f, &m.nc, 1);
  wv(f, m.ptr);
  wv(f, m.col);
  wv(f, m.val);
}
void rcsr(std::ifstream& f, Csr& m) {
  rd(f, &m.nr, 1);
  rd(f, &m.nc, 1);
  rv(f, m.ptr);
  rv(f, m.col);
  rv(f, m.val);
}
const char kMagic[8] = {'I', 'G', 'H', '1', 0, 0, 0, 2};  // last byte: version
}  // namespace

extern "C" {

int igh_write(const igh_case* c, const char* path) {
  if (!c || !path) return fail("igh_write: null argument");
  if (c->geometric) return fail("igh_write: a geometry-only case (igh_build_geometry) has no hierarchy to write");
  try {
    std::ofstream f(path, std::ios::binary);
    if (!f) return fail(std::string("igh_write: cannot open ") + path);
    wr(f, kMagic, 8);
    const int32_t L = static_cast<int32_t>(c->A.size());
    wr(f, &L, 1);
    wr(f, &c->info, 1);
    for (int l = 0; l < L; ++l) {
      wcsr(f, c->A[l]);
      wcsr(f, c->R[l]);
      wr(f, &c->kind[l], 1);
      wr(f, &c->gamma[l], 1);
      wv(f, c->B[l].owners);
      wv(f, c->B[l].ptr);
      wv(f, c->B[l].dofs);
      wv(f, c->B[l].fptr);
      wv(f, c->B[l].fac);
      wr(f, &c->B[l].max_nk, 1);
      wv(f, c->xyz[l]);
      wv(f, c->B[l].color);
      wr(f, &c->B[l].n_colors, 1);
    }
    wv(f, c->coarseL);
    wv(f, c->piv);
    wr(f, &c->rank, 1);
    wv(f, c->b);
    if (!f) return fail("igh_write: write failed");
    return IG_OK;
  } catch (const std::exception& e) {
    return fail(e.what());
  }
}

int igh_read(const char* path, igh_case** out) {
  try {
    std::ifstream f(path, std::ios::binary);
    if (!f) return fail(std::string("igh_read: cannot open ") + path);
    char mg[8];
    rd(f, mg, 8);
    if (std::memcmp(mg, kMagic, 7) != 0 || (mg[7] != 1 && mg[7] != 2)) return fail("igh_read: bad magic");
    const int version = mg[7];
    auto c = std::make_unique<igh_case>();
    int32_t L = 0;
    rd(f, &L, 1);
    if (L < 1 || L > 16) return fail("igh_read: bad level count");
    igh_info info;
    rd(f, &info, 1);
    c->A.resize(L);
    c->R.resize(L);
    c->B.resize(L);
    c->kind.resize(L);
    c->gamma.resize(L);
    c->xyz.resize(L);
    for (int l = 0; l < L; ++l) {
      rcsr(f, c->A[l]);
      rcsr(f, c->R[l]);
      rd(f, &c->kind[l], 1);
      rd(f, &c->gamma[l], 1);
      rv(f, c->B[l].owners);
      rv(f, c->B[l].ptr);
      rv(f, c->B[l].dofs);
      rv(f, c->B[l].fptr);
      rv(f, c->B[l].fac);
      rd(f, &c->B[l].max_nk, 1);
      rv(f, c->xyz[l]);
      if (version >= 2) {
        rv(f, c->B[l].color);
        rd(f, &c->B[l].n_colors, 1);
      }
    }
    rv(f, c->coarseL);
    rv(f, c->piv);
    rd(f, &c->rank, 1);
    rv(f, c->b);
    c->wire();
    c->info = info;
    *out = c.release();
    return IG_OK;
  } catch (const std::exception& e) {
    return fail(e.what());
  }
}

}  // extern "C"
