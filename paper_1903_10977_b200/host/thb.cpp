// Truncated hierarchical B-splines (THB) on a trimmed hierarchical 2D mesh:
// the setup side of BASELINE.json configs[4] (C5).  Restates
//   HierarchicalMesh::refine / refine_by_box / coarsen  proj/src/mesh.cpp:35-89
//   trim on hierarchical meshes                          proj/src/mesh.cpp:91-111
//   build_space for Family::THB                          proj/src/basis.cpp:23-64, 91-316
//   evaluate_basis                                       proj/src/basis.cpp:318-341
//   restriction_matrix, THB branch                       proj/src/basis.cpp:433-581
//   assemble (Poisson, penalty)                          proj/src/assembly.cpp:36-183
// with per-element extraction rows (a THB element carries the truncated
// functions of several levels, so the tensor-class shortcuts of space.cpp do
// not apply).
#include <algorithm>
#include <cmath>
#include <map>
#include <set>

#include "host.hpp"
#include "thb.hpp"

namespace igh {

// ------------------------------------------------------------------ mesh ---

void HMesh::cell_box(int l, int ix, int iy, double* lo, double* hi) const {
  const double dx = g.extent[0] / cells_x(l), dy = g.extent[1] / cells_y(l);
  lo[0] = g.origin[0] + ix * dx;
  lo[1] = g.origin[1] + iy * dy;
  hi[0] = lo[0] + dx;
  hi[1] = lo[1] + dy;
}

bool HMesh::active(int l, int ix, int iy) const {
  if (l < 0 || l >= static_cast<int>(lv.size())) return false;
  return lv[l].count({ix, iy}) > 0;
}

HMesh HMesh::uniform(const Grid& g) {
  HMesh m;
  m.g = g;
  m.lv.resize(1);
  for (int i = 0; i < g.res[0]; ++i)
    for (int j = 0; j < g.res[1]; ++j) m.lv[0].insert({i, j});
  return m;
}

void HMesh::refine(const std::vector<std::array<int, 3>>& targets) {
  for (const auto& t : targets)
    if (!active(t[0], t[1], t[2])) throw SetupError("refine: target is not active");
  for (const auto& t : targets) {
    lv[t[0]].erase({t[1], t[2]});
    if (t[0] + 1 >= static_cast<int>(lv.size())) lv.resize(t[0] + 2);
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) lv[t[0] + 1].insert({2 * t[1] + a, 2 * t[2] + b});
  }
  while (lv.size() > 1 && lv.back().empty()) lv.pop_back();
}

std::vector<std::array<int, 3>> HMesh::elements() const {
  std::vector<std::array<int, 3>> out;
  for (int l = 0; l < static_cast<int>(lv.size()); ++l)
    for (const auto& [i, j] : lv[l]) out.push_back({l, i, j});
  return out;
}

void HMesh::refine_by_box(const double* box) {
  // Box::overlaps (common.hpp:30-32): strict interior overlap.
  std::vector<std::array<int, 3>> t;
  for (const auto& e : elements()) {
    double lo[2], hi[2];
    cell_box(e[0], e[1], e[2], lo, hi);
    if (lo[0] < box[2] && box[0] < hi[0] && lo[1] < box[3] && box[1] < hi[1]) t.push_back(e);
  }
  refine(t);
}

void HMesh::refine_near_circle(double cx, double cy, double r, double dist) {
  // max(0, d_min - R, R - d_max) <= dist, applied to the
  // elements of the current finest level (one pass per call).
  const int l = max_level();
  std::vector<std::array<int, 3>> t;
  for (const auto& [i, j] : lv[l]) {
    double lo[2], hi[2];
    cell_box(l, i, j, lo, hi);
    const double nx = std::max(lo[0], std::min(cx, hi[0])), ny = std::max(lo[1], std::min(cy, hi[1]));
    const double dmin = std::hypot(nx - cx, ny - cy);
    const double fx = std::max(std::fabs(lo[0] - cx), std::fabs(hi[0] - cx));
    const double fy = std::max(std::fabs(lo[1] - cy), std::fabs(hi[1] - cy));
    const double dmax = std::hypot(fx, fy);
    if (std::max(0.0, std::max(dmin - r, r - dmax)) <= dist) t.push_back({l, i, j});
  }
  refine(t);
}

HMesh coarsen(const HMesh& fine) {
  // Paper Algorithm 2 (mesh.cpp:58-89).
  if (fine.g.res[0] % 2 != 0 || fine.g.res[1] % 2 != 0) throw SetupError("coarsen: base resolution must be even");
  Grid cg = fine.g;
  cg.res[0] /= 2;
  cg.res[1] /= 2;
  HMesh coarse = HMesh::uniform(cg);
  const int fmax = fine.max_level();
  std::vector<std::set<std::pair<int, int>>> trigger(std::max(fmax, 1));
  for (int l = 1; l <= fmax; ++l)
    for (const auto& [a, b] : fine.lv[l])
      for (int m = 0; m < l && m < static_cast<int>(trigger.size()); ++m) {
        const int shift = l - m + 1;
        trigger[m].insert({a >> shift, b >> shift});
      }
  for (int m = 0; m < static_cast<int>(trigger.size()); ++m) {
    std::vector<std::array<int, 3>> t;
    for (const auto& [i, j] : trigger[m])
      if (coarse.active(m, i, j)) t.push_back({m, i, j});
    coarse.refine(t);
  }
  return coarse;
}

// ----------------------------------------------------------------- space ---

namespace {

enum class CellState : uint8_t { Active, FineCovered, CoarseCovered };

void fn_spans(int a, int p, int cells, int& lo, int& hi) {
  lo = std::max(a - p, 0);
  hi = std::min(a, cells - 1);
}

Mat block(const Mat& M, int r0, int c0, int nr, int nc) {
  Mat B(nr, nc);
  for (int j = 0; j < nc; ++j)
    for (int i = 0; i < nr; ++i) B(i, j) = M(r0 + i, c0 + j);
  return B;
}

}  // namespace

int GSpace::element_index(int l, int ix, int iy) const {
  auto it = el_index.find(std::array<int, 3>{l, ix, iy});
  return it == el_index.end() ? -1 : it->second;
}

std::unique_ptr<GSpace> build_thb(const HMesh& mesh, const LevelSet& ls, int p, int classify_depth, int threads) {
  if (p < 1 || p > 4) throw SetupError("build_space: degree must be in 1..4");
  auto sp = std::make_unique<GSpace>();
  GSpace& S = *sp;
  S.mesh = mesh;
  S.ls = ls;
  S.p = p;
  S.classify_depth = classify_depth;
  const int M = mesh.max_level();

  // --- trim (mesh.cpp:91-111): classify every active element -------------
  const auto all = mesh.elements();
  std::vector<uint8_t> tag(all.size(), kOutside);
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads)
  for (int64_t k = 0; k < static_cast<int64_t>(all.size()); ++k) {
    double lo[2], hi[2];
    mesh.cell_box(all[k][0], all[k][1], all[k][2], lo, hi);
    const CellClass cc = classify_cell(ls, lo, hi, 2, classify_depth);
    tag[k] = cc == CellClass::Inside ? kInside : (cc == CellClass::Cut ? kCut : kOutside);
  }
  std::map<std::array<int, 3>, uint8_t> tags;
  for (size_t k = 0; k < all.size(); ++k) tags[all[k]] = tag[k];
  if (std::none_of(tag.begin(), tag.end(), [](uint8_t t) { return t != kOutside; }))
    throw SetupError("trim: no element intersects the domain");

  // --- per-level function grids ------------------------------------------
  S.fn_nx.resize(M + 1);
  S.fn_ny.resize(M + 1);
  S.knx.resize(M + 1);
  S.kny.resize(M + 1);
  for (int l = 0; l <= M; ++l) {
    const int cx = mesh.cells_x(l), cy = mesh.cells_y(l);
    S.fn_nx[l] = cx + p;
    S.fn_ny[l] = cy + p;
    S.knx[l] = spline::open_uniform_knots(mesh.g.origin[0], mesh.g.origin[0] + mesh.g.extent[0], cx, p);
    S.kny[l] = spline::open_uniform_knots(mesh.g.origin[1], mesh.g.origin[1] + mesh.g.extent[1], cy, p);
  }
  // cell_states (basis.cpp:23-50)
  std::vector<std::vector<CellState>> st(M + 1);
  for (int l = 0; l <= M; ++l) {
    const int cx = mesh.cells_x(l), cy = mesh.cells_y(l);
    st[l].assign(static_cast<size_t>(cx) * cy, CellState::FineCovered);
    for (int iy = 0; iy < cy; ++iy)
      for (int ix = 0; ix < cx; ++ix) {
        CellState s = CellState::FineCovered;
        if (mesh.active(l, ix, iy)) {
          s = CellState::Active;
        } else {
          for (int k = 1; k <= l; ++k)
            if (mesh.active(l - k, ix >> k, iy >> k)) {
              s = CellState::CoarseCovered;
              break;
            }
        }
        st[l][static_cast<size_t>(iy) * cx + ix] = s;
      }
  }
  // active functions and untrimmed ordinals (basis.cpp:141-162)
  S.active_fn.resize(M + 1);
  S.ordinal.resize(M + 1);
  for (int l = 0; l <= M; ++l) {
    const int cx = mesh.cells_x(l), cy = mesh.cells_y(l);
    const int nfx = S.fn_nx[l], nfy = S.fn_ny[l];
    S.active_fn[l].assign(static_cast<size_t>(nfx) * nfy, 0);
    S.ordinal[l].assign(static_cast<size_t>(nfx) * nfy, -1);
    for (int ay = 0; ay < nfy; ++ay)
      for (int ax = 0; ax < nfx; ++ax) {
        int xlo, xhi, ylo, yhi;
        fn_spans(ax, p, cx, xlo, xhi);
        fn_spans(ay, p, cy, ylo, yhi);
        bool any_active = false, any_coarse = false;
        for (int sy = ylo; sy <= yhi && !any_coarse; ++sy)
          for (int sx = xlo; sx <= xhi; ++sx) {
            const CellState cs = st[l][static_cast<size_t>(sy) * cx + sx];
            if (cs == CellState::Active) any_active = true;
            if (cs == CellState::CoarseCovered) {
              any_coarse = true;
              break;
            }
          }
        if (any_active && !any_coarse) {
          S.active_fn[l][static_cast<size_t>(ay) * nfx + ax] = 1;
          S.ordinal[l][static_cast<size_t>(ay) * nfx + ax] = static_cast<int>(S.all_anchors.size());
          S.all_anchors.push_back({l, ax, ay});
        }
      }
  }
  // per-level per-cell span extraction
  std::vector<std::vector<Mat>> Ex(M + 1), Ey(M + 1);
  for (int l = 0; l <= M; ++l) {
    const int cx = mesh.cells_x(l), cy = mesh.cells_y(l);
    Ex[l].resize(cx);
    Ey[l].resize(cy);
    for (int c = 0; c < cx; ++c) Ex[l][c] = spline::span_extraction(S.knx[l], p, c + p);
    for (int c = 0; c < cy; ++c) Ey[l][c] = spline::span_extraction(S.kny[l], p, c + p);
  }
  // two-scale matrices and their nonzero column ranges
  std::vector<Mat> Tx(M), Ty(M);
  std::vector<std::vector<std::pair<int, int>>> crx(M), cry(M);
  auto col_ranges = [](const Mat& T) {
    std::vector<std::pair<int, int>> r(T.r);
    for (int i = 0; i < T.r; ++i) {
      int lo = -1, hi = -1;
      for (int j = 0; j < T.c; ++j)
        if (T(i, j) != 0.0) {
          if (lo < 0) lo = j;
          hi = j;
        }
      r[i] = {lo, hi};
    }
    return r;
  };
  for (int m = 0; m < M; ++m) {
    Tx[m] = spline::dyadic_refine_matrix(mesh.cells_x(m), p);
    Ty[m] = spline::dyadic_refine_matrix(mesh.cells_y(m), p);
    crx[m] = col_ranges(Tx[m]);
    cry[m] = col_ranges(Ty[m]);
  }

  // --- truncated chains and element extraction rows (basis.cpp:217-280) ---
  const int q = p + 1, nb = q * q;
  std::map<std::array<int, 3>, std::pair<std::vector<int>, std::vector<double>>> eb;  // anchors, rows (nb each)
  S.chains.resize(S.all_anchors.size());
  for (int f = 0; f < static_cast<int>(S.all_anchors.size()); ++f) {
    const auto a = S.all_anchors[f];
    int i0 = a[1], i1 = a[1], j0 = a[2], j1 = a[2];
    Mat C(1, 1);
    C(0, 0) = 1.0;
    for (int m = a[0]; m <= M; ++m) {
      const int cx = mesh.cells_x(m), cy = mesh.cells_y(m);
      for (int sx = std::max(i0 - p, 0); sx <= std::min(i1, cx - 1); ++sx)
        for (int sy = std::max(j0 - p, 0); sy <= std::min(j1, cy - 1); ++sy) {
          auto it = tags.find({m, sx, sy});
          if (it == tags.end() || it->second == kOutside) continue;
          Mat Cl(q, q);
          bool any = false;
          for (int ia = 0; ia <= p; ++ia)
            for (int jb = 0; jb <= p; ++jb) {
              const int gx = sx + ia, gy = sy + jb;
              if (gx < i0 || gx > i1 || gy < j0 || gy > j1) continue;
              const double c = C(gx - i0, gy - j0);
              if (c != 0.0) {
                Cl(ia, jb) = c;
                any = true;
              }
            }
          if (!any) continue;
          const Mat coeffs = matmul(matmul(transpose(Ex[m][sx]), Cl), Ey[m][sy]);  // (jx, jy)
          auto& entry = eb[{m, sx, sy}];
          entry.first.push_back(f);
          for (int jy = 0; jy <= p; ++jy)
            for (int jx = 0; jx <= p; ++jx) entry.second.push_back(coeffs(jx, jy));  // x fastest
        }
      if (m == M) {
        S.chains[f] = {i0, j0, C};
        break;
      }
      const int fi0 = crx[m][i0].first, fi1 = crx[m][i1].second;
      const int fj0 = cry[m][j0].first, fj1 = cry[m][j1].second;
      C = matmul(matmul(transpose(block(Tx[m], i0, fi0, i1 - i0 + 1, fi1 - fi0 + 1)), C),
                 block(Ty[m], j0, fj0, j1 - j0 + 1, fj1 - fj0 + 1));
      const int nfx = S.fn_nx[m + 1];
      for (int af = 0; af < C.r; ++af)
        for (int bf = 0; bf < C.c; ++bf)
          if (S.active_fn[m + 1][static_cast<size_t>(fj0 + bf) * nfx + (fi0 + af)]) C(af, bf) = 0.0;
      i0 = fi0;
      i1 = fi1;
      j0 = fj0;
      j1 = fj1;
    }
  }
  (void)nb;

  // --- trimming: keep anchors with at least one row (basis.cpp:293-309) ---
  const int nall = static_cast<int>(S.all_anchors.size());
  S.kept.assign(nall, -1);
  for (const auto& [e, rows] : eb)
    for (int aa : rows.first) S.kept[aa] = 0;
  int next = 0;
  for (int aa = 0; aa < nall; ++aa)
    if (S.kept[aa] == 0) {
      S.kept[aa] = next++;
      S.anchors.push_back(S.all_anchors[aa]);
    }
  S.supp.assign(next, {});
  for (const auto& [e, rows] : eb) {
    GSpace::El el;
    el.l = e[0];
    el.ix = e[1];
    el.iy = e[2];
    el.tag = tags[e];
    for (int aa : rows.first) el.anchors.push_back(S.kept[aa]);
    el.E = rows.second;
    const int idx = static_cast<int>(S.el.size());
    S.el_index[e] = idx;
    for (int a : el.anchors) S.supp[a].push_back(idx);
    S.el.push_back(std::move(el));
  }
  // Inside/Cut elements with no rows (possible only for fully truncated
  // coverage) still count for trimming order; they carry no DOFs.
  return sp;
}

// ------------------------------------------------------------- assembly ---

namespace {

void eval_el(const GSpace& s, const GSpace::El& e, double u, double v, double hx, double hy, double* val,
             double* gx, double* gy) {
  const int p = s.p, q = p + 1, nb = q * q;
  double bu[8], du[8], bv[8], dv[8];
  spline::bernstein(p, u, bu, du);
  spline::bernstein(p, v, bv, dv);
  double bval[64], bgx[64], bgy[64];
  for (int jy = 0; jy < q; ++jy)
    for (int jx = 0; jx < q; ++jx) {
      const int k = jy * q + jx;
      bval[k] = bu[jx] * bv[jy];
      bgx[k] = du[jx] * bv[jy];
      bgy[k] = bu[jx] * dv[jy];
    }
  const int nr = static_cast<int>(e.anchors.size());
  for (int r = 0; r < nr; ++r) {
    double a = 0.0, b = 0.0, c = 0.0;
    const double* row = e.E.data() + static_cast<size_t>(r) * nb;
    for (int k = 0; k < nb; ++k) {
      a += row[k] * bval[k];
      b += row[k] * bgx[k];
      c += row[k] * bgy[k];
    }
    val[r] = a;
    gx[r] = b / hx;
    gy[r] = c / hy;
  }
}

}  // namespace

Assembled assemble_g(const GSpace& s, const ProblemConfig& prob, const QuadConfig& qc, int threads) {
  const HMesh& mesh = s.mesh;
  const int M = mesh.max_level();
  const double hmin = std::min(mesh.g.extent[0] / mesh.cells_x(M), mesh.g.extent[1] / mesh.cells_y(M));
  const double beta = prob.beta > 0.0 ? prob.beta : 2.0 / hmin;  // default_penalty at the finest level
  const int ne = static_cast<int>(s.el.size());
  std::vector<std::vector<double>> K(ne), F(ne);
  double eta = 1.0;
  int64_t ncut = 0;
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads) reduction(min : eta) reduction(+ : ncut)
  for (int e = 0; e < ne; ++e) {
    const GSpace::El& el = s.el[e];
    const int nl = static_cast<int>(el.anchors.size());
    K[e].assign(static_cast<size_t>(nl) * nl, 0.0);
    F[e].assign(nl, 0.0);
    double lo[2], hi[2];
    mesh.cell_box(el.l, el.ix, el.iy, lo, hi);
    const double sx = hi[0] - lo[0], sy = hi[1] - lo[1];
    std::vector<double> val(nl), gx(nl), gy(nl);
    auto at = [&](double x, double y) { eval_el(s, el, (x - lo[0]) / sx, (y - lo[1]) / sy, sx, sy, val.data(), gx.data(), gy.data()); };
    const bool cut = el.tag == kCut;
    const QuadRule2 vr = volume_rule2(s.ls, lo, hi, cut ? kCut : kInside, qc);
    double vol = 0.0;
    for (size_t k = 0; k < vr.size(); ++k) {
      const double w = vr.w[k];
      vol += w;
      at(vr.px[k], vr.py[k]);
      for (int i = 0; i < nl; ++i)
        for (int j = 0; j < nl; ++j) K[e][i * nl + j] += w * (gx[i] * gx[j] + gy[i] * gy[j]);
      if (prob.body_force != 0.0)
        for (int i = 0; i < nl; ++i) F[e][i] += w * prob.body_force * val[i];
    }
    if (cut) {
      ++ncut;
      eta = std::min(eta, vol / (sx * sy));
      const QuadRule2 br = boundary_rule2(s.ls, lo, hi, qc);
      for (size_t k = 0; k < br.size(); ++k) {
        at(br.px[k], br.py[k]);
        const double wb = br.w[k] * beta;
        for (int i = 0; i < nl; ++i)
          for (int j = 0; j < nl; ++j) K[e][i * nl + j] += wb * (val[i] * val[j]);
      }
    }
    if (prob.dirichlet_box_sides) {
      const int cx = mesh.cells_x(el.l), cy = mesh.cells_y(el.l);
      int sd[4], ns = 0;
      if (el.iy == 0) sd[ns++] = 0;
      if (el.ix == cx - 1) sd[ns++] = 1;
      if (el.iy == cy - 1) sd[ns++] = 2;
      if (el.ix == 0) sd[ns++] = 3;
      for (int t = 0; t < ns; ++t) {
        const QuadRule2 sr = side_rule2(s.ls, lo, hi, sd[t], qc);
        for (size_t k = 0; k < sr.size(); ++k) {
          at(sr.px[k], sr.py[k]);
          const double wb = sr.w[k] * beta;
          for (int i = 0; i < nl; ++i)
            for (int j = 0; j < nl; ++j) K[e][i * nl + j] += wb * (val[i] * val[j]);
        }
      }
    }
  }
  // Row gather in element order (setFromTriplets order), exact zeros dropped.
  Assembled out;
  out.eta = eta;
  out.cut_elements = ncut;
  const int n = s.n();
  out.b.assign(n, 0.0);
  std::vector<std::vector<std::pair<int32_t, double>>> rows(n);
#pragma omp parallel for schedule(dynamic, 256) num_threads(threads)
  for (int a = 0; a < n; ++a) {
    auto& row = rows[a];
    double bsum = 0.0;
    for (int e : s.supp[a]) {
      const GSpace::El& el = s.el[e];
      const int nl = static_cast<int>(el.anchors.size());
      const int li = static_cast<int>(std::find(el.anchors.begin(), el.anchors.end(), a) - el.anchors.begin());
      bsum += F[e][li];
      for (int lj = 0; lj < nl; ++lj) {
        const double v = K[e][li * nl + lj];
        if (v == 0.0) continue;
        const int32_t c = el.anchors[lj];
        auto it = std::find_if(row.begin(), row.end(), [c](const auto& pr) { return pr.first == c; });
        if (it == row.end())
          row.push_back({c, v});
        else
          it->second = it->second + v;
      }
    }
    out.b[a] = bsum;
    std::sort(row.begin(), row.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
  }
  Csr& A = out.A;
  A.nr = A.nc = n;
  A.ptr.assign(static_cast<size_t>(n) + 1, 0);
  for (int a = 0; a < n; ++a) A.ptr[a + 1] = A.ptr[a] + static_cast<int32_t>(rows[a].size());
  A.col.resize(A.ptr[n]);
  A.val.resize(A.ptr[n]);
  for (int a = 0; a < n; ++a)
    for (size_t k = 0; k < rows[a].size(); ++k) {
      A.col[A.ptr[a] + k] = rows[a][k].first;
      A.val[A.ptr[a] + k] = rows[a][k].second;
    }
  std::vector<double> sym(A.val.size());
  for (int i = 0; i < n; ++i)
    for (int32_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      const int32_t j = A.col[k];
      const int32_t* b = A.col.data() + A.ptr[j];
      const int32_t* e = A.col.data() + A.ptr[j + 1];
      const int32_t* it = std::lower_bound(b, e, i);
      if (it == e || *it != i) throw SetupError("assemble: unsymmetric pattern");
      sym[k] = 0.5 * (A.val[k] + A.val[it - A.col.data()]);
    }
  A.val.swap(sym);
  return out;
}

// ------------------------------------------------------------ blocks -------

Blocks select_blocks_g(const GSpace& s) {
  // smoothers.cpp:20-67: candidates = anchors on the owner's support
  // elements, members = candidates whose support is a subset (std::includes
  // on element ids, ascending == element index order).
  const int n = s.n();
  Blocks B;
  std::vector<uint8_t> covered(n, 0);
  for (int j = 0; j < n; ++j) {
    const auto& supj = s.supp[j];
    std::set<int> cands;
    for (int e : supj)
      for (int k : s.el[e].anchors) cands.insert(k);
    B.owners.push_back(j);
    for (int k : cands)
      if (std::includes(supj.begin(), supj.end(), s.supp[k].begin(), s.supp[k].end())) {
        B.dofs.push_back(k);
        covered[k] = 1;
      }
    B.ptr.push_back(static_cast<int32_t>(B.dofs.size()));
  }
  for (int d = 0; d < n; ++d)
    if (!covered[d]) throw SetupError("select_blocks: uncovered THB DOF");  // cannot happen: owner in own block
  return B;
}

int max_blocks_per_element_g(const Blocks& b, const GSpace& s) {
  const int ne = static_cast<int>(s.el.size());
  std::vector<int32_t> cnt(ne, 0), mark(ne, -1);
  for (int k = 0; k < static_cast<int>(b.owners.size()); ++k)
    for (int32_t q = b.ptr[k]; q < b.ptr[k + 1]; ++q)
      for (int e : s.supp[b.dofs[q]])
        if (mark[e] != k) {
          mark[e] = k;
          ++cnt[e];
        }
  int mx = 0;
  for (int e = 0; e < ne; ++e) mx = std::max(mx, cnt[e]);
  return mx;
}

// --------------------------------------------------------- restriction -----

namespace {

// Least squares A x = b (m >= n) by Householder QR with column pivoting
// (Eigen colPivHouseholderQr semantics up to rounding).
std::vector<double> qr_solve(Mat A, std::vector<double> b) {
  const int m = A.r, n = A.c;
  std::vector<int> perm(n);
  for (int j = 0; j < n; ++j) perm[j] = j;
  const int kmax = std::min(m, n);
  std::vector<double> diag(kmax, 0.0);
  int rank = kmax;
  double maxnorm = 0.0;
  for (int k = 0; k < kmax; ++k) {
    int piv = k;
    double best = -1.0;
    for (int j = k; j < n; ++j) {
      double s = 0.0;
      for (int i = k; i < m; ++i) s += A(i, j) * A(i, j);
      if (s > best) {
        best = s;
        piv = j;
      }
    }
    if (k == 0) maxnorm = std::sqrt(best);
    if (std::sqrt(best) <= 1e-13 * maxnorm) {
      rank = k;
      break;
    }
    if (piv != k) {
      for (int i = 0; i < m; ++i) std::swap(A(i, k), A(i, piv));
      std::swap(perm[k], perm[piv]);
    }
    double norm = 0.0;
    for (int i = k; i < m; ++i) norm += A(i, k) * A(i, k);
    norm = std::sqrt(norm);
    const double alpha = A(k, k) > 0 ? -norm : norm;
    std::vector<double> v(m, 0.0);
    for (int i = k; i < m; ++i) v[i] = A(i, k);
    v[k] -= alpha;
    double vn = 0.0;
    for (int i = k; i < m; ++i) vn += v[i] * v[i];
    if (vn > 0.0) {
      for (int j = k; j < n; ++j) {
        double d = 0.0;
        for (int i = k; i < m; ++i) d += v[i] * A(i, j);
        d = 2.0 * d / vn;
        for (int i = k; i < m; ++i) A(i, j) -= d * v[i];
      }
      double d = 0.0;
      for (int i = k; i < m; ++i) d += v[i] * b[i];
      d = 2.0 * d / vn;
      for (int i = k; i < m; ++i) b[i] -= d * v[i];
    }
    diag[k] = A(k, k);
  }
  std::vector<double> z(n, 0.0);
  for (int k = rank - 1; k >= 0; --k) {
    double s = b[k];
    for (int j = k + 1; j < rank; ++j) s -= A(k, j) * z[j];
    z[k] = s / A(k, k);
  }
  std::vector<double> x(n, 0.0);
  for (int j = 0; j < n; ++j) x[perm[j]] = z[j];
  return x;
}

}  // namespace

Csr restriction_thb(const GSpace& fine, const GSpace& coarse, int threads) {
  const int p = fine.p;
  const HMesh& fmesh = fine.mesh;
  const int Mf = fmesh.max_level();
  const int ffx = fine.fn_nx[Mf], ffy = fine.fn_ny[Mf];
  const auto& fknx = fine.knx[Mf];
  const auto& fkny = fine.kny[Mf];
  std::map<int, Mat> tcache;
  auto twoscale = [&](int cells) -> const Mat& {
    auto it = tcache.find(cells);
    if (it == tcache.end()) it = tcache.emplace(cells, spline::dyadic_refine_matrix(cells, p)).first;
    return it->second;
  };
  std::vector<double> cheb(p + 1);
  for (int k = 0; k <= p; ++k) cheb[k] = 0.5 - 0.5 * std::cos(M_PI * (2.0 * k + 1.0) / (2.0 * (p + 1)));

  Csr R;
  R.nr = coarse.n();
  R.nc = fine.n();
  R.ptr.assign(static_cast<size_t>(R.nr) + 1, 0);
  std::vector<std::vector<std::pair<int32_t, double>>> rows(R.nr);
  const int cMax = coarse.mesh.max_level();
  // Two-scale matrices needed by the promotion loop, built before the
  // parallel region (read-only inside).
  for (int cx = coarse.mesh.cells_x(cMax), cy = coarse.mesh.cells_y(cMax); cx < fmesh.cells_x(Mf); cx *= 2, cy *= 2) {
    twoscale(cx);
    twoscale(cy);
  }
  int err = 0;
#pragma omp parallel num_threads(threads)
  {
  std::vector<double> r(static_cast<size_t>(ffx) * ffy);
#pragma omp for schedule(dynamic, 16)
  for (int ca = 0; ca < coarse.n(); ++ca) {
    const auto A = coarse.anchors[ca];
    const int cord = coarse.ordinal[A[0]][static_cast<size_t>(A[2]) * coarse.fn_nx[A[0]] + A[1]];
    const GSpace::Chain& ch = coarse.chains[cord];
    int i0 = ch.fi0, j0 = ch.fj0;
    Mat C = ch.C;
    int cellsx = coarse.mesh.cells_x(cMax), cellsy = coarse.mesh.cells_y(cMax);
    while (cellsx < fmesh.cells_x(Mf)) {
      const Mat& Tx = twoscale(cellsx);
      const Mat& Ty = twoscale(cellsy);
      int fi0 = -1, fi1 = -1, fj0 = -1, fj1 = -1;
      for (int i = 0; i < C.r; ++i)
        for (int j = 0; j < Tx.c; ++j)
          if (Tx(i0 + i, j) != 0.0) {
            if (fi0 < 0 || j < fi0) fi0 = j;
            fi1 = std::max(fi1, j);
          }
      for (int i = 0; i < C.c; ++i)
        for (int j = 0; j < Ty.c; ++j)
          if (Ty(j0 + i, j) != 0.0) {
            if (fj0 < 0 || j < fj0) fj0 = j;
            fj1 = std::max(fj1, j);
          }
      C = matmul(matmul(transpose(block(Tx, i0, fi0, C.r, fi1 - fi0 + 1)), C), block(Ty, j0, fj0, C.c, fj1 - fj0 + 1));
      i0 = fi0;
      j0 = fj0;
      cellsx *= 2;
      cellsy *= 2;
    }
    std::fill(r.begin(), r.end(), 0.0);
    double rmax0 = 0.0;
    for (int a = 0; a < C.r; ++a)
      for (int b = 0; b < C.c; ++b) {
        r[static_cast<size_t>(j0 + b) * ffx + (i0 + a)] = C(a, b);
        rmax0 = std::max(rmax0, std::fabs(C(a, b)));
      }
    int rx0 = std::max(i0 - p, 0), rx1 = std::min(i0 + C.r - 1, fmesh.cells_x(Mf) - 1);
    int ry0 = std::max(j0 - p, 0), ry1 = std::min(j0 + C.c - 1, fmesh.cells_y(Mf) - 1);
    std::map<int, double> assigned;
    for (int l = 0; l <= Mf; ++l) {
      const int shift = Mf - l;
      const int nfx = fine.fn_nx[l];
      const auto& knx = fine.knx[l];
      const auto& kny = fine.kny[l];
      std::vector<int> lvl_assigned;
      // Active level-l cells overlapping the residual rectangle, visited in
      // the reference's std::set order (ix, then iy) -- only the rectangle
      // is scanned instead of every cell of the level.
      const int ixa = rx0 >> shift, ixb = rx1 >> shift, iya = ry0 >> shift, iyb = ry1 >> shift;
      for (int ix = ixa; ix <= ixb; ++ix)
        for (int iy = iya; iy <= iyb; ++iy) {
        if (!fmesh.active(l, ix, iy)) continue;
        if ((ix << shift) > rx1 || ((ix + 1) << shift) - 1 < rx0) continue;
        if ((iy << shift) > ry1 || ((iy + 1) << shift) - 1 < ry0) continue;
        std::vector<int> unk;
        for (int b = iy; b <= iy + p; ++b)
          for (int a = ix; a <= ix + p; ++a)
            if (fine.active_fn[l][static_cast<size_t>(b) * nfx + a]) unk.push_back(a + b * nfx);
        if (unk.empty()) continue;
        double lo[2], hi[2];
        fmesh.cell_box(l, ix, iy, lo, hi);
        const int npts = (p + 1) * (p + 1);
        Mat Am(npts, static_cast<int>(unk.size()));
        std::vector<double> rhs(npts);
        double vx[8], dxv[8], vy[8], dyv[8];
        for (int ky = 0, row = 0; ky <= p; ++ky)
          for (int kx = 0; kx <= p; ++kx, ++row) {
            const double ptx = lo[0] + cheb[kx] * (hi[0] - lo[0]), pty = lo[1] + cheb[ky] * (hi[1] - lo[1]);
            spline::eval_nonzero(knx, p, ptx, ix + p, vx, dxv);
            spline::eval_nonzero(kny, p, pty, iy + p, vy, dyv);
            for (int u = 0; u < static_cast<int>(unk.size()); ++u) {
              const int a = unk[u] % nfx, b = unk[u] / nfx;
              Am(row, u) = vx[a - ix] * vy[b - iy];
            }
            const int sxf = spline::find_span(fknx, p, ptx);
            const int syf = spline::find_span(fkny, p, pty);
            spline::eval_nonzero(fknx, p, ptx, sxf, vx, dxv);
            spline::eval_nonzero(fkny, p, pty, syf, vy, dyv);
            double val = 0.0;
            for (int jb = 0; jb <= p; ++jb)
              for (int ia = 0; ia <= p; ++ia)
                val += r[static_cast<size_t>(syf - p + jb) * ffx + (sxf - p + ia)] * vx[ia] * vy[jb];
            rhs[row] = val;
          }
        const std::vector<double> x = qr_solve(Am, rhs);
        for (int u = 0; u < static_cast<int>(unk.size()); ++u) {
          const int a = unk[u] % nfx, b = unk[u] / nfx;
          const int ford = fine.ordinal[l][static_cast<size_t>(b) * nfx + a];
          if (!assigned.count(ford)) {
            assigned.emplace(ford, x[u]);
            lvl_assigned.push_back(ford);
          }
        }
      }
      for (int ford : lvl_assigned) {
        const double xv = assigned[ford];
        if (xv == 0.0) continue;
        const GSpace::Chain& fc = fine.chains[ford];
        for (int a = 0; a < fc.C.r; ++a)
          for (int b = 0; b < fc.C.c; ++b) r[static_cast<size_t>(fc.fj0 + b) * ffx + (fc.fi0 + a)] -= xv * fc.C(a, b);
        rx0 = std::min(rx0, std::max(fc.fi0 - p, 0));
        rx1 = std::max(rx1, std::min(fc.fi0 + fc.C.r - 1, fmesh.cells_x(Mf) - 1));
        ry0 = std::min(ry0, std::max(fc.fj0 - p, 0));
        ry1 = std::max(ry1, std::min(fc.fj0 + fc.C.c - 1, fmesh.cells_y(Mf) - 1));
      }
    }
    double rmax = 0.0;
    for (double v : r) rmax = std::max(rmax, std::fabs(v));
    if (rmax > 1e-8 * std::max(rmax0, 1e-300)) {
#pragma omp atomic write
      err = 1;
      continue;
    }
    for (const auto& [ford, xv] : assigned) {
      if (xv == 0.0) continue;
      const int fk = fine.kept[ford];
      if (fk >= 0 && std::fabs(xv) > 1e-14) rows[ca].push_back({fk, xv});
    }
    std::sort(rows[ca].begin(), rows[ca].end(), [](const auto& x, const auto& y) { return x.first < y.first; });
  }
  }
  if (err) throw SetupError("restriction_matrix: coarse function not representable (hierarchy not nested)");
  for (int ca = 0; ca < R.nr; ++ca) R.ptr[ca + 1] = R.ptr[ca] + static_cast<int32_t>(rows[ca].size());
  R.col.resize(R.ptr.back());
  R.val.resize(R.ptr.back());
  for (int ca = 0; ca < R.nr; ++ca)
    for (size_t k = 0; k < rows[ca].size(); ++k) {
      R.col[R.ptr[ca] + k] = rows[ca][k].first;
      R.val[R.ptr[ca] + k] = rows[ca][k].second;
    }
  return R;
}

}  // namespace igh
