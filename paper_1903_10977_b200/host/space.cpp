// Trimmed uniform mesh + Lagrange / B-spline space, 2D and 3D.
// 2D restates proj/src/mesh.cpp:91-111 (trim) and proj/src/basis.cpp:91-316
// for unrefined meshes (M = 0); 3D is the same construction with a third
// tensor axis (no reference counterpart).
#include <algorithm>
#include <cmath>

#include "host.hpp"

namespace igh {

void Grid::cell_box(int ix, int iy, int iz, double* lo, double* hi) const {
  // EmbeddingGrid::cell_box (mesh.hpp:34-38): lo = origin + i*d, hi = lo + d.
  const int idx[3] = {ix, iy, iz};
  for (int d = 0; d < dim; ++d) {
    const double cs = extent[d] / res[d];
    lo[d] = origin[d] + idx[d] * cs;
    hi[d] = lo[d] + cs;
  }
}

void Space::element_anchors(int e, int32_t* out) const {
  const int q = p + 1;
  const int a0 = first_anchor(el_ix[e]);
  const int b0 = first_anchor(el_iy[e]);
  if (grid.dim == 2) {
    int r = 0;
    for (int jb = 0; jb < q; ++jb)
      for (int ia = 0; ia < q; ++ia) out[r++] = kept[untrimmed(a0 + ia, b0 + jb, 0)];
  } else {
    const int c0 = first_anchor(el_iz[e]);
    int r = 0;
    for (int kc = 0; kc < q; ++kc)
      for (int jb = 0; jb < q; ++jb)
        for (int ia = 0; ia < q; ++ia) out[r++] = kept[untrimmed(a0 + ia, b0 + jb, c0 + kc)];
  }
}

// Cells (per axis) whose local anchors include anchor index a.
void anchor_cells(Family fam, int a, int p, int cells, int& lo, int& hi) {
  if (fam == Family::Bspline) {  // fn_spans (basis.cpp:66-70)
    lo = std::max(a - p, 0);
    hi = std::min(a, cells - 1);
  } else {  // node_elems (basis.cpp:73-78)
    lo = std::max(0, (a - 1) / p);
    if (a == 0) lo = 0;
    hi = std::min(cells - 1, a / p);
  }
}

namespace {

// Deduplicate per-cell extraction matrices into classes (max |diff| <= 1e-13
// relative): interior spans of a uniform knot vector share one matrix.
void classify_extractions(const std::vector<Mat>& per_cell, std::vector<int32_t>& cls,
                          std::vector<Mat>& reps) {
  cls.assign(per_cell.size(), -1);
  reps.clear();
  for (size_t c = 0; c < per_cell.size(); ++c) {
    const Mat& m = per_cell[c];
    int found = -1;
    for (size_t k = 0; k < reps.size() && found < 0; ++k) {
      double diff = 0.0;
      for (size_t i = 0; i < m.a.size(); ++i) diff = std::max(diff, std::fabs(m.a[i] - reps[k].a[i]));
      if (diff <= 1e-13) found = static_cast<int>(k);
    }
    if (found < 0) {
      found = static_cast<int>(reps.size());
      reps.push_back(m);
    }
    cls[c] = found;
  }
}

}  // namespace

std::unique_ptr<Space> build_space(const Grid& g, const LevelSet& ls, Family fam, int p,
                                   int classify_depth, int threads) {
  if (p < 1 || p > 4) throw SetupError("build_space: degree must be in 1..4");
  if (g.dim != 2 && g.dim != 3) throw SetupError("build_space: dim must be 2 or 3");
  if (fam == Family::Lagrange && g.dim != 2) throw SetupError("build_space: Lagrange is 2D only");
  auto s = std::make_unique<Space>();
  Space& S = *s;
  S.grid = g;
  S.family = fam;
  S.p = p;
  S.ls = ls;
  S.classify_depth = classify_depth;
  const int dim = g.dim;
  for (int d = 0; d < 3; ++d) S.nf[d] = 1;
  for (int d = 0; d < dim; ++d) S.nf[d] = fam == Family::Bspline ? g.res[d] + p : p * g.res[d] + 1;

  // --- trim: classify every cell (mesh.cpp:91-111) -------------------------
  const int64_t ncell = g.num_cells();
  S.cell_tag.assign(static_cast<size_t>(ncell), kOutside);
  const int rx = g.res[0], ry = g.res[1], rz = dim == 3 ? g.res[2] : 1;
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads)
  for (int64_t c = 0; c < ncell; ++c) {
    int ix, iy, iz = 0;
    if (dim == 2) {
      ix = static_cast<int>(c / ry);
      iy = static_cast<int>(c % ry);
    } else {
      ix = static_cast<int>(c / (static_cast<int64_t>(ry) * rz));
      iy = static_cast<int>((c / rz) % ry);
      iz = static_cast<int>(c % rz);
    }
    double lo[3], hi[3];
    g.cell_box(ix, iy, iz, lo, hi);
    const CellClass cc = classify_cell(ls, lo, hi, dim, classify_depth);
    S.cell_tag[c] = cc == CellClass::Inside ? kInside : (cc == CellClass::Cut ? kCut : kOutside);
  }
  S.cell_to_el.assign(static_cast<size_t>(ncell), -1);
  for (int64_t c = 0; c < ncell; ++c) {
    if (S.cell_tag[c] == kOutside) continue;
    S.cell_to_el[c] = static_cast<int32_t>(S.el_ix.size());
    if (dim == 2) {
      S.el_ix.push_back(static_cast<int32_t>(c / ry));
      S.el_iy.push_back(static_cast<int32_t>(c % ry));
      S.el_iz.push_back(0);
    } else {
      S.el_ix.push_back(static_cast<int32_t>(c / (static_cast<int64_t>(ry) * rz)));
      S.el_iy.push_back(static_cast<int32_t>((c / rz) % ry));
      S.el_iz.push_back(static_cast<int32_t>(c % rz));
    }
    S.el_tag.push_back(S.cell_tag[c]);
  }
  if (S.el_ix.empty()) throw SetupError("trim: no element intersects the domain");

  // --- per-axis extraction (basis.cpp:185-198) -------------------------------
  for (int d = 0; d < dim; ++d) {
    std::vector<Mat> per_cell(static_cast<size_t>(g.res[d]));
    if (fam == Family::Lagrange) {
      const Mat lag = spline::lagrange_extraction(p);
      for (auto& m : per_cell) m = lag;
    } else {
      const auto t = spline::open_uniform_knots(g.origin[d], g.origin[d] + g.extent[d], g.res[d], p);
      for (int c = 0; c < g.res[d]; ++c) per_cell[c] = spline::span_extraction(t, p, c + p);
    }
    classify_extractions(per_cell, S.ext_cls[d], S.ext[d]);
  }

  // --- kept anchors: those on at least one active element (basis.cpp:293-309)
  const int64_t nall = static_cast<int64_t>(S.nf[0]) * S.nf[1] * S.nf[2];
  std::vector<uint8_t> on(static_cast<size_t>(nall), 0);
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t u = 0; u < nall; ++u) {
    const int ax = static_cast<int>(u % S.nf[0]);
    const int ay = static_cast<int>((u / S.nf[0]) % S.nf[1]);
    const int az = static_cast<int>(u / (static_cast<int64_t>(S.nf[0]) * S.nf[1]));
    int xl, xh, yl, yh, zl = 0, zh = 0;
    anchor_cells(fam, ax, p, rx, xl, xh);
    anchor_cells(fam, ay, p, ry, yl, yh);
    if (dim == 3) anchor_cells(fam, az, p, rz, zl, zh);
    bool any = false;
    for (int ex = xl; ex <= xh && !any; ++ex)
      for (int ey = yl; ey <= yh && !any; ++ey)
        for (int ez = zl; ez <= zh && !any; ++ez)
          if (S.cell_to_el[g.cell_linear(ex, ey, ez)] >= 0) any = true;
    on[u] = any;
  }
  S.kept.assign(static_cast<size_t>(nall), -1);
  for (int64_t u = 0; u < nall; ++u)
    if (on[u]) {
      S.kept[u] = static_cast<int32_t>(S.anchors.size());
      S.anchors.push_back(u);
    }

  // --- physical supports in element order (basis.cpp:312-313) -------------
  const int n = S.n();
  std::vector<int32_t> cnt(static_cast<size_t>(n), 0);
  auto for_support = [&](int a, auto&& fn) {
    const int64_t u = S.anchors[a];
    const int ax = static_cast<int>(u % S.nf[0]);
    const int ay = static_cast<int>((u / S.nf[0]) % S.nf[1]);
    const int az = static_cast<int>(u / (static_cast<int64_t>(S.nf[0]) * S.nf[1]));
    int xl, xh, yl, yh, zl = 0, zh = 0;
    anchor_cells(fam, ax, p, rx, xl, xh);
    anchor_cells(fam, ay, p, ry, yl, yh);
    if (dim == 3) anchor_cells(fam, az, p, rz, zl, zh);
    for (int ex = xl; ex <= xh; ++ex)  // (ix, iy, iz) lexicographic == element order
      for (int ey = yl; ey <= yh; ++ey)
        for (int ez = zl; ez <= zh; ++ez) {
          const int32_t e = S.cell_to_el[g.cell_linear(ex, ey, ez)];
          if (e >= 0) fn(e);
        }
  };
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int a = 0; a < n; ++a) {
    int c = 0;
    for_support(a, [&](int32_t) { ++c; });
    cnt[a] = c;
  }
  S.supp_ptr.assign(static_cast<size_t>(n) + 1, 0);
  for (int a = 0; a < n; ++a) S.supp_ptr[a + 1] = S.supp_ptr[a] + cnt[a];
  S.supp_el.resize(static_cast<size_t>(S.supp_ptr[n]));
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int a = 0; a < n; ++a) {
    int64_t o = S.supp_ptr[a];
    for_support(a, [&](int32_t e) { S.supp_el[o++] = e; });
  }
  return s;
}

}  // namespace igh
