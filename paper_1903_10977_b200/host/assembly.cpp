// Poisson assembly with penalty Dirichlet: restates proj/src/assembly.cpp
// (default_penalty :7-10, assemble :36-183, scatter + setFromTriplets +
// symmetrisation :164-180) for the Poisson / scalar case.
//
// Element matrices:
//   * 2D cut elements and elements on the embedding-box boundary: the
//     reference's point quadrature (quad2d.cpp) evaluated exactly as
//     assembly.cpp:66-160 does;
//   * Inside elements without box-side terms: computed once per extraction
//     class in reference coordinates (identical mathematics; avoids 10^6
//     repeated quadratures);
//   * 3D cut elements (no reference): octree bisection to `depth`, Kuhn
//     6-tetrahedra per cut leaf clipped against psi >= 0 (edge roots by the
//     reference's bisection intersect_edge), polynomial moments of the cut
//     volume and interface, contracted with the tensor extraction.
// Global assembly gathers, for every row, the element contributions in
// ascending element order -- the order in which Eigen's setFromTriplets sums
// the reference's duplicate triplets -- dropping exact zeros (assembly.cpp:171).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>

#include "host.hpp"

namespace igh {

namespace {

constexpr int kMaxP = 4;
constexpr int kMaxQ = kMaxP + 1;
constexpr int kMaxM = 2 * kMaxP + 1;  // moment index range per axis

double default_penalty(const Grid& g) {
  double hmin = g.h(0);
  for (int d = 1; d < g.dim; ++d) hmin = std::min(hmin, g.h(d));
  return 2.0 / hmin;
}

struct ElemData {
  std::vector<double> K;  // nloc x nloc, row-major
  std::vector<double> F;  // nloc
  double volume = 0.0;    // physical measure of K ∩ domain (cut elements)
};

// ------------------------------------------------------------------ 2D ----

// Full nloc x nloc extraction for classes (cx, cy) (basis.cpp:204-214).
Mat extraction2(const Space& s, int cx, int cy) {
  const int q = s.p + 1, nl = q * q;
  const Mat& Rx = s.ext[0][cx];
  const Mat& Ry = s.ext[1][cy];
  Mat E(nl, nl);
  int r = 0;
  for (int jb = 0; jb < q; ++jb)
    for (int ia = 0; ia < q; ++ia, ++r)
      for (int jy = 0; jy < q; ++jy)
        for (int jx = 0; jx < q; ++jx) E(r, jy * q + jx) = Rx(ia, jx) * Ry(jb, jy);
  return E;
}

// evaluate_basis (basis.cpp:318-341) at reference point (u, v).
void eval2(const Mat& E, int p, double u, double v, double hx, double hy, double* val, double* gx,
           double* gy) {
  const int q = p + 1, nl = q * q;
  double bu[kMaxQ], du[kMaxQ], bv[kMaxQ], dv[kMaxQ];
  spline::bernstein(p, u, bu, du);
  spline::bernstein(p, v, bv, dv);
  double bval[kMaxQ * kMaxQ], bgx[kMaxQ * kMaxQ], bgy[kMaxQ * kMaxQ];
  for (int jy = 0; jy < q; ++jy)
    for (int jx = 0; jx < q; ++jx) {
      const int k = jy * q + jx;
      bval[k] = bu[jx] * bv[jy];
      bgx[k] = du[jx] * bv[jy];
      bgy[k] = bu[jx] * dv[jy];
    }
  for (int r = 0; r < nl; ++r) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (int k = 0; k < nl; ++k) {
      a += E(r, k) * bval[k];
      b += E(r, k) * bgx[k];
      c += E(r, k) * bgy[k];
    }
    val[r] = a;
    gx[r] = b / hx;
    gy[r] = c / hy;
  }
}

// Box sides of a cell on the embedding-box boundary (assembly.cpp:24-33).
int box_sides(const Grid& g, int ix, int iy, int* out) {
  int n = 0;
  if (iy == 0) out[n++] = 0;
  if (ix == g.res[0] - 1) out[n++] = 1;
  if (iy == g.res[1] - 1) out[n++] = 2;
  if (ix == 0) out[n++] = 3;
  return n;
}

// Reference element loop body for one 2D element (assembly.cpp:55-162).
ElemData element2(const Space& s, int e, const ProblemConfig& prob, const QuadConfig& qc,
                  double beta, bool cut, bool sides) {
  const Grid& g = s.grid;
  const int p = s.p, q = p + 1, nl = q * q;
  const Mat E = extraction2(s, s.ext_cls[0][s.el_ix[e]], s.ext_cls[1][s.el_iy[e]]);
  double lo[3], hi[3];
  g.cell_box(s.el_ix[e], s.el_iy[e], 0, lo, hi);
  const double sx = hi[0] - lo[0], sy = hi[1] - lo[1];
  ElemData d;
  d.K.assign(static_cast<size_t>(nl) * nl, 0.0);
  d.F.assign(nl, 0.0);
  double val[kMaxQ * kMaxQ], gx[kMaxQ * kMaxQ], gy[kMaxQ * kMaxQ];
  auto at = [&](double x, double y) { eval2(E, p, (x - lo[0]) / sx, (y - lo[1]) / sy, sx, sy, val, gx, gy); };

  const QuadRule2 vr = volume_rule2(s.ls, lo, hi, cut ? kCut : kInside, qc);
  for (size_t k = 0; k < vr.size(); ++k) {
    const double w = vr.w[k];
    d.volume += w;
    at(vr.px[k], vr.py[k]);
    for (int i = 0; i < nl; ++i)
      for (int j = 0; j < nl; ++j) d.K[i * nl + j] += w * (gx[i] * gx[j] + gy[i] * gy[j]);
    if (prob.body_force != 0.0)
      for (int i = 0; i < nl; ++i) d.F[i] += w * prob.body_force * val[i];
  }
  auto boundary_point = [&](double x, double y, double w) {
    // Dirichlet piece, g = 0 (assembly.cpp:123-131): Ke += (w*beta) v v^T.
    at(x, y);
    const double wb = w * beta;
    for (int i = 0; i < nl; ++i)
      for (int j = 0; j < nl; ++j) d.K[i * nl + j] += wb * (val[i] * val[j]);
  };
  if (cut) {
    const QuadRule2 br = boundary_rule2(s.ls, lo, hi, qc);
    for (size_t k = 0; k < br.size(); ++k) boundary_point(br.px[k], br.py[k], br.w[k]);
  }
  if (sides) {
    int sd[4];
    const int ns = box_sides(g, s.el_ix[e], s.el_iy[e], sd);
    for (int i = 0; i < ns; ++i) {
      const QuadRule2 sr = side_rule2(s.ls, lo, hi, sd[i], qc);
      for (size_t k = 0; k < sr.size(); ++k) boundary_point(sr.px[k], sr.py[k], sr.w[k]);
    }
  }
  return d;
}

// ------------------------------------------------------------------ 3D ----
// Stable point evaluation: 1D local functions of an extraction class are
// non-negative combinations of Bernstein polynomials (span_extraction), so
// values/derivatives at a point carry no cancellation, and every diagonal
// contribution w*|grad phi|^2 is >= 0 -- essential for slivers whose
// diagonal is 1e-30 of the interior one.

inline void eval1d(const Mat& E, int p, double u, double* v, double* d) {
  double b[kMaxQ], db[kMaxQ];
  spline::bernstein(p, u, b, db);
  for (int i = 0; i <= p; ++i) {
    double a = 0.0, c = 0.0;
    for (int k = 0; k <= p; ++k) {
      a += E(i, k) * b[k];
      c += E(i, k) * db[k];
    }
    v[i] = a;
    d[i] = c;
  }
}

struct Elem3 {
  const Mat* E[3];
  int p;
  double h[3];
  double beta, f;
  double* K;  // nl x nl row-major (upper triangle accumulated, mirrored at the end)
  double* F;
  double vol;  // reference-units volume integrated (fraction of the cell)
};

// Volume point u (reference coords), reference weight w.
void add_vol_point(Elem3& e, const double* u, double w) {
  const int p = e.p, q = p + 1, nl = q * q * q;
  double v[3][kMaxQ], d[3][kMaxQ];
  for (int a = 0; a < 3; ++a) eval1d(*e.E[a], p, u[a], v[a], d[a]);
  const double jac = e.h[0] * e.h[1] * e.h[2];
  const double wp = w * jac;
  double phi[kMaxQ * kMaxQ * kMaxQ], gx[kMaxQ * kMaxQ * kMaxQ], gy[kMaxQ * kMaxQ * kMaxQ],
      gz[kMaxQ * kMaxQ * kMaxQ];
  for (int ic = 0, i = 0; ic < q; ++ic)
    for (int ib = 0; ib < q; ++ib)
      for (int ia = 0; ia < q; ++ia, ++i) {
        phi[i] = v[0][ia] * v[1][ib] * v[2][ic];
        gx[i] = d[0][ia] * v[1][ib] * v[2][ic] / e.h[0];
        gy[i] = v[0][ia] * d[1][ib] * v[2][ic] / e.h[1];
        gz[i] = v[0][ia] * v[1][ib] * d[2][ic] / e.h[2];
      }
  for (int i = 0; i < nl; ++i) {
    double* Ki = e.K + static_cast<size_t>(i) * nl;
    const double a = wp * gx[i], b = wp * gy[i], c = wp * gz[i];
    for (int j = i; j < nl; ++j) Ki[j] += a * gx[j] + b * gy[j] + c * gz[j];
    if (e.f != 0.0) e.F[i] += wp * e.f * phi[i];
  }
  e.vol += w;
}

// Interface point (reference coords, reference-area weight w): penalty term.
void add_surf_point(Elem3& e, const double* u, double w) {
  const int p = e.p, q = p + 1, nl = q * q * q;
  double v[3][kMaxQ], d[3][kMaxQ];
  for (int a = 0; a < 3; ++a) eval1d(*e.E[a], p, u[a], v[a], d[a]);
  const double wb = w * e.h[0] * e.h[0] * e.beta;  // cubic cells: dS = h^2 dS_ref
  double phi[kMaxQ * kMaxQ * kMaxQ];
  for (int ic = 0, i = 0; ic < q; ++ic)
    for (int ib = 0; ib < q; ++ib)
      for (int ia = 0; ia < q; ++ia, ++i) phi[i] = v[0][ia] * v[1][ib] * v[2][ic];
  for (int i = 0; i < nl; ++i) {
    double* Ki = e.K + static_cast<size_t>(i) * nl;
    const double a = wb * phi[i];
    for (int j = i; j < nl; ++j) Ki[j] += a * phi[j];
  }
}

// Axis box [a, b] (reference coords): exact tensor integration with (p+1)-point
// Gauss per axis (the 1D integrands have degree <= 2p).
void add_box(Elem3& e, const double* a, const double* b) {
  const int p = e.p, q = p + 1, nl = q * q * q;
  std::vector<double> gn, gw;
  gauss_legendre(q, gn, gw);
  double Ivv[3][kMaxQ][kMaxQ] = {}, Idd[3][kMaxQ][kMaxQ] = {}, Iv[3][kMaxQ] = {};
  for (int ax = 0; ax < 3; ++ax) {
    const double L = b[ax] - a[ax];
    if (!(L > 0.0)) return;
    for (int g = 0; g < q; ++g) {
      const double u = a[ax] + 0.5 * (gn[g] + 1.0) * L, w = 0.5 * gw[g] * L;
      double v[kMaxQ], d[kMaxQ];
      eval1d(*e.E[ax], p, u, v, d);
      for (int i = 0; i < q; ++i) {
        Iv[ax][i] += w * v[i];
        for (int j = 0; j < q; ++j) {
          Ivv[ax][i][j] += w * v[i] * v[j];
          Idd[ax][i][j] += w * d[i] * d[j];
        }
      }
    }
  }
  const double jac = e.h[0] * e.h[1] * e.h[2];
  const double cx = jac / (e.h[0] * e.h[0]), cy = jac / (e.h[1] * e.h[1]), cz = jac / (e.h[2] * e.h[2]);
  for (int i = 0; i < nl; ++i) {
    const int ia = i % q, ib = (i / q) % q, ic = i / (q * q);
    double* Ki = e.K + static_cast<size_t>(i) * nl;
    for (int j = i; j < nl; ++j) {
      const int ja = j % q, jb = (j / q) % q, jc = j / (q * q);
      Ki[j] += cx * Idd[0][ia][ja] * Ivv[1][ib][jb] * Ivv[2][ic][jc] +
               cy * Ivv[0][ia][ja] * Idd[1][ib][jb] * Ivv[2][ic][jc] +
               cz * Ivv[0][ia][ja] * Ivv[1][ib][jb] * Idd[2][ic][jc];
    }
    if (e.f != 0.0) e.F[i] += e.f * jac * Iv[0][ia] * Iv[1][ib] * Iv[2][ic];
  }
  e.vol += (b[0] - a[0]) * (b[1] - a[1]) * (b[2] - a[2]);
}

void finish3(Elem3& e) {
  const int q = e.p + 1, nl = q * q * q;
  for (int i = 0; i < nl; ++i)
    for (int j = 0; j < i; ++j) e.K[static_cast<size_t>(i) * nl + j] = e.K[static_cast<size_t>(j) * nl + i];
}

struct Rule1 {
  std::vector<double> x, w;  // on [0,1]
};
Rule1 gauss01(int n) {
  Rule1 r;
  std::vector<double> nd, wt;
  gauss_legendre(n, nd, wt);
  for (int i = 0; i < n; ++i) {
    r.x.push_back(0.5 * (nd[i] + 1.0));
    r.w.push_back(0.5 * wt[i]);
  }
  return r;
}

// Collapsed (Duffy) rule on tetrahedron v0..v3 (reference coords):
// x = v0 + a[(v1-v0) + b((v2-v1) + c(v3-v2))], |J| = 6 V a^2 b.
void tet_points(Elem3& e, const double v[4][3], const Rule1& g) {
  double e1[3], e2[3], e3[3];
  for (int k = 0; k < 3; ++k) {
    e1[k] = v[1][k] - v[0][k];
    e2[k] = v[2][k] - v[1][k];
    e3[k] = v[3][k] - v[2][k];
  }
  const double det = e1[0] * (e2[1] * e3[2] - e2[2] * e3[1]) - e1[1] * (e2[0] * e3[2] - e2[2] * e3[0]) +
                     e1[2] * (e2[0] * e3[1] - e2[1] * e3[0]);
  const double vol6 = std::fabs(det);
  if (!(vol6 > 0.0)) return;
  const size_t n = g.x.size();
  for (size_t ia = 0; ia < n; ++ia)
    for (size_t ib = 0; ib < n; ++ib)
      for (size_t ic = 0; ic < n; ++ic) {
        const double a = g.x[ia], b = g.x[ib], c = g.x[ic];
        double u[3];
        for (int k = 0; k < 3; ++k) u[k] = v[0][k] + a * (e1[k] + b * (e2[k] + c * e3[k]));
        add_vol_point(e, u, vol6 * a * a * b * g.w[ia] * g.w[ib] * g.w[ic]);
      }
}

// Triangle v0..v2 (reference coords, area in reference units).
void tri_points(Elem3& e, const double v[3][3], const Rule1& g) {
  double e1[3], e2[3];
  for (int k = 0; k < 3; ++k) {
    e1[k] = v[1][k] - v[0][k];
    e2[k] = v[2][k] - v[1][k];
  }
  const double cx = e1[1] * e2[2] - e1[2] * e2[1], cy = e1[2] * e2[0] - e1[0] * e2[2],
               cz = e1[0] * e2[1] - e1[1] * e2[0];
  const double area2 = std::sqrt(cx * cx + cy * cy + cz * cz);
  if (!(area2 > 0.0)) return;
  const size_t n = g.x.size();
  for (size_t ia = 0; ia < n; ++ia)
    for (size_t ib = 0; ib < n; ++ib) {
      const double a = g.x[ia], b = g.x[ib];
      double u[3];
      for (int k = 0; k < 3; ++k) u[k] = v[0][k] + a * (e1[k] + b * e2[k]);
      add_surf_point(e, u, area2 * a * g.w[ia] * g.w[ib]);
    }
}

struct Cut3Ctx {
  const LevelSet* ls;
  const double* elo;  // element box lo (physical)
  QuadConfig qc;
  Rule1 gt, gs;  // tetrahedron / triangle 1D factors
  Elem3* e;
};

void to_ref(const Cut3Ctx& c, const double* x, double* u) {
  for (int k = 0; k < 3; ++k) u[k] = (x[k] - c.elo[k]) / c.e->h[k];
}

// Clip tetrahedron (physical vertices x, values f) to psi >= 0; interface
// facets are the clip planes through the (bisection) edge roots.
void clip_tet(Cut3Ctx& c, const double x[4][3], const double f[4]) {
  int in[4], out[4], ni = 0, no = 0;
  for (int k = 0; k < 4; ++k) {
    if (f[k] >= 0.0)
      in[ni++] = k;
    else
      out[no++] = k;
  }
  if (ni == 0) return;
  auto ref = [&](const double* p, double* u) { to_ref(c, p, u); };
  auto cross = [&](int a, int b, double* u) {
    double r[3];
    intersect_edge(*c.ls, x[a], x[b], 3, c.qc.edge_tol, r);
    ref(r, u);
  };
  double T[4][3];
  if (ni == 4) {
    for (int k = 0; k < 4; ++k) ref(x[k], T[k]);
    tet_points(*c.e, T, c.gt);
    return;
  }
  if (ni == 1) {
    const int a = in[0];
    double P[3][3];
    for (int k = 0; k < 3; ++k) cross(a, out[k], P[k]);
    ref(x[a], T[0]);
    for (int k = 0; k < 3; ++k)
      for (int d = 0; d < 3; ++d) T[k + 1][d] = P[k][d];
    tet_points(*c.e, T, c.gt);
    tri_points(*c.e, P, c.gs);
    return;
  }
  if (ni == 3) {
    const int a = out[0];
    double bot[3][3], top[3][3];
    for (int k = 0; k < 3; ++k) {
      ref(x[in[k]], bot[k]);
      cross(in[k], a, top[k]);
    }
    const double* Pr[3][4] = {{bot[0], bot[1], bot[2], top[0]},
                              {bot[1], bot[2], top[0], top[1]},
                              {bot[2], top[0], top[1], top[2]}};
    for (auto& t : Pr) {
      for (int k = 0; k < 4; ++k)
        for (int d = 0; d < 3; ++d) T[k][d] = t[k][d];
      tet_points(*c.e, T, c.gt);
    }
    tri_points(*c.e, top, c.gs);
    return;
  }
  const int a = in[0], b = in[1];
  double pa[3], pb[3], xa0[3], xa1[3], xb0[3], xb1[3];
  ref(x[a], pa);
  ref(x[b], pb);
  cross(a, out[0], xa0);
  cross(a, out[1], xa1);
  cross(b, out[0], xb0);
  cross(b, out[1], xb1);
  const double* Pr[3][4] = {{pa, xa0, xa1, pb}, {xa0, xa1, pb, xb0}, {xa1, pb, xb0, xb1}};
  for (auto& t : Pr) {
    for (int k = 0; k < 4; ++k)
      for (int d = 0; d < 3; ++d) T[k][d] = t[k][d];
    tet_points(*c.e, T, c.gt);
  }
  double t1[3][3], t2[3][3];
  for (int d = 0; d < 3; ++d) {
    t1[0][d] = xa0[d];
    t1[1][d] = xb0[d];
    t1[2][d] = xb1[d];
    t2[0][d] = xa0[d];
    t2[1][d] = xb1[d];
    t2[2][d] = xa1[d];
  }
  tri_points(*c.e, t1, c.gs);
  tri_points(*c.e, t2, c.gs);
}

// Kuhn decomposition: 6 tetrahedra sharing the diagonal 0 -> 7 (corner = x + 2y + 4z).
const int kKuhn[6][4] = {{0, 1, 3, 7}, {0, 1, 5, 7}, {0, 2, 3, 7},
                         {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 4, 6, 7}};

void cut_leaf3(Cut3Ctx& c, const double* lo, const double* hi) {
  double x[8][3], f[8];
  for (int k = 0; k < 8; ++k) {
    x[k][0] = (k & 1) ? hi[0] : lo[0];
    x[k][1] = (k & 2) ? hi[1] : lo[1];
    x[k][2] = (k & 4) ? hi[2] : lo[2];
    f[k] = (*c.ls)(x[k]);
  }
  for (const auto& t : kKuhn) {
    double tx[4][3], tf[4];
    for (int k = 0; k < 4; ++k) {
      for (int d = 0; d < 3; ++d) tx[k][d] = x[t[k]][d];
      tf[k] = f[t[k]];
    }
    clip_tet(c, tx, tf);
  }
}

// Octree analogue of recurse_cut (quadrature.cpp:266-290).
void recurse3(Cut3Ctx& c, const double* lo, const double* hi, int depth) {
  switch (classify_cell(*c.ls, lo, hi, 3, c.qc.classify_depth)) {
    case CellClass::Outside: return;
    case CellClass::Inside: {
      double a[3], b[3];
      to_ref(c, lo, a);
      to_ref(c, hi, b);
      add_box(*c.e, a, b);
      return;
    }
    case CellClass::Cut: break;
  }
  if (depth == 0) {
    cut_leaf3(c, lo, hi);
    return;
  }
  double mid[3];
  for (int k = 0; k < 3; ++k) mid[k] = 0.5 * (lo[k] + hi[k]);
  for (int k = 0; k < 8; ++k) {
    double l[3], hh[3];
    for (int d = 0; d < 3; ++d) {
      const bool up = (k >> d) & 1;
      l[d] = up ? mid[d] : lo[d];
      hh[d] = up ? hi[d] : mid[d];
    }
    recurse3(c, l, hh, depth - 1);
  }
}

// Element data for a 3D element: cut (octree + clipped tets) or full box.
ElemData element3(const Space& s, int cx, int cy, int cz, const double* lo, const double* hi, bool cut,
                  const QuadConfig& qc, double beta, double f) {
  const int q = s.p + 1, nl = q * q * q;
  ElemData d;
  d.K.assign(static_cast<size_t>(nl) * nl, 0.0);
  d.F.assign(nl, 0.0);
  Elem3 e{{&s.ext[0][cx], &s.ext[1][cy], &s.ext[2][cz]}, s.p, {s.grid.h(0), s.grid.h(1), s.grid.h(2)},
          beta, f, d.K.data(), d.F.data(), 0.0};
  if (cut) {
    Cut3Ctx c{&s.ls, lo, qc, gauss01(2), gauss01(3), &e};
    recurse3(c, lo, hi, qc.depth);
  } else {
    const double a[3] = {0, 0, 0}, b[3] = {1, 1, 1};
    add_box(e, a, b);
  }
  finish3(e);
  d.volume = e.vol;
  return d;
}
}  // namespace

Assembled assemble(const Space& s, const ProblemConfig& prob, const QuadConfig& qc, int threads, bool numeric) {
  const Grid& g = s.grid;
  const int dim = g.dim, p = s.p, nl = s.nloc();
  const double beta = prob.beta > 0.0 ? prob.beta : default_penalty(g);
  const int ne = static_cast<int>(s.el_ix.size());
  Assembled out;
  const bool timing = std::getenv("IG_TIMING") != nullptr;
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  auto secs = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
  const auto ta0 = tnow();

  // --- element data -------------------------------------------------------
  // Elements needing individual treatment: cut, or (2D) box-boundary sides.
  std::vector<int32_t> special(static_cast<size_t>(ne), -1);
  std::vector<int> special_list;
  for (int e = 0; e < ne; ++e) {
    bool sp = s.el_tag[e] == kCut;
    if (prob.dirichlet_box_sides) {
      if (dim == 3) {
        const int idx[3] = {s.el_ix[e], s.el_iy[e], s.el_iz[e]};
        for (int d = 0; d < 3; ++d)
          if (idx[d] == 0 || idx[d] == g.res[d] - 1)
            throw SetupError("assemble: Dirichlet on 3D box faces is not supported");
      } else {
        int sd[4];
        if (box_sides(g, s.el_ix[e], s.el_iy[e], sd) > 0) sp = true;
      }
    }
    if (sp) {
      special[e] = static_cast<int32_t>(special_list.size());
      special_list.push_back(e);
    }
  }
  out.cut_elements = 0;
  for (int e = 0; e < ne; ++e) out.cut_elements += s.el_tag[e] == kCut;

  std::vector<ElemData> sdata(special_list.size());
  // Class data for plain Inside elements.
  const int ncx = static_cast<int>(s.ext[0].size()), ncy = static_cast<int>(s.ext[1].size());
  const int ncz = dim == 3 ? static_cast<int>(s.ext[2].size()) : 1;
  std::vector<ElemData> cdata(static_cast<size_t>(ncx) * ncy * ncz);
  const double h3[3] = {g.h(0), g.h(1), dim == 3 ? g.h(2) : 1.0};
  if (dim == 3 && (std::fabs(h3[0] - h3[1]) > 1e-14 * h3[0] || std::fabs(h3[0] - h3[2]) > 1e-14 * h3[0]))
    throw SetupError("assemble: 3D cells must be cubic");

  // Inside classes: reference-coordinate integration.
  std::vector<uint8_t> class_used(cdata.size(), 0);
  for (int e = 0; e < ne; ++e)
    if (special[e] < 0) {
      const int cx = s.ext_cls[0][s.el_ix[e]], cy = s.ext_cls[1][s.el_iy[e]];
      const int cz = dim == 3 ? s.ext_cls[2][s.el_iz[e]] : 0;
      class_used[(static_cast<size_t>(cz) * ncy + cy) * ncx + cx] = 1;
    }
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
  for (int64_t ci = 0; ci < static_cast<int64_t>(cdata.size()); ++ci) {
    if (!class_used[ci]) continue;
    const int cx = static_cast<int>(ci % ncx), cy = static_cast<int>((ci / ncx) % ncy),
              cz = static_cast<int>(ci / (static_cast<int64_t>(ncx) * ncy));
    ElemData& d = cdata[ci];
    if (dim == 2) {
      const Mat E = extraction2(s, cx, cy);
      std::vector<double> gn, gw;
      gauss_legendre(qc.gauss_order, gn, gw);
      d.K.assign(static_cast<size_t>(nl) * nl, 0.0);
      d.F.assign(nl, 0.0);
      double val[kMaxQ * kMaxQ], gx[kMaxQ * kMaxQ], gy[kMaxQ * kMaxQ];
      for (int j = 0; j < qc.gauss_order; ++j)
        for (int i = 0; i < qc.gauss_order; ++i) {
          const double w = gw[i] * gw[j] * 0.25 * h3[0] * h3[1];
          eval2(E, p, 0.5 * (gn[i] + 1.0), 0.5 * (gn[j] + 1.0), h3[0], h3[1], val, gx, gy);
          for (int a = 0; a < nl; ++a)
            for (int b = 0; b < nl; ++b) d.K[a * nl + b] += w * (gx[a] * gx[b] + gy[a] * gy[b]);
          if (prob.body_force != 0.0)
            for (int a = 0; a < nl; ++a) d.F[a] += w * prob.body_force * val[a];
        }
    } else {
      d = element3(s, cx, cy, cz, nullptr, nullptr, false, qc, beta, prob.body_force);
    }
  }

  // Special elements.
  double eta = 1.0;
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads) reduction(min : eta)
  for (int64_t k = 0; k < (numeric ? static_cast<int64_t>(special_list.size()) : 0); ++k) {
    const int e = special_list[k];
    const bool cut = s.el_tag[e] == kCut;
    if (dim == 2) {
      sdata[k] = element2(s, e, prob, qc, beta, cut, prob.dirichlet_box_sides);
      if (cut) {
        double lo[3], hi[3];
        g.cell_box(s.el_ix[e], s.el_iy[e], 0, lo, hi);
        eta = std::min(eta, sdata[k].volume / ((hi[0] - lo[0]) * (hi[1] - lo[1])));
      }
    } else {
      double lo[3], hi[3];
      g.cell_box(s.el_ix[e], s.el_iy[e], s.el_iz[e], lo, hi);
      const int cx = s.ext_cls[0][s.el_ix[e]], cy = s.ext_cls[1][s.el_iy[e]], cz = s.ext_cls[2][s.el_iz[e]];
      sdata[k] = element3(s, cx, cy, cz, lo, hi, true, qc, beta, prob.body_force);
      eta = std::min(eta, sdata[k].volume);  // reference units: fraction of the cell
    }
  }
  out.eta = eta;
  out.el_vol.assign(static_cast<size_t>(ne), 1.0);
  for (size_t k = 0; k < special_list.size(); ++k) {
    const int e = special_list[k];
    if (s.el_tag[e] != kCut) continue;
    if (dim == 2) {
      double lo[3], hi[3];
      g.cell_box(s.el_ix[e], s.el_iy[e], 0, lo, hi);
      out.el_vol[e] = sdata[k].volume / ((hi[0] - lo[0]) * (hi[1] - lo[1]));
    } else {
      out.el_vol[e] = sdata[k].volume;
    }
  }
  const auto ta1 = tnow();

  // Element tables for the device row gather (same data, flattened).
  {
    const int ncls = static_cast<int>(cdata.size());
    out.n_tables = ncls + static_cast<int32_t>(sdata.size());
    out.tabK.assign(static_cast<size_t>(out.n_tables) * nl * nl, 0.0);
    out.tabF.assign(static_cast<size_t>(out.n_tables) * nl, 0.0);
    auto put = [&](int t, const ElemData& d) {
      if (d.K.size() == static_cast<size_t>(nl) * nl)
        std::copy(d.K.begin(), d.K.end(), out.tabK.begin() + static_cast<size_t>(t) * nl * nl);
      if (d.F.size() == static_cast<size_t>(nl)) std::copy(d.F.begin(), d.F.end(), out.tabF.begin() + static_cast<size_t>(t) * nl);
    };
    for (int t = 0; t < ncls; ++t)
      if (class_used[t]) put(t, cdata[t]);
    for (size_t k = 0; k < sdata.size(); ++k) put(ncls + static_cast<int>(k), sdata[k]);
    out.el_table.resize(static_cast<size_t>(ne));
    for (int e = 0; e < ne; ++e) {
      if (special[e] >= 0) {
        out.el_table[e] = ncls + special[e];
      } else {
        const int cx = s.ext_cls[0][s.el_ix[e]], cy = s.ext_cls[1][s.el_iy[e]];
        const int cz = dim == 3 ? s.ext_cls[2][s.el_iz[e]] : 0;
        out.el_table[e] = (cz * ncy + cy) * ncx + cx;
      }
    }
  }

  if (!numeric) {  // geometric half: no row gather, no symmetrisation
    out.A.nr = out.A.nc = s.n();
    out.A.ptr.assign(static_cast<size_t>(s.n()) + 1, 0);
    out.b.assign(static_cast<size_t>(s.n()), 0.0);
    return out;
  }

  auto elem = [&](int e) -> const ElemData& {
    if (special[e] >= 0) return sdata[special[e]];
    const int cx = s.ext_cls[0][s.el_ix[e]], cy = s.ext_cls[1][s.el_iy[e]];
    const int cz = dim == 3 ? s.ext_cls[2][s.el_iz[e]] : 0;
    return cdata[(static_cast<size_t>(cz) * ncy + cy) * ncx + cx];
  };

  // --- row-gather assembly -------------------------------------------------
  const int n = s.n();
  const int q = p + 1;
  const int W = 2 * p + 1;  // column window per axis (B-spline and Lagrange)
  const int wz = dim == 3 ? W : 1;
  const int wsize = W * W * wz;
  std::vector<int32_t> rowlen(static_cast<size_t>(n), 0);
  out.b.assign(n, 0.0);

  // Pass 1 computes row patterns + values into per-row scratch, twice
  // (count, then fill) to avoid storing triplets.
  auto row_work = [&](int a, double* acc, uint8_t* touched, int32_t* cols, double* vals,
                      bool fill) -> int {
    const int64_t u = s.anchors[a];
    const int ax = static_cast<int>(u % s.nf[0]);
    const int ay = static_cast<int>((u / s.nf[0]) % s.nf[1]);
    const int az = static_cast<int>(u / (static_cast<int64_t>(s.nf[0]) * s.nf[1]));
    std::fill(touched, touched + wsize, 0);
    double bsum = 0.0;
    for (int64_t k = s.supp_ptr[a]; k < s.supp_ptr[a + 1]; ++k) {
      const int e = s.supp_el[k];
      const ElemData& d = elem(e);
      const int x0 = s.first_anchor(s.el_ix[e]), y0 = s.first_anchor(s.el_iy[e]);
      const int z0 = dim == 3 ? s.first_anchor(s.el_iz[e]) : 0;
      const int li = dim == 3 ? ((az - z0) * q + (ay - y0)) * q + (ax - x0) : (ay - y0) * q + (ax - x0);
      if (fill) bsum += d.F[li];
      const double* Krow = d.K.data() + static_cast<size_t>(li) * nl;
      for (int lj = 0; lj < nl; ++lj) {
        const double v = Krow[lj];
        if (v == 0.0) continue;
        const int jx = x0 + lj % q, jy = y0 + (lj / q) % q, jz = dim == 3 ? z0 + lj / (q * q) : 0;
        const int w = ((dim == 3 ? (jz - az + p) : 0) * W + (jy - ay + p)) * W + (jx - ax + p);
        if (!touched[w]) {
          touched[w] = 1;
          acc[w] = v;  // 0 + v == v
        } else {
          acc[w] = acc[w] + v;
        }
      }
    }
    int cnt = 0;
    for (int w = 0; w < wsize; ++w) {
      if (!touched[w]) continue;
      if (fill) {
        const int dx = w % W - p, dy = (w / W) % W - p, dz = dim == 3 ? w / (W * W) - p : 0;
        cols[cnt] = s.kept[s.untrimmed(ax + dx, ay + dy, az + dz)];
        vals[cnt] = acc[w];
      }
      ++cnt;
    }
    if (fill) out.b[a] = bsum;
    return cnt;
  };
  // bsum: b[gi] starts at 0 and receives Fe contributions in element order.
#pragma omp parallel num_threads(threads)
  {
    std::vector<double> acc(wsize);
    std::vector<uint8_t> touched(wsize);
#pragma omp for schedule(dynamic, 512)
    for (int a = 0; a < n; ++a) rowlen[a] = row_work(a, acc.data(), touched.data(), nullptr, nullptr, false);
  }
  Csr& A = out.A;
  A.nr = A.nc = n;
  A.ptr.assign(static_cast<size_t>(n) + 1, 0);
  for (int a = 0; a < n; ++a) {
    const int64_t nx = static_cast<int64_t>(A.ptr[a]) + rowlen[a];
    if (nx > INT32_MAX) throw SetupError("assemble: nnz exceeds int32");
    A.ptr[a + 1] = static_cast<int32_t>(nx);
  }
  A.col.resize(A.ptr[n]);
  A.val.resize(A.ptr[n]);
#pragma omp parallel num_threads(threads)
  {
    std::vector<double> acc(wsize);
    std::vector<uint8_t> touched(wsize);
#pragma omp for schedule(dynamic, 512)
    for (int a = 0; a < n; ++a)
      row_work(a, acc.data(), touched.data(), A.col.data() + A.ptr[a], A.val.data() + A.ptr[a], true);
  }
  // Columns come out in window order; kept numbering is monotone in
  // (az, ay, ax), so window order is ascending column order.

  const auto ta2 = tnow();
  // --- symmetrise: A = 0.5 (A + A^T) (assembly.cpp:177-180) ----------------
  std::vector<double> sym(A.val.size());
  int unsym = 0;
#pragma omp parallel for schedule(dynamic, 512) num_threads(threads) reduction(+ : unsym)
  for (int i = 0; i < n; ++i)
    for (int32_t k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
      const int32_t j = A.col[k];
      const int32_t* b = A.col.data() + A.ptr[j];
      const int32_t* e = A.col.data() + A.ptr[j + 1];
      const int32_t* it = std::lower_bound(b, e, i);
      if (it == e || *it != i) {
        ++unsym;
        continue;
      }
      sym[k] = 0.5 * (A.val[k] + A.val[it - A.col.data()]);
    }
  if (unsym) throw SetupError("assemble: unsymmetric pattern");
  A.val.swap(sym);
  if (timing)
    std::fprintf(stderr, "assemble: element data %.3f s (%zu special), row gather %.3f s, symmetrise %.3f s\n",
                 secs(ta0, ta1), special_list.size(), secs(ta1, ta2), secs(ta2, tnow()));
  return out;
}

}  // namespace igh
