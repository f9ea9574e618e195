// cutquad2.cuh — the reference's 2D cut-cell quadrature on the device
// (ig_cut2, ig_gpu.h): the element integration of assemble()
// (proj/src/assembly.cpp:55-162) for the individually integrated elements of
// a uniform 2D case -- cut elements (recurse_cut with leaf_polygons,
// refine_chords, fan_triangulate / interface_segments,
// proj/src/quadrature.cpp:128-335) and elements with embedding-box sides
// (side_rule, :337-372) -- restated operation for operation from
// host/quad2d.cpp and host/assembly.cpp element2, so the element matrices are
// bit-identical to the host's.  Three kernels, one CTA per element:
// k_cq2_points<false> counts every element's quadrature points (volume points
// of its quadtree leaves in depth-first order, then interface points, then
// box-side points), k_cq2_points<true> writes them, k_cq2_integrate evaluates
// the basis per point (eval2: Bernstein x full 2D extraction) in shared memory
// and every thread accumulates its K / F entries over the points in order.
#pragma once

#include <cstdint>

#include "cutquad.cuh"

namespace igk {

constexpr int kCq2Threads = 128;
constexpr int kCq2MaxQ = 5;  // p <= 4
constexpr int kCq2Batch = 32;

struct V2d {
  double x, y;
};
__device__ __forceinline__ V2d v2add(V2d a, V2d b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ V2d v2sub(V2d a, V2d b) { return {a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ V2d v2mul(double s, V2d a) { return {s * a.x, s * a.y}; }
__device__ __forceinline__ double v2norm(V2d a) { return sqrt(a.x * a.x + a.y * a.y); }

struct Box2d {
  V2d lo, hi;
  __device__ V2d center() const { return v2mul(0.5, v2add(lo, hi)); }
  __device__ V2d size() const { return v2sub(hi, lo); }
  __device__ bool contains(V2d p) const { return p.x >= lo.x && p.x <= hi.x && p.y >= lo.y && p.y <= hi.y; }
  __device__ V2d corner(int k) const {
    switch (k & 3) {
      case 0: return lo;
      case 1: return {hi.x, lo.y};
      case 2: return hi;
      default: return {lo.x, hi.y};
    }
  }
};

__device__ __forceinline__ double cq2_ls(const ig_cut2& I, V2d p) {
  const double q[3] = {p.x, p.y, 0.0};
  return ls_eval(I.prog, I.prog_len, q);
}
// intersect_edge in 2D (host/levelset.cpp, dim 2)
__device__ V2d cq2_isect(const ig_cut2& I, V2d a, V2d b) {
  const double p0[2] = {a.x, a.y}, p1[2] = {b.x, b.y};
  double f0 = cq2_ls(I, a);
  double t0 = 0.0, t1 = 1.0;
  while (t1 - t0 > I.edge_tol) {
    const double tm = 0.5 * (t0 + t1);
    const V2d q{p0[0] + tm * (p1[0] - p0[0]), p0[1] + tm * (p1[1] - p0[1])};
    const double fm = cq2_ls(I, q);
    if (f0 * fm <= 0.0) {
      t1 = tm;
    } else {
      t0 = tm;
      f0 = fm;
    }
  }
  const double tm = 0.5 * (t0 + t1);
  return {p0[0] + tm * (p1[0] - p0[0]), p0[1] + tm * (p1[1] - p0[1])};
}
// classify_cell in 2D
__device__ int cq2_classify(const ig_cut2& I, const Box2d& b) {
  const double lo[3] = {b.lo.x, b.lo.y, 0.0}, hi[3] = {b.hi.x, b.hi.y, 0.0};
  double vmin, vmax;
  ls_bounds(I.prog, I.prog_len, lo, hi, 2, vmin, vmax);
  double scale = 0;
  for (int k = 0; k < 2; ++k) scale = cq_max(scale, fabs(lo[k]) + fabs(hi[k]));
  const double margin = 1e-9 * (1.0 + scale);
  if (vmin > margin) return 0;
  if (vmax < -margin) return 1;
  const int n = (1 << I.classify_depth) + 1;
  bool any_in = false, any_out = false;
  double d[2];
  for (int k = 0; k < 2; ++k) d[k] = (hi[k] - lo[k]) / static_cast<double>(n - 1);
  double p[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      p[0] = lo[0] + i * d[0];
      p[1] = lo[1] + j * d[1];
      if (ls_eval(I.prog, I.prog_len, p) >= 0.0)
        any_in = true;
      else
        any_out = true;
      if (any_in && any_out) return 2;
    }
  return any_in ? 0 : 1;
}

// A quadrature point sink: counts, or writes (x, y, w, kind) records.
template <bool W>
struct Cq2Sink {
  double* out;  // 4 doubles per point
  int n;
  __device__ void put(V2d p, double w) {
    if (W) {
      double* o = out + 4 * static_cast<int64_t>(n);
      o[0] = p.x;
      o[1] = p.y;
      o[2] = w;
      o[3] = 0.0;
    }
    ++n;
  }
};

constexpr int kCq2MaxPoly = 20;
struct Poly2 {
  V2d v[kCq2MaxPoly];
  bool cr[kCq2MaxPoly];
  int n;
};

__device__ int cq2_leaf_polygons(const ig_cut2& I, const Box2d& cell, Poly2 out[2]) {
  V2d c[4];
  double f[4];
  bool in[4];
  int n_in = 0;
  for (int k = 0; k < 4; ++k) {
    c[k] = cell.corner(k);
    f[k] = cq2_ls(I, c[k]);
    in[k] = f[k] >= 0.0;
    n_in += in[k];
  }
  if (n_in == 0) return 0;
  if (n_in == 4) {
    for (int k = 0; k < 4; ++k) {
      out[0].v[k] = c[k];
      out[0].cr[k] = false;
    }
    out[0].n = 4;
    return 1;
  }
  const bool saddle = in[0] == in[2] && in[1] == in[3] && in[0] != in[1];
  if (saddle && cq2_ls(I, cell.center()) < 0.0) {
    int np = 0;
    for (int k = 0; k < 4; ++k) {
      if (!in[k]) continue;
      const V2d xin = cq2_isect(I, c[k], c[(k + 3) % 4]);
      const V2d xout = cq2_isect(I, c[k], c[(k + 1) % 4]);
      out[np].v[0] = xin;
      out[np].v[1] = c[k];
      out[np].v[2] = xout;
      out[np].cr[0] = true;
      out[np].cr[1] = false;
      out[np].cr[2] = true;
      out[np].n = 3;
      ++np;
    }
    return np;
  }
  Poly2& p = out[0];
  p.n = 0;
  for (int k = 0; k < 4; ++k) {
    const int k1 = (k + 1) % 4;
    if (in[k]) {
      p.v[p.n] = c[k];
      p.cr[p.n++] = false;
    }
    if (in[k] != in[k1]) {
      p.v[p.n] = cq2_isect(I, c[k], c[k1]);
      p.cr[p.n++] = true;
    }
  }
  return 1;
}

__device__ V2d cq2_centroid(const Poly2& p) {
  V2d s{0.0, 0.0};
  for (int k = 0; k < p.n; ++k) s = v2add(s, p.v[k]);
  const double n = static_cast<double>(p.n);
  return {s.x / n, s.y / n};
}

__device__ void cq2_refine_chords(const ig_cut2& I, const Box2d& leaf, Poly2& p) {
  const int n = p.n;
  if (n < 3) return;
  Poly2 o;
  o.n = 0;
  for (int i = 0; i < n; ++i) {
    o.v[o.n] = p.v[i];
    o.cr[o.n++] = p.cr[i];
    const int j = (i + 1) % n;
    if (!p.cr[i] || !p.cr[j]) continue;
    const V2d a = p.v[i], b = p.v[j];
    const V2d d = v2sub(b, a);
    const double len = v2norm(d);
    if (!(len > 0.0)) continue;
    const V2d nrm{d.y / len, -d.x / len};
    const V2d m = v2mul(0.5, v2add(a, b));
    const double fm = cq2_ls(I, m);
    bool found = false;
    V2d refined{0, 0};
    if (fm == 0.0) {
      refined = m;
      found = true;
    } else {
      for (double t = len / 64.0; t <= 0.25 * len && !found; t *= 2.0) {
        for (int sgn = 0; sgn < 2; ++sgn) {
          const double s = sgn == 0 ? t : -t;
          const V2d q = v2add(m, v2mul(s, nrm));
          if (!leaf.contains(q) || fm * cq2_ls(I, q) > 0.0) continue;
          refined = cq2_isect(I, m, q);
          found = true;
          break;
        }
      }
    }
    if (found) {
      o.v[o.n] = refined;
      o.cr[o.n++] = true;
    }
  }
  p = o;
}

// tensor_rule (q-point Gauss per axis): j outer, i inner.
template <bool W>
__device__ void cq2_tensor(const ig_cut2& I, const Box2d& cell, Cq2Sink<W>& sk) {
  const int q = I.gauss_order;
  const double* n = I.gauss_q;
  const double* w = I.gauss_q + q;
  const V2d c = cell.center();
  const V2d h = v2mul(0.5, cell.size());
  for (int j = 0; j < q; ++j)
    for (int i = 0; i < q; ++i) sk.put({c.x + h.x * n[i], c.y + h.y * n[j]}, w[i] * w[j] * h.x * h.y);
}

// triangle_rule: Dunavant (q <= 3) or collapsed Gauss (q > 3).
template <bool W>
__device__ void cq2_triangle(const ig_cut2& I, V2d v0, V2d v1, V2d v2, Cq2Sink<W>& sk) {
  const int q = I.gauss_order;
  const V2d e1 = v2sub(v1, v0), e2 = v2sub(v2, v0);
  const double area = 0.5 * fabs(e1.x * e2.y - e1.y * e2.x);
  if (!(area > 0.0)) return;
  if (q <= 3) {
    double B[7][4];
    int nb = 0;
    auto orbit = [&](double a, double w) {
      const double b = 1.0 - 2.0 * a;
      B[nb][0] = a; B[nb][1] = a; B[nb][2] = b; B[nb][3] = w; ++nb;
      B[nb][0] = a; B[nb][1] = b; B[nb][2] = a; B[nb][3] = w; ++nb;
      B[nb][0] = b; B[nb][1] = a; B[nb][2] = a; B[nb][3] = w; ++nb;
    };
    if (q == 1) {
      B[0][0] = B[0][1] = B[0][2] = 1.0 / 3.0;
      B[0][3] = 1.0;
      nb = 1;
    } else if (q == 2) {
      orbit(0.445948490915965, 0.223381589678011);
      orbit(0.091576213509771, 0.109951743655322);
    } else {
      B[0][0] = B[0][1] = B[0][2] = 1.0 / 3.0;
      B[0][3] = 0.225;
      nb = 1;
      orbit(0.470142064105115, 0.132394152788506);
      orbit(0.101286507323456, 0.125939180544827);
    }
    for (int k = 0; k < nb; ++k)
      sk.put(v2add(v2add(v2mul(B[k][0], v0), v2mul(B[k][1], v1)), v2mul(B[k][2], v2)), B[k][3] * area);
    return;
  }
  const double* nu = I.gauss_q1;
  const double* wu = I.gauss_q1 + (q + 1);
  const double* nv = I.gauss_q;
  const double* wv = I.gauss_q + q;
  for (int j = 0; j < q; ++j) {
    const double v = 0.5 * (nv[j] + 1.0), dv = 0.5 * wv[j];
    for (int i = 0; i <= q; ++i) {
      const double u = 0.5 * (nu[i] + 1.0), du = 0.5 * wu[i];
      sk.put(v2add(v0, v2mul(u, v2add(v2mul(1.0 - v, e1), v2mul(v, e2)))), 2.0 * area * u * du * dv);
    }
  }
}

template <bool W>
__device__ void cq2_interface(const ig_cut2& I, const Poly2& p, Cq2Sink<W>& sk) {
  const int q = I.gauss_order;
  const double* gn = I.gauss_q;
  const double* gw = I.gauss_q + q;
  for (int i = 0; i < p.n; ++i) {
    const int j = (i + 1) % p.n;
    if (!p.cr[i] || !p.cr[j]) continue;
    const V2d d = v2sub(p.v[j], p.v[i]);
    const double len = v2norm(d);
    if (!(len > 0.0)) continue;
    for (int g = 0; g < q; ++g) {
      const double t = 0.5 * (gn[g] + 1.0);
      sk.put(v2add(p.v[i], v2mul(t, d)), 0.5 * gw[g] * len);
    }
  }
}

// Leaf `leaf` of the quadtree (digits in recurse_cut's child order: SW, SE,
// NE, NW): its volume points (vol = true) or interface points (vol = false).
template <bool W>
__device__ void cq2_leaf(const ig_cut2& I, const Box2d& root, int leaf, int D, bool vol, Cq2Sink<W>& sk) {
  Box2d cell = root;
  for (int d = 0; d <= D; ++d) {
    if (d > 0) {
      const int kd = (leaf >> (2 * (D - d))) & 3;
      const V2d m = cell.center();
      Box2d k;
      switch (kd) {
        case 0: k = {cell.lo, m}; break;
        case 1: k = {{m.x, cell.lo.y}, {cell.hi.x, m.y}}; break;
        case 2: k = {m, cell.hi}; break;
        default: k = {{cell.lo.x, m.y}, {m.x, cell.hi.y}}; break;
      }
      cell = k;
    }
    const int cls = cq2_classify(I, cell);
    if (cls == 1) return;
    if (cls == 0) {
      if (vol && (leaf & ((1 << (2 * (D - d))) - 1)) == 0) cq2_tensor<W>(I, cell, sk);
      return;
    }
    if (d == D) {
      Poly2 polys[2];
      const int np = cq2_leaf_polygons(I, cell, polys);
      for (int i = 0; i < np; ++i) {
        cq2_refine_chords(I, cell, polys[i]);
        if (vol) {
          const V2d ctr = cq2_centroid(polys[i]);
          for (int k = 0; k < polys[i].n; ++k)
            cq2_triangle<W>(I, ctr, polys[i].v[k], polys[i].v[(k + 1) % polys[i].n], sk);
        } else {
          cq2_interface<W>(I, polys[i], sk);
        }
      }
      return;
    }
  }
}

// side_rule: nseg = 2^depth segments of box side `side`.
template <bool W>
__device__ void cq2_side(const ig_cut2& I, const Box2d& cell, int side, Cq2Sink<W>& sk) {
  const V2d a = cell.corner(side);
  const V2d b = cell.corner((side + 1) % 4);
  const int q = I.gauss_order;
  const double* gn = I.gauss_q;
  const double* gw = I.gauss_q + q;
  const int nseg = 1 << I.depth;
  auto add_segment = [&](V2d p0, V2d p1) {
    const V2d d = v2sub(p1, p0);
    const double len = v2norm(d);
    if (!(len > 0.0)) return;
    for (int g = 0; g < q; ++g) {
      const double t = 0.5 * (gn[g] + 1.0);
      sk.put(v2add(p0, v2mul(t, d)), 0.5 * gw[g] * len);
    }
  };
  for (int s = 0; s < nseg; ++s) {
    const double t0 = static_cast<double>(s) / nseg;
    const double t1 = static_cast<double>(s + 1) / nseg;
    const V2d p0 = v2add(a, v2mul(t0, v2sub(b, a)));
    const V2d p1 = v2add(a, v2mul(t1, v2sub(b, a)));
    const double f0 = cq2_ls(I, p0), f1 = cq2_ls(I, p1);
    const bool in0 = f0 >= 0.0, in1 = f1 >= 0.0;
    if (in0 && in1) {
      add_segment(p0, p1);
    } else if (in0 != in1) {
      const V2d x = cq2_isect(I, p0, p1);
      if (in0)
        add_segment(p0, x);
      else
        add_segment(x, p1);
    }
  }
}

// Points of element e: [volume points | interface points | side points].
// npt[3 e + k]: counts (W = false); off: per-element point offsets (W = true).
template <bool W>
__global__ void __launch_bounds__(kCq2Threads) k_cq2_points(ig_cut2 I0, const int64_t* __restrict__ off,
                                                           int64_t* npt, double* pts, const double* eprog,
                                                           const int* elen) {
  const int e = blockIdx.x;
  if (e >= I0.n_elem) return;
  const Box2d root{{I0.lo[2 * e], I0.lo[2 * e + 1]}, {I0.hi[2 * e], I0.hi[2 * e + 1]}};
  // The element's specialised level-set program (cutquad.cuh k_ls_specialize).
  ig_cut2 I = I0;
  I.prog = eprog + static_cast<int64_t>(e) * I0.prog_len;
  I.prog_len = elen[e];
  const bool cut = I.cut[e] != 0;
  const int D = I.depth;
  const int nleaf = 1 << (2 * D);
  const int l0 = static_cast<int>(static_cast<int64_t>(nleaf) * threadIdx.x / blockDim.x);
  const int l1 = static_cast<int>(static_cast<int64_t>(nleaf) * (threadIdx.x + 1) / blockDim.x);
  __shared__ int sv[kCq2Threads], sb[kCq2Threads];
  Cq2Sink<false> cv{nullptr, 0}, cb{nullptr, 0};
  if (cut) {
    for (int l = l0; l < l1; ++l) {
      cq2_leaf<false>(I, root, l, D, true, cv);
      cq2_leaf<false>(I, root, l, D, false, cb);
    }
  } else if (threadIdx.x == 0) {
    cq2_tensor<false>(I, root, cv);  // volume_rule on an Inside element
  }
  sv[threadIdx.x] = cv.n;
  sb[threadIdx.x] = cb.n;
  __syncthreads();
  int nside = 0;
  if (threadIdx.x == 0) {
    Cq2Sink<false> cs{nullptr, 0};
    for (int k = 0; k < 4; ++k)
      if ((I.sides[e] >> k) & 1) cq2_side<false>(I, root, k, cs);
    nside = cs.n;
  }
  if (!W) {
    if (threadIdx.x == 0) {
      int64_t tv = 0, tb = 0;
      for (int k = 0; k < blockDim.x; ++k) {
        tv += sv[k];
        tb += sb[k];
      }
      npt[3 * e] = tv;
      npt[3 * e + 1] = tb;
      npt[3 * e + 2] = nside;
    }
    return;
  }
  int bv = 0, bb = 0, tv = 0, tb = 0;
  for (int k = 0; k < static_cast<int>(blockDim.x); ++k) {
    if (k < static_cast<int>(threadIdx.x)) {
      bv += sv[k];
      bb += sb[k];
    }
    tv += sv[k];
    tb += sb[k];
  }
  double* base = pts + 4 * off[e];
  Cq2Sink<true> wv{base, bv}, wb{base, tv + bb};
  if (cut) {
    for (int l = l0; l < l1; ++l) cq2_leaf<true>(I, root, l, D, true, wv);
    for (int l = l0; l < l1; ++l) cq2_leaf<true>(I, root, l, D, false, wb);
  } else if (threadIdx.x == 0) {
    cq2_tensor<true>(I, root, wv);
  }
  if (threadIdx.x == 0) {
    Cq2Sink<true> ws{base, tv + tb};
    for (int k = 0; k < 4; ++k)
      if ((I.sides[e] >> k) & 1) cq2_side<true>(I, root, k, ws);
  }
}

// Element matrices: volume points add w (gx_i gx_j + gy_i gy_j) and w f val_i;
// interface and side points add (w beta) val_i val_j (assembly.cpp:66-131).
// spline::bernstein (host/spline_linalg.cpp)
__device__ __forceinline__ void cq2_bernstein(int p, double x, double* val, double* der) {
  double lower[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  val[0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    if (j == p)
      for (int k = 0; k < p; ++k) lower[k] = val[k];
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      const double temp = val[r];
      val[r] = saved + (1.0 - x) * temp;
      saved = x * temp;
    }
    val[j] = saved;
  }
  der[0] = -p * lower[0];
  for (int r = 1; r < p; ++r) der[r] = p * (lower[r - 1] - lower[r]);
  der[p] = p * lower[p - 1];
}

template <int NL>
__global__ void __launch_bounds__(kCq2Threads) k_cq2_integrate(ig_cut2 I, const int64_t* __restrict__ off,
                                                              const int64_t* __restrict__ npt,
                                                              const double* __restrict__ pts, double* Kout,
                                                              double* Fout, double* vout) {
  constexpr int PER = (NL * NL + kCq2Threads - 1) / kCq2Threads;
  const int e = blockIdx.x;
  if (e >= I.n_elem) return;
  const int p = I.p, q = p + 1;
  const double* Rx = I.ext[0] + static_cast<int64_t>(I.cls[2 * e]) * q * q;
  const double* Ry = I.ext[1] + static_cast<int64_t>(I.cls[2 * e + 1]) * q * q;
  const double lo0 = I.lo[2 * e], lo1 = I.lo[2 * e + 1];
  const double sx = I.hi[2 * e] - lo0, sy = I.hi[2 * e + 1] - lo1;
  __shared__ double Em[NL * NL];  // extraction2: E(r = jb q + ia, jy q + jx) = Rx(ia, jx) Ry(jb, jy)
  __shared__ double bas[kCq2Batch][3][NL];
  __shared__ double bb[kCq2Batch][3][NL];
  for (int t = threadIdx.x; t < NL * NL; t += blockDim.x) {
    const int r = t / NL, k = t % NL;
    const int jb = r / q, ia = r % q, jy = k / q, jx = k % q;
    Em[r * NL + k] = Rx[jx * q + ia] * Ry[jy * q + jb];
  }
  int ei[PER], ej[PER];
  double acc[PER];
#pragma unroll
  for (int s = 0; s < PER; ++s) {
    const int idx = threadIdx.x + s * kCq2Threads;
    acc[s] = 0.0;
    ei[s] = idx < NL * NL ? idx / NL : -1;
    ej[s] = idx < NL * NL ? idx % NL : -1;
  }
  double facc = 0.0, vol = 0.0;
  const int64_t nvol = npt[3 * e], ntot = npt[3 * e] + npt[3 * e + 1] + npt[3 * e + 2];
  const double* P = pts + 4 * off[e];
  __syncthreads();
  for (int64_t b0 = 0; b0 < ntot; b0 += kCq2Batch) {
    const int nb = static_cast<int>(ntot - b0 < kCq2Batch ? ntot - b0 : kCq2Batch);
    // Bernstein products per point (bval, bgx, bgy over k = jy q + jx)
    for (int t = threadIdx.x; t < nb; t += blockDim.x) {
      const double* pt = P + 4 * (b0 + t);
      const double u = (pt[0] - lo0) / sx, v = (pt[1] - lo1) / sy;
      double bu[kCq2MaxQ], du[kCq2MaxQ], bv[kCq2MaxQ], dv[kCq2MaxQ];
      auto bern = [&](double x, double* val, double* der) {  // spline::bernstein
        double lower[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        val[0] = 1.0;
        for (int j = 1; j <= p; ++j) {
          if (j == p)
            for (int k = 0; k < p; ++k) lower[k] = val[k];
          double saved = 0.0;
          for (int r = 0; r < j; ++r) {
            const double temp = val[r];
            val[r] = saved + (1.0 - x) * temp;
            saved = x * temp;
          }
          val[j] = saved;
        }
        der[0] = -p * lower[0];
        for (int r = 1; r < p; ++r) der[r] = p * (lower[r - 1] - lower[r]);
        der[p] = p * lower[p - 1];
      };
      bern(u, bu, du);
      bern(v, bv, dv);
      for (int jy = 0; jy < q; ++jy)
        for (int jx = 0; jx < q; ++jx) {
          const int k = jy * q + jx;
          bb[t][0][k] = bu[jx] * bv[jy];
          bb[t][1][k] = du[jx] * bv[jy];
          bb[t][2][k] = bu[jx] * dv[jy];
        }
    }
    __syncthreads();
    // val, gx, gy per point and local function (ascending k sums)
    for (int t = threadIdx.x; t < nb * NL; t += blockDim.x) {
      const int pi = t / NL, r = t % NL;
      double a = 0.0, b = 0.0, c = 0.0;
      for (int k = 0; k < NL; ++k) {
        a += Em[r * NL + k] * bb[pi][0][k];
        b += Em[r * NL + k] * bb[pi][1][k];
        c += Em[r * NL + k] * bb[pi][2][k];
      }
      bas[pi][0][r] = a;
      bas[pi][1][r] = b / sx;
      bas[pi][2][r] = c / sy;
    }
    __syncthreads();
    for (int k = 0; k < nb; ++k) {
      const int64_t g = b0 + k;
      const double w = P[4 * g + 2];
      if (g < nvol) {
#pragma unroll
        for (int s = 0; s < PER; ++s)
          if (ei[s] >= 0)
            acc[s] += w * (bas[k][1][ei[s]] * bas[k][1][ej[s]] + bas[k][2][ei[s]] * bas[k][2][ej[s]]);
        if (threadIdx.x < NL && I.f != 0.0) facc += w * I.f * bas[k][0][threadIdx.x];
        if (threadIdx.x == 0) vol += w;
      } else {
        const double wb = w * I.beta;
#pragma unroll
        for (int s = 0; s < PER; ++s)
          if (ei[s] >= 0) acc[s] += wb * (bas[k][0][ei[s]] * bas[k][0][ej[s]]);
      }
    }
    __syncthreads();
  }
  double* K = Kout + static_cast<int64_t>(e) * NL * NL;
#pragma unroll
  for (int s = 0; s < PER; ++s)
    if (ei[s] >= 0) K[ei[s] * NL + ej[s]] = acc[s];
  if (threadIdx.x < NL) Fout[static_cast<int64_t>(e) * NL + threadIdx.x] = facc;
  if (threadIdx.x == 0 && vout) vout[e] = vol;
}

// ------------------------------------------------------------ THB -------
// Element integration of a THB element (host/thb.cpp assemble_g): the
// element's truncated functions are `nl` rows of Bernstein coefficients
// (eval_el), every element is integrated with the ig_cut2 point rules; K is
// the full nl x nl element matrix (shared-memory accumulators, one owner per
// entry), F nl values.  Elements with more than kThbMaxRows rows set *bad.
constexpr int kThbMaxRows = 32;
constexpr int kThbBatch = 16;
__global__ void __launch_bounds__(kCq2Threads) k_thb_integrate(ig_cut2 I, const int32_t* __restrict__ erow_ptr,
                                                              const double* __restrict__ Eall,
                                                              const int64_t* __restrict__ off,
                                                              const int64_t* __restrict__ npt,
                                                              const double* __restrict__ pts,
                                                              const int64_t* __restrict__ koff, double* Kout,
                                                              double* Fout, int* bad) {
  const int e = blockIdx.x;
  if (e >= I.n_elem) return;
  const int p = I.p, q = p + 1, nb = q * q;
  const int nl = erow_ptr[e + 1] - erow_ptr[e];
  if (nl > kThbMaxRows) {
    if (threadIdx.x == 0) atomicAdd(bad, 1);
    return;
  }
  const double lo0 = I.lo[2 * e], lo1 = I.lo[2 * e + 1];
  const double sx = I.hi[2 * e] - lo0, sy = I.hi[2 * e + 1] - lo1;
  __shared__ double Es[kThbMaxRows * kCq2MaxQ * kCq2MaxQ];
  __shared__ double Ks[kThbMaxRows * kThbMaxRows];
  __shared__ double bb[kThbBatch][3][kCq2MaxQ * kCq2MaxQ];
  __shared__ double bas[kThbBatch][3][kThbMaxRows];
  const double* E = Eall + static_cast<int64_t>(erow_ptr[e]) * nb;
  for (int t = threadIdx.x; t < nl * nb; t += blockDim.x) Es[t] = E[t];
  for (int t = threadIdx.x; t < nl * nl; t += blockDim.x) Ks[t] = 0.0;
  double facc = 0.0;
  const int64_t nvol = npt[3 * e], ntot = npt[3 * e] + npt[3 * e + 1] + npt[3 * e + 2];
  const double* P = pts + 4 * off[e];
  __syncthreads();
  for (int64_t b0 = 0; b0 < ntot; b0 += kThbBatch) {
    const int nbt = static_cast<int>(ntot - b0 < kThbBatch ? ntot - b0 : kThbBatch);
    for (int t = threadIdx.x; t < nbt; t += blockDim.x) {
      const double* pt = P + 4 * (b0 + t);
      const double u = (pt[0] - lo0) / sx, v = (pt[1] - lo1) / sy;
      double bu[kCq2MaxQ], du[kCq2MaxQ], bv[kCq2MaxQ], dv[kCq2MaxQ];
      cq2_bernstein(p, u, bu, du);
      cq2_bernstein(p, v, bv, dv);
      for (int jy = 0; jy < q; ++jy)
        for (int jx = 0; jx < q; ++jx) {
          const int k = jy * q + jx;
          bb[t][0][k] = bu[jx] * bv[jy];
          bb[t][1][k] = du[jx] * bv[jy];
          bb[t][2][k] = bu[jx] * dv[jy];
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nbt * nl; t += blockDim.x) {
      const int pi = t / nl, r = t % nl;
      double a = 0.0, b = 0.0, c = 0.0;
      for (int k = 0; k < nb; ++k) {
        a += Es[r * nb + k] * bb[pi][0][k];
        b += Es[r * nb + k] * bb[pi][1][k];
        c += Es[r * nb + k] * bb[pi][2][k];
      }
      bas[pi][0][r] = a;
      bas[pi][1][r] = b / sx;
      bas[pi][2][r] = c / sy;
    }
    __syncthreads();
    for (int k = 0; k < nbt; ++k) {
      const int64_t g = b0 + k;
      const double w = P[4 * g + 2];
      if (g < nvol) {
        for (int t = threadIdx.x; t < nl * nl; t += blockDim.x) {
          const int i = t / nl, j = t % nl;
          Ks[t] += w * (bas[k][1][i] * bas[k][1][j] + bas[k][2][i] * bas[k][2][j]);
        }
        if (threadIdx.x < nl && I.f != 0.0) facc += w * I.f * bas[k][0][threadIdx.x];
      } else {
        const double wb = w * I.beta;
        for (int t = threadIdx.x; t < nl * nl; t += blockDim.x) {
          const int i = t / nl, j = t % nl;
          Ks[t] += wb * (bas[k][0][i] * bas[k][0][j]);
        }
      }
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < nl * nl; t += blockDim.x) Kout[koff[e] + t] = Ks[t];
  if (threadIdx.x < nl) Fout[erow_ptr[e] + threadIdx.x] = facc;
}

// Row gather of the THB assembly (assemble_g): DOF a walks its support in
// ascending element order, adds its element row's nonzero entries to a list in
// first-appearance order (exact zeros dropped), b_a sums its F entries; the
// list is then sorted by column.  FILL = false: counts; FILL = true: CSR.
constexpr int kThbMaxCols = 160;
template <bool FILL>
__global__ void __launch_bounds__(128) k_thb_rows(int32_t n, const int64_t* __restrict__ supp_ptr,
                                                 const int32_t* __restrict__ supp_el,
                                                 const int32_t* __restrict__ supp_li,
                                                 const int32_t* __restrict__ erow_ptr,
                                                 const int32_t* __restrict__ anchors,
                                                 const int64_t* __restrict__ koff, const double* __restrict__ K,
                                                 const double* __restrict__ F, int32_t* cnt, const int64_t* rowoff,
                                                 int32_t* col, double* val, double* b, int* bad) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  int32_t cs[kThbMaxCols];
  double vs[kThbMaxCols];
  int m = 0;
  double bsum = 0.0;
  for (int64_t s = supp_ptr[a]; s < supp_ptr[a + 1]; ++s) {
    const int e = supp_el[s], li = supp_li[s];
    const int r0 = erow_ptr[e], nl = erow_ptr[e + 1] - r0;
    bsum += F[r0 + li];
    const double* Ke = K + koff[e] + static_cast<int64_t>(li) * nl;
    for (int lj = 0; lj < nl; ++lj) {
      const double v = Ke[lj];
      if (v == 0.0) continue;
      const int32_t c = anchors[r0 + lj];
      int k = 0;
      while (k < m && cs[k] != c) ++k;
      if (k < m) {
        vs[k] = vs[k] + v;
      } else if (m < kThbMaxCols) {
        cs[m] = c;
        vs[m] = v;
        ++m;
      } else {
        atomicAdd(bad, 1);
      }
    }
  }
  if (!FILL) {
    cnt[a] = m;
    return;
  }
  for (int i = 1; i < m; ++i) {  // insertion sort by column (columns are distinct)
    const int32_t c = cs[i];
    const double v = vs[i];
    int j = i - 1;
    while (j >= 0 && cs[j] > c) {
      cs[j + 1] = cs[j];
      vs[j + 1] = vs[j];
      --j;
    }
    cs[j + 1] = c;
    vs[j + 1] = v;
  }
  const int64_t o = rowoff[a];
  for (int k = 0; k < m; ++k) {
    col[o + k] = cs[k];
    val[o + k] = vs[k];
  }
  b[a] = bsum;
}

}  // namespace igk
