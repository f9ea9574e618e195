// cutquad.cuh — cut-element quadrature of the 3D uniform B-spline case on the
// device (ig_cut3, ig_gpu.h).  The host's element3(cut = true)
// (host/assembly.cpp: recurse3, cut_leaf3, clip_tet, tet_points, tri_points,
// add_box, add_vol_point, add_surf_point, finish3) restated operation for
// operation, so every element matrix is bit-identical (-fmad=false here,
// -ffp-contract=off there).  Three kernels, one CTA per cut element:
//   k_cq_prims<false>  counts the primitives of every element (octree walk:
//                      classify_cell per cell, cut leaves -> clipped Kuhn
//                      tetrahedra + interface triangles, inside cells -> boxes);
//   k_cq_prims<true>   writes them in the host's depth-first order (thread t
//                      owns a contiguous range of leaves; a block scan over
//                      the per-thread counts gives every primitive its slot);
//   k_cq_integrate     expands the primitives into quadrature points in
//                      batches of 32, evaluates the 27 basis functions per
//                      point cooperatively in shared memory, and every thread
//                      accumulates its own K / F entries over the points in
//                      order -- the host's summation order per entry.
#pragma once

#include <cstdint>

#include "ig_gpu.h"

namespace igk {

constexpr int kCqThreads = 128;
constexpr int kCqMaxQ = 4;          // p <= 3
constexpr int kCqPrim = 14;         // doubles per primitive: type, npts, 12 coordinates
constexpr int kCqBatch = 32;        // points per integration batch

// ------------------------------------------------------------ level set ----
__device__ __forceinline__ double cq_min(double a, double b) { return (b < a) ? b : a; }  // std::min
__device__ __forceinline__ double cq_max(double a, double b) { return (a < b) ? b : a; }  // std::max

__device__ double ls_eval(const double* P, int len, const double* p) {
  double st[16];
  int sp = 0;
  for (int k = 0; k < len;) {
    const int op = static_cast<int>(P[k]);
    switch (op) {
      case 0: st[sp++] = P[k + 1]; k += 2; break;
      case 1: {
        const int dim = static_cast<int>(P[k + 5]);
        st[sp++] = dim == 2 ? P[k + 1] * p[0] + P[k + 2] * p[1] + P[k + 4]
                            : P[k + 1] * p[0] + P[k + 2] * p[1] + P[k + 3] * p[2] + P[k + 4];
        k += 6;
        break;
      }
      case 2: {
        const int dim = static_cast<int>(P[k + 5]);
        const double dx = p[0] - P[k + 1], dy = p[1] - P[k + 2];
        if (dim == 2) {
          st[sp++] = P[k + 4] - sqrt(dx * dx + dy * dy);
        } else {
          const double dz = p[2] - P[k + 3];
          st[sp++] = P[k + 4] - sqrt(dx * dx + dy * dy + dz * dz);
        }
        k += 6;
        break;
      }
      case 3: {
        const double* lo = P + k + 1;
        const double* hi = P + k + 4;
        double v = cq_min(cq_min(p[0] - lo[0], hi[0] - p[0]), cq_min(p[1] - lo[1], hi[1] - p[1]));
        if (static_cast<int>(P[k + 7]) == 3) v = cq_min(v, cq_min(p[2] - lo[2], hi[2] - p[2]));
        st[sp++] = v;
        k += 8;
        break;
      }
      case 4: --sp; st[sp - 1] = cq_min(st[sp - 1], st[sp]); k += 1; break;
      case 5: --sp; st[sp - 1] = cq_max(st[sp - 1], st[sp]); k += 1; break;
      default: st[sp - 1] = -st[sp - 1]; k += 1; break;
    }
  }
  return st[0];
}

// LsNode::bounds over an axis box (every node of a device program has one).
__device__ void ls_bounds(const double* P, int len, const double* lo, const double* hi, int dim,
                          double& a, double& b) {
  double sa[16], sb[16];
  int sp = 0;
  for (int k = 0; k < len;) {
    const int op = static_cast<int>(P[k]);
    switch (op) {
      case 0: sa[sp] = sb[sp] = P[k + 1]; ++sp; k += 2; break;
      case 1: {
        const int nd = static_cast<int>(P[k + 5]);
        double x = P[k + 4], y = P[k + 4];
        for (int d = 0; d < nd; ++d) {
          const double u = P[k + 1 + d] * lo[d], v = P[k + 1 + d] * hi[d];
          x += cq_min(u, v);
          y += cq_max(u, v);
        }
        sa[sp] = x;
        sb[sp] = y;
        ++sp;
        k += 6;
        break;
      }
      case 2: {
        const int nd = static_cast<int>(P[k + 5]);
        double dmin2 = 0, dmax2 = 0;
        for (int d = 0; d < nd; ++d) {
          const double l = lo[d] - P[k + 1 + d], h = hi[d] - P[k + 1 + d];
          const double nr = (l > 0) ? l : (h < 0 ? -h : 0.0);
          const double fr = cq_max(fabs(l), fabs(h));
          dmin2 += nr * nr;
          dmax2 += fr * fr;
        }
        sa[sp] = P[k + 4] - sqrt(dmax2);
        sb[sp] = P[k + 4] - sqrt(dmin2);
        ++sp;
        k += 6;
        break;
      }
      case 3: {
        const int nd = static_cast<int>(P[k + 7]);
        double x = 1e300, y = 1e300;
        for (int d = 0; d < nd; ++d) {
          x = cq_min(x, cq_min(lo[d] - P[k + 1 + d], P[k + 4 + d] - hi[d]));
          y = cq_min(y, cq_min(hi[d] - P[k + 1 + d], P[k + 4 + d] - lo[d]));
        }
        sa[sp] = x;
        sb[sp] = y;
        ++sp;
        k += 8;
        break;
      }
      case 4:
        --sp;
        sa[sp - 1] = cq_min(sa[sp - 1], sa[sp]);
        sb[sp - 1] = cq_min(sb[sp - 1], sb[sp]);
        k += 1;
        break;
      case 5:
        --sp;
        sa[sp - 1] = cq_max(sa[sp - 1], sa[sp]);
        sb[sp - 1] = cq_max(sb[sp - 1], sb[sp]);
        k += 1;
        break;
      default: {
        const double x = -sb[sp - 1], y = -sa[sp - 1];
        sa[sp - 1] = x;
        sb[sp - 1] = y;
        k += 1;
        break;
      }
    }
  }
  a = sa[0];
  b = sb[0];
}

// The program specialised to an axis box: a min (max) node whose child B
// lies, over the whole box, strictly above (below) its other child A by more
// than a rounding margin is replaced by A -- min(a, b) returns a bit for bit
// wherever b > a, so every value (and every ls_bounds interval of a sub-box)
// the specialised program produces inside the box equals the full program's.
// A union of 64 discs (C3) keeps the one or two discs near an element.
// Returns the specialised length (<= len) written to out.
__device__ int ls_specialize(const double* P, int len, const double* lo, const double* hi, int dim,
                             double* out) {
  double sa[16], sb[16];
  int ss[16];
  int sp = 0, o = 0;
  double scale = 0.0;
  for (int d = 0; d < dim; ++d) scale = cq_max(scale, fabs(lo[d]) + fabs(hi[d]));
  const double m = 1e-9 * (1.0 + scale);
  for (int k = 0; k < len;) {
    const int op = static_cast<int>(P[k]);
    if (op <= 3) {  // primitive: copy, and its interval over the box
      const int sz = op == 0 ? 2 : (op == 3 ? 8 : 6);
      ls_bounds(P + k, sz, lo, hi, dim, sa[sp], sb[sp]);
      ss[sp++] = o;
      for (int t = 0; t < sz; ++t) out[o++] = P[k + t];
      k += sz;
      continue;
    }
    if (op == 6) {  // negation
      const double a = -sb[sp - 1], b = -sa[sp - 1];
      sa[sp - 1] = a;
      sb[sp - 1] = b;
      out[o++] = 6.0;
      k += 1;
      continue;
    }
    --sp;  // min / max of A = [sp - 1] and B = [sp] (B's code follows A's)
    const bool mn = op == 4;
    const bool dropB = mn ? (sa[sp] > sb[sp - 1] + m) : (sb[sp] < sa[sp - 1] - m);
    const bool dropA = mn ? (sa[sp - 1] > sb[sp] + m) : (sb[sp - 1] < sa[sp] - m);
    if (dropB) {
      o = ss[sp];
    } else if (dropA) {
      const int n = o - ss[sp];
      for (int t = 0; t < n; ++t) out[ss[sp - 1] + t] = out[ss[sp] + t];
      o = ss[sp - 1] + n;
      sa[sp - 1] = sa[sp];
      sb[sp - 1] = sb[sp];
    } else {
      sa[sp - 1] = mn ? cq_min(sa[sp - 1], sa[sp]) : cq_max(sa[sp - 1], sa[sp]);
      sb[sp - 1] = mn ? cq_min(sb[sp - 1], sb[sp]) : cq_max(sb[sp - 1], sb[sp]);
      out[o++] = static_cast<double>(op);
    }
    k += 1;
  }
  return o;
}

// classify_cell (host/levelset.cpp): 0 Inside, 1 Outside, 2 Cut.
__device__ int cq_classify(const double* P, int len, const double* lo, const double* hi, int depth) {
  double vmin, vmax;
  ls_bounds(P, len, lo, hi, 3, vmin, vmax);
  double scale = 0;
  for (int k = 0; k < 3; ++k) scale = cq_max(scale, fabs(lo[k]) + fabs(hi[k]));
  const double margin = 1e-9 * (1.0 + scale);
  if (vmin > margin) return 0;
  if (vmax < -margin) return 1;
  const int n = (1 << depth) + 1;
  bool any_in = false, any_out = false;
  double d[3];
  for (int k = 0; k < 3; ++k) d[k] = (hi[k] - lo[k]) / static_cast<double>(n - 1);
  double p[3];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        p[0] = lo[0] + i * d[0];
        p[1] = lo[1] + j * d[1];
        p[2] = lo[2] + k * d[2];
        if (ls_eval(P, len, p) >= 0.0)
          any_in = true;
        else
          any_out = true;
        if (any_in && any_out) return 2;
      }
  return any_in ? 0 : 1;
}

// intersect_edge (host/levelset.cpp): bisection to tol.
__device__ void cq_isect(const double* P, int len, const double* p0, const double* p1, double tol, double* out) {
  double f0 = ls_eval(P, len, p0);
  double t0 = 0.0, t1 = 1.0;
  double q[3];
  while (t1 - t0 > tol) {
    const double tm = 0.5 * (t0 + t1);
    for (int k = 0; k < 3; ++k) q[k] = p0[k] + tm * (p1[k] - p0[k]);
    const double fm = ls_eval(P, len, q);
    if (f0 * fm <= 0.0) {
      t1 = tm;
    } else {
      t0 = tm;
      f0 = fm;
    }
  }
  const double tm = 0.5 * (t0 + t1);
  for (int k = 0; k < 3; ++k) out[k] = p0[k] + tm * (p1[k] - p0[k]);
}

// ------------------------------------------------------------ primitives ---
// Kuhn decomposition (host kKuhn): 6 tetrahedra sharing the diagonal 0 -> 7.
__constant__ int kCqKuhn[6][4] = {{0, 1, 3, 7}, {0, 1, 5, 7}, {0, 2, 3, 7}, {0, 2, 6, 7}, {0, 4, 5, 7}, {0, 4, 6, 7}};

// Emits primitives (or only counts them with W = false) in the host order.
template <bool W>
struct CqSink {
  double* out;
  int n;
  __device__ void put(int type, const double* c, int nc) {
    if (W) {
      double* o = out + static_cast<int64_t>(n) * kCqPrim;
      o[0] = type;
      o[1] = 0.0;
      for (int k = 0; k < 12; ++k) o[2 + k] = k < nc ? c[k] : 0.0;
    }
    ++n;
  }
};

struct CqCtx {
  const ig_cut3* in;
  const double* elo;   // element lower corner (physical)
  const double* prog;  // level-set program (the element's specialisation)
  int prog_len;
};

__device__ __forceinline__ void cq_ref(const CqCtx& c, const double* x, double* u) {
  for (int k = 0; k < 3; ++k) u[k] = (x[k] - c.elo[k]) / c.in->h[k];
}

template <bool W>
__device__ void cq_clip_tet(const CqCtx& c, const double x[4][3], const double f[4], CqSink<W>& sk) {
  int in[4], out[4], ni = 0, no = 0;
  for (int k = 0; k < 4; ++k) {
    if (f[k] >= 0.0)
      in[ni++] = k;
    else
      out[no++] = k;
  }
  if (ni == 0) return;
  const ig_cut3& I = *c.in;
  auto cross = [&](int a, int b, double* u) {
    double r[3];
    if (W) cq_isect(c.prog, c.prog_len, x[a], x[b], I.edge_tol, r);
    else r[0] = r[1] = r[2] = 0.0;
    cq_ref(c, r, u);
  };
  double buf[12];
  if (ni == 4) {
    for (int k = 0; k < 4; ++k) cq_ref(c, x[k], buf + 3 * k);
    sk.put(1, buf, 12);
    return;
  }
  if (ni == 1) {
    const int a = in[0];
    double Pp[3][3];
    for (int k = 0; k < 3; ++k) cross(a, out[k], Pp[k]);
    cq_ref(c, x[a], buf);
    for (int k = 0; k < 3; ++k)
      for (int d = 0; d < 3; ++d) buf[3 * (k + 1) + d] = Pp[k][d];
    sk.put(1, buf, 12);
    for (int k = 0; k < 3; ++k)
      for (int d = 0; d < 3; ++d) buf[3 * k + d] = Pp[k][d];
    sk.put(2, buf, 9);
    return;
  }
  if (ni == 3) {
    const int a = out[0];
    double bot[3][3], top[3][3];
    for (int k = 0; k < 3; ++k) {
      cq_ref(c, x[in[k]], bot[k]);
      cross(in[k], a, top[k]);
    }
    const double* Pr[3][4] = {{bot[0], bot[1], bot[2], top[0]},
                              {bot[1], bot[2], top[0], top[1]},
                              {bot[2], top[0], top[1], top[2]}};
    for (int t = 0; t < 3; ++t) {
      for (int k = 0; k < 4; ++k)
        for (int d = 0; d < 3; ++d) buf[3 * k + d] = Pr[t][k][d];
      sk.put(1, buf, 12);
    }
    for (int k = 0; k < 3; ++k)
      for (int d = 0; d < 3; ++d) buf[3 * k + d] = top[k][d];
    sk.put(2, buf, 9);
    return;
  }
  const int a = in[0], b = in[1];
  double pa[3], pb[3], xa0[3], xa1[3], xb0[3], xb1[3];
  cq_ref(c, x[a], pa);
  cq_ref(c, x[b], pb);
  cross(a, out[0], xa0);
  cross(a, out[1], xa1);
  cross(b, out[0], xb0);
  cross(b, out[1], xb1);
  const double* Pr[3][4] = {{pa, xa0, xa1, pb}, {xa0, xa1, pb, xb0}, {xa1, pb, xb0, xb1}};
  for (int t = 0; t < 3; ++t) {
    for (int k = 0; k < 4; ++k)
      for (int d = 0; d < 3; ++d) buf[3 * k + d] = Pr[t][k][d];
    sk.put(1, buf, 12);
  }
  for (int d = 0; d < 3; ++d) {
    buf[d] = xa0[d];
    buf[3 + d] = xb0[d];
    buf[6 + d] = xb1[d];
  }
  sk.put(2, buf, 9);
  for (int d = 0; d < 3; ++d) {
    buf[d] = xa0[d];
    buf[3 + d] = xb1[d];
    buf[6 + d] = xa1[d];
  }
  sk.put(2, buf, 9);
}

template <bool W>
__device__ void cq_cut_leaf(const CqCtx& c, const double* lo, const double* hi, CqSink<W>& sk) {
  const ig_cut3& I = *c.in;
  double x[8][3], f[8];
  for (int k = 0; k < 8; ++k) {
    x[k][0] = (k & 1) ? hi[0] : lo[0];
    x[k][1] = (k & 2) ? hi[1] : lo[1];
    x[k][2] = (k & 4) ? hi[2] : lo[2];
    f[k] = ls_eval(c.prog, c.prog_len, x[k]);
  }
  for (int t = 0; t < 6; ++t) {
    double tx[4][3], tf[4];
    for (int k = 0; k < 4; ++k) {
      for (int d = 0; d < 3; ++d) tx[k][d] = x[kCqKuhn[t][k]][d];
      tf[k] = f[kCqKuhn[t][k]];
    }
    cq_clip_tet<W>(c, tx, tf, sk);
  }
}

// The primitives of leaf `leaf` (digits k_1 .. k_D, k_1 most significant) in
// the host's recurse3 order: the cell at each level is classified; an Inside
// cell emits its box once (from its first leaf), Outside nothing, Cut
// recurses; a Cut leaf emits its clipped tetrahedra / triangles.
template <bool W>
__device__ void cq_leaf(const CqCtx& c, int leaf, int D, CqSink<W>& sk) {
  const ig_cut3& I = *c.in;
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) {
    lo[k] = c.elo[k];
    hi[k] = c.elo[k] + I.h[k];
  }
  for (int d = 0; d <= D; ++d) {
    if (d > 0) {  // the child of the current cell along digit k_d
      const int kd = (leaf >> (3 * (D - d))) & 7;
      double mid[3];
      for (int k = 0; k < 3; ++k) mid[k] = 0.5 * (lo[k] + hi[k]);
      for (int k = 0; k < 3; ++k) {
        const bool up = (kd >> k) & 1;
        if (up)
          lo[k] = mid[k];
        else
          hi[k] = mid[k];
      }
    }
    const int cls = cq_classify(c.prog, c.prog_len, lo, hi, I.classify_depth);
    if (cls == 1) return;
    if (cls == 0) {
      const int rest = leaf & ((1 << (3 * (D - d))) - 1);
      if (rest == 0) {
        double b[6];
        cq_ref(c, lo, b);
        cq_ref(c, hi, b + 3);
        sk.put(0, b, 6);
      }
      return;
    }
    if (d == D) {
      cq_cut_leaf<W>(c, lo, hi, sk);
      return;
    }
  }
}

// Counts (W = false: count[e]) or writes (W = true: from prim + off[e])
// the primitives of every cut element; one CTA per element.
// Per-element specialised programs (ls_specialize), one thread per element:
// element e's program at out + e * len (len = the full program's length, an
// upper bound), its length in olen[e].  3D: the cell [lo, lo + h]; 2D: the
// box [lo, hi]; both grown by half the cell size on every side (every point
// the element's leaves, chords and bisections evaluate lies inside).
__global__ void k_ls_specialize(const double* __restrict__ P, int len, int n, int dim, const double* __restrict__ elo,
                                const double* __restrict__ ehi, const double* h3, double* out, int* olen) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  for (int k = 0; k < dim; ++k) {
    const double a = elo[static_cast<int64_t>(dim) * e + k];
    const double b = ehi ? ehi[static_cast<int64_t>(dim) * e + k] : a + h3[k];
    const double g = 0.5 * (b - a);
    lo[k] = a - g;
    hi[k] = b + g;
  }
  olen[e] = ls_specialize(P, len, lo, hi, dim, out + static_cast<int64_t>(e) * len);
}

template <bool W>
__global__ void __launch_bounds__(kCqThreads) k_cq_prims(ig_cut3 I, const int64_t* __restrict__ off,
                                                        int64_t* count, double* prim, const double* eprog,
                                                        const int* elen) {
  const int e = blockIdx.x;
  if (e >= I.n_cut) return;
  const int sl = elen[e];
  CqCtx c{&I, I.lo + 3 * static_cast<int64_t>(e), eprog + static_cast<int64_t>(e) * I.prog_len, sl};
  const int D = I.depth;
  const int nleaf = 1 << (3 * D);
  const int l0 = static_cast<int>(static_cast<int64_t>(nleaf) * threadIdx.x / blockDim.x);
  const int l1 = static_cast<int>(static_cast<int64_t>(nleaf) * (threadIdx.x + 1) / blockDim.x);
  CqSink<false> cnt{nullptr, 0};
  for (int l = l0; l < l1; ++l) cq_leaf<false>(c, l, D, cnt);
  __shared__ int sc[kCqThreads];
  sc[threadIdx.x] = cnt.n;
  __syncthreads();
  if (!W) {
    if (threadIdx.x == 0) {
      int64_t t = 0;
      for (int k = 0; k < blockDim.x; ++k) t += sc[k];
      count[e] = t;
    }
    return;
  }
  int base = 0;
  for (int k = 0; k < static_cast<int>(threadIdx.x); ++k) base += sc[k];
  CqSink<true> sk{prim + off[e] * kCqPrim, base};
  for (int l = l0; l < l1; ++l) cq_leaf<true>(c, l, D, sk);
}

// ------------------------------------------------------------ integrate ----
// eval1d (host/assembly.cpp): Bernstein values / derivatives at u, then the
// extraction rows E(i, k) (column-major q x q).
__device__ __forceinline__ void cq_eval1d(const double* __restrict__ E, int p, double u, double* v, double* dv) {
  double b[kCqMaxQ], db[kCqMaxQ];
  double lower[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  b[0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    if (j == p)
      for (int k = 0; k < p; ++k) lower[k] = b[k];
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      const double temp = b[r];
      b[r] = saved + (1.0 - u) * temp;
      saved = u * temp;
    }
    b[j] = saved;
  }
  db[0] = -p * lower[0];
  for (int r = 1; r < p; ++r) db[r] = p * (lower[r - 1] - lower[r]);
  db[p] = p * lower[p - 1];
  const int q = p + 1;
  for (int i = 0; i <= p; ++i) {
    double a = 0.0, c = 0.0;
    for (int k = 0; k <= p; ++k) {
      a += E[k * q + i] * b[k];
      c += E[k * q + i] * db[k];
    }
    v[i] = a;
    dv[i] = c;
  }
}

// A batch entry: a volume point (kind 1), an interface point (2) or a box (0).
struct CqPoint {
  double u[3];
  double w;
  double b[3];  // box upper corner (kind 0)
  int kind;
};

template <int NL>
__global__ void __launch_bounds__(kCqThreads) k_cq_integrate(ig_cut3 I, const int64_t* __restrict__ off,
                                                            const double* __restrict__ prim, double* Kout,
                                                            double* Fout, double* vout) {
  constexpr int NE = NL * (NL + 1) / 2;                 // upper-triangle entries
  constexpr int PER = (NE + kCqThreads - 1) / kCqThreads;
  const int e = blockIdx.x;
  if (e >= I.n_cut) return;
  const int p = I.p, q = p + 1;
  const double* E[3];
  for (int d = 0; d < 3; ++d) E[d] = I.ext[d] + static_cast<int64_t>(I.cls[3 * e + d]) * q * q;
  const double h0 = I.h[0], h1 = I.h[1], h2 = I.h[2];
  const double jac = h0 * h1 * h2;
  const int64_t p0 = off[e], np = off[e + 1] - off[e];
  const double* pr = prim + p0 * kCqPrim;

  __shared__ CqPoint pts[kCqBatch];
  __shared__ double vd[kCqBatch][3][2][kCqMaxQ];             // eval1d values / derivatives per point and axis
  __shared__ double bas[kCqBatch][4][NL];                    // phi, gx, gy, gz
  __shared__ double mom[kCqBatch > 0 ? 1 : 1][3][2 * kCqMaxQ * kCqMaxQ + kCqMaxQ];  // box moments
  __shared__ int pstart[513];

  // my K entries (upper triangle, row-major enumeration)
  int ei[PER], ej[PER];
  double acc[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    int idx = threadIdx.x + k * kCqThreads, i = 0;
    acc[k] = 0.0;
    ei[k] = -1;
    ej[k] = -1;
    if (idx < NE) {
      while (idx >= NL - i) {
        idx -= NL - i;
        ++i;
      }
      ei[k] = i;
      ej[k] = i + idx;
    }
  }
  double facc = 0.0, vol = 0.0;
  const int tix = threadIdx.x;

  // Primitive point counts: box 1, tetrahedron 8 (0 if degenerate), triangle 9 (0 if degenerate).
  // Processed in windows of 512 primitives.
  for (int64_t w0 = 0; w0 < np; w0 += 512) {
    const int nw = static_cast<int>(np - w0 < 512 ? np - w0 : 512);
    __syncthreads();
    for (int k = tix; k < nw; k += blockDim.x) {
      const double* P = pr + (w0 + k) * kCqPrim;
      const int type = static_cast<int>(P[0]);
      int n = 1;
      if (type == 1) {
        const double* v = P + 2;
        double e1[3], e2[3], e3[3];
        for (int d = 0; d < 3; ++d) {
          e1[d] = v[3 + d] - v[d];
          e2[d] = v[6 + d] - v[3 + d];
          e3[d] = v[9 + d] - v[6 + d];
        }
        const double det = e1[0] * (e2[1] * e3[2] - e2[2] * e3[1]) - e1[1] * (e2[0] * e3[2] - e2[2] * e3[0]) +
                           e1[2] * (e2[0] * e3[1] - e2[1] * e3[0]);
        n = fabs(det) > 0.0 ? 8 : 0;
      } else if (type == 2) {
        const double* v = P + 2;
        double e1[3], e2[3];
        for (int d = 0; d < 3; ++d) {
          e1[d] = v[3 + d] - v[d];
          e2[d] = v[6 + d] - v[3 + d];
        }
        const double cx = e1[1] * e2[2] - e1[2] * e2[1], cy = e1[2] * e2[0] - e1[0] * e2[2],
                     cz = e1[0] * e2[1] - e1[1] * e2[0];
        n = sqrt(cx * cx + cy * cy + cz * cz) > 0.0 ? 9 : 0;
      }
      pstart[k + 1] = n;
    }
    __syncthreads();
    if (tix == 0) {
      pstart[0] = 0;
      for (int k = 0; k < nw; ++k) pstart[k + 1] += pstart[k];
    }
    __syncthreads();
    const int npts = pstart[nw];
    for (int b0 = 0; b0 < npts; b0 += kCqBatch) {
      const int nb = npts - b0 < kCqBatch ? npts - b0 : kCqBatch;
      // (1) point coordinates and weights (host tet_points / tri_points order)
      if (tix < nb) {
        const int g = b0 + tix;
        int lo = 0, hi = nw - 1;  // primitive k with pstart[k] <= g < pstart[k+1]
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (pstart[mid] <= g) lo = mid;
          else hi = mid - 1;
        }
        const double* P = pr + (w0 + lo) * kCqPrim;
        const int type = static_cast<int>(P[0]);
        const int j = g - pstart[lo];
        CqPoint pt;
        pt.kind = type == 0 ? 0 : (type == 1 ? 1 : 2);
        const double* v = P + 2;
        if (type == 0) {
          for (int d = 0; d < 3; ++d) {
            pt.u[d] = v[d];
            pt.b[d] = v[3 + d];
          }
          pt.w = 0.0;
        } else if (type == 1) {
          double e1[3], e2[3], e3[3];
          for (int d = 0; d < 3; ++d) {
            e1[d] = v[3 + d] - v[d];
            e2[d] = v[6 + d] - v[3 + d];
            e3[d] = v[9 + d] - v[6 + d];
          }
          const double det = e1[0] * (e2[1] * e3[2] - e2[2] * e3[1]) - e1[1] * (e2[0] * e3[2] - e2[2] * e3[0]) +
                             e1[2] * (e2[0] * e3[1] - e2[1] * e3[0]);
          const double vol6 = fabs(det);
          const int ia = j / 4, ib = (j / 2) % 2, ic = j % 2;
          const double a = I.gauss_tet[ia], bb = I.gauss_tet[ib], cc = I.gauss_tet[ic];
          for (int d = 0; d < 3; ++d) pt.u[d] = v[d] + a * (e1[d] + bb * (e2[d] + cc * e3[d]));
          pt.w = vol6 * a * a * bb * I.gauss_tet[2 + ia] * I.gauss_tet[2 + ib] * I.gauss_tet[2 + ic];
        } else {
          double e1[3], e2[3];
          for (int d = 0; d < 3; ++d) {
            e1[d] = v[3 + d] - v[d];
            e2[d] = v[6 + d] - v[3 + d];
          }
          const double cx = e1[1] * e2[2] - e1[2] * e2[1], cy = e1[2] * e2[0] - e1[0] * e2[2],
                       cz = e1[0] * e2[1] - e1[1] * e2[0];
          const double area2 = sqrt(cx * cx + cy * cy + cz * cz);
          const int ia = j / 3, ib = j % 3;
          const double a = I.gauss_tri[ia], bb = I.gauss_tri[ib];
          for (int d = 0; d < 3; ++d) pt.u[d] = v[d] + a * (e1[d] + bb * e2[d]);
          pt.w = area2 * a * I.gauss_tri[3 + ia] * I.gauss_tri[3 + ib];
        }
        pts[tix] = pt;
      }
      __syncthreads();
      // (2) 1D evaluations per point and axis; box entries: their tensor moments
      for (int t = tix; t < nb * 3; t += blockDim.x) {
        const int k = t / 3, ax = t % 3;
        const CqPoint& pt = pts[k];
        if (pt.kind != 0) {
          cq_eval1d(E[ax], p, pt.u[ax], vd[k][ax][0], vd[k][ax][1]);
        }
      }
      __syncthreads();
      // (3) basis functions per point (ia fastest, then ib, ic: host order)
      for (int t = tix; t < nb * NL; t += blockDim.x) {
        const int k = t / NL, i = t % NL;
        const CqPoint& pt = pts[k];
        if (pt.kind == 0) continue;
        const int ia = i % q, ib = (i / q) % q, ic = i / (q * q);
        const double v0 = vd[k][0][0][ia], v1 = vd[k][1][0][ib], v2 = vd[k][2][0][ic];
        bas[k][0][i] = v0 * v1 * v2;
        if (pt.kind == 1) {
          bas[k][1][i] = vd[k][0][1][ia] * v1 * v2 / h0;
          bas[k][2][i] = v0 * vd[k][1][1][ib] * v2 / h1;
          bas[k][3][i] = v0 * v1 * vd[k][2][1][ic] / h2;
        }
      }
      __syncthreads();
      // (4) accumulate in point order; a box entry is applied in place
      for (int k = 0; k < nb; ++k) {
        const CqPoint& pt = pts[k];
        if (pt.kind == 0) {
          // add_box: 1D moments per axis over q Gauss points (axis loop, then g, i, j)
          bool ok = true;
          for (int ax = 0; ax < 3; ++ax) ok = ok && (pt.b[ax] - pt.u[ax] > 0.0);
          __syncthreads();
          if (ok && tix < 3) {
            const int ax = tix;
            double* M = mom[0][ax];  // [Iv (q) | Ivv (q x q) | Idd (q x q)]
            for (int z = 0; z < q + 2 * q * q; ++z) M[z] = 0.0;
            const double L = pt.b[ax] - pt.u[ax];
            for (int g = 0; g < q; ++g) {
              const double u = pt.u[ax] + 0.5 * (I.gauss_box[g] + 1.0) * L, w = 0.5 * I.gauss_box[q + g] * L;
              double v[kCqMaxQ], dv[kCqMaxQ];
              cq_eval1d(E[ax], p, u, v, dv);
              for (int i = 0; i < q; ++i) {
                M[i] += w * v[i];
                for (int j = 0; j < q; ++j) {
                  M[q + i * q + j] += w * v[i] * v[j];
                  M[q + q * q + i * q + j] += w * dv[i] * dv[j];
                }
              }
            }
          }
          __syncthreads();
          if (ok) {
            const double cx = jac / (h0 * h0), cy = jac / (h1 * h1), cz = jac / (h2 * h2);
            const double* M0 = mom[0][0];
            const double* M1 = mom[0][1];
            const double* M2 = mom[0][2];
#pragma unroll
            for (int s = 0; s < PER; ++s) {
              if (ei[s] < 0) continue;
              const int i = ei[s], j = ej[s];
              const int ia = i % q, ib = (i / q) % q, ic = i / (q * q);
              const int ja = j % q, jb = (j / q) % q, jc = j / (q * q);
              const double Ivv0 = M0[q + ia * q + ja], Ivv1 = M1[q + ib * q + jb], Ivv2 = M2[q + ic * q + jc];
              const double Idd0 = M0[q + q * q + ia * q + ja], Idd1 = M1[q + q * q + ib * q + jb],
                           Idd2 = M2[q + q * q + ic * q + jc];
              acc[s] += cx * Idd0 * Ivv1 * Ivv2 + cy * Ivv0 * Idd1 * Ivv2 + cz * Ivv0 * Ivv1 * Idd2;
            }
            if (tix < NL && I.f != 0.0) {
              const int ia = tix % q, ib = (tix / q) % q, ic = tix / (q * q);
              facc += I.f * jac * M0[ia] * M1[ib] * M2[ic];
            }
            if (tix == 0) vol += (pt.b[0] - pt.u[0]) * (pt.b[1] - pt.u[1]) * (pt.b[2] - pt.u[2]);
          }
          continue;
        }
        if (pt.kind == 1) {  // add_vol_point
          const double wp = pt.w * jac;
#pragma unroll
          for (int s = 0; s < PER; ++s) {
            if (ei[s] < 0) continue;
            const int i = ei[s], j = ej[s];
            const double a = wp * bas[k][1][i], b = wp * bas[k][2][i], c = wp * bas[k][3][i];
            acc[s] += a * bas[k][1][j] + b * bas[k][2][j] + c * bas[k][3][j];
          }
          if (tix < NL && I.f != 0.0) facc += wp * I.f * bas[k][0][tix];
          if (tix == 0) vol += pt.w;
        } else {  // add_surf_point
          const double wb = pt.w * h0 * h0 * I.beta;
#pragma unroll
          for (int s = 0; s < PER; ++s) {
            if (ei[s] < 0) continue;
            const int i = ei[s], j = ej[s];
            const double a = wb * bas[k][0][i];
            acc[s] += a * bas[k][0][j];
          }
        }
      }
      __syncthreads();
    }
  }
  // finish3: K symmetric from the upper triangle
  double* K = Kout + static_cast<int64_t>(e) * NL * NL;
#pragma unroll
  for (int s = 0; s < PER; ++s) {
    if (ei[s] < 0) continue;
    K[ei[s] * NL + ej[s]] = acc[s];
    K[ej[s] * NL + ei[s]] = acc[s];
  }
  if (tix < NL) Fout[static_cast<int64_t>(e) * NL + tix] = facc;
  if (tix == 0 && vout) vout[e] = vol;
}

}  // namespace igk
