// Small dense/sparse linear algebra (the Eigen pieces the setup needs) and the
// 1D spline machinery of proj/src/spline1d.cpp (:11-158).
#include <algorithm>
#include <cmath>

#include "host.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace igh {

// ------------------------------------------------------------- sparse -----

double Csr::coeff(int32_t i, int32_t j) const {
  const int32_t* b = col.data() + ptr[i];
  const int32_t* e = col.data() + ptr[i + 1];
  const int32_t* it = std::lower_bound(b, e, j);
  return (it != e && *it == j) ? val[it - col.data()] : 0.0;
}

Csr transpose(const Csr& a) {
  Csr t;
  t.nr = a.nc;
  t.nc = a.nr;
  t.ptr.assign(static_cast<size_t>(t.nr) + 1, 0);
  for (int32_t c : a.col) ++t.ptr[c + 1];
  for (int32_t i = 0; i < t.nr; ++i) t.ptr[i + 1] += t.ptr[i];
  t.col.resize(a.col.size());
  t.val.resize(a.val.size());
  std::vector<int32_t> next(t.ptr.begin(), t.ptr.end() - 1);
  for (int32_t i = 0; i < a.nr; ++i)
    for (int32_t k = a.ptr[i]; k < a.ptr[i + 1]; ++k) {
      const int32_t pos = next[a.col[k]]++;
      t.col[pos] = i;  // rows visited ascending -> columns of t ascending
      t.val[pos] = a.val[k];
    }
  return t;
}

Csr spgemm(const Csr& a, const Csr& b, int threads) {
  if (a.nc != b.nr) throw SetupError("spgemm: inner dimension mismatch");
  Csr c;
  c.nr = a.nr;
  c.nc = b.nc;
  std::vector<int32_t> cnt(static_cast<size_t>(a.nr), 0);
  // Pass 1: row pattern sizes.
#pragma omp parallel num_threads(threads)
  {
    std::vector<int32_t> mark(static_cast<size_t>(b.nc), -1);
#pragma omp for schedule(dynamic, 256)
    for (int32_t i = 0; i < a.nr; ++i) {
      int32_t n = 0;
      for (int32_t k = a.ptr[i]; k < a.ptr[i + 1]; ++k) {
        const int32_t r = a.col[k];
        for (int32_t q = b.ptr[r]; q < b.ptr[r + 1]; ++q)
          if (mark[b.col[q]] != i) {
            mark[b.col[q]] = i;
            ++n;
          }
      }
      cnt[i] = n;
    }
  }
  c.ptr.assign(static_cast<size_t>(a.nr) + 1, 0);
  for (int32_t i = 0; i < a.nr; ++i) {
    const int64_t nx = static_cast<int64_t>(c.ptr[i]) + cnt[i];
    if (nx > INT32_MAX) throw SetupError("spgemm: nnz exceeds int32");
    c.ptr[i + 1] = static_cast<int32_t>(nx);
  }
  c.col.resize(c.ptr.back());
  c.val.resize(c.ptr.back());
  // Pass 2: values; acc[col] accumulates in ascending k (inner index) order.
#pragma omp parallel num_threads(threads)
  {
    std::vector<int32_t> pos(static_cast<size_t>(b.nc), -1);
    std::vector<double> acc(static_cast<size_t>(b.nc), 0.0);
    std::vector<int32_t> cols;
#pragma omp for schedule(dynamic, 256)
    for (int32_t i = 0; i < a.nr; ++i) {
      cols.clear();
      for (int32_t k = a.ptr[i]; k < a.ptr[i + 1]; ++k) {
        const int32_t r = a.col[k];
        const double av = a.val[k];
        for (int32_t q = b.ptr[r]; q < b.ptr[r + 1]; ++q) {
          const int32_t j = b.col[q];
          const double prod = av * b.val[q];
          if (pos[j] < 0) {
            pos[j] = 1;
            acc[j] = prod;
            cols.push_back(j);
          } else {
            acc[j] = acc[j] + prod;
          }
        }
      }
      std::sort(cols.begin(), cols.end());
      int32_t o = c.ptr[i];
      for (int32_t j : cols) {
        c.col[o] = j;
        c.val[o] = acc[j];
        ++o;
        pos[j] = -1;
      }
    }
  }
  return c;
}

// -------------------------------------------------------------- dense -----

Mat matmul(const Mat& A, const Mat& B) {
  Mat C(A.r, B.c);
  for (int j = 0; j < B.c; ++j)
    for (int i = 0; i < A.r; ++i) {
      double s = 0.0;
      for (int k = 0; k < A.c; ++k) s += A(i, k) * B(k, j);
      C(i, j) = s;
    }
  return C;
}

Mat transpose(const Mat& A) {
  Mat T(A.c, A.r);
  for (int j = 0; j < A.c; ++j)
    for (int i = 0; i < A.r; ++i) T(j, i) = A(i, j);
  return T;
}

Mat lu_solve(Mat A, Mat B) {
  const int n = A.r;
  std::vector<int> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = std::fabs(A(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(A(i, k)) > best) {
        best = std::fabs(A(i, k));
        piv = i;
      }
    if (piv != k) {
      for (int j = 0; j < n; ++j) std::swap(A(k, j), A(piv, j));
      for (int j = 0; j < B.c; ++j) std::swap(B(k, j), B(piv, j));
    }
    for (int i = k + 1; i < n; ++i) {
      const double f = A(i, k) / A(k, k);
      A(i, k) = f;
      for (int j = k + 1; j < n; ++j) A(i, j) -= f * A(k, j);
      for (int j = 0; j < B.c; ++j) B(i, j) -= f * B(k, j);
    }
  }
  for (int j = 0; j < B.c; ++j)
    for (int i = n - 1; i >= 0; --i) {
      double s = B(i, j);
      for (int k = i + 1; k < n; ++k) s -= A(i, k) * B(k, j);
      B(i, j) = s / A(i, i);
    }
  return B;
}

// ------------------------------------------------------------ spline1d ----
namespace spline {

std::vector<double> open_uniform_knots(double x0, double x1, int n_cells, int p) {
  if (n_cells < 1 || p < 1) throw SetupError("open_uniform_knots: bad sizes");
  std::vector<double> t;
  t.reserve(static_cast<size_t>(n_cells) + 2 * p + 1);
  for (int i = 0; i < p; ++i) t.push_back(x0);
  for (int i = 0; i <= n_cells; ++i) t.push_back(x0 + (x1 - x0) * static_cast<double>(i) / n_cells);
  for (int i = 0; i < p; ++i) t.push_back(x1);
  return t;
}

int find_span(const std::vector<double>& t, int p, double x) {
  const int n = static_cast<int>(t.size()) - p - 1;
  if (x >= t[n]) return n - 1;
  if (x <= t[p]) return p;
  auto it = std::upper_bound(t.begin() + p, t.begin() + n, x);
  return static_cast<int>(it - t.begin()) - 1;
}

void eval_nonzero(const std::vector<double>& t, int p, double x, int span, double* val,
                  double* der) {
  double left[8], right[8], ndu[8][8];
  ndu[0][0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    left[j] = x - t[span + 1 - j];
    right[j] = t[span + j] - x;
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      ndu[j][r] = right[r + 1] + left[j - r];  // ndu(j, r): knot differences
      const double temp = ndu[r][j - 1] / ndu[j][r];
      ndu[r][j] = saved + right[r + 1] * temp;
      saved = left[j - r] * temp;
    }
    ndu[j][j] = saved;
  }
  for (int i = 0; i <= p; ++i) val[i] = ndu[i][p];
  for (int r = 0; r <= p; ++r) {
    double d = 0.0;
    if (r > 0) d += ndu[r - 1][p - 1] / ndu[p][r - 1];
    if (r < p) d -= ndu[r][p - 1] / ndu[p][r];
    der[r] = d * p;
  }
}

void bernstein(int p, double u, double* val, double* der) {
  double lower[8] = {0};
  val[0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    if (j == p)
      for (int k = 0; k < p; ++k) lower[k] = val[k];
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      const double temp = val[r];
      val[r] = saved + (1.0 - u) * temp;
      saved = u * temp;
    }
    val[j] = saved;
  }
  der[0] = -p * lower[0];
  for (int r = 1; r < p; ++r) der[r] = p * (lower[r - 1] - lower[r]);
  der[p] = p * lower[p - 1];
}

namespace {
std::vector<double> collocation_points(int p) {
  std::vector<double> u(p + 1);
  for (int k = 0; k <= p; ++k) u[k] = 0.5 - 0.5 * std::cos(M_PI * (2.0 * k + 1.0) / (2.0 * (p + 1)));
  return u;
}
Mat bernstein_collocation(int p, const std::vector<double>& u) {
  Mat B(p + 1, p + 1);
  double v[8], d[8];
  for (int k = 0; k <= p; ++k) {
    bernstein(p, u[k], v, d);
    for (int j = 0; j <= p; ++j) B(k, j) = v[j];
  }
  return B;
}
}  // namespace

Mat span_extraction(const std::vector<double>& t, int p, int span) {
  const auto u = collocation_points(p);
  const double a = t[span], b = t[span + 1];
  Mat Vs(p + 1, p + 1);
  double v[8], d[8];
  for (int k = 0; k <= p; ++k) {
    eval_nonzero(t, p, a + u[k] * (b - a), span, v, d);
    for (int i = 0; i <= p; ++i) Vs(k, i) = v[i];
  }
  return transpose(lu_solve(bernstein_collocation(p, u), Vs));
}

Mat lagrange_extraction(int p) {
  const auto u = collocation_points(p);
  Mat Vs(p + 1, p + 1);
  for (int k = 0; k <= p; ++k)
    for (int i = 0; i <= p; ++i) {
      double val = 1.0;
      for (int j = 0; j <= p; ++j) {
        if (j == i) continue;
        val *= (u[k] - static_cast<double>(j) / p) /
               (static_cast<double>(i) / p - static_cast<double>(j) / p);
      }
      Vs(k, i) = val;
    }
  return transpose(lu_solve(bernstein_collocation(p, u), Vs));
}

Mat dyadic_refine_matrix(int n_cells_coarse, int p) {
  // Boehm insertion of every span midpoint (spline1d.cpp:131-158).  The
  // product T*step is banded, so it is formed sparsely row by row.
  std::vector<double> t = open_uniform_knots(0.0, 1.0, n_cells_coarse, p);
  const int n0 = n_cells_coarse + p;
  Mat T(n0, n0);
  for (int i = 0; i < n0; ++i) T(i, i) = 1.0;
  for (int s = 0; s < n_cells_coarse; ++s) {
    const double u = (s + 0.5) / n_cells_coarse;
    const int n = static_cast<int>(t.size()) - p - 1;
    const int l = find_span(t, p, u);
    std::vector<double> a(static_cast<size_t>(n) + 1);
    for (int i = 0; i <= n; ++i) {
      if (i <= l - p)
        a[i] = 1.0;
      else if (i <= l)
        a[i] = (u - t[i]) / (t[i + p] - t[i]);
      else
        a[i] = 0.0;
    }
    // T_new(r, j) = sum_i T(r, i) * step(i, j), step(i,i) = a_i, step(i,i+1) = 1 - a_{i+1}
    Mat Tn(n0, n + 1);
    for (int r = 0; r < n0; ++r)
      for (int j = 0; j <= n; ++j) {
        double v = 0.0;
        // Eigen's dense product sums over i ascending; only i = j-1 and i = j contribute.
        if (j - 1 >= 0 && j - 1 < n) v += T(r, j - 1) * (1.0 - a[j]);
        if (j < n) {
          // keep ascending-i order: term i=j-1 first, then i=j
          v += T(r, j) * a[j];
        }
        Tn(r, j) = v;
      }
    T = std::move(Tn);
    t.insert(std::upper_bound(t.begin(), t.end(), u), u);
  }
  return T;
}

}  // namespace spline
}  // namespace igh
