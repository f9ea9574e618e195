// Level sets, cell classification and edge intersection.
// Restates proj/src/geometry.cpp (node types :10-141, classify_cell :143-155,
// intersect_edge :157-175) and the expression language of
// proj/src/config.cpp:32-132, extended with 3D primitives.
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <functional>

#include "host.hpp"

namespace igh {

struct LsNode {
  virtual ~LsNode() = default;
  virtual double eval(const double* p) const = 0;
  virtual bool bounds(const double*, const double*, int, double&, double&) const {
    return false;
  }
  // Postfix program for the device evaluator (ig_gpu.h ig_cut3: op codes
  // 0 const, 1 linear, 2 ball, 3 box, 4 min, 5 max, 6 neg); false for nodes
  // without a bit-exact device form (star: atan2 / sin; affine).
  virtual bool emit(std::vector<double>&) const { return false; }
};

namespace {

struct ConstNode final : LsNode {
  double v;
  explicit ConstNode(double v_) : v(v_) {}
  bool emit(std::vector<double>& o) const override {
    o.insert(o.end(), {0.0, v});
    return true;
  }
  double eval(const double*) const override { return v; }
  bool bounds(const double*, const double*, int, double& a, double& b) const override {
    a = b = v;
    return true;
  }
};

// a*x + b*y (+ c*z) + d
struct LinearNode final : LsNode {
  double c[3], d;
  int dim;
  bool emit(std::vector<double>& o) const override {
    o.insert(o.end(), {1.0, c[0], c[1], c[2], d, static_cast<double>(dim)});
    return true;
  }
  double eval(const double* p) const override {
    return dim == 2 ? c[0] * p[0] + c[1] * p[1] + d : c[0] * p[0] + c[1] * p[1] + c[2] * p[2] + d;
  }
  bool bounds(const double* lo, const double* hi, int, double& a, double& b) const override {
    a = b = d;
    for (int k = 0; k < dim; ++k) {
      const double u = c[k] * lo[k], v = c[k] * hi[k];
      a += std::min(u, v);
      b += std::max(u, v);
    }
    return true;
  }
};

// r - |p - c|  (disc in 2D, sphere in 3D)
struct BallNode final : LsNode {
  double c[3], r;
  int dim;
  bool emit(std::vector<double>& o) const override {
    o.insert(o.end(), {2.0, c[0], c[1], c[2], r, static_cast<double>(dim)});
    return true;
  }
  double eval(const double* p) const override {
    const double dx = p[0] - c[0], dy = p[1] - c[1];
    if (dim == 2) return r - std::sqrt(dx * dx + dy * dy);
    const double dz = p[2] - c[2];
    return r - std::sqrt(dx * dx + dy * dy + dz * dz);
  }
  bool bounds(const double* lo, const double* hi, int, double& a, double& b) const override {
    double dmin2 = 0, dmax2 = 0;
    for (int k = 0; k < dim; ++k) {
      const double l = lo[k] - c[k], h = hi[k] - c[k];
      const double near = (l > 0) ? l : (h < 0 ? -h : 0.0);
      const double far = std::max(std::fabs(l), std::fabs(h));
      dmin2 += near * near;
      dmax2 += far * far;
    }
    a = r - std::sqrt(dmax2);
    b = r - std::sqrt(dmin2);
    return true;
  }
};

struct StarNode final : LsNode {
  double cx, cy, r0, amp;
  int k;
  double eval(const double* p) const override {
    const double dx = p[0] - cx, dy = p[1] - cy;
    const double r = std::hypot(dx, dy);
    const double theta = (dx == 0.0 && dy == 0.0) ? 0.0 : std::atan2(dy, dx);
    return r0 + amp * std::sin(k * theta) - r;
  }
};

// min over axes of (x - lo, hi - x)
struct BoxNode final : LsNode {
  double lo[3], hi[3];
  int dim;
  bool emit(std::vector<double>& o) const override {
    o.insert(o.end(), {3.0, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], static_cast<double>(dim)});
    return true;
  }
  double eval(const double* p) const override {
    double v = std::min(std::min(p[0] - lo[0], hi[0] - p[0]), std::min(p[1] - lo[1], hi[1] - p[1]));
    if (dim == 3) v = std::min(v, std::min(p[2] - lo[2], hi[2] - p[2]));
    return v;
  }
  bool bounds(const double* bl, const double* bh, int, double& a, double& b) const override {
    a = 1e300;
    b = 1e300;
    for (int k = 0; k < dim; ++k) {
      a = std::min(a, std::min(bl[k] - lo[k], hi[k] - bh[k]));
      b = std::min(b, std::min(bh[k] - lo[k], hi[k] - bl[k]));
    }
    return true;
  }
};

struct AffineNode final : LsNode {
  std::shared_ptr<const LsNode> sub;
  double A[4], bb[2];
  double eval(const double* p) const override {
    const double q[2] = {A[0] * p[0] + A[1] * p[1] + bb[0], A[2] * p[0] + A[3] * p[1] + bb[1]};
    return sub->eval(q);
  }
};

enum class Comb { Min, Max, Neg };
struct CombineNode final : LsNode {
  Comb op;
  std::shared_ptr<const LsNode> a, b;
  bool emit(std::vector<double>& o) const override {
    if (!a->emit(o)) return false;
    if (op != Comb::Neg && !b->emit(o)) return false;
    o.push_back(op == Comb::Min ? 4.0 : (op == Comb::Max ? 5.0 : 6.0));
    return true;
  }
  double eval(const double* p) const override {
    switch (op) {
      case Comb::Min: return std::min(a->eval(p), b->eval(p));
      case Comb::Max: return std::max(a->eval(p), b->eval(p));
      default: return -a->eval(p);
    }
  }
  bool bounds(const double* lo, const double* hi, int dim, double& x, double& y) const override {
    double a0, a1, b0, b1;
    if (!a->bounds(lo, hi, dim, a0, a1)) return false;
    if (op == Comb::Neg) {
      x = -a1;
      y = -a0;
      return true;
    }
    if (!b->bounds(lo, hi, dim, b0, b1)) return false;
    if (op == Comb::Min) {
      x = std::min(a0, b0);
      y = std::min(a1, b1);
    } else {
      x = std::max(a0, b0);
      y = std::max(a1, b1);
    }
    return true;
  }
};

// ---- recursive-descent parser (config.cpp:32-132 grammar) ----------------
struct Parser {
  const std::string& s;
  size_t i = 0;
  explicit Parser(const std::string& str) : s(str) {}
  [[noreturn]] void fail(const std::string& m) {
    throw SetupError("parse_levelset: " + m + " at offset " + std::to_string(i) + " in '" + s + "'");
  }
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  bool peek(char c) {
    ws();
    return i < s.size() && s[i] == c;
  }
  void expect(char c) {
    if (!peek(c)) fail(std::string("expected '") + c + "'");
    ++i;
  }
  std::string ident() {
    ws();
    size_t j = i;
    while (j < s.size() && (std::isalnum(static_cast<unsigned char>(s[j])) || s[j] == '_')) ++j;
    if (j == i) fail("expected identifier");
    std::string r = s.substr(i, j - i);
    i = j;
    return r;
  }
  bool number_ahead() {
    ws();
    if (i >= s.size()) return false;
    const char c = s[i];
    return std::isdigit(static_cast<unsigned char>(c)) || c == '-' || c == '+' || c == '.';
  }
  double number() {
    ws();
    const char* b = s.c_str() + i;
    char* e = nullptr;
    const double v = std::strtod(b, &e);
    if (e == b) fail("expected number");
    i += static_cast<size_t>(e - b);
    return v;
  }
  std::shared_ptr<const LsNode> expr() {
    const std::string name = ident();
    expect('(');
    std::vector<double> nums;
    std::vector<std::shared_ptr<const LsNode>> subs;
    if (!peek(')')) {
      while (true) {
        if (number_ahead())
          nums.push_back(number());
        else
          subs.push_back(expr());
        if (peek(',')) {
          ++i;
          continue;
        }
        break;
      }
    }
    expect(')');
    auto need = [&](size_t nn, size_t ns) {
      if (nums.size() != nn || subs.size() != ns)
        fail(name + ": wrong number of arguments");
    };
    if (name == "constant") {
      need(1, 0);
      return std::make_shared<ConstNode>(nums[0]);
    }
    if (name == "halfplane") {
      need(3, 0);
      auto n = std::make_shared<LinearNode>();
      n->dim = 2;
      n->c[0] = nums[0];
      n->c[1] = nums[1];
      n->c[2] = 0;
      n->d = nums[2];
      return n;
    }
    if (name == "halfspace") {
      need(4, 0);
      auto n = std::make_shared<LinearNode>();
      n->dim = 3;
      for (int k = 0; k < 3; ++k) n->c[k] = nums[k];
      n->d = nums[3];
      return n;
    }
    if (name == "disc") {
      need(3, 0);
      auto n = std::make_shared<BallNode>();
      n->dim = 2;
      n->c[0] = nums[0];
      n->c[1] = nums[1];
      n->c[2] = 0;
      n->r = nums[2];
      return n;
    }
    if (name == "sphere") {
      need(4, 0);
      auto n = std::make_shared<BallNode>();
      n->dim = 3;
      for (int k = 0; k < 3; ++k) n->c[k] = nums[k];
      n->r = nums[3];
      return n;
    }
    if (name == "star") {
      need(5, 0);
      auto n = std::make_shared<StarNode>();
      n->cx = nums[0];
      n->cy = nums[1];
      n->r0 = nums[2];
      n->amp = nums[3];
      n->k = static_cast<int>(nums[4]);
      return n;
    }
    if (name == "box") {
      need(4, 0);
      auto n = std::make_shared<BoxNode>();
      n->dim = 2;
      n->lo[0] = nums[0];
      n->lo[1] = nums[1];
      n->hi[0] = nums[2];
      n->hi[1] = nums[3];
      n->lo[2] = n->hi[2] = 0;
      return n;
    }
    if (name == "box3") {
      need(6, 0);
      auto n = std::make_shared<BoxNode>();
      n->dim = 3;
      for (int k = 0; k < 3; ++k) {
        n->lo[k] = nums[k];
        n->hi[k] = nums[3 + k];
      }
      return n;
    }
    if (name == "union" || name == "intersect") {
      if (!nums.empty() || subs.empty()) fail(name + ": expects level-set arguments");
      std::shared_ptr<const LsNode> acc = subs[0];
      for (size_t k = 1; k < subs.size(); ++k) {
        auto c = std::make_shared<CombineNode>();
        c->op = name == "union" ? Comb::Max : Comb::Min;
        c->a = acc;
        c->b = subs[k];
        acc = c;
      }
      return acc;
    }
    if (name == "complement") {
      need(0, 1);
      auto c = std::make_shared<CombineNode>();
      c->op = Comb::Neg;
      c->a = subs[0];
      c->b = subs[0];
      return c;
    }
    if (name == "affine") {
      need(6, 1);
      auto n = std::make_shared<AffineNode>();
      for (int k = 0; k < 4; ++k) n->A[k] = nums[k];
      n->bb[0] = nums[4];
      n->bb[1] = nums[5];
      n->sub = subs[0];
      return n;
    }
    fail("unknown primitive '" + name + "'");
  }
};

}  // namespace

LevelSet::LevelSet() : node_(std::make_shared<ConstNode>(1.0)) {}
double LevelSet::operator()(const double* p) const { return node_->eval(p); }
bool LevelSet::program(std::vector<double>& out) const {
  out.clear();
  return node_->emit(out);
}
bool LevelSet::bounds(const double* lo, const double* hi, int dim, double& a, double& b) const {
  return node_->bounds(lo, hi, dim, a, b);
}

LevelSet parse_levelset(const std::string& expr) {
  Parser ps(expr);
  auto n = ps.expr();
  ps.ws();
  if (ps.i != expr.size()) ps.fail("trailing characters");
  return LevelSet(n);
}

CellClass classify_cell(const LevelSet& ls, const double* lo, const double* hi, int dim,
                        int depth) {
  // Exact shortcut: if psi is provably one-signed over the cell (with a
  // margin far above rounding), every lattice sample has that sign and the
  // sampling below would return the same class.
  double vmin, vmax;
  if (ls.bounds(lo, hi, dim, vmin, vmax)) {
    double scale = 0;
    for (int k = 0; k < dim; ++k) scale = std::max(scale, std::fabs(lo[k]) + std::fabs(hi[k]));
    const double margin = 1e-9 * (1.0 + scale);
    if (vmin > margin) return CellClass::Inside;
    if (vmax < -margin) return CellClass::Outside;
  }
  const int n = (1 << depth) + 1;
  bool any_in = false, any_out = false;
  double d[3];
  for (int k = 0; k < dim; ++k) d[k] = (hi[k] - lo[k]) / static_cast<double>(n - 1);
  double p[3] = {0, 0, 0};
  if (dim == 2) {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        p[0] = lo[0] + i * d[0];
        p[1] = lo[1] + j * d[1];
        (ls(p) >= 0.0 ? any_in : any_out) = true;
        if (any_in && any_out) return CellClass::Cut;
      }
  } else {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k) {
          p[0] = lo[0] + i * d[0];
          p[1] = lo[1] + j * d[1];
          p[2] = lo[2] + k * d[2];
          (ls(p) >= 0.0 ? any_in : any_out) = true;
          if (any_in && any_out) return CellClass::Cut;
        }
  }
  return any_in ? CellClass::Inside : CellClass::Outside;
}

void intersect_edge(const LevelSet& ls, const double* p0, const double* p1, int dim, double tol,
                    double* out) {
  double f0 = ls(p0);
  double f1 = ls(p1);
  if (f0 * f1 > 0.0) throw SetupError("intersect_edge: no sign change on segment");
  double t0 = 0.0, t1 = 1.0;
  double q[3] = {0, 0, 0};
  auto at = [&](double t, double* o) {
    for (int k = 0; k < dim; ++k) o[k] = p0[k] + t * (p1[k] - p0[k]);
  };
  while (t1 - t0 > tol) {
    const double tm = 0.5 * (t0 + t1);
    at(tm, q);
    const double fm = ls(q);
    if (f0 * fm <= 0.0) {
      t1 = tm;
      f1 = fm;
    } else {
      t0 = tm;
      f0 = fm;
    }
  }
  at(0.5 * (t0 + t1), out);
}

}  // namespace igh
