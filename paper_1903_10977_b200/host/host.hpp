// Host-side setup for the solve phase: everything the reference runs ONCE,
// before the hot path, to build the algebraic multigrid hierarchy that crosses
// the C-ABI (include/ig_gpu.h).  Restates, in flat arrays instead of
// std::map/std::set, the reference modules
//   geometry   proj/src/geometry.cpp        level sets, classify_cell, intersect_edge
//   mesh       proj/src/mesh.cpp            uniform grid, coarsen, trim
//   quadrature proj/src/quadrature.cpp      cut-cell rules (2D, literal)
//   spline1d   proj/src/spline1d.cpp        knots, Cox-de Boor, Bernstein, two-scale
//   basis      proj/src/basis.cpp:91-316    Lagrange / B-spline spaces, trimming
//              proj/src/basis.cpp:376-432   restriction matrices
//   assembly   proj/src/assembly.cpp        Poisson + penalty Dirichlet
//   smoothers  proj/src/smoothers.cpp:20-162,216-241  blocks, gamma, filter+LLT
//   multigrid  proj/src/multigrid.cpp:12-75 Galerkin hierarchy + dpstrf
// and extends them to 3D (no reference counterpart).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace igh {

// ---------------------------------------------------------------- basics --

// splitmix64, bit-identical to immergrid::Rng (proj/include/immergrid/common.hpp:43-58).
struct Rng {
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double a, double b) { return a + (b - a) * uniform(); }
};

// Row-major compressed sparse matrix (== Eigen RowMajor SpMat, int32 indices).
struct Csr {
  int32_t nr = 0, nc = 0;
  std::vector<int32_t> ptr{0}, col;
  std::vector<double> val;
  int64_t nnz() const { return static_cast<int64_t>(col.size()); }
  // A.coeff(i, j): stored value or 0 (binary search in row i).
  double coeff(int32_t i, int32_t j) const;
};

Csr transpose(const Csr& a);
// C = A * B, row-wise Gustavson: each output entry accumulates in ascending
// order of the inner index k (documented order; Eigen's is not observable).
Csr spgemm(const Csr& a, const Csr& b, int threads);

// Column-major dense matrix.
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int r_, int c_) : r(r_), c(c_), a(static_cast<size_t>(r_) * c_, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(j) * r + i]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(j) * r + i]; }
};
Mat matmul(const Mat& A, const Mat& B);
Mat transpose(const Mat& A);
// Solve A X = B with partial-pivot LU (Eigen partialPivLu semantics).
Mat lu_solve(Mat A, Mat B);

struct SetupError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------- level sets --

// Expression-tree level set; physical domain = { psi >= 0 } (geometry.hpp:18-23).
// 2D primitives as parse_levelset (config.hpp:21-31) plus 3D primitives
// sphere(cx,cy,cz,r), box3(x0,y0,z0,x1,y1,z1), halfspace(a,b,c,d).
struct LsNode;
class LevelSet {
 public:
  LevelSet();  // constant +1
  explicit LevelSet(std::shared_ptr<const LsNode> n) : node_(std::move(n)) {}
  double operator()(const double* p) const;  // p has 2 or 3 coordinates
  double at(double x, double y, double z = 0.0) const {
    const double p[3] = {x, y, z};
    return (*this)(p);
  }
  // Exact-bound fast path for classification: returns true and sets lo/hi
  // if the node can bound psi over an axis box (used only to skip sampling
  // when every lattice sample provably has one sign).
  bool bounds(const double* lo, const double* hi, int dim, double& vmin, double& vmax) const;
  // Postfix program for the device evaluator (ig_cut3); false if a node has
  // no bit-exact device form.
  bool program(std::vector<double>& out) const;
  const std::shared_ptr<const LsNode>& node() const { return node_; }

 private:
  std::shared_ptr<const LsNode> node_;
};
LevelSet parse_levelset(const std::string& expr);

enum class CellClass : uint8_t { Inside = 0, Outside = 1, Cut = 2 };
// Samples psi on the (2^depth+1)^dim lattice (geometry.cpp:143-155).
CellClass classify_cell(const LevelSet& ls, const double* lo, const double* hi, int dim,
                        int depth);
// Bisection root on p0..p1 (geometry.cpp:157-175); throws on no sign change.
void intersect_edge(const LevelSet& ls, const double* p0, const double* p1, int dim,
                    double tol, double* out);

// --------------------------------------------------------------- spline1d --
namespace spline {
std::vector<double> open_uniform_knots(double x0, double x1, int n_cells, int p);
int find_span(const std::vector<double>& t, int p, double x);
void eval_nonzero(const std::vector<double>& t, int p, double x, int span, double* val,
                  double* der);
void bernstein(int p, double u, double* val, double* der);
Mat span_extraction(const std::vector<double>& t, int p, int span);
Mat lagrange_extraction(int p);
Mat dyadic_refine_matrix(int n_cells_coarse, int p);
}  // namespace spline

// ------------------------------------------------------------ mesh + space --

enum class Family : int { Lagrange = 0, Bspline = 1 };
enum ElemTag : uint8_t { kInside = 0, kCut = 1, kOutside = 2 };

struct Grid {
  int dim = 2;
  double origin[3] = {0, 0, 0};
  double extent[3] = {1, 1, 1};
  int res[3] = {1, 1, 1};
  double h(int d) const { return extent[d] / res[d]; }
  int64_t num_cells() const {
    int64_t n = 1;
    for (int d = 0; d < dim; ++d) n *= res[d];
    return n;
  }
  // Reference element order (mesh.cpp:7-14, std::set<pair> ordering): x-major.
  int64_t cell_linear(int ix, int iy, int iz) const {
    return dim == 2 ? static_cast<int64_t>(ix) * res[1] + iy
                    : (static_cast<int64_t>(ix) * res[1] + iy) * res[2] + iz;
  }
  void cell_box(int ix, int iy, int iz, double* lo, double* hi) const;
};

// Uniform trimmed mesh + Lagrange/B-spline space on it (basis.cpp:91-316 for
// M = 0).  Anchors: ordered (az, ay, ax), ax fastest (basis.hpp:35).
struct Space {
  Grid grid;
  Family family = Family::Bspline;
  int p = 2;
  int nf[3] = {1, 1, 1};  // functions per axis
  // Active (Inside/Cut) elements in reference id order.
  std::vector<int32_t> el_ix, el_iy, el_iz;
  std::vector<uint8_t> el_tag;
  std::vector<int32_t> cell_to_el;  // num_cells -> active index or -1
  std::vector<uint8_t> cell_tag;    // num_cells -> ElemTag
  // Untrimmed anchor linear index (az*nfy+ay)*nfx+ax <-> kept index.
  std::vector<int32_t> kept;     // untrimmed -> kept or -1
  std::vector<int64_t> anchors;  // kept -> untrimmed linear
  // Physical support per kept anchor: active element indices, ascending.
  std::vector<int64_t> supp_ptr;
  std::vector<int32_t> supp_el;
  // Per-axis extraction: ext_cls[d][cell] -> class id; ext[d][class] the
  // (p+1)x(p+1) local-function -> Bernstein map (span_extraction).
  std::vector<int32_t> ext_cls[3];
  std::vector<Mat> ext[3];
  LevelSet ls;
  int classify_depth = 2;

  int n() const { return static_cast<int>(anchors.size()); }
  int nloc() const {
    int k = 1;
    for (int d = 0; d < grid.dim; ++d) k *= p + 1;
    return k;
  }
  int64_t untrimmed(int ax, int ay, int az) const {
    return (static_cast<int64_t>(az) * nf[1] + ay) * nf[0] + ax;
  }
  // Local anchors of active element e in reference row order (basis.cpp:204-214):
  // z outer, then y, x fastest.  Writes kept indices.
  void element_anchors(int e, int32_t* out) const;
  // First anchor index per axis of element cell c: ex (spline) or p*ex (Lagrange).
  int first_anchor(int cell) const { return family == Family::Bspline ? cell : p * cell; }
};

// Cells [lo, hi] along one axis whose local anchors include anchor index a:
// fn_spans (basis.cpp:66-70) for B-splines, node_elems (basis.cpp:73-78) for Lagrange.
void anchor_cells(Family fam, int a, int p, int cells, int& lo, int& hi);

// trim + build_space (mesh.cpp:91-111, basis.cpp:91-316).
std::unique_ptr<Space> build_space(const Grid& g, const LevelSet& ls, Family fam, int p,
                                   int classify_depth, int threads);

// ------------------------------------------------------------- assembly ---

struct QuadConfig {
  int depth = 3;
  int gauss_order = 3;
  int classify_depth = 2;
  double edge_tol = 1e-12;
};

struct ProblemConfig {
  double body_force = 1.0;
  double beta = 0.0;               // 0 = default 2/h (assembly.cpp:7-10)
  bool dirichlet_box_sides = true; // boundary pieces also on embedding-box sides
};

struct Assembled {
  Csr A;
  std::vector<double> b;
  double eta = 1.0;  // min volume fraction (quadrature.cpp:363-371)
  int64_t cut_elements = 0;
  // Element tables the row gather consumed (device assembly payload,
  // ig_assembly): table t holds K (nloc x nloc, row-major) and F (nloc);
  // element e uses table el_table[e] (Inside classes first, then the
  // individually integrated elements).
  std::vector<double> tabK, tabF;
  std::vector<int32_t> el_table;
  int32_t n_tables = 0;
  // Physical volume fraction of every active element's cell (1 for Inside).
  std::vector<double> el_vol;
};

// numeric = false: the geometric half only (igh_build_geometry) -- element
// classes, Inside-class tables and the element -> table map; the individually
// integrated elements' tables stay zero (the device fills them), A is an
// empty n x n pattern and b zeros (no row gather, no symmetrisation).
Assembled assemble(const Space& s, const ProblemConfig& prob, const QuadConfig& q,
                   int threads, bool numeric = true);

// ------------------------------------------------------- 2D quadrature ----
struct QuadRule2 {
  std::vector<double> px, py, w, nx, ny;
  size_t size() const { return w.size(); }
};
void gauss_legendre(int q, std::vector<double>& nodes, std::vector<double>& weights);
QuadRule2 volume_rule2(const LevelSet& ls, const double* lo, const double* hi, ElemTag tag,
                       const QuadConfig& cfg);
QuadRule2 boundary_rule2(const LevelSet& ls, const double* lo, const double* hi,
                         const QuadConfig& cfg);
QuadRule2 side_rule2(const LevelSet& ls, const double* lo, const double* hi, int side,
                     const QuadConfig& cfg);

// --------------------------------------------------------- hierarchy ------

Csr restriction_matrix(const Space& fine, const Space& coarse);

struct Blocks {
  std::vector<int32_t> owners;
  std::vector<int32_t> ptr{0};
  std::vector<int32_t> dofs;
  std::vector<int64_t> fptr{0};
  std::vector<double> fac;  // s x s column-major lower factors
  int max_nk = 0;
  int64_t filtered_dofs = 0;
  std::vector<int32_t> color;  // multiplicative sweeps: colour per block (pre-filter)
  int n_colors = 0;
};
Blocks select_blocks(const Space& s, int threads);
int max_blocks_per_element(const Blocks& b, const Space& s);
// Greedy colouring in block (owner) order; blocks are adjacent when the
// physical supports of their members share an element (smoothers.cpp:99-122).
// supp(d, f) calls f(e) for every element of DOF d's physical support.
template <typename SuppFn>
void color_blocks(Blocks& b, int n_elements, SuppFn supp) {
  constexpr int kW = 8;  // up to 512 colours
  std::vector<uint64_t> used(static_cast<size_t>(n_elements) * kW, 0);
  const int nb = static_cast<int>(b.owners.size());
  b.color.assign(static_cast<size_t>(nb), 0);
  b.n_colors = 0;
  std::vector<int> els;
  for (int k = 0; k < nb; ++k) {
    els.clear();
    for (int32_t q = b.ptr[k]; q < b.ptr[k + 1]; ++q) supp(b.dofs[q], [&](int e) { els.push_back(e); });
    uint64_t m[kW] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int e : els)
      for (int w = 0; w < kW; ++w) m[w] |= used[static_cast<size_t>(e) * kW + w];
    int col = 0;
    while (col < kW * 64 && ((m[col >> 6] >> (col & 63)) & 1u)) ++col;
    if (col >= kW * 64) throw std::runtime_error("color_blocks: more than 512 colours");
    b.color[k] = col;
    b.n_colors = std::max(b.n_colors, col + 1);
    for (int e : els) used[static_cast<size_t>(e) * kW + (col >> 6)] |= uint64_t(1) << (col & 63);
  }
}
void factorize_blocks(const Csr& A, Blocks& b, double filter_ratio, int threads);

// LAPACK dpstrf('L') restatement (unblocked dpstf2 order).  a: n x n col-major,
// overwritten with L in its lower triangle; piv 1-based; returns rank.
int pstrf_lower(int n, double* a, int32_t* piv, double tol);

}  // namespace igh
