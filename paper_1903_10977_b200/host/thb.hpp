// THB spaces on trimmed hierarchical 2D meshes (see thb.cpp).
#pragma once

#include <array>
#include <map>
#include <memory>
#include <set>
#include <vector>

#include "host.hpp"

namespace igh {

// HierarchicalMesh (proj/include/immergrid/mesh.hpp:51-76): active cells per
// level in std::set order ((ix, iy) lexicographic), level m cells of size
// extent / (res << m).
struct HMesh {
  Grid g;
  std::vector<std::set<std::pair<int, int>>> lv;
  static HMesh uniform(const Grid& g);
  int max_level() const { return static_cast<int>(lv.size()) - 1; }
  int cells_x(int l) const { return g.res[0] << l; }
  int cells_y(int l) const { return g.res[1] << l; }
  bool active(int l, int ix, int iy) const;
  std::vector<std::array<int, 3>> elements() const;  // sorted (level, ix, iy)
  void cell_box(int l, int ix, int iy, double* lo, double* hi) const;
  void refine(const std::vector<std::array<int, 3>>& targets);
  void refine_by_box(const double* box);  // x0, y0, x1, y1
  void refine_near_circle(double cx, double cy, double r, double dist);
};
HMesh coarsen(const HMesh& fine);

// General (per-element extraction) 2D spline space; built for THB.
struct GSpace {
  HMesh mesh;
  LevelSet ls;
  int p = 2;
  int classify_depth = 2;
  struct El {
    int l = 0, ix = 0, iy = 0;
    uint8_t tag = kInside;
    std::vector<int32_t> anchors;  // kept indices, in the reference's row order
    std::vector<double> E;         // rows x (p+1)^2 Bernstein coefficients, x fastest
  };
  std::vector<El> el;  // Inside/Cut elements with rows, sorted (level, ix, iy)
  std::map<std::array<int, 3>, int> el_index;
  std::vector<std::array<int, 3>> anchors;  // kept (level, ax, ay)
  std::vector<std::vector<int32_t>> supp;   // per kept anchor, ascending element index
  // THB bookkeeping (basis.cpp:14-34 SpaceData)
  std::vector<int> fn_nx, fn_ny;
  std::vector<std::vector<double>> knx, kny;
  std::vector<std::vector<uint8_t>> active_fn;
  std::vector<std::vector<int>> ordinal;
  std::vector<std::array<int, 3>> all_anchors;
  std::vector<int> kept;
  struct Chain {
    int fi0 = 0, fj0 = 0;
    Mat C;
  };
  std::vector<Chain> chains;
  int n() const { return static_cast<int>(anchors.size()); }
  int element_index(int l, int ix, int iy) const;
};

std::unique_ptr<GSpace> build_thb(const HMesh& mesh, const LevelSet& ls, int p, int classify_depth, int threads);
Assembled assemble_g(const GSpace& s, const ProblemConfig& prob, const QuadConfig& qc, int threads);
Csr restriction_thb(const GSpace& fine, const GSpace& coarse, int threads);
Blocks select_blocks_g(const GSpace& s);
int max_blocks_per_element_g(const Blocks& b, const GSpace& s);

}  // namespace igh
