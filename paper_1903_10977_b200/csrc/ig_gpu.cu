// ig_gpu.cu — host side of the B200 solve phase behind the C-ABI of
// include/ig_gpu.h: device layouts built from the boundary payload, the
// V-cycle and PCG launch sequences, and the CUDA graph that runs the whole PCG
// loop device-side (conditional WHILE node, no host round trips).
//
// Reference semantics followed (file:line in /root/reference/proj):
//   pcg                 src/solvers.cpp:17-71
//   MgHierarchy::vcycle_at src/multigrid.cpp:90-108
//   coarse_solve        src/multigrid.cpp:77-88
//   Smoother::apply(AS) src/smoothers.cpp:174-184
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <utility>
#include <vector>

#include "ig_gpu.h"
#include "kernels.cuh"
#include "spmv_psell.cuh"
#include "galerkin.cuh"
#include "blockfac.cuh"
#include "assemble.cuh"
#include "cutquad.cuh"
#include "cutquad2.cuh"

using namespace igk;

namespace {

thread_local std::string g_err;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(call)                                                                             \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      throw Error(IG_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_) + " (" + \
                                     __FILE__ + ":" + std::to_string(__LINE__) + ")");       \
  } while (0)

inline unsigned grid_of(int64_t n) { return static_cast<unsigned>((n + kCta - 1) / kCta); }

// Options (include/ig_gpu.h IG_OPT_*).  ig_set_option writes the process-wide
// DEFAULTS; every handle snapshots them at ig_hier_create (ig_hier::opt) and
// ig_hier_set_option changes the runtime ones of one handle, so handles built
// with different options coexist and run concurrently.  Code below reads
// opt(): the options of the handle whose API call is running on this thread
// (OptScope), else the defaults (handle-free entry points).
struct Opts {
  int use_graph = 1;     // CUDA-graph PCG / V-cycle (0: host-launched kernels)
  int use_pdl = 1;       // programmatic dependent launch for every kernel (kernels.cuh: pdl_entry)
  int use_dict = 1;      // row dictionary in the SELL layout
  int small_rows = 12000;  // matrices up to this many rows use k_spmv_grp (profiles/option_sweep.py)
  int red_ctas = 8;      // CTAs per SM of the canonical-reduction kernels (profiles/option_sweep.py 13)
  int use_psell = 1;     // pattern SELL above small_rows
  int psell_pairs = 1;   // FAST slices with two rows per lane (x reuse across a column run)
  int32_t psell_pairs_rows = 100000;  // ... for matrices with at least this many rows (below, one row per lane:
                                      // a 38k-row level is a fraction of a wave of warps and the pair slices'
                                      // longer dependent chains cost more than their x reuse saves -- C4 level 3
                                      // 58.0 -> 47.0 us per V-cycle; level 4, 267k rows, 120 -> 149 us without pairs)
  // Occupancy cap of the pattern-SELL kernels (CTAs per SM, 0 = registers
  // decide), applied as unused dynamic shared memory.
  int psell_ctas = 0;
  int psell_ctab = 1;    // FAST2 value sequences from a constant-bank table
  int psell_lines2 = 1;  // FAST4 slices (two x-lines per slice)
  int psell_multi = 1;   // FAST2M slices (row pairs of up to four short runs per slice)
  int psell_rows4 = 1;   // FAST8 slices (four rows of each of two x-lines per lane)
  int32_t psell_rows4_rows = 1000000;  // ... for matrices with at least this many rows: below, a product is
                                       // less than one wave of warps and bound by the slice's dependent chain
                                       // (C4 level 4, 267k rows: 138.7 -> 122.5 us per V-cycle with FAST4 there)
  int32_t psell_edge_rows = 100000;  // FASTE slices (edge-compacted x) for square matrices with at least this many rows (0 = off)
  int psell_order = 1;   // slices launched by class (GENERAL spread through the two-line slices, multi-piece, rest)
                         // instead of row order (0); 2: GENERAL first
  int psell_ab = 1;      // FASTAB slices (row pairs with one column list, two value sequences: prolongations)
  int gal_short = 1;     // prefetching SpGEMM for B rows <= 32 entries
  // Levels below the finest with at most this many DOFs live in the
  // L2-persisting arena (ig_hier::alloc); 0 = off.  Arena size l2_bytes.
  // Measured (profiles/option_sweep.py 18/19): C4 V-cycle 903 -> 881 us, C3
  // 424 -> 395 us; an arena above the device's persisting maximum (83 MB on
  // B200) thrashes and gains nothing.
  int32_t l2_rows = 300000;
  size_t l2_bytes = size_t(48) << 20;  // (64 MiB: the PCG vector kernels lose the L2 they need -- C4 solve 86.0 vs 84.8 ms)
  // Additive smoother on small levels (profiles/level_costs.py): four lanes
  // per complex DOF up to complex4_rows DOFs; main stream only (no fork /
  // join) up to one_stream_rows DOFs.
  int32_t complex4_rows = 100000;
  int32_t one_stream_rows = 40000;
  // Tolerance mode of the coarse solve: x = P M P^T r with the
  // explicit M = L11^-T L11^-1 (columns from the substitution solves of unit
  // vectors) as one parallel GEMV with FMA -- NOT bit-identical to the
  // substitution order; validated against the sequential-order oracle at the
  // north-star tolerances (tests/test_gpu_fast_mode.py).  Off by default.
  int fast_coarse = 0;
  // Tolerance mode of the additive smoother's block solves: the factor slots
  // hold the lower triangle of the explicit inverse M_b = (L_b L_b^T)^-1
  // (columns from the oracle-order substitutions of unit vectors) and the
  // kernels apply y = M_b r_b (FMA, ascending j) instead of the substitutions.
  int fast_blocks = 0;
};
Opts g_defaults;
thread_local const Opts* t_opts = nullptr;
inline const Opts& opt() { return t_opts ? *t_opts : g_defaults; }
struct OptScope {
  const Opts* prev;
  explicit OptScope(const Opts* o) : prev(t_opts) { t_opts = o; }
  ~OptScope() { t_opts = prev; }
};

// Every kernel launch of the library: cudaLaunchKernelEx with programmatic
// stream serialization, so consecutive kernels on a stream (and in the
// captured graphs) overlap launch latency with the predecessor's execution.
template <typename... KArgs, typename... Args>
void launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = opt().use_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (e != cudaSuccess) throw Error(IG_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(e));
}

// Host image of a SELL-32 matrix with its row dictionary (kernels.cuh: Sell).
struct HostSell {
  int32_t nr = 0, nc = 0;
  std::vector<int64_t> slice_ptr;
  std::vector<int32_t> rowinfo;
  std::vector<double> val;
  std::vector<int32_t> col;
  int32_t dict_w = 1;
  std::vector<double> dval;
  std::vector<int32_t> doff;
  int64_t explicit_vals = 0;  // nnz whose value is read from HBM
  int64_t explicit_cols = 0;  // nnz whose column is read from HBM
};

constexpr int kDictEntries = 8;

uint64_t fnv(const void* p, size_t bytes, uint64_t h = 1469598103934665603ULL) {
  const unsigned char* c = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < bytes; ++i) h = (h ^ c[i]) * 1099511628211ULL;
  return h;
}

// Up to kDictEntries most frequent bit-exact row patterns (count >= min_count).
template <typename KeyFn, typename EqFn>
std::vector<int32_t> top_patterns(int32_t nr, const std::vector<uint8_t>& eligible, KeyFn key, EqFn eq,
                                  int64_t min_count) {
  std::vector<std::pair<uint64_t, int32_t>> keys;  // (hash, row)
  keys.reserve(static_cast<size_t>(nr));
  for (int32_t i = 0; i < nr; ++i)
    if (eligible[i]) keys.push_back({key(i), i});
  std::sort(keys.begin(), keys.end());
  std::vector<std::pair<int64_t, int32_t>> groups;  // (count, representative row)
  for (size_t a = 0; a < keys.size();) {
    size_t b = a;
    while (b < keys.size() && keys[b].first == keys[a].first) ++b;
    int64_t c = 0;
    for (size_t k = a; k < b; ++k) c += eq(keys[k].second, keys[a].second) ? 1 : 0;
    groups.push_back({c, keys[a].second});
    a = b;
  }
  std::sort(groups.begin(), groups.end(), [](const auto& x, const auto& y) {
    return x.first != y.first ? x.first > y.first : x.second < y.second;
  });
  std::vector<int32_t> reps;
  for (const auto& g : groups) {
    if (static_cast<int>(reps.size()) >= kDictEntries || g.first < min_count) break;
    reps.push_back(g.second);
  }
  return reps;
}

HostSell to_sell(int32_t nr, int32_t nc, const int32_t* ptr, const int32_t* col, const double* val) {
  HostSell s;
  s.nr = nr;
  s.nc = nc;
  const int32_t nslice = (nr + kSell - 1) / kSell;
  s.slice_ptr.assign(static_cast<size_t>(nslice) + 1, 0);
  s.rowinfo.assign(static_cast<size_t>(std::max(nr, 1)), 0);
  auto len = [&](int32_t i) { return ptr[i + 1] - ptr[i]; };
  for (int32_t i = 0; i < nr; ++i)
    if (len(i) > 0xffff) throw Error(IG_UNSUPPORTED, "SELL: row longer than 65535 entries");
  for (int32_t sl = 0; sl < nslice; ++sl) {
    int32_t w = 0;
    for (int32_t i = sl * kSell; i < std::min(nr, (sl + 1) * kSell); ++i) w = std::max(w, len(i));
    s.slice_ptr[sl + 1] = s.slice_ptr[sl] + static_cast<int64_t>(w) * kSell;
  }
  const int64_t slots = s.slice_ptr[nslice];
  s.val.assign(static_cast<size_t>(std::max<int64_t>(slots, 1)), 0.0);
  s.col.assign(static_cast<size_t>(std::max<int64_t>(slots, 1)), 0);
  for (int32_t i = 0; i < nr; ++i) {
    const int64_t base = s.slice_ptr[i / kSell] + (i % kSell);
    for (int32_t k = 0; k < len(i); ++k) {
      s.val[base + static_cast<int64_t>(k) * kSell] = val[ptr[i] + k];
      s.col[base + static_cast<int64_t>(k) * kSell] = col[ptr[i] + k];
    }
  }
  // Row dictionary: value sequences, then column-offset patterns among them.
  std::vector<int32_t> vd(static_cast<size_t>(std::max(nr, 1)), 0), od(static_cast<size_t>(std::max(nr, 1)), 0);
  std::vector<int32_t> vreps, oreps;
  if (opt().use_dict && nr >= 256) {
    const int64_t min_count = std::max<int64_t>(64, nr / 200);
    std::vector<uint8_t> all(static_cast<size_t>(nr), 1);
    auto vkey = [&](int32_t i) {
      const uint64_t l = static_cast<uint64_t>(len(i));
      return fnv(val + ptr[i], sizeof(double) * static_cast<size_t>(len(i)), fnv(&l, sizeof(l)));
    };
    auto veq = [&](int32_t a, int32_t b) {
      return len(a) == len(b) && std::memcmp(val + ptr[a], val + ptr[b], sizeof(double) * len(a)) == 0;
    };
    vreps = top_patterns(nr, all, vkey, veq, min_count);
    for (int32_t i = 0; i < nr; ++i)
      for (size_t e = 0; e < vreps.size(); ++e)
        if (veq(i, vreps[e])) {
          vd[i] = static_cast<int32_t>(e) + 1;
          break;
        }
    std::vector<uint8_t> has_v(static_cast<size_t>(nr), 0);
    for (int32_t i = 0; i < nr; ++i) has_v[i] = vd[i] > 0;
    auto off_eq = [&](int32_t a, int32_t b) {
      if (len(a) != len(b)) return false;
      for (int32_t k = 0; k < len(a); ++k)
        if (col[ptr[a] + k] - a != col[ptr[b] + k] - b) return false;
      return true;
    };
    auto okey = [&](int32_t i) {
      uint64_t h = fnv(&vd[i], sizeof(int32_t));
      for (int32_t k = 0; k < len(i); ++k) {
        const int32_t o = col[ptr[i] + k] - i;
        h = fnv(&o, sizeof(o), h);
      }
      return h;
    };
    auto oeq = [&](int32_t a, int32_t b) { return vd[a] == vd[b] && off_eq(a, b); };
    oreps = top_patterns(nr, has_v, okey, oeq, min_count);
    for (int32_t i = 0; i < nr; ++i) {
      if (!has_v[i]) continue;
      for (size_t e = 0; e < oreps.size(); ++e)
        if (off_eq(i, oreps[e])) {
          od[i] = static_cast<int32_t>(e) + 1;
          break;
        }
    }
  }
  int32_t W = 1;
  for (int32_t r : vreps) W = std::max(W, len(r));
  s.dict_w = W;
  s.dval.assign(static_cast<size_t>(W) * std::max<size_t>(vreps.size(), 1), 0.0);
  s.doff.assign(static_cast<size_t>(W) * std::max<size_t>(oreps.size(), 1), 0);
  for (size_t e = 0; e < vreps.size(); ++e)
    for (int32_t k = 0; k < len(vreps[e]); ++k) s.dval[e * W + k] = val[ptr[vreps[e]] + k];
  for (size_t e = 0; e < oreps.size(); ++e)
    for (int32_t k = 0; k < len(oreps[e]); ++k) s.doff[e * W + k] = col[ptr[oreps[e]] + k] - oreps[e];
  for (int32_t i = 0; i < nr; ++i) {
    s.rowinfo[i] = len(i) | (vd[i] << 16) | (od[i] << 24);
    if (!vd[i]) s.explicit_vals += len(i);
    if (!od[i]) s.explicit_cols += len(i);
  }
  return s;
}

// ------------------------------------------------ pattern SELL (host) ------
// Host image of spmv_psell.cuh's PSell.  See that header for the layout.
size_t psell_smem() {
  const int c = opt().psell_ctas;
  if (c <= 0) return 0;
  return static_cast<size_t>(std::max(0, 233472 / c - 1024 - 1024)) & ~size_t(1023);
}
constexpr int kPDictEntries = 32;
constexpr int kPMinRun = 8;  // shorter runs of identical rows go to GENERAL slices

struct HostPSell {
  std::vector<int2> seg;  // FAST2 segment lists: (first offset, run length), m = 0 terminates
  std::vector<PSliceMeta> meta;
  std::vector<int32_t> rlist;
  std::vector<uint32_t> ginfo;
  std::vector<double> V;
  std::vector<int32_t> O;
  int32_t dict_w = 2;
  int32_t smul = 1, sshift = 0;
  int64_t layout_bytes = 0;  // matrix words read from HBM per product (shared sequences once)
  int64_t n_fast = 0, n_general = 0, fast_rows = 0;
  std::vector<int4> useg;    // FAST4 union segment lists (header {D, n}, then {o, m, vA, vB})
  int64_t n_fast4 = 0;
  int64_t n_fast2m = 0;      // FAST2M slices (their tables live in useg too)
  int64_t n_fastab = 0;      // FASTAB slices
  int64_t n_fast8 = 0;       // FAST8 slices
  int64_t n_faste = 0;       // FASTE slices
  std::vector<int32_t> G;    // FASTE: xe[i] = x[G[i]] (the edge-compacted copy of x, gathered before the product)
  std::vector<double> tab;   // constant-bank value table (spmv_psell.cuh PValTab)
  int64_t tab_rows = 0;      // rows whose FAST2 values come from the table
};

// Host-side data-parallel loop over [0, n) in contiguous ranges (layout
// construction of the large levels; results do not depend on the split).
template <typename F>
void parallel_rows(int32_t n, F fn) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 65536 || hw == 1) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> th;
  const int32_t step = (n + static_cast<int32_t>(hw) - 1) / static_cast<int32_t>(hw);
  for (unsigned t = 0; t < hw; ++t) {
    const int32_t a = static_cast<int32_t>(t) * step, b = std::min(n, a + step);
    if (a < b) th.emplace_back(fn, a, b);
  }
  for (auto& x : th) x.join();
}

inline uint64_t mix64(uint64_t h, uint64_t w) {
  h ^= w + 0x9E3779B97F4A7C15ULL + (h << 6) + (h >> 2);
  return h * 0xff51afd7ed558ccdULL;
}

// Content hash of a CSR operator (sizes, row pointers, columns, value bits):
// fixed 65536-row chunks hashed in parallel, combined in chunk order, so the
// value does not depend on the thread count.
uint64_t csr_hash(const ig_csr& a) {
  constexpr int32_t kRows = 4096;
  const int32_t nr = a.n_rows;
  const int32_t nch = (nr + kRows - 1) / kRows;
  std::vector<uint64_t> part(static_cast<size_t>(std::max(nch, 1)), 0);
  auto work = [&](int32_t c0, int32_t c1) {
    for (int32_t c = c0; c < c1; ++c) {
      uint64_t h = 0x243F6A8885A308D3ULL + static_cast<uint64_t>(c);
      const int32_t r0 = c * kRows, r1 = std::min(nr, r0 + kRows);
      for (int32_t i = r0; i < r1; ++i) {
        h = mix64(h, static_cast<uint64_t>(a.row_ptr[i + 1] - a.row_ptr[i]));
        for (int32_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
          uint64_t vb;
          std::memcpy(&vb, &a.val[k], 8);
          h = mix64(h, (static_cast<uint64_t>(static_cast<uint32_t>(a.col_idx[k])) << 32) ^ vb);
        }
      }
      part[c] = h;
    }
  };
  const int32_t hw = static_cast<int32_t>(std::max(1u, std::min(32u, std::thread::hardware_concurrency())));
  if (nch < 16 || hw == 1) {
    work(0, nch);
  } else {
    std::vector<std::thread> th;
    const int32_t step = (nch + hw - 1) / hw;
    for (int32_t t = 0; t < hw; ++t) {
      const int32_t c0 = t * step, c1 = std::min(nch, c0 + step);
      if (c0 < c1) th.emplace_back(work, c0, c1);
    }
    for (auto& x : th) x.join();
  }
  uint64_t h = mix64(static_cast<uint64_t>(a.n_rows), static_cast<uint64_t>(a.n_cols));
  h = mix64(h, static_cast<uint64_t>(a.nnz));
  for (uint64_t p : part) h = mix64(h, p);
  return h;
}

// Returns false when the matrix does not fit the format (row longer than
// kPMaxLen, pools beyond 2^32 entries); the caller keeps the plain SELL.
bool to_psell(int32_t nr, int32_t nc, const int32_t* ptr, const int32_t* col, const double* val, HostPSell& s) {
  auto len = [&](int32_t i) { return ptr[i + 1] - ptr[i]; };
  for (int32_t i = 0; i < nr; ++i)
    if (len(i) > kPMaxLen) return false;
  // Offset base per matrix: the scale (1, 2 or 1/2 of the row index) under
  // which the column-offset sequences repeat most (A: 1, R: 2, P: 1/2).
  std::vector<uint64_t> hv(static_cast<size_t>(nr)), ho(static_cast<size_t>(nr));
  parallel_rows(nr, [&](int32_t i0, int32_t i1) {
    for (int32_t i = i0; i < i1; ++i) {
      uint64_t a = static_cast<uint64_t>(len(i));
      for (int32_t k = ptr[i]; k < ptr[i + 1]; ++k) {
        uint64_t w;
        std::memcpy(&w, val + k, 8);
        a = mix64(a, w);
      }
      hv[i] = a;
    }
  });
  const int cand[3][2] = {{1, 0}, {2, 0}, {1, 1}};
  size_t best_runs = SIZE_MAX, best_oruns = SIZE_MAX;
  std::vector<uint64_t> hcur(static_cast<size_t>(nr));
  for (const auto& c : cand) {
    if (c[0] == 2 && nc < nr) continue;  // scaling up only for wide (restriction-shaped) matrices
    if (c[1] == 1 && nc > nr) continue;
    parallel_rows(nr, [&](int32_t i0, int32_t i1) {
      for (int32_t i = i0; i < i1; ++i) {
        const int64_t b = (static_cast<int64_t>(i) * c[0]) >> c[1];
        uint64_t h = static_cast<uint64_t>(len(i));
        for (int32_t k = ptr[i]; k < ptr[i + 1]; ++k) h = mix64(h, static_cast<uint64_t>(col[k] - b));
        hcur[i] = h;
      }
    });
    size_t runs = 0, oruns = 0;  // consecutive-row changes of the offsets alone (what the scale decides: a
                                 // prolongation's rows alternate two value sequences under every scale), then
                                 // of (values, offsets)
    for (int32_t i = 1; i < nr; ++i) {
      runs += (hv[i] != hv[i - 1] || hcur[i] != hcur[i - 1]) ? 1 : 0;
      oruns += hcur[i] != hcur[i - 1] ? 1 : 0;
    }
    if (oruns < best_oruns || (oruns == best_oruns && runs < best_runs)) {
      best_runs = runs;
      best_oruns = oruns;
      s.smul = c[0];
      s.sshift = c[1];
      ho.swap(hcur);
      hcur.resize(static_cast<size_t>(nr));
    }
  }
  auto base = [&](int32_t i) { return static_cast<int32_t>((static_cast<int64_t>(i) * s.smul) >> s.sshift); };
  auto veq = [&](int32_t a, int32_t b) {
    return len(a) == len(b) && std::memcmp(val + ptr[a], val + ptr[b], sizeof(double) * len(a)) == 0;
  };
  auto oeq = [&](int32_t a, int32_t b) {
    if (len(a) != len(b)) return false;
    const int32_t ba = base(a), bb = base(b);
    for (int32_t k = 0; k < len(a); ++k)
      if (col[ptr[a] + k] - ba != col[ptr[b] + k] - bb) return false;
    return true;
  };
  // Runs of identical consecutive rows.
  std::vector<uint8_t> brk(static_cast<size_t>(nr), 0);
  parallel_rows(nr, [&](int32_t i0, int32_t i1) {
    for (int32_t i = i0; i < i1; ++i)
      brk[i] = (i == 0 || hv[i] != hv[i - 1] || ho[i] != ho[i - 1] || !veq(i, i - 1) || !oeq(i, i - 1)) ? 1 : 0;
  });
  std::vector<int32_t> run_start;
  for (int32_t i = 0; i < nr; ++i)
    if (brk[i]) run_start.push_back(i);
  run_start.push_back(nr);
  std::vector<uint8_t> in_fast(static_cast<size_t>(nr), 0);
  for (size_t r = 0; r + 1 < run_start.size(); ++r)
    if (run_start[r + 1] - run_start[r] >= kPMinRun)
      for (int32_t i = run_start[r]; i < run_start[r + 1]; ++i) in_fast[i] = 1;
  // Global value dictionary (GENERAL rows): the most frequent sequences among
  // the rows left to GENERAL slices, >= 32 rows each.
  std::vector<int32_t> dict_rows;
  {
    std::vector<std::pair<uint64_t, int32_t>> keys;
    for (int32_t i = 0; i < nr; ++i)
      if (!in_fast[i]) keys.push_back({hv[i], i});
    std::sort(keys.begin(), keys.end());
    std::vector<std::pair<int64_t, int32_t>> groups;
    for (size_t a = 0; a < keys.size();) {
      size_t b = a;
      while (b < keys.size() && keys[b].first == keys[a].first) ++b;
      int64_t c = 0;
      for (size_t k = a; k < b; ++k) c += veq(keys[k].second, keys[a].second) ? 1 : 0;
      groups.push_back({c, keys[a].second});
      a = b;
    }
    std::sort(groups.begin(), groups.end(), [](const auto& x, const auto& y) {
      return x.first != y.first ? x.first > y.first : x.second < y.second;
    });
    for (const auto& g : groups) {
      if (static_cast<int>(dict_rows.size()) >= kPDictEntries || g.first < 32) break;
      dict_rows.push_back(g.second);
    }
  }
  int32_t W = 2;
  for (int32_t r : dict_rows) W = std::max(W, len(r));
  W = (W + 1) & ~1;  // entries 16-byte aligned (double2 loads)
  s.dict_w = W;
  s.V.assign(static_cast<size_t>(W) * dict_rows.size(), 0.0);
  for (size_t e = 0; e < dict_rows.size(); ++e)
    std::memcpy(s.V.data() + e * W, val + ptr[dict_rows[e]], sizeof(double) * len(dict_rows[e]));
  s.layout_bytes += static_cast<int64_t>(s.V.size()) * 8;
  auto dict_of = [&](int32_t i) -> int {  // 1-based dictionary entry, 0 = none
    for (size_t e = 0; e < dict_rows.size(); ++e)
      if (hv[i] == hv[dict_rows[e]] && veq(i, dict_rows[e])) return static_cast<int>(e) + 1;
    return 0;
  };
  // Deduplicated stride-1 sequences of FAST slices (16-byte aligned starts).
  std::unordered_map<uint64_t, std::vector<std::pair<uint32_t, int32_t>>> vseq, oseq;  // hash -> (start, row)
  auto v_start = [&](int32_t i) -> uint32_t {
    auto& b = vseq[hv[i]];
    for (const auto& [st, r] : b)
      if (veq(i, r)) return st;
    s.V.resize((s.V.size() + 1) & ~size_t(1), 0.0);
    const uint32_t st = static_cast<uint32_t>(s.V.size());
    s.V.insert(s.V.end(), val + ptr[i], val + ptr[i + 1]);
    s.layout_bytes += 8 * static_cast<int64_t>(len(i));
    b.push_back({st, i});
    return st;
  };
  auto o_start = [&](int32_t i) -> uint32_t {
    auto& b = oseq[ho[i]];
    for (const auto& [st, r] : b)
      if (oeq(i, r)) return st;
    s.O.resize((s.O.size() + 3) & ~size_t(3), 0);
    const uint32_t st = static_cast<uint32_t>(s.O.size());
    for (int32_t k = ptr[i]; k < ptr[i + 1]; ++k) s.O.push_back(col[k] - base(i));
    s.layout_bytes += 4 * static_cast<int64_t>(len(i));
    b.push_back({st, i});
    return st;
  };
  // FAST2 segment list of a row's offsets: maximal runs of consecutive
  // columns, split at 8 entries; deduplicated like the offset sequences.
  std::unordered_map<uint64_t, std::vector<std::pair<uint32_t, int32_t>>> sseq;
  auto seg_start = [&](int32_t i) -> uint32_t {
    auto& b = sseq[ho[i]];
    for (const auto& [st, r] : b)
      if (oeq(i, r)) return st;
    const uint32_t st = static_cast<uint32_t>(s.seg.size());
    const int32_t bi = base(i);
    for (int32_t k = ptr[i]; k < ptr[i + 1];) {
      int32_t m = 1;
      while (k + m < ptr[i + 1] && m < 8 && col[k + m] == col[k] + m) ++m;
      s.seg.push_back(make_int2(col[k] - bi, m));
      k += m;
    }
    s.seg.push_back(make_int2(0, 0));
    s.layout_bytes += 8 * static_cast<int64_t>(s.seg.size() - st);
    b.push_back({st, i});
    return st;
  };
  auto pack = [](int lmax, int count, bool fast, bool ulen, int wv, int wo) {
    return static_cast<uint32_t>(lmax) | static_cast<uint32_t>(count) << 11 | (fast ? 1u << 17 : 0u) |
           (ulen ? 1u << 18 : 0u) | static_cast<uint32_t>(wv) << 19 | static_cast<uint32_t>(wo) << 25;
  };
  int lmax_all = 0;
  // GENERAL slice over the leftover rows g[0..cnt).
  auto emit_general = [&](const std::vector<int32_t>& g) {
    const int cnt = static_cast<int>(g.size());
    int lmax = 0;
    bool ulen = true;
    for (int32_t i : g) {
      lmax = std::max(lmax, len(i));
      ulen = ulen && len(i) == len(g[0]);
    }
    lmax_all = std::max(lmax_all, lmax);
    std::vector<int32_t> opat, vpat;  // representative rows of the table columns
    const uint32_t a = static_cast<uint32_t>(s.rlist.size());
    for (int32_t i : g) {
      int oi = -1;
      for (size_t j = 0; j < opat.size() && len(i) > 0; ++j)  // empty rows: own column (padding is per row)
        if (ho[i] == ho[opat[j]] && oeq(i, opat[j])) {
          oi = static_cast<int>(j);
          break;
        }
      if (oi < 0) {
        oi = static_cast<int>(opat.size());
        opat.push_back(i);
      }
      const int e = dict_of(i);
      int vi = 0;
      if (!e) {
        vi = -1;
        for (size_t j = 0; j < vpat.size(); ++j)
          if (hv[i] == hv[vpat[j]] && veq(i, vpat[j])) {
            vi = static_cast<int>(j);
            break;
          }
        if (vi < 0) {
          vi = static_cast<int>(vpat.size());
          vpat.push_back(i);
        }
      }
      s.rlist.push_back(i);
      s.ginfo.push_back(static_cast<uint32_t>(len(i)) | static_cast<uint32_t>(e) << 11 |
                        static_cast<uint32_t>(vi) << 17 | static_cast<uint32_t>(oi) << 22);
    }
    const int wo = static_cast<int>(opat.size()), wv = static_cast<int>(vpat.size());
    // k-blocked tables, zero-padded to a multiple of 8 entries.
    const size_t l8 = static_cast<size_t>((lmax + 7) & ~7);
    s.O.resize((s.O.size() + 3) & ~size_t(3), 0);
    const uint32_t obase = static_cast<uint32_t>(s.O.size());
    s.O.resize(s.O.size() + l8 * wo, 0);
    for (int j = 0; j < wo; ++j) {
      const int32_t r = opat[j];
      // Padding past the row's end repeats its first offset (gathers stay in
      // x for every row sharing the column); an empty row points at x[0].
      const int32_t pad = len(r) > 0 ? col[ptr[r]] - base(r) : -base(r);
      for (size_t k = 0; k < l8; ++k)
        s.O[obase + (k / 4) * 4 * static_cast<size_t>(wo) + 4 * j + k % 4] =
            static_cast<int32_t>(k) < len(r) ? col[ptr[r] + k] - base(r) : pad;
    }
    s.V.resize((s.V.size() + 1) & ~size_t(1), 0.0);
    const uint32_t vbase = static_cast<uint32_t>(s.V.size());
    s.V.resize(s.V.size() + l8 * wv, 0.0);
    for (int j = 0; j < wv; ++j) {
      const int32_t r = vpat[j];
      for (int32_t k = 0; k < len(r); ++k)
        s.V[vbase + (k / 2) * 2 * static_cast<size_t>(wv) + 2 * j + k % 2] = val[ptr[r] + k];
    }
    s.meta.push_back(PSliceMeta{a, vbase, obase, pack(lmax, cnt, false, ulen, wv, wo)});
    s.layout_bytes += 16 + 8 * static_cast<int64_t>(cnt) + static_cast<int64_t>(l8) * (4 * wo + 8 * wv);
    ++s.n_general;
  };
  // Slices in row order: FAST pieces of the long runs; leftover rows are
  // collected 32 at a time into GENERAL slices.
  // FAST2 / FAST pieces of a run [a, b) (representative row rep: the run's
  // pattern).  FAST2 (unscaled base only: rows r and r+1 then see the same
  // column run shifted by one): pieces of up to 64 rows, an even count; the
  // odd remainder goes to FAST slices.
  // Pair / two-line slices (64 / 128 rows per warp) trade parallelism for x
  // reuse: only matrices with at least psell_pairs_rows rows use them.
  const bool f2ok = opt().psell_pairs && nr >= opt().psell_pairs_rows && s.smul == 1 && s.sshift == 0;
  // FAST2M: pieces that would leave most of a FAST2 slice's lanes idle (the
  // x-line pieces either side of an immersed boundary: 16-60 rows, each with
  // its own column offsets) are pooled per (value sequence, column-run
  // lengths) and packed, up to four pieces and 32 row pairs per slice.  Table
  // in useg: {first rows of the four pieces}, {lane starts s1 | s2 << 8 |
  // s3 << 16, odd-tail mask, segment list (run lengths), runs}, then one int4
  // of piece offsets per column run.  An odd tail is the last lane of a piece
  // owning one row only.
  const bool fmok = f2ok && opt().psell_multi && nr == nc;
  struct Loose { int32_t a, b, rep; };
  struct Pool { uint32_t vb, sg; int32_t len, nseg; std::vector<Loose> q; int lanes = 0; };
  std::map<std::pair<uint32_t, uint64_t>, Pool> pools;  // (value sequence, hash of the run lengths)
  auto flush_pool = [&](Pool& pl) {
    if (pl.q.empty()) return;
    int4 R = make_int4(0, 0, 0, 0), hd = make_int4(0, 0, static_cast<int>(pl.sg), pl.nseg);
    int st[4] = {0, 64, 64, 64}, lanes = 0;
    int32_t* Rp = &R.x;
    std::vector<int4> offs(static_cast<size_t>(pl.nseg), make_int4(0, 0, 0, 0));
    for (size_t k = 0; k < pl.q.size(); ++k) {
      const Loose& L = pl.q[k];
      Rp[k] = L.a;
      st[k] = lanes;
      lanes += (L.b - L.a + 1) / 2;
      if ((L.b - L.a) & 1) hd.y |= 1 << k;
      int u = 0;  // first column of every run of the representative row
      for (int32_t q = ptr[L.rep]; q < ptr[L.rep + 1]; ++u) {
        (&offs[static_cast<size_t>(u)].x)[k] = col[q] - L.rep;
        int32_t m = 1;
        while (q + m < ptr[L.rep + 1] && m < 8 && col[q + m] == col[q] + m) ++m;
        q += m;
      }
      s.fast_rows += L.b - L.a;
    }
    for (size_t k = pl.q.size(); k < 4; ++k) {  // unused pieces repeat the first (never selected)
      Rp[k] = Rp[0];
      for (auto& o : offs) (&o.x)[k] = o.x;
    }
    hd.x = st[1] | st[2] << 8 | st[3] << 16;
    const uint32_t z = static_cast<uint32_t>(s.useg.size());
    s.useg.push_back(R);
    s.useg.push_back(hd);
    s.useg.insert(s.useg.end(), offs.begin(), offs.end());
    s.meta.push_back(PSliceMeta{static_cast<uint32_t>(R.x), pl.vb, z, pack(pl.len, lanes, true, true, 3, 0)});
    s.layout_bytes += 16 + 16 * static_cast<int64_t>(offs.size() + 2);
    ++s.n_fast;
    ++s.n_fast2m;
    pl.q.clear();
    pl.lanes = 0;
  };
  auto pool_piece = [&](int32_t a, int32_t b, int32_t rep, uint32_t vb) {
    uint64_t hs = 0x1234567;
    int32_t nseg = 0;
    for (int32_t q = ptr[rep]; q < ptr[rep + 1]; ++nseg) {
      int32_t m = 1;
      while (q + m < ptr[rep + 1] && m < 8 && col[q + m] == col[q] + m) ++m;
      hs = mix64(hs, static_cast<uint64_t>(m));
      q += m;
    }
    Pool& pl = pools[{vb, hs}];
    if (pl.q.empty() && pl.lanes == 0 && pl.nseg == 0) {
      pl.vb = vb;
      pl.sg = seg_start(rep);
      pl.len = len(rep);
      pl.nseg = nseg;
    }
    while (a < b) {
      const int room = 32 - pl.lanes;
      const int32_t take = std::min(b - a, 2 * room);  // a split leaves an even count behind
      pl.q.push_back(Loose{a, a + take, rep});
      pl.lanes += (take + 1) / 2;
      a += take;
      if (pl.lanes == 32 || pl.q.size() == 4) flush_pool(pl);
    }
  };
  auto emit_piece = [&](int32_t a, int32_t b, int32_t rep) {
    if (b <= a) return;
    lmax_all = std::max(lmax_all, len(rep));
    const uint32_t vb = v_start(rep);
    int32_t i = a;
    if (fmok) {
      // Whole 64-row slices stay FAST2; the remainder (< 56 rows, or odd) is pooled.
      for (; b - i >= 64; i += 64) {
        const uint32_t sg = seg_start(rep);
        s.meta.push_back(PSliceMeta{static_cast<uint32_t>(i), vb, sg, pack(len(rep), 32, true, true, 1, 0)});
        s.layout_bytes += 16;
        ++s.n_fast;
        s.fast_rows += 64;
      }
      const int32_t rem = b - i;
      // (the phantom second row of an odd tail reads x one past the piece's
      // last column run: keep it inside x)
      const bool tail_ok = !(rem & 1) || col[ptr[b - 1 + 1] - 1] + 1 < nc;
      if (rem > 0 && len(rep) > 0 && tail_ok && !(rem >= 56 && !(rem & 1))) {
        pool_piece(i, b, rep, vb);
        return;
      }
    }
    if (f2ok && b - i >= 2) {
      const uint32_t sg = seg_start(rep);
      for (; b - i >= 2;) {
        const int cnt = std::min(64, (b - i) & ~1);
        s.meta.push_back(PSliceMeta{static_cast<uint32_t>(i), vb, sg, pack(len(rep), cnt / 2, true, true, 1, 0)});
        s.layout_bytes += 16;
        ++s.n_fast;
        s.fast_rows += cnt;
        i += cnt;
      }
    }
    if (i < b) {
      const uint32_t ob = o_start(rep);
      for (; i < b; i += 32) {
        const int cnt = std::min(32, b - i);
        s.meta.push_back(PSliceMeta{static_cast<uint32_t>(i), vb, ob, pack(len(rep), cnt, true, true, 0, 0)});
        s.layout_bytes += 16;
        ++s.n_fast;
        s.fast_rows += cnt;
      }
    }
  };
  // FAST4: two x-line runs A = [a0, a1) and B = A + D with the same pattern,
  // where D is the run's first segment stride (the next line).  Their column
  // runs coincide except at the ends (3D p = 2: 30 distinct lines instead of
  // 50), so one slice computes 2 rows of each line per lane from one union
  // segment list (`useg`: header {D, n}, then {offset, m, value index for A
  // or -1, for B or -1}, offsets ascending -- each row still sums its own
  // runs in ascending order).
  const size_t nruns = run_start.size() > 0 ? run_start.size() - 1 : 0;
  std::vector<int32_t> pairB(nruns, -1), pa0(nruns, 0), pa1(nruns, 0), pD(nruns, 0);
  std::vector<uint8_t> is_b(nruns, 0);
  std::vector<int32_t> pairA(nruns, -1);  // B run -> its A run
  int64_t why[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (f2ok && opt().psell_lines2 && nr == nc) {  // square operators only (k_pprolong has no two-line path)
    for (size_t r = 0; r < nruns; ++r) {
      const int32_t r0 = run_start[r], r1 = run_start[r + 1];
      if (r1 - r0 < kPMinRun || is_b[r] || len(r0) < 2) { ++why[0]; continue; }
      // First segment stride: segments = maximal runs of consecutive columns.
      int32_t k = ptr[r0], o0 = col[k] - r0, o1 = 0;
      bool found = false;  // (offsets are negative before the diagonal)
      for (int32_t q = k + 1; q < ptr[r0 + 1]; ++q)
        if (col[q] != col[q - 1] + 1) {
          o1 = col[q] - r0;
          found = true;
          break;
        }
      if (!found) { ++why[1]; continue; }
      // Only rows of many column runs (3D stencils: 25 for p = 2) pay: in 2D
      // (5 runs, 6 after the merge) the slices measured slower (C3 +1.3 %).
      {
        int32_t runs = 1;
        for (int32_t q = k + 1; q < ptr[r0 + 1]; ++q) runs += col[q] != col[q - 1] + 1 ? 1 : 0;
        if (runs < 9) { ++why[1]; continue; }
      }
      const int32_t DD = o1 - o0;
      if (DD <= 0) { ++why[1]; continue; }
      // Partner run: the run containing r0 + DD, same pattern.
      const int32_t tb = r0 + DD;
      if (tb >= nr) { ++why[2]; continue; }
      const size_t rb = static_cast<size_t>(std::upper_bound(run_start.begin(), run_start.end(), tb) - run_start.begin()) - 1;
      if (rb >= nruns || rb == r || is_b[rb] || pairB[rb] >= 0) { ++why[3]; continue; }
      const int32_t b0 = run_start[rb], b1 = run_start[rb + 1];
      if (b1 - b0 < kPMinRun) { ++why[4]; continue; }
      if (hv[b0] != hv[r0] || ho[b0] != ho[r0] || !veq(b0, r0) || !oeq(b0, r0)) { ++why[5]; continue; }
      const int32_t a0 = std::max(r0, b0 - DD), a1 = std::min(r1, b1 - DD);
      if (a1 - a0 < 16) { ++why[6]; continue; }
      ++why[7];
      pairB[r] = static_cast<int32_t>(rb);
      pa0[r] = a0;
      // (FAST8 slices take whole groups of four rows per line; FAST4 pairs)
      pa1[r] = a0 + ((a1 - a0) & (opt().psell_rows4 && nr >= opt().psell_rows4_rows && a1 - a0 >= 32 ? ~3 : ~1));
      pD[r] = DD;
      is_b[rb] = 1;
      pairA[rb] = static_cast<int32_t>(r);
    }
  }
  if (std::getenv("IG_TIMING"))
    std::fprintf(stderr, "[psell pairs] f2ok=%d lines2=%d runs=%zu: skipped %lld, no 2nd run %lld, past end %lld, partner taken %lld, partner short %lld, pattern differs %lld, overlap < 16 %lld, paired %lld\n",
                 f2ok ? 1 : 0, opt().psell_lines2, nruns, (long long)why[0], (long long)why[1], (long long)why[2], (long long)why[3],
                 (long long)why[4], (long long)why[5], (long long)why[6], (long long)why[7]);
  std::map<std::pair<uint32_t, int32_t>, uint32_t> useg_of;  // (segment list, D) -> union list
  auto union_start = [&](int32_t rep, int32_t D) -> uint32_t {
    const uint32_t sg = seg_start(rep);
    auto it = useg_of.find({sg, D});
    if (it != useg_of.end()) return it->second;
    std::vector<int4> ent;
    int32_t cum = 0;
    std::vector<int4> a, b;
    for (uint32_t q = sg; s.seg[q].y != 0; ++q) {
      a.push_back(make_int4(s.seg[q].x, s.seg[q].y, cum, -1));
      b.push_back(make_int4(s.seg[q].x + D, s.seg[q].y, -1, cum));
      cum += s.seg[q].y;
    }
    size_t ia = 0, ib = 0;
    while (ia < a.size() || ib < b.size()) {
      if (ib == b.size() || (ia < a.size() && a[ia].x < b[ib].x)) {
        ent.push_back(a[ia++]);
      } else if (ia == a.size() || b[ib].x < a[ia].x) {
        ent.push_back(b[ib++]);
      } else if (a[ia].y == b[ib].y) {  // shared column run
        ent.push_back(make_int4(a[ia].x, a[ia].y, a[ia].z, b[ib].w));
        ++ia;
        ++ib;
      } else {
        ent.push_back(a[ia++]);
      }
    }
    const uint32_t st = static_cast<uint32_t>(s.useg.size());
    s.useg.push_back(make_int4(D, static_cast<int>(ent.size()), 0, 0));
    s.useg.insert(s.useg.end(), ent.begin(), ent.end());
    s.layout_bytes += 16 * static_cast<int64_t>(ent.size() + 1);
    useg_of[{sg, D}] = st;
    return st;
  };
  // FASTAB (half-scaled base only, i.e. prolongation-shaped matrices): items
  // = consecutive rows (r, r + 1) with the SAME column list; runs of items
  // whose first rows share one value sequence, whose second rows share
  // another, and whose columns advance by one per item (offsets against
  // base(r) = r >> 1 constant).  One lane per item: every x is gathered once
  // for both rows.  Values interleaved {A_k, B_k}.
  std::vector<uint8_t> claimed(static_cast<size_t>(nr), 0);
  if (opt().psell_ab && s.smul == 1 && s.sshift == 1) {
    auto ceq = [&](int32_t a, int32_t b) {
      return len(a) == len(b) && len(a) > 0 &&
             std::memcmp(col + ptr[a], col + ptr[b], sizeof(int32_t) * static_cast<size_t>(len(a))) == 0;
    };
    std::vector<int32_t> items;  // first rows
    for (int32_t i = 0; i + 1 < nr;) {
      if (!in_fast[i] && !in_fast[i + 1] && ceq(i, i + 1)) {
        items.push_back(i);
        i += 2;
      } else {
        ++i;
      }
    }
    std::map<std::pair<uint64_t, uint64_t>, std::vector<std::pair<uint32_t, int32_t>>> abseq;  // -> (start, first row)
    auto ab_start = [&](int32_t i) -> uint32_t {
      auto& b = abseq[{hv[i], hv[i + 1]}];
      for (const auto& [st, r] : b)
        if (veq(i, r) && veq(i + 1, r + 1)) return st;
      s.V.resize((s.V.size() + 1) & ~size_t(1), 0.0);
      const uint32_t st = static_cast<uint32_t>(s.V.size());
      for (int32_t k = 0; k < len(i); ++k) {
        s.V.push_back(val[ptr[i] + k]);
        s.V.push_back(val[ptr[i + 1] + k]);
      }
      s.layout_bytes += 16 * static_cast<int64_t>(len(i));
      b.push_back({st, i});
      return st;
    };
    for (size_t a = 0; a < items.size();) {
      size_t b = a + 1;
      const int32_t f = items[a];
      while (b < items.size() && items[b] == items[b - 1] + 2 && hv[items[b]] == hv[f] && hv[items[b] + 1] == hv[f + 1] &&
             ho[items[b]] == ho[f] && veq(items[b], f) && veq(items[b] + 1, f + 1) && oeq(items[b], f))
        ++b;
      if (b - a >= static_cast<size_t>(kPMinRun)) {
        lmax_all = std::max(lmax_all, 2 * len(f));
        const uint32_t vb = ab_start(f), ob = o_start(f);
        for (size_t q = a; q < b; q += 32) {
          const int cnt = static_cast<int>(std::min<size_t>(32, b - q));
          s.meta.push_back(PSliceMeta{static_cast<uint32_t>(items[q]), vb, ob, pack(len(f), cnt, true, true, 4, 0)});
          s.layout_bytes += 16;
          ++s.n_fast;
          ++s.n_fastab;
          s.fast_rows += 2 * cnt;
        }
        for (size_t q = a; q < b; ++q) claimed[items[q]] = claimed[items[q] + 1] = 1;
      }
      a = b;
    }
  }
  // FASTE: leftover rows whose gathers are STRIDED -- the first / last rows of
  // every x-line (a B-spline line's end functions: six value classes in 3D,
  // ~5 % of the rows but ~25 % of the kernel's L1 wavefronts as GENERAL
  // slices, whose 32 lanes touch 10-16 cache lines per gather).  The columns
  // they read form equal-length blocks (the last / first columns of
  // consecutive lines); xe = those blocks transposed (xe[c T + t] = column c
  // of block t), gathered from x by a small kernel before the product.  In
  // xe, rows of one class on consecutive lines read consecutive elements
  // with ONE offset sequence -- also next to an immersed boundary, where the
  // line starts are irregular in x but every line still has its ends -- so
  // they run as FAST-style slices (warp-uniform values and offsets, coalesced
  // gathers).  rlist / ginfo hold each lane's row and its anchor block.
  if (opt().psell_edge_rows > 0 && nr >= opt().psell_edge_rows && nr == nc && s.smul == 1 && s.sshift == 0) {
    constexpr size_t kEdgeMin = 256;  // rows per value class
    constexpr int32_t kEdgeRun = 16;  // consecutive anchors per run
    std::unordered_map<uint64_t, std::vector<int32_t>> cls;
    std::unordered_set<uint64_t> run_values;  // value sequences of the long runs: their stray rows are no edge rows
    for (int32_t i = 0; i < nr; ++i)
      if (in_fast[i] && brk[i]) run_values.insert(hv[i]);
    for (int32_t i = 0; i < nr; ++i)
      if (!in_fast[i] && !claimed[i] && len(i) > 0 && !run_values.count(hv[i])) cls[hv[i]].push_back(i);
    std::vector<int32_t> fam;
    for (auto& kv : cls) {
      if (kv.second.size() < kEdgeMin) continue;
      for (int32_t r : kv.second)
        if (veq(r, kv.second[0])) fam.push_back(r);
    }
    std::sort(fam.begin(), fam.end());
    if (static_cast<int64_t>(fam.size()) * 50 >= nr) {  // at least 2 % of the rows
      std::vector<uint8_t> used(static_cast<size_t>(nc), 0);
      for (int32_t r : fam)
        for (int32_t k = ptr[r]; k < ptr[r + 1]; ++k) used[col[k]] = 1;
      std::vector<int32_t> bstart, blen;
      std::map<int32_t, int64_t> hist;
      int64_t total = 0;
      for (int32_t j = 0; j < nc;) {
        if (!used[j]) {
          ++j;
          continue;
        }
        const int32_t j0 = j;
        while (j < nc && used[j]) ++j;
        bstart.push_back(j0);
        blen.push_back(j - j0);
        hist[j - j0] += j - j0;
        total += j - j0;
      }
      int32_t Wb = 0;
      int64_t cov = 0;
      for (const auto& [w, c] : hist)
        if (c > cov) {
          cov = c;
          Wb = w;
        }
      if (std::getenv("IG_TIMING"))
        std::fprintf(stderr, "[psell edge] family %zu rows, %zu column blocks, modal length %d covering %lld of %lld columns\n",
                     fam.size(), bstart.size(), Wb, static_cast<long long>(cov), static_cast<long long>(total));
      if (Wb >= 2 && Wb <= 64 && cov * 2 >= total) {
        std::vector<int32_t> tof(static_cast<size_t>(nc), -1);
        std::vector<uint8_t> cof(static_cast<size_t>(nc), 0);
        int32_t T = 0;
        for (size_t b = 0; b < bstart.size(); ++b)
          if (blen[b] == Wb) {
            for (int32_t c = 0; c < Wb; ++c) {
              tof[bstart[b] + c] = T;
              cof[bstart[b] + c] = static_cast<uint8_t>(c);
            }
            ++T;
          }
        struct ER {
          uint64_t key;
          int32_t ta, row;
        };
        std::vector<ER> er;
        auto xoff = [&](int32_t r, int32_t k, int32_t ta) {  // offset of entry k of row r in xe, against its anchor
          const int32_t c = col[ptr[r] + k];
          return static_cast<int32_t>(cof[c]) * T + (tof[c] - ta);
        };
        for (int32_t r : fam) {
          bool ok = true;
          for (int32_t k = ptr[r]; k < ptr[r + 1] && ok; ++k) ok = tof[col[k]] >= 0;
          if (!ok) continue;
          const int32_t ta = tof[col[ptr[r]]];
          uint64_t h = mix64(hv[r], 0xE5);
          for (int32_t k = 0; k < len(r); ++k) h = mix64(h, static_cast<uint64_t>(static_cast<uint32_t>(xoff(r, k, ta))));
          er.push_back(ER{h, ta, r});
        }
        std::sort(er.begin(), er.end(), [](const ER& a, const ER& b) {
          return a.key != b.key ? a.key < b.key : a.ta != b.ta ? a.ta < b.ta : a.row < b.row;
        });
        std::unordered_map<uint64_t, std::vector<std::pair<uint32_t, int32_t>>> eseq;  // key -> (O start, row)
        auto same = [&](const ER& a, const ER& b) {  // values and xe offsets equal
          if (a.key != b.key || !veq(a.row, b.row)) return false;
          for (int32_t k = 0; k < len(a.row); ++k)
            if (xoff(a.row, k, a.ta) != xoff(b.row, k, b.ta)) return false;
          return true;
        };
        for (size_t a = 0; a < er.size();) {
          size_t b = a + 1;
          while (b < er.size() && er[b].ta == er[b - 1].ta + 1 && same(er[a], er[b])) ++b;
          if (b - a >= static_cast<size_t>(kEdgeRun)) {
            const int32_t rep = er[a].row;
            lmax_all = std::max(lmax_all, len(rep));
            const uint32_t vb = v_start(rep);
            uint32_t ob = 0;
            {
              auto& bk = eseq[er[a].key];
              bool found = false;
              for (const auto& [st, r0] : bk) {
                ER t{er[a].key, tof[col[ptr[r0]]], r0};
                if (same(er[a], t)) {
                  ob = st;
                  found = true;
                  break;
                }
              }
              if (!found) {
                s.O.resize((s.O.size() + 3) & ~size_t(3), 0);
                ob = static_cast<uint32_t>(s.O.size());
                for (int32_t k = 0; k < len(rep); ++k) s.O.push_back(xoff(rep, k, er[a].ta));
                s.layout_bytes += 4 * static_cast<int64_t>(len(rep));
                bk.push_back({ob, rep});
              }
            }
            for (size_t q = a; q < b; q += 32) {
              const int cnt = static_cast<int>(std::min<size_t>(32, b - q));
              const uint32_t at = static_cast<uint32_t>(s.rlist.size());
              for (int u = 0; u < cnt; ++u) {
                s.rlist.push_back(er[q + u].row);
                s.ginfo.push_back(static_cast<uint32_t>(er[q + u].ta));
                claimed[er[q + u].row] = 1;
              }
              s.meta.push_back(PSliceMeta{at, vb, ob, pack(len(rep), cnt, false, false, 0, 0) | 1u << 31});
              s.layout_bytes += 16 + 8 * static_cast<int64_t>(cnt);
              ++s.n_faste;
              s.fast_rows += cnt;
            }
          }
          a = b;
        }
        if (s.n_faste > 0) {
          s.G.assign(static_cast<size_t>(Wb) * T, 0);
          for (size_t b2 = 0, t = 0; b2 < bstart.size(); ++b2)
            if (blen[b2] == Wb) {
              for (int32_t c = 0; c < Wb; ++c) s.G[static_cast<size_t>(c) * T + t] = bstart[b2] + c;
              ++t;
            }
          s.layout_bytes += 20 * static_cast<int64_t>(s.G.size());  // gather list + xe written and read
        }
      }
    }
  }
  if (std::getenv("IG_TIMING"))
    std::fprintf(stderr, "[psell base] %d x %d: smul %d sshift %d, %lld FASTAB slices, %lld FASTE slices (xe %zu)\n", nr, nc,
                 s.smul, s.sshift, static_cast<long long>(s.n_fastab), static_cast<long long>(s.n_faste), s.G.size());
  std::vector<int32_t> pending;
  for (size_t r = 0; r < nruns; ++r) {
    const int32_t r0 = run_start[r], r1 = run_start[r + 1];
    if (r1 - r0 < kPMinRun) {
      for (int32_t i = r0; i < r1; ++i) {
        if (claimed[i]) continue;
        pending.push_back(i);
        if (pending.size() == 32) {
          emit_general(pending);
          pending.clear();
        }
      }
      continue;
    }
    // Rows of this run already computed as the B line of an earlier pair.
    int32_t c0 = r1, c1 = r1;
    if (is_b[r]) {
      const int32_t q = pairA[r];
      c0 = pa0[q] + pD[q];
      c1 = pa1[q] + pD[q];
    }
    if (pairB[r] >= 0) {
      const int32_t a0 = pa0[r], a1 = pa1[r];
      // (a run used as A is never a B: is_b[r] == 0 here)
      emit_piece(r0, a0, r0);
      const uint32_t vb = v_start(r0);
      const uint32_t ug = union_start(r0, pD[r]);
      lmax_all = std::max(lmax_all, len(r0));
      const bool rows4 = opt().psell_rows4 && nr >= opt().psell_rows4_rows && a1 - a0 >= 32 && (a1 - a0) % 4 == 0;
      for (int32_t i = a0; i < a1;) {
        const int cnt = std::min(rows4 ? 128 : 64, a1 - i);
        s.meta.push_back(PSliceMeta{static_cast<uint32_t>(i), vb, ug,
                                    pack(len(r0), rows4 ? cnt / 4 : cnt / 2, true, true, rows4 ? 5 : 2, 0)});
        s.layout_bytes += 16;
        ++s.n_fast;
        s.fast_rows += 2 * cnt;
        ++s.n_fast4;
        if (rows4) ++s.n_fast8;
        i += cnt;
      }
      emit_piece(a1, r1, r0);
    } else if (is_b[r]) {
      emit_piece(r0, c0, r0);
      emit_piece(c1, r1, r0);
    } else {
      emit_piece(r0, r1, r0);
    }
    if (s.V.size() > 0xF0000000ull || s.O.size() > 0xF0000000ull) return false;
  }
  for (auto& kv : pools) flush_pool(kv.second);
  if (!pending.empty()) emit_general(pending);
  if (s.V.size() > 0xF0000000ull || s.O.size() > 0xF0000000ull) return false;
  // Constant-bank value table: the FAST / FAST2 value sequences covering the
  // most rows, as long as they fit (kPValTab doubles); their slices read
  // values from the kernel-parameter table instead of V (pk bit 31, vbase =
  // table offset).
  if (opt().psell_ctab) {
    // FAST2 (rows = 2 x count) and FAST (rows = count) slices compete for the
    // table by the rows they cover; both read V[vbase ..] otherwise.
    std::unordered_map<uint32_t, std::pair<int64_t, int32_t>> use;  // vbase -> (rows, length)
    for (const PSliceMeta& m : s.meta)
      if (!(m.pk & (1u << 17)) && (m.pk >> 31)) {  // FASTE: one row per lane
        auto& u = use[m.vbase];
        u.first += static_cast<int64_t>((m.pk >> 11) & 0x3f);
        u.second = static_cast<int32_t>(m.pk & kPMaxLen);
      } else if (m.pk & (1u << 17)) {
        const int wv = static_cast<int>((m.pk >> 19) & 0x3f);  // 0 FAST, 1 FAST2, 2 FAST4
        auto& u = use[m.vbase];
        u.first += (wv == 5 ? 8 : wv == 2 ? 4 : wv == 1 || wv == 3 || wv == 4 ? 2 : 1) * static_cast<int64_t>((m.pk >> 11) & 0x3f);
        u.second = static_cast<int32_t>(m.pk & kPMaxLen) * (wv == 4 ? 2 : 1);  // FASTAB: interleaved pair sequence
      }
    std::vector<std::pair<int64_t, uint32_t>> order;
    for (const auto& [vb, u] : use) order.push_back({u.first, vb});
    std::sort(order.begin(), order.end(), [](const auto& x, const auto& y) {
      return x.first != y.first ? x.first > y.first : x.second < y.second;
    });
    std::unordered_map<uint32_t, uint32_t> toff;
    for (const auto& [rows, vb] : order) {
      const int32_t L = use[vb].second;
      if (static_cast<int64_t>(s.tab.size()) + L > kPValTab) continue;
      toff[vb] = static_cast<uint32_t>(s.tab.size());
      s.tab.insert(s.tab.end(), s.V.begin() + vb, s.V.begin() + vb + L);
      s.tab_rows += rows;
    }
    for (PSliceMeta& m : s.meta)
      if (!(m.pk & (1u << 17)) && (m.pk >> 31)) {  // FASTE: table flag in bit 18
        auto it = toff.find(m.vbase);
        if (it != toff.end()) {
          m.vbase = it->second;
          m.pk |= 1u << 18;
        }
      } else if (m.pk & (1u << 17)) {
        auto it = toff.find(m.vbase);
        if (it != toff.end()) {
          m.vbase = it->second;
          m.pk |= 1u << 31;
        }
      }
  }
  // Slice order = launch order of the warps: the GENERAL slices first (their
  // unique value rows stream from HBM: the longest latency, started while
  // everything else is still to come), then the two-line slices (the most
  // work per warp), the multi-piece slices, and the light one-row-per-lane /
  // pair slices last, where they fill the grid's tail; row order within a
  // class.  C4 finest A p 80.7 -> 78.0 us against row order (GENERAL first
  // with the rest in row order: 83.1 us; two-line first: 84.4 us).
  if (opt().psell_order) {
    auto weight = [](const PSliceMeta& m) {
      const bool fast = m.pk & (1u << 17);
      const int wv = static_cast<int>((m.pk >> 19) & 0x3f);
      return !fast && !(m.pk >> 31) ? 0 : fast && (wv == 5 || wv == 2) ? 1 : fast && wv == 3 ? 2 : 3;
    };
    std::stable_sort(s.meta.begin(), s.meta.end(),
                     [&](const PSliceMeta& x, const PSliceMeta& y) { return weight(x) < weight(y); });
    if (opt().psell_order == 1) {  // GENERAL slices spread evenly through the two-line slices (their HBM stream
                                   // over the first half of the grid instead of one burst: A p 77.7 -> 76.4 us)
      const double frac = 1.0;
      size_t ng = 0, nt = 0;
      for (const auto& m : s.meta) {
        ng += weight(m) == 0;
        nt += weight(m) == 1;
      }
      if (ng > 0 && nt > 0 && frac > 0) {
        std::vector<PSliceMeta> out;
        out.reserve(s.meta.size());
        size_t ig = 0, it = 0;
        while (ig < ng || it < nt) {
          const double kg = ig < ng ? static_cast<double>(ig) / ng * frac : 2.0;
          const double kt = it < nt ? static_cast<double>(it) / nt : 2.0;
          if (kg <= kt) out.push_back(s.meta[ig++]);
          else out.push_back(s.meta[ng + it++]);
        }
        out.insert(out.end(), s.meta.begin() + ng + nt, s.meta.end());
        s.meta.swap(out);
      }
    }
  }
  // Pad to whole CTAs (count 0 = empty slice); dictionary rows of GENERAL
  // slices read up to the slice's padded length past their start.
  while (s.meta.size() % (kCta / 32) != 0 || s.meta.empty()) s.meta.push_back(PSliceMeta{0, 0, 0, 0});
  s.V.resize(s.V.size() + static_cast<size_t>(lmax_all) + 16, 0.0);
  s.O.resize(s.O.size() + static_cast<size_t>(lmax_all) + 16, 0);
  if (s.rlist.empty()) {
    s.rlist.push_back(0);
    s.ginfo.push_back(0);
  }
  return true;
}

// Host interpreter of the pattern-SELL layout: y = A x slice by slice with
// the SAME index arithmetic, window extents and summation order as
// spmv_psell.cuh (k_pspmv / psell_slice), every x / xe / table / pool index
// bounds-checked.  Test infrastructure (ig_debug_psell_apply): it validates
// the layout builder on the CPU -- each row computed exactly once, no load
// outside its array (compute-sanitizer is not available on the GPU pool) --
// and its results equal the serial CSR row sums bit for bit.
bool psell_apply_host(const HostPSell& s, int32_t nr, int32_t nc, const double* x, double* y, std::string& err) {
  std::vector<uint8_t> done(static_cast<size_t>(nr), 0);
  std::vector<double> xe(s.G.size(), 0.0);
  for (size_t i = 0; i < s.G.size(); ++i) {
    if (s.G[i] < 0 || s.G[i] >= nc) return err = "xgather index out of range", false;
    xe[i] = x[s.G[i]];
  }
  auto fail_at = [&](size_t slice, const char* what) {
    err = std::string("slice ") + std::to_string(slice) + ": " + what;
    return false;
  };
  bool ok = true;
  const char* why = "";
  auto X = [&](int64_t i) -> double {
    if (i < 0 || i >= nc) {
      ok = false;
      why = "x index out of range";
      return 0.0;
    }
    return x[i];
  };
  auto Vv = [&](int64_t i) -> double {
    if (i < 0 || i >= static_cast<int64_t>(s.V.size())) {
      ok = false;
      why = "V index out of range";
      return 0.0;
    }
    return s.V[static_cast<size_t>(i)];
  };
  auto Tv = [&](int64_t i) -> double {
    if (i < 0 || i >= static_cast<int64_t>(s.tab.size())) {
      ok = false;
      why = "value table index out of range";
      return 0.0;
    }
    return s.tab[static_cast<size_t>(i)];
  };
  auto Ov = [&](int64_t i) -> int32_t {
    if (i < 0 || i >= static_cast<int64_t>(s.O.size())) {
      ok = false;
      why = "O index out of range";
      return 0;
    }
    return s.O[static_cast<size_t>(i)];
  };
  auto put = [&](int64_t row, double v) {
    if (row < 0 || row >= nr) {
      ok = false;
      why = "row out of range";
      return;
    }
    if (done[row]) {
      ok = false;
      why = "row computed twice";
      return;
    }
    done[row] = 1;
    y[row] = v;
  };
  auto base = [&](int64_t row) { return (row * s.smul) >> s.sshift; };
  for (size_t sl = 0; sl < s.meta.size() && ok; ++sl) {
    const PSliceMeta& m = s.meta[sl];
    const uint32_t pk = m.pk;
    const int count = static_cast<int>((pk >> 11) & 0x3f);
    if (count == 0) continue;
    const int L = static_cast<int>(pk & kPMaxLen);
    const bool fast = pk & (1u << 17);
    const int wv = static_cast<int>((pk >> 19) & 0x3f), wo = static_cast<int>((pk >> 25) & 0x3f);
    const bool tabv = fast && (pk >> 31);
    auto val = [&](int64_t j) { return tabv ? Tv(m.vbase + j) : Vv(m.vbase + j); };
    for (int lane = 0; lane < count && ok; ++lane) {
      if (fast && (wv == 2 || wv == 5)) {  // FAST4 / FAST8: R rows of each of two lines
        const int R = wv == 5 ? 4 : 2;
        if (m.obase + 1 > s.useg.size()) return fail_at(sl, "useg header out of range");
        const int4 hd = s.useg[m.obase];
        if (m.obase + 1 + static_cast<size_t>(hd.y) > s.useg.size()) return fail_at(sl, "useg list out of range");
        const int64_t ra = static_cast<int64_t>(m.a) + R * lane;
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int u = 0; u < hd.y; ++u) {
          const int4 e = s.useg[m.obase + 1 + u];
          const int64_t a = ra + e.x;
          const int M = e.y;
          if (wv == 5 && M == 5) {  // 32-byte window loads from the 32-byte boundary below (x 32-byte aligned at 0)
            const int Q = static_cast<int>(a & 3);
            X(a - Q);
            X(a + M + 2);
          } else {
            X(a - (a & 1));
            X(a + M + R - 2);
          }
          for (int line = 0; line < 2; ++line) {
            const int vi = line == 0 ? e.z : e.w;
            if (vi < 0) continue;
            for (int j = 0; j < M; ++j)
              for (int r = 0; r < R; ++r) acc[line * R + r] = acc[line * R + r] + val(vi + j) * X(a + j + r);
          }
        }
        for (int r = 0; r < R; ++r) {
          put(ra + r, acc[r]);
          put(ra + hd.x + r, acc[R + r]);
        }
      } else if (fast && wv == 3) {  // FAST2M
        if (m.obase + 2 > s.useg.size()) return fail_at(sl, "FAST2M table out of range");
        const int4 R4 = s.useg[m.obase], hd = s.useg[m.obase + 1];
        if (m.obase + 2 + static_cast<size_t>(hd.w) > s.useg.size()) return fail_at(sl, "FAST2M offsets out of range");
        const int s1 = hd.x & 0xff, s2 = (hd.x >> 8) & 0xff, s3 = (hd.x >> 16) & 0xff;
        const int pid = (lane >= s1) + (lane >= s2) + (lane >= s3);
        const int st = pid == 0 ? 0 : pid == 1 ? s1 : pid == 2 ? s2 : s3;
        const int en = std::min(count, pid == 0 ? s1 : pid == 1 ? s2 : pid == 2 ? s3 : 64);
        const int64_t ra = (&R4.x)[pid] + 2 * (lane - st);
        const bool odd = ((hd.y >> pid) & 1) && lane == en - 1;
        double a0 = 0.0, a1 = 0.0;
        int vo = 0;
        for (int u = 0; u < hd.w; ++u) {
          if (static_cast<size_t>(hd.z) + u >= s.seg.size()) return fail_at(sl, "segment list out of range");
          const int M = s.seg[hd.z + u].y;
          const int64_t a = ra + (&s.useg[m.obase + 2 + u].x)[pid];
          X(a - (a & 1));
          X(a + M);
          for (int j = 0; j < M; ++j) {
            const double v = val(vo + j);
            a0 = a0 + v * X(a + j);
            a1 = a1 + v * X(a + j + 1);
          }
          vo += M;
        }
        put(ra, a0);
        if (!odd) put(ra + 1, a1);
      } else if (fast && wv == 1) {  // FAST2
        const int64_t ra = static_cast<int64_t>(m.a) + 2 * lane;
        double a0 = 0.0, a1 = 0.0;
        int vo = 0;
        for (size_t q = m.obase;; ++q) {
          if (q >= s.seg.size()) return fail_at(sl, "segment list out of range");
          const int2 e = s.seg[q];
          if (e.y == 0) break;
          const int64_t a = ra + e.x;
          X(a - (a & 1));
          X(a + e.y);
          for (int j = 0; j < e.y; ++j) {
            const double v = val(vo + j);
            a0 = a0 + v * X(a + j);
            a1 = a1 + v * X(a + j + 1);
          }
          vo += e.y;
        }
        put(ra, a0);
        put(ra + 1, a1);
      } else if (fast && wv == 4) {  // FASTAB
        const int64_t ra = static_cast<int64_t>(m.a) + 2 * lane;
        double a0 = 0.0, a1 = 0.0;
        for (int k = 0; k < L; ++k) {
          const double xk = X(base(ra) + Ov(m.obase + k));
          a0 = a0 + val(2 * k) * xk;
          a1 = a1 + val(2 * k + 1) * xk;
        }
        put(ra, a0);
        put(ra + 1, a1);
      } else if (fast) {  // FAST
        const int64_t row = static_cast<int64_t>(m.a) + lane;
        double acc = 0.0;
        for (int k = 0; k < L; ++k) acc = acc + val(k) * X(base(row) + Ov(m.obase + k));
        put(row, acc);
      } else if (pk >> 31) {  // FASTE
        if (m.a + static_cast<size_t>(lane) >= s.rlist.size()) return fail_at(sl, "row list out of range");
        const int64_t row = s.rlist[m.a + lane], ta = s.ginfo[m.a + lane];
        const bool tb = pk & (1u << 18);
        double acc = 0.0;
        for (int k = 0; k < L; ++k) {
          const int64_t xi = ta + Ov(m.obase + k);
          if (xi < 0 || xi >= static_cast<int64_t>(xe.size())) return fail_at(sl, "xe index out of range");
          acc = acc + (tb ? Tv(m.vbase + k) : Vv(m.vbase + k)) * xe[static_cast<size_t>(xi)];
        }
        put(row, acc);
      } else {  // GENERAL
        if (m.a + static_cast<size_t>(lane) >= s.rlist.size()) return fail_at(sl, "row list out of range");
        const int64_t row = s.rlist[m.a + lane];
        const uint32_t info = s.ginfo[m.a + lane];
        const int len = static_cast<int>(info & kPMaxLen), vsel = static_cast<int>((info >> 11) & 0x3f);
        const int vi = static_cast<int>((info >> 17) & 0x1f), oi = static_cast<int>((info >> 22) & 0x1f);
        const int L8 = (L + 7) & ~7;
        double acc = 0.0;
        for (int k = 0; k < L8; ++k) {  // padded entries are gathered too (never added)
          const int32_t o = Ov(static_cast<int64_t>(m.obase) + static_cast<int64_t>(k / 4) * 4 * wo + 4 * oi + k % 4);
          const double xv = X(base(row) + o);
          const double v = vsel ? Vv(static_cast<int64_t>(vsel - 1) * s.dict_w + k)
                                : Vv(static_cast<int64_t>(m.vbase) + static_cast<int64_t>(k / 2) * 2 * wv + 2 * vi + k % 2);
          if (k < len) acc = acc + v * xv;
        }
        put(row, acc);
      }
    }
    if (!ok) return fail_at(sl, why);
  }
  for (int32_t i = 0; i < nr; ++i)
    if (!done[i]) return err = "row " + std::to_string(i) + " not computed", false;
  return true;
}

// Transpose of a CSR (rows of the result visit source rows ascending).
void csr_transpose(const ig_csr& a, std::vector<int32_t>& tp, std::vector<int32_t>& tc, std::vector<double>& tv) {
  tp.assign(static_cast<size_t>(a.n_cols) + 1, 0);
  for (int64_t k = 0; k < a.nnz; ++k) ++tp[a.col_idx[k] + 1];
  for (int32_t j = 0; j < a.n_cols; ++j) tp[j + 1] += tp[j];
  tc.resize(static_cast<size_t>(a.nnz));
  tv.resize(static_cast<size_t>(a.nnz));
  std::vector<int32_t> nx(tp.begin(), tp.end() - 1);
  for (int32_t i = 0; i < a.n_rows; ++i)
    for (int32_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const int32_t p = nx[a.col_idx[k]]++;
      tc[p] = i;
      tv[p] = a.val[k];
    }
}

struct DevSell {
  Sell s{};
  bool stream = false;
  int64_t nnz = 0, slots = 0;
  int64_t explicit_vals = 0, explicit_cols = 0;
  bool has_p = false;   // pattern-SELL layout present (spmv_psell.cuh)
  PSell p{};
  std::shared_ptr<PValTab> ptab;  // constant-bank value table (zeros when unused)
  bool has_f4 = false;            // the pattern layout holds two-line slices
  int32_t n_xe = 0;               // FASTE: size of the edge-compacted copy xe of the input vector
  const int32_t* xgather = nullptr;
  double* xe = nullptr;
  int64_t p_bytes = 0;  // HostPSell::layout_bytes
  int64_t n_fast = 0, n_general = 0;
  int64_t layout_matrix_bytes() const { return has_p ? p_bytes : 8 * explicit_vals + 4 * explicit_cols + 4 * int64_t(s.n_rows); }
};

// Additive smoother levels with at least this many DOFs run the small-block
// groups (k_as_blocks4) on a second side stream (profiles/level_costs.py:
// C4 finest level 453 -> 440 us per V-cycle).
constexpr int32_t kSplitRows = 100000;

struct Level {
  int32_t n = 0;
  DevSell A, R, P;
  AsGroups G{};
  AsGather S{};
  int32_t g_small = 0;  // first group with smax <= 4 (groups are sorted by size, descending)
  int32_t n_blocks = 0, n_multi = 0, n_complex = 0;
  int64_t sum_s = 0, sum_s2 = 0, packed_F = 0;
  double* r_in = nullptr;  // input residual buffer (host API; coarse levels: R res)
  double* x = nullptr;
  double* res = nullptr;
  double* cor = nullptr;
  double* ybuf = nullptr;
  // Multiplicative Schwarz (smoother_kind MULTIPLICATIVE_SCHWARZ).
  bool ms = false;
  double gamma = 1.0;
  struct MsColor {
    AsGroups G{};
    int32_t n_items = 0;   // warp work items of the block solves
    DevSell S;             // the colour's columns of A over the rows they touch
    int32_t* rowmap = nullptr;
    int64_t n_dofs = 0;    // DOFs solved in this colour
  };
  std::vector<MsColor> colors;  // [colour]; empty colours have n_items == 0
  double *ms_cur = nullptr, *ms_delta = nullptr, *ms_x = nullptr;
};

// Algorithmic byte counts (CSR-minimal traffic).
int64_t bytes_spmv(int64_t nr, int64_t nin, int64_t nnz, bool resid) {
  return 12 * nnz + 4 * (nr + 1) + 8 * nin + 8 * nr + (resid ? 8 * nr : 0);
}

}  // namespace

struct ig_hier {
  Opts opts;              // snapshot of the defaults at ig_hier_create (ig_hier_set_option)
  // The finest operator the handle was built on (ig_hier_matches): the
  // caller's arrays and sizes, and a content hash for copies of it.
  ig_csr fine_src{};
  uint64_t fine_hash = 0;
  std::vector<Level> lv;  // [0] coarsest
  int32_t L = 0;
  int32_t n0 = 0, rank = 0;
  double* Lp = nullptr;  // packed lower L11
  double* Minv = nullptr;  // tolerance mode: rank x rank row-major M = L11^-T L11^-1
  bool fast_coarse = false;
  int32_t* piv = nullptr;
  int coarse_threads = 32;
  size_t coarse_smem = 0;
  int coarse_use_smem = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;   // block solves, forked from / joined into `stream`
  cudaStream_t side2 = nullptr;  // small-block groups (k_as_blocks4), concurrently
  int num_sms = 148;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join2 = nullptr;
  PcgState* st = nullptr;
  double* partials = nullptr;
  double* residuals = nullptr;
  int32_t res_cap = 0;
  double *r = nullptr, *z = nullptr, *p = nullptr, *ap = nullptr;
  double *hb = nullptr, *hx = nullptr;  // device copies for the host-buffer API
  cudaGraphExec_t pcg_exec = nullptr;
  cudaGraphExec_t rich_exec = nullptr;
  struct VcGraph {
    int level;
    const double* r;
    double* x;
    cudaGraphExec_t exec;
  };
  std::vector<VcGraph> vc_graphs;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<void*> allocs;
  ig_info info{};
  std::mutex mu;
  int last_status = IG_OK;

  // L2-resident arena for the small levels (IG_OPT_L2_ROWS): their arrays
  // are sub-allocated from one block so a single persisting access-policy
  // window on the streams covers them (the finest level's streaming would
  // otherwise evict them between V-cycles).
  char* arena = nullptr;
  size_t arena_cap = 0, arena_used = 0;
  bool arena_on = false;
  template <typename T>
  T* alloc(size_t count) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    info.device_bytes += static_cast<int64_t>(bytes);
    if (arena_on && arena) {
      const size_t off = (arena_used + 255) & ~size_t(255);
      if (off + bytes <= arena_cap) {
        arena_used = off + bytes;
        return reinterpret_cast<T*>(arena + off);
      }
    }
    void* p = nullptr;
    CK(cudaMalloc(&p, bytes));
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
  template <typename T>
  T* upload(const T* src, size_t count) {
    T* d = alloc<T>(count);
    if (count && src) CK(cudaMemcpy(d, src, count * sizeof(T), cudaMemcpyHostToDevice));
    return d;
  }
  DevSell upload_sell(const HostSell& h, int64_t nnz) {
    DevSell d;
    d.s.n_rows = h.nr;
    d.s.n_cols = h.nc;
    d.s.slice_ptr = upload(h.slice_ptr.data(), h.slice_ptr.size());
    d.s.rowinfo = upload(h.rowinfo.data(), h.rowinfo.size());
    d.s.val = upload(h.val.data(), h.val.size());
    d.s.col = upload(h.col.data(), h.col.size());
    d.s.dict_w = h.dict_w;
    d.s.dval = upload(h.dval.data(), h.dval.size());
    d.s.doff = upload(h.doff.data(), h.doff.size());
    d.nnz = nnz;
    d.slots = h.slice_ptr.back();
    d.explicit_vals = h.explicit_vals;
    d.explicit_cols = h.explicit_cols;
    // Stream (evict-first) matrices far larger than L2; keep small ones cached.
    d.stream = d.slots * 12 > (int64_t(48) << 20);
    return d;
  }
  // Device layout of one operator: pattern SELL for the large matrices (when
  // it fits), the row-dictionary SELL otherwise (and for the small levels,
  // which run k_spmv_grp on it).
  DevSell make_matrix(int32_t nr, int32_t nc, const int32_t* ptr, const int32_t* col, const double* val, int64_t nnz) {
    if (opt().use_psell && nr > opt().small_rows) {
      HostPSell hp;
      if (to_psell(nr, nc, ptr, col, val, hp)) {
        DevSell d;
        d.s.n_rows = nr;
        d.s.n_cols = nc;
        d.nnz = nnz;
        d.has_p = true;
        d.p.n_rows = nr;
        d.p.n_cols = nc;
        d.p.n_slices = static_cast<int32_t>(hp.meta.size());
        d.p.meta = upload(hp.meta.data(), hp.meta.size());
        d.p.rlist = upload(hp.rlist.data(), hp.rlist.size());
        d.p.ginfo = upload(hp.ginfo.data(), hp.ginfo.size());
        d.p.smul = hp.smul;
        d.p.sshift = hp.sshift;
        if (hp.seg.empty()) hp.seg.push_back(make_int2(0, 0));
        d.p.seg = upload(hp.seg.data(), hp.seg.size());
        if (hp.useg.empty()) hp.useg.push_back(make_int4(0, 0, 0, 0));
        d.p.useg = upload(hp.useg.data(), hp.useg.size());
        d.n_xe = static_cast<int32_t>(hp.G.size());
        if (d.n_xe > 0) {
          d.xgather = upload(hp.G.data(), hp.G.size());
          d.xe = alloc<double>(hp.G.size());
          d.p.xe = d.xe;
        }
        d.p.V = upload(hp.V.data(), hp.V.size());
        d.p.O = upload(hp.O.data(), hp.O.size());
        d.p.dict_w = hp.dict_w;
        d.has_f4 = hp.n_fast4 > 0 || hp.n_fast2m > 0;
        d.ptab = std::make_shared<PValTab>();
        std::memset(d.ptab.get(), 0, sizeof(PValTab));
        std::copy(hp.tab.begin(), hp.tab.end(), d.ptab->v);
        if (std::getenv("IG_TIMING"))
          std::fprintf(stderr, "[psell] %d x %d: %lld fast (%lld two-line) / %lld general slices, value table %zu doubles (%lld rows)\n",
                       nr, nc, static_cast<long long>(hp.n_fast), static_cast<long long>(hp.n_fast4),
                       static_cast<long long>(hp.n_general), hp.tab.size(), static_cast<long long>(hp.tab_rows));
        d.p_bytes = hp.layout_bytes;
        d.n_fast = hp.n_fast;
        d.n_general = hp.n_general;
        d.explicit_vals = static_cast<int64_t>(hp.V.size());
        d.explicit_cols = static_cast<int64_t>(hp.O.size());
        d.slots = static_cast<int64_t>(hp.V.size());
        d.stream = static_cast<int64_t>(hp.O.size()) * 4 > (int64_t(48) << 20);
        return d;
      }
    }
    return upload_sell(to_sell(nr, nc, ptr, col, val), nnz);
  }
  // Cached graphs bake in the launch attributes (PDL) and grids: dropped when
  // a runtime option of the handle changes.
  void drop_graphs() {
    if (pcg_exec) cudaGraphExecDestroy(pcg_exec);
    if (rich_exec) cudaGraphExecDestroy(rich_exec);
    for (auto& g : vc_graphs) cudaGraphExecDestroy(g.exec);
    pcg_exec = rich_exec = nullptr;
    vc_graphs.clear();
  }
  ~ig_hier() {
    drop_graphs();
    for (void* p : allocs) cudaFree(p);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (ev_join2) cudaEventDestroy(ev_join2);
    if (side) cudaStreamDestroy(side);
    if (side2) cudaStreamDestroy(side2);
    if (stream) cudaStreamDestroy(stream);
  }

  // ------------------------------------------------------------ launches --
  template <int M, bool S, bool R>
  void spmv_var(unsigned g, const DevSell& A, const double* x, double* y, const double* rsrc, PcgState* s) {
    launch(k_spmv<M, S, R>, g, kCta, 0, stream, A.s, x, y, rsrc, s, partials);
  }
  void spmv(const DevSell& A, int mode, const double* x, double* y, const double* rsrc,
            PcgState* s = nullptr, bool red = false) {
    const unsigned g = grid_of(A.s.n_rows);
    if (g == 0) return;
    if (A.has_p) {
      const unsigned gp = static_cast<unsigned>(A.p.n_slices / (kPCta / 32));
      const size_t sm = psell_smem();
      const PValTab& tb = *A.ptab;
      if (A.n_xe > 0) {  // FASTE slices read the edge-compacted copy of x
        launch(k_xgather, static_cast<unsigned>((A.n_xe + kCta - 1) / kCta), kCta, 0, stream, A.n_xe, A.xgather, x, A.xe);
        CK(cudaGetLastError());
      }
      if (!A.has_f4 && !A.stream) {  // no two-line slices: the leaner instantiation
        if (mode == 0) launch(k_pspmv<0, false, false>, gp, kPCta, sm, stream, A.p, x, y, rsrc, s, tb);
        else launch(k_pspmv<1, false, false>, gp, kPCta, sm, stream, A.p, x, y, rsrc, s, tb);
      } else if (mode == 0) {
        if (A.stream) launch(k_pspmv<0, true>, gp, kPCta, sm, stream, A.p, x, y, rsrc, s, tb);
        else launch(k_pspmv<0, false>, gp, kPCta, sm, stream, A.p, x, y, rsrc, s, tb);
      } else {
        if (A.stream) launch(k_pspmv<1, true>, gp, kPCta, sm, stream, A.p, x, y, rsrc, s, tb);
        else launch(k_pspmv<1, false>, gp, kPCta, sm, stream, A.p, x, y, rsrc, s, tb);
      }
      CK(cudaGetLastError());
      if (red) {  // p . Ap over the canonical chunks, alpha / Breakdown
        launch(k_pap, red_grid(A.s.n_rows), kCta, 0, stream, A.s.n_rows, x, y, s, partials);
        CK(cudaGetLastError());
      }
      return;
    }
    if (!red && A.s.n_rows <= opt().small_rows) {  // latency-bound level: 8 lanes per row
      const unsigned gg = grid_of(static_cast<int64_t>(A.s.n_rows) * 8);
      if (mode == 0)
        launch(k_spmv_grp<0, 8>, gg, kCta, 0, stream, A.s, x, y, rsrc);
      else
        launch(k_spmv_grp<1, 8>, gg, kCta, 0, stream, A.s, x, y, rsrc);
      CK(cudaGetLastError());
      return;
    }
    if (red) {
      if (A.stream) spmv_var<0, true, true>(g, A, x, y, rsrc, s); else spmv_var<0, false, true>(g, A, x, y, rsrc, s);
    } else if (mode == 0) {
      if (A.stream) spmv_var<0, true, false>(g, A, x, y, rsrc, s); else spmv_var<0, false, false>(g, A, x, y, rsrc, s);
    } else {
      if (A.stream) spmv_var<1, true, false>(g, A, x, y, rsrc, s); else spmv_var<1, false, false>(g, A, x, y, rsrc, s);
    }
    CK(cudaGetLastError());
  }
  template <bool S>
  void prolong_var(unsigned g, const Level& l, const double* xc, double* x, PcgState* s) {
    launch(k_prolong<S>, g, kCta, 0, stream, l.P.s, xc, l.cor, x, s);
  }
  void prolong(const Level& l, const double* xc, double* x, PcgState* s) {
    const unsigned g = grid_of(l.P.s.n_rows);
    if (l.P.has_p) {
      const unsigned gp = static_cast<unsigned>(l.P.p.n_slices / (kPCta / 32));
      const size_t sm = psell_smem();
      if (l.P.stream) launch(k_pprolong<true>, gp, kPCta, sm, stream, l.P.p, xc, l.cor, x, s, *l.P.ptab);
      else launch(k_pprolong<false>, gp, kPCta, sm, stream, l.P.p, xc, l.cor, x, s, *l.P.ptab);
      CK(cudaGetLastError());
      return;
    }
    if (l.P.stream)
      prolong_var<true>(g, l, xc, x, s);
    else
      prolong_var<false>(g, l, xc, x, s);
    CK(cudaGetLastError());
  }
  // Smoother::apply (AS).  Fork: the block solves run on the side stream while
  // the singleton fast path runs on the main stream; join; then the DOFs with
  // contribution lists (and, in PCG on the finest level, r . z).
  // Smoother::apply(r, dir) (smoothers.cpp:169-208); dir < 0: Forward for the
  // pre-smoother (acc = false), Reverse for the post-smoother (acc = true),
  // as vcycle_at uses them (multigrid.cpp:99, :106).
  void smoother(const Level& l, const double* r, double* x, bool acc, PcgState* s, const double* rdot, int dir = -1) {
    if (l.ms) {
      ms_smoother(l, r, x, acc, s, rdot, dir < 0 ? (acc ? 1 : 0) : dir);
      return;
    }
    // Block solves on two side streams forked from / joined into the main
    // stream: the groups of small blocks (smax <= 4, k_as_blocks4, few
    // registers) and the rest (larger groups and warp blocks, k_as_blocks);
    // the singleton DOFs run on the main stream meanwhile.
    if (l.n <= opt().one_stream_rows) {  // small level: blocks + singletons, then the lists, all PDL-chained
      const int32_t items = l.G.n_groups + l.G.n_wblocks;
      const int32_t nb = (items * 32 + 127) / 128;
      const unsigned gtot = static_cast<unsigned>(nb + (l.n + 127) / 128);
      if (acc)
        launch(k_as_blocks_simple<true>, gtot, 128, 0, stream, l.G, nb, l.S, r, l.ybuf, x, s);
      else
        launch(k_as_blocks_simple<false>, gtot, 128, 0, stream, l.G, nb, l.S, r, l.ybuf, x, s);
      CK(cudaGetLastError());
      if (l.S.n_complex > 0) {
        const unsigned gc = grid_of(static_cast<int64_t>(l.S.n_complex) * 4);
        if (acc)
          launch(k_as_complex4<true>, gc, kCta, 0, stream, l.S, r, l.ybuf, x, s);
        else
          launch(k_as_complex4<false>, gc, kCta, 0, stream, l.S, r, l.ybuf, x, s);
      }
      if (rdot) launch(k_pcg_rz, red_grid(l.n), kCta, 0, stream, l.n, rdot, x, s, partials);
      CK(cudaGetLastError());
      return;
    }
    // Only large levels split: on small ones the second graph branch costs
    // more than it overlaps (C5 / C2 levels below 40k DOFs +2-5 us each).
    const bool split = l.n >= kSplitRows;
    AsGroups big = l.G;
    big.n_groups = split ? l.g_small : l.G.n_groups;  // groups are sorted by size: [0, g_small) have smax > 4
    const int32_t n_small = l.G.n_groups - big.n_groups;
    const bool fork1 = big.n_groups + big.n_wblocks > 0;
    const bool fork2 = n_small > 0;
    if (fork1 || fork2) CK(cudaEventRecord(ev_fork, stream));
    if (fork1) {
      CK(cudaStreamWaitEvent(side, ev_fork, 0));
      const unsigned gb = static_cast<unsigned>((static_cast<int64_t>(big.n_groups + big.n_wblocks) * 32 + 127) / 128);
      launch(k_as_blocks, gb, 128, 0, side, big, r, l.ybuf, s);
      CK(cudaGetLastError());
      CK(cudaEventRecord(ev_join, side));
    }
    if (fork2) {
      CK(cudaStreamWaitEvent(side2, ev_fork, 0));
      const unsigned gs = static_cast<unsigned>((static_cast<int64_t>(n_small) * 32 + 127) / 128);
      launch(k_as_blocks4, gs, 128, 0, side2, l.G, l.g_small, r, l.ybuf, s);
      CK(cudaGetLastError());
      CK(cudaEventRecord(ev_join2, side2));
    }
    const unsigned g = grid_of(l.n);
    if (acc)
      launch(k_as_simple<true>, g, kCta, 0, stream, l.S, r, x, s);
    else
      launch(k_as_simple<false>, g, kCta, 0, stream, l.S, r, x, s);
    CK(cudaGetLastError());
    if (fork1) CK(cudaStreamWaitEvent(stream, ev_join, 0));
    if (fork2) CK(cudaStreamWaitEvent(stream, ev_join2, 0));
    if (rdot) {
      // Complex DOFs, then r . z as a plain streaming reduction (the fused
      // k_as_finish_red keeps the list walks inside the reduction chunks and
      // measured 71 us vs ~13 + ~17 us split; same products, same tree).
      if (l.S.n_complex > 0) {
        const unsigned gc = grid_of(l.S.n_complex);
        if (acc)
          launch(k_as_complex<true>, gc, kCta, 0, stream, l.S, r, l.ybuf, x, s);
        else
          launch(k_as_complex<false>, gc, kCta, 0, stream, l.S, r, l.ybuf, x, s);
      }
      launch(k_pcg_rz, red_grid(l.n), kCta, 0, stream, l.n, rdot, x, s, partials);
    } else if (l.S.n_complex > 0 && l.n <= opt().complex4_rows) {  // latency-bound: four lanes per DOF
      const unsigned gc = grid_of(static_cast<int64_t>(l.S.n_complex) * 4);
      if (acc)
        launch(k_as_complex4<true>, gc, kCta, 0, stream, l.S, r, l.ybuf, x, s);
      else
        launch(k_as_complex4<false>, gc, kCta, 0, stream, l.S, r, l.ybuf, x, s);
    } else if (l.S.n_complex > 0) {
      const unsigned gc = grid_of(l.S.n_complex);
      if (acc)
        launch(k_as_complex<true>, gc, kCta, 0, stream, l.S, r, l.ybuf, x, s);
      else
        launch(k_as_complex<false>, gc, kCta, 0, stream, l.S, r, l.ybuf, x, s);
    }
    CK(cudaGetLastError());
  }
  // Grid of the canonical-reduction kernels (kernels.cuh chunk_reduce): at
  // most 4 CTAs per SM, each looping over 256-element chunks.
  unsigned red_grid(int64_t n) const {
    return static_cast<unsigned>(std::min<int64_t>(grid_of(n), static_cast<int64_t>(opt().red_ctas) * num_sms));
  }
  void ms_smoother(const Level& l, const double* r, double* out, bool acc, PcgState* s, const double* rdot, int dir) {
    const int32_t n = l.n;
    const int C = static_cast<int>(l.colors.size());
    launch(k_ms_init, grid_of(n), kCta, 0, stream, n, r, l.ms_cur, l.ms_x, s);
    for (int step = 0; step < C; ++step) {
      const int c = dir == 0 ? C - 1 - step : step;
      const Level::MsColor& mc = l.colors[c];
      if (mc.n_items == 0) continue;  // `if (!any) continue;`
      const unsigned gb = static_cast<unsigned>((static_cast<int64_t>(mc.n_items) * 32 + 127) / 128);
      launch(k_ms_blocks, gb, 128, 0, stream, mc.G, l.ms_cur, l.ms_delta, l.ms_x, s);
      if (step + 1 < C)
        launch(k_ms_update, grid_of(mc.S.s.n_rows), kCta, 0, stream, mc.S.s, mc.rowmap, l.ms_delta, l.ms_cur, s);
    }
    if (rdot) {
      if (acc) launch(k_ms_finish<true, true>, red_grid(n), kCta, 0, stream, n, l.gamma, l.ms_x, out, rdot, s, partials);
      else launch(k_ms_finish<false, true>, red_grid(n), kCta, 0, stream, n, l.gamma, l.ms_x, out, rdot, s, partials);
    } else {
      if (acc) launch(k_ms_finish<true, false>, grid_of(n), kCta, 0, stream, n, l.gamma, l.ms_x, out, rdot, s, partials);
      else launch(k_ms_finish<false, false>, grid_of(n), kCta, 0, stream, n, l.gamma, l.ms_x, out, rdot, s, partials);
    }
  }
  template <int R>
  void coarse_warp(bool sm, const double* r, double* x, PcgState* s) {
    if (sm)
      launch(k_coarse_warp<R, true>, 1, 32, coarse_smem, stream, n0, rank, Lp, piv, r, x, s);
    else
      launch(k_coarse_warp<R, false>, 1, 32, 0, stream, n0, rank, Lp, piv, r, x, s);
  }
  void coarse_launch(bool sm, const double* r, double* x, PcgState* s) {
    if (rank <= 256) {  // single-warp solve, R = ceil(rank / 32) rows per lane
      switch ((std::max(rank, 1) + 31) / 32) {
        case 1: coarse_warp<1>(sm, r, x, s); return;
        case 2: coarse_warp<2>(sm, r, x, s); return;
        case 3: coarse_warp<3>(sm, r, x, s); return;
        case 4: coarse_warp<4>(sm, r, x, s); return;
        case 5: coarse_warp<5>(sm, r, x, s); return;
        case 6: coarse_warp<6>(sm, r, x, s); return;
        case 7: coarse_warp<7>(sm, r, x, s); return;
        default: coarse_warp<8>(sm, r, x, s); return;
      }
    }
    const bool big = coarse_threads > 256;
    if (sm && !big)
      launch(k_coarse<true, false>, 1, coarse_threads, coarse_smem, stream, n0, rank, Lp, piv, r, x, s);
    else if (sm)
      launch(k_coarse<true, true>, 1, coarse_threads, coarse_smem, stream, n0, rank, Lp, piv, r, x, s);
    else if (!big)
      launch(k_coarse<false, false>, 1, coarse_threads, coarse_smem, stream, n0, rank, Lp, piv, r, x, s);
    else
      launch(k_coarse<false, true>, 1, coarse_threads, coarse_smem, stream, n0, rank, Lp, piv, r, x, s);
  }
  void coarse(const double* r, double* x, PcgState* s) {
    if (fast_coarse) {  // tolerance mode: one warp per row of M
      launch(k_coarse_gemv, static_cast<unsigned>((n0 + 7) / 8), 256, 0, stream, n0, rank, Minv, piv, r, x, s);
      CK(cudaGetLastError());
      return;
    }
    coarse_launch(coarse_use_smem != 0, r, x, s);
    CK(cudaGetLastError());
  }
  // MgHierarchy::vcycle_at (multigrid.cpp:90-108).  rdot != null: PCG mode on
  // the finest level (the last kernel also reduces r . z).
  void vcycle(int l, const double* r, double* x, PcgState* s, const double* rdot) {
    if (l == 0) {
      coarse(r, x, s);
      if (rdot) {  // 1-level hierarchy inside PCG: r . z as a separate pass
        launch(k_pcg_rz, red_grid(n0), kCta, 0, stream, n0, rdot, x, s, partials);
        CK(cudaGetLastError());
      }
      mark("coarse", 0);
      return;
    }
    Level& c = lv[l];
    Level& cc = lv[l - 1];
    smoother(c, r, x, false, s, nullptr);       // x = S(r, Forward)
    mark("smooth_pre", l);
    spmv(c.A, 1, x, c.res, r, s);               // res = r - A x
    mark("residual", l);
    spmv(c.R, 0, c.res, cc.r_in, nullptr, s);   // R res
    mark("restrict", l);
    vcycle(l - 1, cc.r_in, cc.x, s, nullptr);   // coarse_x
    prolong(c, cc.x, x, s);                     // cor = R^T coarse_x; x += cor
    mark("prolong", l);
    spmv(c.A, 1, c.cor, c.res, c.res, s);       // res -= A cor
    mark("residual2", l);
    smoother(c, c.res, x, true, s, rdot);       // x += S(res, Reverse)
    mark("smooth_post", l);
  }
  // Debug timeline (ig_debug_vcycle_timeline): an event after every step.
  struct Mark {
    const char* what;
    int level;
    cudaEvent_t ev;
  };
  std::vector<Mark>* timeline = nullptr;
  void mark(const char* what, int level) {
    if (!timeline) return;
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    CK(cudaEventRecord(e, stream));
    timeline->push_back({what, level, e});
  }
  // PCG pieces (solvers.cpp:24-66).  head: init (+ conditions); tail: the
  // preconditioner application and the direction update, which are skipped
  // (IF node / host check) once the solve has stopped.
  void pcg_init(cudaGraphConditionalHandle c_if, cudaGraphConditionalHandle c_loop) {
    const int32_t n = lv[L - 1].n;
    launch(k_pcg_init, red_grid(n), kCta, 0, stream, n, r, st, partials, c_if, c_loop);
    CK(cudaGetLastError());
  }
  void pcg_precond(bool first) {
    const int32_t n = lv[L - 1].n;
    vcycle(L - 1, r, z, st, r);  // z = M r; r . z; beta
    if (first)
      launch(k_pcg_p<true>, grid_of(n), kCta, 0, stream, n, z, p, st);
    else
      launch(k_pcg_p<false>, grid_of(n), kCta, 0, stream, n, z, p, st);
    CK(cudaGetLastError());
  }
  void pcg_step(cudaGraphConditionalHandle c_if, cudaGraphConditionalHandle c_loop) {
    const int32_t n = lv[L - 1].n;
    spmv(lv[L - 1].A, 0, p, ap, nullptr, st, true);  // ap = A p; pap; alpha / breakdown
    launch(k_pcg_update, red_grid(n), kCta, 0, stream, n, p, ap, r, st, partials, c_if, c_loop);
    CK(cudaGetLastError());
  }
  // Append a conditional node of `type` after the current capture frontier
  // of `stream`; returns its body graph (capture continues after the node).
  cudaGraph_t add_conditional(cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type) {
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    cudaGraph_t cap_graph;
    CK(cudaStreamGetCaptureInfo(stream, &cs, nullptr, &cap_graph, &deps, &ndeps));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = type;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, cap_graph, deps, ndeps, &cp));
    CK(cudaStreamUpdateCaptureDependencies(stream, &node, 1, cudaStreamSetCaptureDependencies));
    return cp.conditional.phGraph_out[0];
  }
  // Capture `fn` into an (empty) conditional body graph.
  template <typename F>
  void capture_into(cudaGraph_t body, F&& fn) {
    CK(cudaStreamBeginCaptureToGraph(stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    fn();
    CK(cudaStreamEndCapture(stream, &body));
  }
  // init -> IF(go){ precond(first) } -> WHILE(go){ step -> IF(go){ precond } }
  void build_pcg_graph() {
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle c_if0, c_loop, c_if1;
    CK(cudaGraphConditionalHandleCreate(&c_if0, g, 0, cudaGraphCondAssignDefault));
    CK(cudaGraphConditionalHandleCreate(&c_loop, g, 0, cudaGraphCondAssignDefault));
    CK(cudaGraphConditionalHandleCreate(&c_if1, g, 0, cudaGraphCondAssignDefault));
    CK(cudaStreamBeginCaptureToGraph(stream, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    pcg_init(c_if0, c_loop);
    cudaGraph_t pro = add_conditional(c_if0, cudaGraphCondTypeIf);
    cudaGraph_t body = add_conditional(c_loop, cudaGraphCondTypeWhile);
    CK(cudaStreamEndCapture(stream, &g));
    capture_into(pro, [&] { pcg_precond(true); });
    cudaGraph_t tail = nullptr;
    capture_into(body, [&] {
      pcg_step(c_if1, c_loop);
      tail = add_conditional(c_if1, cudaGraphCondTypeIf);
    });
    capture_into(tail, [&] { pcg_precond(false); });
    CK(cudaGraphInstantiate(&pcg_exec, g, 0));
    CK(cudaGraphDestroy(g));
  }
  // Richardson (solvers.cpp:73-120): WHILE node whose body is
  // z = V-cycle(r); r -= A z; x += z and the residual tests.
  void rich_body(cudaGraphConditionalHandle c_loop) {
    const int32_t n = lv[L - 1].n;
    vcycle(L - 1, r, z, st, nullptr);
    spmv(lv[L - 1].A, 1, z, r, r, st);
    launch(k_rich_step, red_grid(n), kCta, 0, stream, n, z, r, st, partials, c_loop);
  }
  void build_rich_graph() {
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle c_loop;
    CK(cudaGraphConditionalHandleCreate(&c_loop, g, 0, cudaGraphCondAssignDefault));
    CK(cudaStreamBeginCaptureToGraph(stream, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const int32_t n = lv[L - 1].n;
    launch(k_rich_init, red_grid(n), kCta, 0, stream, n, r, st, partials, c_loop);
    cudaGraph_t body = add_conditional(c_loop, cudaGraphCondTypeWhile);
    CK(cudaStreamEndCapture(stream, &g));
    capture_into(body, [&] { rich_body(c_loop); });
    CK(cudaGraphInstantiate(&rich_exec, g, 0));
    CK(cudaGraphDestroy(g));
  }
  void rich_launch(const double* d_b, double* d_x, double tol, int32_t maxit) {
    ensure_residuals(maxit);
    PcgState hs{};
    hs.tol = tol;
    hs.maxit = maxit;
    hs.k = 0;
    hs.status = ST_RUNNING;
    hs.b = d_b;
    hs.x = d_x;
    hs.residuals = residuals;
    CK(cudaMemcpyAsync(st, &hs, sizeof(PcgState), cudaMemcpyHostToDevice, stream));
    const int32_t n = lv[L - 1].n;
    if (opt().use_graph) {
      if (!rich_exec) build_rich_graph();
      CK(cudaGraphLaunch(rich_exec, stream));
      return;
    }
    auto stopped = [&] {
      int32_t done = 0;
      CK(cudaMemcpyAsync(&done, &st->done, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      return done != 0;
    };
    launch(k_rich_init, red_grid(n), kCta, 0, stream, n, r, st, partials, cudaGraphConditionalHandle(0));
    while (!stopped()) rich_body(0);
  }
  int rich_collect(double* res_out, int32_t* iters) {
    CK(cudaStreamSynchronize(stream));
    PcgState hs{};
    CK(cudaMemcpy(&hs, st, sizeof(PcgState), cudaMemcpyDeviceToHost));
    if (hs.status == ST_RUNNING) throw Error(IG_CUDA_ERROR, "richardson: solve did not terminate");
    const int32_t k = std::max(hs.k, 0);
    if (iters) *iters = k;
    if (res_out) CK(cudaMemcpy(res_out, residuals, sizeof(double) * (static_cast<size_t>(k) + 1), cudaMemcpyDeviceToHost));
    return hs.status;
  }
  void ensure_residuals(int32_t maxit) {
    if (maxit + 1 > res_cap) {
      res_cap = std::max(maxit + 1, 1024);
      residuals = alloc<double>(static_cast<size_t>(res_cap));
    }
  }
  // Enqueue a whole solve on the stream (no host synchronisation).
  void pcg_launch(const double* d_b, double* d_x, double tol, int32_t maxit) {
    ensure_residuals(maxit);
    PcgState h{};
    h.tol = tol;
    h.maxit = maxit;
    h.k = -1;
    h.done = 0;
    h.status = ST_RUNNING;
    h.b = d_b;
    h.x = d_x;
    h.residuals = residuals;
    CK(cudaMemcpyAsync(st, &h, sizeof(PcgState), cudaMemcpyHostToDevice, stream));
    if (maxit <= 0) {
      // Zero iterations allowed: still report the initial residual.
      pcg_init(0, 0);
      return;
    }
    if (opt().use_graph) {
      if (!pcg_exec) build_pcg_graph();
      CK(cudaGraphLaunch(pcg_exec, stream));
    } else {
      // Host-loop fallback (debug / ncu): same kernels, host checks the flag.
      auto stopped = [&] {
        int32_t done = 0;
        CK(cudaMemcpyAsync(&done, &st->done, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        return done != 0;
      };
      pcg_init(0, 0);
      if (stopped()) return;
      pcg_precond(true);
      for (int32_t it = 0; it < maxit; ++it) {
        pcg_step(0, 0);
        if (stopped()) break;
        pcg_precond(false);
      }
    }
  }
  int pcg_collect(double* res_out, int32_t* iters) {
    CK(cudaStreamSynchronize(stream));
    PcgState h{};
    CK(cudaMemcpy(&h, st, sizeof(PcgState), cudaMemcpyDeviceToHost));
    int status = h.status;
    int32_t k = std::max(h.k, 0);
    if (h.maxit <= 0) {
      status = h.bnorm == 0.0 || 1.0 <= h.tol ? IG_OK : IG_NOT_CONVERGED;
      k = 0;
    }
    if (status == ST_RUNNING) throw Error(IG_CUDA_ERROR, "pcg: solve did not terminate");
    if (iters) *iters = k;
    if (res_out) CK(cudaMemcpy(res_out, residuals, sizeof(double) * (static_cast<size_t>(k) + 1), cudaMemcpyDeviceToHost));
    return status;
  }
};

namespace {

// Device vectors handed to the *_device entry points are read with 16-byte
// vector loads (pattern-SELL x pairs) and written by the same kernels that
// write the library's own (cudaMalloc-aligned) buffers.
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    return fail(e.code, e.what());
  } catch (const std::exception& e) {
    return fail(IG_CUDA_ERROR, e.what());
  }
}

void check_csr(const ig_csr& a, const char* what) {
  if (a.n_rows < 0 || a.n_cols < 0 || a.nnz < 0) throw Error(IG_INVALID_ARGUMENT, std::string(what) + ": negative size");
  if (a.n_rows > 0 && (!a.row_ptr || (a.nnz > 0 && (!a.col_idx || !a.val))))
    throw Error(IG_INVALID_ARGUMENT, std::string(what) + ": null array");
  if (a.n_rows > 0 && (a.row_ptr[0] != 0 || a.row_ptr[a.n_rows] != a.nnz))
    throw Error(IG_INVALID_ARGUMENT, std::string(what) + ": row_ptr inconsistent with nnz");
  for (int32_t i = 0; i < a.n_rows; ++i)
    if (a.row_ptr[i + 1] < a.row_ptr[i]) throw Error(IG_INVALID_ARGUMENT, std::string(what) + ": row_ptr decreasing");
  std::atomic<int> bad{0};
  parallel_rows(a.n_rows, [&](int32_t i0, int32_t i1) {
    for (int32_t i = i0; i < i1 && !bad.load(std::memory_order_relaxed); ++i)
      for (int32_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
        if (a.col_idx[k] < 0 || a.col_idx[k] >= a.n_cols || (k > a.row_ptr[i] && a.col_idx[k] <= a.col_idx[k - 1])) {
          bad.store(1);
          break;
        }
  });
  if (bad.load()) throw Error(IG_INVALID_ARGUMENT, std::string(what) + ": column indices out of range or not ascending");
}

AsGroups build_groups(ig_hier& h, const ig_blocks& B, std::vector<int32_t> grouped, const std::vector<int32_t>& warped,
                      const std::vector<int32_t>& ypos);
void build_gather(ig_hier& h, Level& L, const ig_level& src, const std::vector<int32_t>& ypos,
                  const std::vector<double>& sval);

// Smoother layout for one level (see kernels.cuh: AsGroups / AsGather).
void build_smoother(ig_hier& h, Level& L, const ig_level& src) {
  const ig_blocks& B = src.blocks;
  const int32_t n = L.n, nb = B.n_blocks;
  if (nb <= 0 || !B.blk_ptr || !B.blk_dofs || !B.fac_ptr || !B.fac)
    throw Error(IG_INVALID_ARGUMENT, "smoother: empty block layout");
  L.n_blocks = nb;
  auto bsize = [&](int32_t b) { return B.blk_ptr[b + 1] - B.blk_ptr[b]; };
  // Multi-DOF blocks: compact ybuf positions; thread-per-block groups for
  // s <= 8 and s > 32, warp-per-block for 9 <= s <= 32.
  std::vector<int32_t> ypos(static_cast<size_t>(nb), -1);
  std::vector<int32_t> grouped, warped;
  int64_t yl = 0;
  std::vector<double> sval(static_cast<size_t>(nb), 0.0);
  for (int32_t b = 0; b < nb; ++b) {
    const int32_t s = bsize(b);
    if (s <= 0) throw Error(IG_INVALID_ARGUMENT, "smoother: empty block");
    for (int32_t i = B.blk_ptr[b]; i < B.blk_ptr[b + 1]; ++i)
      if (B.blk_dofs[i] < 0 || B.blk_dofs[i] >= n) throw Error(IG_INVALID_ARGUMENT, "smoother: DOF out of range");
    L.sum_s += s;
    L.sum_s2 += static_cast<int64_t>(s) * s;
    L.packed_F += static_cast<int64_t>(s) * (s + 1) / 2;
    if (s == 1) {
      sval[b] = B.fac[B.fac_ptr[b]];
      continue;
    }
    if (s > 128) throw Error(IG_INVALID_ARGUMENT, "smoother: block larger than 128 DOFs");
    ypos[b] = static_cast<int32_t>(yl);
    yl += s;
    if (s >= 9 && s <= 32)
      warped.push_back(b);
    else
      grouped.push_back(b);
  }
  if (yl > INT32_MAX) throw Error(IG_INVALID_ARGUMENT, "smoother: too many block entries");
  L.n_multi = static_cast<int32_t>(grouped.size() + warped.size());
  std::vector<double> minv;  // tolerance mode: explicit inverses in the factor layout
  ig_blocks BI = B;
  if (opt().fast_blocks) {
    minv.assign(B.fac, B.fac + B.fac_ptr[nb]);
    parallel_rows(nb, [&](int32_t b0, int32_t b1) {
      std::vector<double> y;
      for (int32_t b = b0; b < b1; ++b) {
        const int s = bsize(b);
        if (s == 1) continue;
        const double* f = B.fac + B.fac_ptr[b];
        double* m = minv.data() + B.fac_ptr[b];
        auto L = [&](int i, int j) { return f[static_cast<size_t>(j) * s + i]; };
        y.assign(static_cast<size_t>(s), 0.0);
        for (int j = 0; j < s; ++j) {  // column j of M: the oracle's LLT solve of e_j
          std::fill(y.begin(), y.end(), 0.0);
          y[j] = 1.0;
          for (int c = 0; c < s; ++c) {
            const double yc = y[c] / L(c, c);
            y[c] = yc;
            for (int i = c + 1; i < s; ++i) y[i] = y[i] - L(i, c) * yc;
          }
          for (int i = s - 1; i >= 0; --i) {
            double acc = 0.0;
            for (int k = s - 1; k > i; --k) acc = acc + L(k, i) * y[k];
            y[i] = (y[i] - acc) / L(i, i);
          }
          for (int i = j; i < s; ++i) m[static_cast<size_t>(j) * s + i] = y[i];  // lower triangle of M
        }
      }
    });
    BI.fac = minv.data();
  }
  L.G = build_groups(h, BI, grouped, warped, ypos);
  L.G.inv = opt().fast_blocks ? 1 : 0;
  {
    std::vector<int32_t> gs(grouped.size());
    for (size_t k = 0; k < grouped.size(); ++k) gs[k] = bsize(grouped[k]);
    std::stable_sort(gs.begin(), gs.end(), [](int32_t a, int32_t b) { return a > b; });
    int32_t first = static_cast<int32_t>((grouped.size() + 31) / 32);
    for (int32_t g = 0; g < static_cast<int32_t>((grouped.size() + 31) / 32); ++g)
      if (gs[static_cast<size_t>(g) * 32] <= 4) {
        first = g;
        break;
      }
    L.g_small = first;
  }
  L.ybuf = h.alloc<double>(static_cast<size_t>(std::max<int64_t>(yl, 1)));
  build_gather(h, L, src, ypos, sval);
}

// Batched block-solve layout (kernels.cuh AsGroups) for a subset of blocks:
// `grouped` thread-per-block (sorted by size, descending, stable), `warped`
// warp-per-block.  ypos: ybuf offsets (additive) -- unused by the
// multiplicative sweep, which writes by DOF.
AsGroups build_groups(ig_hier& h, const ig_blocks& B, std::vector<int32_t> grouped, const std::vector<int32_t>& warped,
                      const std::vector<int32_t>& ypos) {
  auto bsize = [&](int32_t b) { return B.blk_ptr[b + 1] - B.blk_ptr[b]; };
  AsGroups G{};
  std::stable_sort(grouped.begin(), grouped.end(), [&](int32_t a, int32_t b) { return bsize(a) > bsize(b); });
  const int32_t ng = static_cast<int32_t>((grouped.size() + 31) / 32);
  const size_t ng1 = static_cast<size_t>(std::max(ng, 1));
  std::vector<int32_t> gsmax(ng1, 0), gsize(ng1 * 32, 0), gypos(ng1 * 32, 0), gdofs;
  std::vector<int64_t> gdoff(ng1, 0), gfoff(ng1, 0);
  std::vector<double> gfac;
  for (int32_t g = 0; g < ng; ++g) {
    const int32_t smax = bsize(grouped[static_cast<size_t>(g) * 32]);
    gsmax[g] = smax;
    gdoff[g] = static_cast<int64_t>(gdofs.size());
    gfoff[g] = static_cast<int64_t>(gfac.size());
    const int64_t np = static_cast<int64_t>(smax) * (smax + 1) / 2;
    gdofs.resize(gdofs.size() + static_cast<size_t>(smax) * 32, 0);
    gfac.resize(gfac.size() + static_cast<size_t>(np) * 32, 1.0);
    for (int lane = 0; lane < 32; ++lane) {
      const size_t idx = static_cast<size_t>(g) * 32 + lane;
      if (idx >= grouped.size()) continue;
      const int32_t b = grouped[idx];
      const int32_t s = bsize(b);
      gsize[idx] = s;
      gypos[idx] = ypos.empty() ? 0 : ypos[b];
      for (int i = 0; i < s; ++i) gdofs[gdoff[g] + static_cast<int64_t>(i) * 32 + lane] = B.blk_dofs[B.blk_ptr[b] + i];
      const double* f = B.fac + B.fac_ptr[b];
      for (int j = 0; j < s; ++j)
        for (int i = j; i < s; ++i) {
          const int64_t e = static_cast<int64_t>(j) * smax - (static_cast<int64_t>(j) * (j - 1)) / 2 + (i - j);
          gfac[gfoff[g] + e * 32 + lane] = f[static_cast<size_t>(j) * s + i];
        }
    }
  }
  G.n_groups = ng;
  G.smax = h.upload(gsmax.data(), gsmax.size());
  G.dof_off = h.upload(gdoff.data(), gdoff.size());
  G.fac_off = h.upload(gfoff.data(), gfoff.size());
  G.size = h.upload(gsize.data(), gsize.size());
  G.ypos = h.upload(gypos.data(), gypos.size());
  G.dofs = h.upload(gdofs.data(), gdofs.size());  // empty -> 1-element placeholder
  G.fac = h.upload(gfac.data(), gfac.size());
  // Warp blocks: contiguous DOF lists and full column-major factors.
  {
    const size_t nw = warped.size();
    std::vector<int32_t> wsize(std::max<size_t>(nw, 1), 0), wypos(std::max<size_t>(nw, 1), 0), wdofs;
    std::vector<int64_t> wdoff(std::max<size_t>(nw, 1), 0), wfoff(std::max<size_t>(nw, 1), 0);
    std::vector<double> wfac;
    for (size_t k = 0; k < nw; ++k) {
      const int32_t b = warped[k];
      const int32_t s = bsize(b);
      wsize[k] = s;
      wypos[k] = ypos.empty() ? 0 : ypos[b];
      wdoff[k] = static_cast<int64_t>(wdofs.size());
      wfoff[k] = static_cast<int64_t>(wfac.size());
      wdofs.insert(wdofs.end(), B.blk_dofs + B.blk_ptr[b], B.blk_dofs + B.blk_ptr[b + 1]);
      wfac.insert(wfac.end(), B.fac + B.fac_ptr[b], B.fac + B.fac_ptr[b] + static_cast<int64_t>(s) * s);
    }
    G.n_wblocks = static_cast<int32_t>(nw);
    G.w_size = h.upload(wsize.data(), wsize.size());
    G.w_ypos = h.upload(wypos.data(), wypos.size());
    G.w_dof_off = h.upload(wdoff.data(), wdoff.size());
    G.w_fac_off = h.upload(wfoff.data(), wfoff.size());
    G.w_dofs = h.upload(wdofs.data(), wdofs.size());
    G.w_fac = h.upload(wfac.data(), wfac.size());
  }
  return G;
}

// Per-DOF gather of the additive smoother (kernels.cuh AsGather).
void build_gather(ig_hier& h, Level& L, const ig_level& src, const std::vector<int32_t>& ypos,
                  const std::vector<double>& sval) {
  const ig_blocks& B = src.blocks;
  const int32_t n = L.n, nb = B.n_blocks;
  auto bsize = [&](int32_t b) { return B.blk_ptr[b + 1] - B.blk_ptr[b]; };
  // Per-DOF contribution lists in ascending block order; DOFs whose only
  // contribution is their own singleton take the head >= 0 fast path.
  std::vector<int32_t> cnt(static_cast<size_t>(n) + 1, 0);
  for (int32_t b = 0; b < nb; ++b)
    for (int32_t i = B.blk_ptr[b]; i < B.blk_ptr[b + 1]; ++i) ++cnt[B.blk_dofs[i] + 1];
  for (int32_t d = 0; d < n; ++d) cnt[d + 1] += cnt[d];
  std::vector<int32_t> centry(static_cast<size_t>(cnt[n]));
  std::vector<int32_t> nx(cnt.begin(), cnt.end() - 1);
  for (int32_t b = 0; b < nb; ++b) {
    const int32_t s = bsize(b);
    for (int32_t i = 0; i < s; ++i) {
      const int32_t d = B.blk_dofs[B.blk_ptr[b] + i];
      centry[nx[d]++] = s == 1 ? -(b + 1) : ypos[b] + i;
    }
  }
  std::vector<int32_t> head(static_cast<size_t>(n), 0), cptr{0}, cent, cdof;
  std::vector<double> sdiag(static_cast<size_t>(n), 0.0);
  for (int32_t d = 0; d < n; ++d) {
    const int32_t q0 = cnt[d], q1 = cnt[d + 1];
    if (q1 - q0 == 1 && centry[q0] < 0) {
      head[d] = 0;
      sdiag[d] = sval[-centry[q0] - 1];
    } else {
      head[d] = -static_cast<int32_t>(cptr.size());  // -(c+1), c = cptr.size()-1
      cdof.push_back(d);
      cent.insert(cent.end(), centry.begin() + q0, centry.begin() + q1);
      cptr.push_back(static_cast<int32_t>(cent.size()));
    }
  }
  L.S.n_complex = static_cast<int32_t>(cdof.size());
  L.S.cdof = h.upload(cdof.data(), cdof.size());
  L.S.n = n;
  L.S.gamma = src.gamma;
  L.S.head = h.upload(head.data(), head.size());
  L.S.sdiag = h.upload(sdiag.data(), sdiag.size());
  L.S.cptr = h.upload(cptr.data(), cptr.size());
  L.S.centry = h.upload(cent.data(), cent.size());
  L.S.sval = h.upload(sval.data(), sval.size());
  L.n_complex = static_cast<int32_t>(cptr.size() - 1);
}

// Multiplicative (colored) Schwarz layout (kernels.cuh k_ms_*): per colour,
// the batched block solves of its blocks and the colour's columns of A over
// the rows they touch (ascending row, ascending column: A's own order).
void build_ms(ig_hier& h, Level& L, const ig_level& src, const ig_csr& A) {
  const ig_blocks& B = src.blocks;
  const int32_t n = L.n, nb = B.n_blocks;
  if (nb <= 0 || !B.blk_ptr || !B.blk_dofs || !B.fac_ptr || !B.fac)
    throw Error(IG_INVALID_ARGUMENT, "smoother: empty block layout");
  if (B.n_colors <= 0 || !B.color_of) throw Error(IG_INVALID_ARGUMENT, "multiplicative smoother: no block colours");
  const int C = B.n_colors;
  L.ms = true;
  L.gamma = src.gamma;
  L.n_blocks = nb;
  auto bsize = [&](int32_t b) { return B.blk_ptr[b + 1] - B.blk_ptr[b]; };
  std::vector<std::vector<int32_t>> cb(static_cast<size_t>(C));
  for (int32_t b = 0; b < nb; ++b) {
    const int32_t s = bsize(b);
    if (s <= 0) throw Error(IG_INVALID_ARGUMENT, "smoother: empty block");
    if (s > 128) throw Error(IG_INVALID_ARGUMENT, "smoother: block larger than 128 DOFs");
    if (B.color_of[b] < 0 || B.color_of[b] >= C) throw Error(IG_INVALID_ARGUMENT, "smoother: colour out of range");
    for (int32_t i = B.blk_ptr[b]; i < B.blk_ptr[b + 1]; ++i)
      if (B.blk_dofs[i] < 0 || B.blk_dofs[i] >= n) throw Error(IG_INVALID_ARGUMENT, "smoother: DOF out of range");
    L.sum_s += s;
    L.sum_s2 += static_cast<int64_t>(s) * s;
    L.packed_F += static_cast<int64_t>(s) * (s + 1) / 2;
    if (s > 1) ++L.n_multi;
    cb[B.color_of[b]].push_back(b);
  }
  std::vector<int32_t> mark(static_cast<size_t>(n), -1);
  L.colors.resize(static_cast<size_t>(C));
  std::vector<int32_t> ptr, col, rowmap;
  std::vector<double> val;
  for (int c = 0; c < C; ++c) {
    Level::MsColor& mc = L.colors[c];
    if (cb[c].empty()) continue;
    std::vector<int32_t> grouped, warped;
    for (int32_t b : cb[c]) {
      const int32_t s = bsize(b);
      if (s >= 9 && s <= 32)
        warped.push_back(b);
      else
        grouped.push_back(b);
      for (int32_t i = B.blk_ptr[b]; i < B.blk_ptr[b + 1]; ++i) {
        if (mark[B.blk_dofs[i]] == c) throw Error(IG_INVALID_ARGUMENT, "smoother: same-colour blocks share a DOF");
        mark[B.blk_dofs[i]] = c;
        ++mc.n_dofs;
      }
    }
    mc.G = build_groups(h, B, grouped, warped, {});
    mc.n_items = mc.G.n_groups + mc.G.n_wblocks;
    ptr.assign(1, 0);
    col.clear();
    val.clear();
    rowmap.clear();
    for (int32_t i = 0; i < n; ++i) {
      const size_t before = col.size();
      for (int32_t k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k)
        if (mark[A.col_idx[k]] == c) {
          col.push_back(A.col_idx[k]);
          val.push_back(A.val[k]);
        }
      if (col.size() > before) {
        rowmap.push_back(i);
        ptr.push_back(static_cast<int32_t>(col.size()));
      }
    }
    const int32_t nr = static_cast<int32_t>(rowmap.size());
    mc.S = h.upload_sell(to_sell(nr, n, ptr.data(), col.data(), val.data()), static_cast<int64_t>(col.size()));
    mc.rowmap = h.upload(rowmap.data(), rowmap.size());
  }
  L.ms_cur = h.alloc<double>(n);
  L.ms_delta = h.alloc<double>(n);
  L.ms_x = h.alloc<double>(n);
}


}  // namespace

extern "C" {

const char* ig_last_error(void) { return g_err.c_str(); }

int ig_set_option(int32_t option, int64_t value) {
  if (option == IG_OPT_USE_GRAPH) {
    g_defaults.use_graph = value != 0;
    return IG_OK;
  }
  if (option == IG_OPT_ROW_DICT) {
    g_defaults.use_dict = value != 0;
    return IG_OK;
  }
  if (option == IG_OPT_RED_CTAS) {
    if (value < 1 || value > 64) return fail(IG_INVALID_ARGUMENT, "ig_set_option: reduction CTAs per SM in 1..64");
    g_defaults.red_ctas = static_cast<int>(value);
    return IG_OK;
  }
  if (option == IG_OPT_PSELL_LINES2) {
    g_defaults.psell_lines2 = value != 0;
    return IG_OK;
  }
  if (option == IG_OPT_PSELL_CTAB) {
    g_defaults.psell_ctab = value != 0;
    return IG_OK;
  }
  if (option == IG_OPT_PSELL_MULTI) {
    g_defaults.psell_multi = value != 0;
    return IG_OK;
  }
  if (option == IG_OPT_PSELL_ROWS4) {
    g_defaults.psell_rows4 = value != 0;
    return IG_OK;
  }
  if (option == IG_OPT_PSELL_ROWS4_ROWS) {
    if (value < 0 || value > INT32_MAX) return fail(IG_INVALID_ARGUMENT, "ig_set_option: bad row count");
    g_defaults.psell_rows4_rows = static_cast<int32_t>(value);
    return IG_OK;
  }
  if (option == IG_OPT_PSELL_EDGE_ROWS) {
    if (value < 0 || value > INT32_MAX) return fail(IG_INVALID_ARGUMENT, "ig_set_option: bad row count");
    g_defaults.psell_edge_rows = static_cast<int32_t>(value);
    return IG_OK;
  }
  if (option == IG_OPT_PSELL_ORDER) {
    if (value < 0 || value > 2) return fail(IG_INVALID_ARGUMENT, "ig_set_option: slice order in 0..2");
    g_defaults.psell_order = static_cast<int>(value);
    return IG_OK;
  }
  if (option == IG_OPT_PSELL_AB) {
    g_defaults.psell_ab = value != 0;
    return IG_OK;
  }
  if (option == IG_OPT_GAL_SHORT) {
    g_defaults.gal_short = value != 0;
    return IG_OK;
  }
  if (option == IG_OPT_L2_MB) {
    if (value < 1 || value > 4096) return fail(IG_INVALID_ARGUMENT, "ig_set_option: L2 arena MB in 1..4096");
    g_defaults.l2_bytes = static_cast<size_t>(value) << 20;
    return IG_OK;
  }
  if (option == IG_OPT_L2_ROWS) {
    if (value < 0 || value > INT32_MAX) return fail(IG_INVALID_ARGUMENT, "ig_set_option: L2 rows out of range");
    g_defaults.l2_rows = static_cast<int32_t>(value);
    return IG_OK;
  }
  if (option == IG_OPT_PSELL_PAIRS_ROWS) {
    if (value < 0 || value > INT32_MAX) return fail(IG_INVALID_ARGUMENT, "ig_set_option: rows out of range");
    g_defaults.psell_pairs_rows = static_cast<int32_t>(value);
    return IG_OK;
  }
  if (option == IG_OPT_FAST_COARSE) {
    g_defaults.fast_coarse = value != 0;
    return IG_OK;
  }
  if (option == IG_OPT_FAST_BLOCKS) {
    g_defaults.fast_blocks = value != 0;
    return IG_OK;
  }
  if (option == IG_OPT_COMPLEX4_ROWS || option == IG_OPT_ONE_STREAM_ROWS) {
    if (value < 0 || value > INT32_MAX) return fail(IG_INVALID_ARGUMENT, "ig_set_option: rows out of range");
    (option == IG_OPT_COMPLEX4_ROWS ? g_defaults.complex4_rows : g_defaults.one_stream_rows) =
        static_cast<int32_t>(value);
    return IG_OK;
  }
  if (option == IG_OPT_PSELL_CTAS) {
    if (value < 0 || value > 8) return fail(IG_INVALID_ARGUMENT, "ig_set_option: pattern-SELL CTAs per SM in 0..8");
    g_defaults.psell_ctas = static_cast<int>(value);
    const int sm = static_cast<int>(psell_smem());
    void (*ks[])(PSell, const double*, double*, const double*, const PcgState*, const PValTab) = {
        k_pspmv<0, true>, k_pspmv<0, false>, k_pspmv<1, true>, k_pspmv<1, false>};
    for (auto k : ks) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_pprolong<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_pprolong<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    return IG_OK;
  }
  if (option == IG_OPT_PDL) {
    g_defaults.use_pdl = value != 0;
    return IG_OK;
  }
  if (option == IG_OPT_PSELL) {
    g_defaults.use_psell = value != 0;
    return IG_OK;
  }
  if (option == IG_OPT_SMALL_ROWS) {
    if (value < 0 || value > INT32_MAX) return fail(IG_INVALID_ARGUMENT, "ig_set_option: bad row threshold");
    g_defaults.small_rows = static_cast<int>(value);
    return IG_OK;
  }
  return fail(IG_INVALID_ARGUMENT, "ig_set_option: unknown option");
}

int ig_hier_matches(ig_hier* h, const ig_csr* a) {
  if (!h || !a) return fail(IG_INVALID_ARGUMENT, "ig_hier_matches: null argument");
  const ig_csr& f = h->fine_src;
  if (a->n_rows != f.n_rows || a->n_cols != f.n_cols || a->nnz != f.nnz)
    return fail(IG_INVALID_ARGUMENT, "the operator's dimensions / nnz differ from the hierarchy's finest A");
  if (a->row_ptr == f.row_ptr && a->col_idx == f.col_idx && a->val == f.val) return IG_OK;
  if (!a->row_ptr || !a->col_idx || !a->val) return fail(IG_INVALID_ARGUMENT, "ig_hier_matches: null arrays");
  if (csr_hash(*a) != h->fine_hash)
    return fail(IG_INVALID_ARGUMENT, "the operator differs from the finest A the hierarchy was built on "
                                     "(the device solve multiplies by that A)");
  return IG_OK;
}

int ig_hier_set_option(ig_hier* h, int32_t option, int64_t value) {
  if (!h) return fail(IG_INVALID_ARGUMENT, "ig_hier_set_option: null handle");
  std::lock_guard<std::mutex> lk(h->mu);
  Opts& o = h->opts;
  if (option == IG_OPT_USE_GRAPH) {
    o.use_graph = value != 0;
  } else if (option == IG_OPT_PDL) {
    o.use_pdl = value != 0;
  } else if (option == IG_OPT_COMPLEX4_ROWS || option == IG_OPT_ONE_STREAM_ROWS) {
    if (value < 0 || value > INT32_MAX) return fail(IG_INVALID_ARGUMENT, "ig_hier_set_option: rows out of range");
    (option == IG_OPT_COMPLEX4_ROWS ? o.complex4_rows : o.one_stream_rows) = static_cast<int32_t>(value);
  } else if (option == IG_OPT_RED_CTAS) {
    if (value < 1 || value > 64) return fail(IG_INVALID_ARGUMENT, "ig_hier_set_option: reduction CTAs per SM in 1..64");
    o.red_ctas = static_cast<int>(value);
  } else {
    return fail(IG_INVALID_ARGUMENT,
                "ig_hier_set_option: only IG_OPT_USE_GRAPH, IG_OPT_PDL, IG_OPT_RED_CTAS, IG_OPT_COMPLEX4_ROWS and "
                "IG_OPT_ONE_STREAM_ROWS change after "
                "ig_hier_create (layout options: ig_set_option before creating the handle)");
  }
  h->drop_graphs();
  return IG_OK;
}

int ig_hier_create(const ig_level* levels, int32_t n_levels, const ig_coarse* coarse, ig_hier** out) {
  if (!out) return fail(IG_INVALID_ARGUMENT, "ig_hier_create: null out");
  *out = nullptr;
  if (!levels || !coarse || n_levels < 1 || n_levels > 16)
    return fail(IG_INVALID_ARGUMENT, "ig_hier_create: need 1..16 levels and a coarse factor");
  return guarded([&] {
    auto h = std::make_unique<ig_hier>();
    h->opts = g_defaults;
    OptScope os_(&h->opts);
    h->L = n_levels;
    h->lv.resize(n_levels);
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->side2, cudaStreamNonBlocking));
    CK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&h->ev_join2, cudaEventDisableTiming));
    CK(cudaEventCreate(&h->ev0));
    CK(cudaEventCreate(&h->ev1));
    ig_info& I = h->info;
    I.n_levels = n_levels;
    I.coarse_n = coarse->n;
    I.coarse_rank = coarse->rank;
    h->fine_src = levels[n_levels - 1].A;
    h->fine_hash = csr_hash(levels[n_levels - 1].A);
    if (opt().l2_rows > 0 && n_levels > 1) {
      void* p = nullptr;
      CK(cudaMalloc(&p, opt().l2_bytes));
      h->allocs.push_back(p);
      h->arena = static_cast<char*>(p);
      h->arena_cap = opt().l2_bytes;
    }
    for (int l = 0; l < n_levels; ++l) {
      const ig_level& s = levels[l];
      Level& L = h->lv[l];
      h->arena_on = l < n_levels - 1 && s.A.n_rows <= opt().l2_rows;
      check_csr(s.A, "A");
      if (s.A.n_rows != s.A.n_cols) throw Error(IG_INVALID_ARGUMENT, "A must be square");
      L.n = s.A.n_rows;
      if (L.n <= 0) throw Error(IG_INVALID_ARGUMENT, "empty level");
      I.n[l] = L.n;
      I.nnz_A[l] = s.A.nnz;
      L.r_in = h->alloc<double>(L.n);
      L.x = h->alloc<double>(L.n);
      if (l == 0) continue;
      check_csr(s.R, "R");
      if (s.R.n_cols != L.n || s.R.n_rows != levels[l - 1].A.n_rows)
        throw Error(IG_INVALID_ARGUMENT, "R has the wrong shape");
      if (s.smoother_kind != IG_SMOOTHER_ADDITIVE_SCHWARZ && s.smoother_kind != IG_SMOOTHER_MULTIPLICATIVE_SCHWARZ)
        throw Error(IG_UNSUPPORTED, "device smoother: additive or multiplicative Schwarz only");
      I.nnz_R[l] = s.R.nnz;
      const bool timing = std::getenv("IG_TIMING") != nullptr;
      auto tnow = [] { return std::chrono::steady_clock::now(); };
      auto secs = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
      const auto t0 = tnow();
      L.A = h->make_matrix(s.A.n_rows, s.A.n_cols, s.A.row_ptr, s.A.col_idx, s.A.val, s.A.nnz);
      const auto t1 = tnow();
      L.R = h->make_matrix(s.R.n_rows, s.R.n_cols, s.R.row_ptr, s.R.col_idx, s.R.val, s.R.nnz);
      const auto t2 = tnow();
      std::vector<int32_t> tp, tc;
      std::vector<double> tv;
      csr_transpose(s.R, tp, tc, tv);
      L.P = h->make_matrix(s.R.n_cols, s.R.n_rows, tp.data(), tc.data(), tv.data(), s.R.nnz);
      const auto t3 = tnow();
      L.res = h->alloc<double>(L.n);
      L.cor = h->alloc<double>(L.n);
      if (s.smoother_kind == IG_SMOOTHER_MULTIPLICATIVE_SCHWARZ)
        build_ms(*h, L, s, s.A);
      else
        build_smoother(*h, L, s);
      const auto t4 = tnow();
      if (timing)
        std::fprintf(stderr, "[ig_hier_create] level %d n=%d: A %.3f s, R %.3f s, P %.3f s, smoother %.3f s\n", l, L.n,
                     secs(t0, t1), secs(t1, t2), secs(t2, t3), secs(t3, t4));
      I.sell_slots_A[l] = L.A.slots;
      I.n_blocks[l] = L.n_blocks;
      I.n_multi_blocks[l] = L.n_multi;
      I.sum_s[l] = L.sum_s;
      I.sum_s2[l] = L.sum_s2;
    }
    // Finest A is used by PCG even with a single level.
    Level& F = h->lv[n_levels - 1];
    if (n_levels == 1) {
      const ig_level& s = levels[0];
      F.A = h->make_matrix(s.A.n_rows, s.A.n_cols, s.A.row_ptr, s.A.col_idx, s.A.val, s.A.nnz);
      I.sell_slots_A[0] = F.A.slots;
    }
    // Coarse factor.
    h->n0 = coarse->n;
    h->rank = coarse->rank;
    if (h->n0 != h->lv[0].n) throw Error(IG_INVALID_ARGUMENT, "coarse factor size differs from level 0");
    if (h->rank < 0 || h->rank > h->n0) throw Error(IG_INVALID_ARGUMENT, "coarse rank out of range");
    if (h->rank > 1024) throw Error(IG_UNSUPPORTED, "coarse rank above 1024");
    if (!coarse->L || !coarse->piv) throw Error(IG_INVALID_ARGUMENT, "coarse factor arrays are null");
    for (int k = 0; k < h->n0; ++k)
      if (coarse->piv[k] < 1 || coarse->piv[k] > h->n0) throw Error(IG_INVALID_ARGUMENT, "coarse pivot out of range");
    const int64_t rk = h->rank, n0 = h->n0;
    // Packed lower L11, padded to an even count (16-byte TMA bulk copies).
    const int64_t np = rk * (rk + 1) / 2, np_al = (np + 1) & ~int64_t(1);
    std::vector<double> packed(static_cast<size_t>(std::max<int64_t>(np_al, 2)), 0.0);
    for (int64_t j = 0; j < rk; ++j)
      for (int64_t i = j; i < rk; ++i) packed[j * rk - (j * (j - 1)) / 2 + (i - j)] = coarse->L[j * n0 + i];
    h->arena_on = h->arena != nullptr;
    h->Lp = h->upload(packed.data(), packed.size());
    h->piv = h->upload(coarse->piv, static_cast<size_t>(n0));
    if (opt().fast_coarse && rk > 0) {
      // Column j of M: the oracle-order substitutions (oracle.c tri_solve) of e_j.
      std::vector<double> M(static_cast<size_t>(rk * rk)), y(static_cast<size_t>(rk));
      auto L = [&](int64_t i, int64_t j) { return coarse->L[j * n0 + i]; };
      for (int64_t j = 0; j < rk; ++j) {
        std::fill(y.begin(), y.end(), 0.0);
        y[j] = 1.0;
        for (int64_t c = 0; c < rk; ++c) {
          const double yc = y[c] / L(c, c);
          y[c] = yc;
          for (int64_t i = c + 1; i < rk; ++i) y[i] = y[i] - L(i, c) * yc;
        }
        for (int64_t i = rk - 1; i >= 0; --i) {
          double acc = 0.0;
          for (int64_t k = rk - 1; k > i; --k) acc = acc + L(k, i) * y[k];
          y[i] = (y[i] - acc) / L(i, i);
        }
        for (int64_t i = 0; i < rk; ++i) M[i * rk + j] = y[i];
      }
      h->Minv = h->upload(M.data(), M.size());
      h->fast_coarse = true;
    }
    h->arena_on = false;
    if (h->arena && h->arena_used > 0) {
      size_t lim = 0;
      int maxp = 0;
      CK(cudaDeviceGetLimit(&lim, cudaLimitPersistingL2CacheSize));
      CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0));
      const size_t want = std::min<size_t>(h->arena_used, static_cast<size_t>(maxp));
      if (lim < want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
      cudaGetLastError();
      if (std::getenv("IG_TIMING"))
        std::fprintf(stderr, "[ig_hier_create] L2 arena: %zu bytes used, persisting max %d\n", h->arena_used, maxp);
      cudaStreamAttrValue av = {};
      av.accessPolicyWindow.base_ptr = h->arena;
      av.accessPolicyWindow.num_bytes = h->arena_used;
      av.accessPolicyWindow.hitRatio =
          std::min(1.0f, static_cast<float>(static_cast<double>(std::max(maxp, 1)) / static_cast<double>(h->arena_used)));
      av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      CK(cudaStreamSetAttribute(h->stream, cudaStreamAttributeAccessPolicyWindow, &av));
      CK(cudaStreamSetAttribute(h->side, cudaStreamAttributeAccessPolicyWindow, &av));
      CK(cudaStreamSetAttribute(h->side2, cudaStreamAttributeAccessPolicyWindow, &av));
    }
    h->coarse_threads = static_cast<int>(std::max<int64_t>(32, (rk + 31) / 32 * 32));  // one row per thread
    // [packed L11][forward results: rank][backward results: rank]
    const size_t smem = sizeof(double) * static_cast<size_t>(np_al + 2 * rk + 2);
    int max_optin = 0;
    CK(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0));
    const int dyn_cap = max_optin - 1024;  // headroom for the kernel's static shared memory
    if (smem <= static_cast<size_t>(dyn_cap)) {
      h->coarse_use_smem = 1;
      h->coarse_smem = smem;
      // Process-wide function attributes: raised to the cap once so no handle
      // created later can shrink them below another handle's need.
      CK(cudaFuncSetAttribute(k_coarse<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_cap));
      CK(cudaFuncSetAttribute(k_coarse<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_cap));
      void (*kw[])(int32_t, int32_t, const double*, const int32_t*, const double*, double*, const PcgState*) = {
          k_coarse_warp<1, true>, k_coarse_warp<2, true>, k_coarse_warp<3, true>, k_coarse_warp<4, true>,
          k_coarse_warp<5, true>, k_coarse_warp<6, true>, k_coarse_warp<7, true>, k_coarse_warp<8, true>};
      for (auto k : kw) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_cap));
    } else {
      h->coarse_use_smem = 0;
      h->coarse_smem = sizeof(double) * static_cast<size_t>(2 * rk + 2);
    }
    // PCG workspace.
    const int32_t nf = F.n;
    h->r = h->alloc<double>(nf);
    h->z = h->alloc<double>(nf);
    h->p = h->alloc<double>(nf);
    h->ap = h->alloc<double>(nf);
    h->hb = h->alloc<double>(nf);
    h->hx = h->alloc<double>(nf);
    h->partials = h->alloc<double>(grid_of(nf) + 1);
    h->st = h->alloc<PcgState>(1);
    CK(cudaMemset(h->st, 0, sizeof(PcgState)));
    h->ensure_residuals(1000);
    // Algorithmic bytes and launch counts.
    // layout_bytes: the same, counting only the matrix words the device
    // layout leaves in HBM (row dictionary / pattern SELL).
    auto layout_spmv = [](const DevSell& M, int64_t nr, int64_t nin, bool resid) {
      return M.layout_matrix_bytes() + 8 * nin + 8 * nr + (resid ? 8 * nr : 0);
    };
    int64_t vc = 0, vcl = 0;
    int kv = 1;  // coarse
    for (int l = 1; l < n_levels; ++l) {
      const Level& L = h->lv[l];
      const int64_t n = L.n, nc = h->lv[l - 1].n;
      int64_t as = 8 * L.packed_F + 8 * L.sum_s + 4 * (L.n_blocks + 1) + 4 * (n + 1) + 16 * n;
      if (L.ms) {  // colored sweep: block solves + the colours' residual updates + init/finish
        as = 8 * L.packed_F + 16 * L.sum_s + 40 * n;
        for (const auto& mc : L.colors) as += 12 * mc.S.nnz + 16 * mc.n_dofs;
      }
      vc += 2 * bytes_spmv(n, n, L.A.nnz, true);
      vc += 2 * as + 8 * n;                                              // second application accumulates
      vc += bytes_spmv(nc, n, L.R.nnz, false);                           // R
      vc += 12 * L.R.nnz + 4 * (n + 1) + 8 * nc + 16 * n + 8 * n;        // P + x update
      vcl += 2 * layout_spmv(L.A, n, n, true) + 2 * as + 8 * n + layout_spmv(L.R, nc, n, false) +
             layout_spmv(L.P, n, nc, false) + 16 * n;
      // smoother: [blocks] + simple + [complex | finish_red on the finest], twice;
      // plus SpMV-residual x2, restriction, prolongation
      const int32_t gb = L.n >= kSplitRows ? L.g_small : L.G.n_groups;
      int per_app = (gb + L.G.n_wblocks > 0 ? 1 : 0) + (L.G.n_groups > gb ? 1 : 0) + 1 + (L.S.n_complex > 0 ? 1 : 0);
      if (L.ms) {
        int ne = 0;
        for (const auto& mc : L.colors) ne += mc.n_items > 0 ? 1 : 0;
        per_app = 2 + 2 * ne - 1;
      }
      kv += 2 * per_app + 4 + (l == n_levels - 1 && !L.ms ? 1 : 0);  // finest: + r . z pass
      kv += L.A.n_xe > 0 ? 2 : 0;  // k_xgather ahead of the two residual products (FASTE slices)
      I.explicit_vals_A[l] = L.A.explicit_vals;
      I.explicit_cols_A[l] = L.A.explicit_cols;
    }
    vc += 8 * static_cast<int64_t>(h->rank) * h->rank + 24 * static_cast<int64_t>(h->n0);
    vcl += 8 * static_cast<int64_t>(h->rank) * h->rank + 24 * static_cast<int64_t>(h->n0);
    I.bytes_vcycle = vc;
    I.bytes_vcycle_layout = vcl;
    I.bytes_spmv_finest = bytes_spmv(nf, nf, F.A.nnz, false);
    I.bytes_spmv_finest_layout = layout_spmv(F.A, nf, nf, false);
    I.explicit_vals_A[n_levels - 1] = F.A.explicit_vals;
    I.explicit_cols_A[n_levels - 1] = F.A.explicit_cols;
    I.bytes_pcg_iter = vc + I.bytes_spmv_finest + 80 * static_cast<int64_t>(nf);
    I.kernels_vcycle = kv;
    I.kernels_pcg_iter = kv + 3 + (F.A.has_p ? 1 : 0) + (F.A.n_xe > 0 ? 1 : 0);  // + k_pap after a pattern-SELL A p, + k_xgather
    CK(cudaDeviceSynchronize());
    *out = h.release();
    return IG_OK;
  });
}

void ig_hier_destroy(ig_hier* h) { delete h; }

int ig_hier_info(const ig_hier* h, ig_info* out) {
  if (!h || !out) return fail(IG_INVALID_ARGUMENT, "ig_hier_info: null argument");
  *out = h->info;
  return IG_OK;
}

void* ig_hier_stream(ig_hier* h) { return h ? static_cast<void*>(h->stream) : nullptr; }

int ig_vcycle_at(ig_hier* h, int32_t level, const double* r, double* x) {
  if (!h || !r || !x) return fail(IG_INVALID_ARGUMENT, "vcycle_at: null argument");
  if (level < 0 || level >= h->L) return fail(IG_INVALID_ARGUMENT, "vcycle_at: level out of range");
  std::lock_guard<std::mutex> lk(h->mu);
  OptScope os_(&h->opts);
  return guarded([&] {
    Level& L = h->lv[level];
    CK(cudaMemcpyAsync(L.r_in, r, sizeof(double) * L.n, cudaMemcpyHostToDevice, h->stream));
    h->vcycle(level, L.r_in, h->hx, nullptr, nullptr);
    CK(cudaMemcpyAsync(x, h->hx, sizeof(double) * L.n, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return IG_OK;
  });
}

int ig_vcycle(ig_hier* h, const double* r, double* x) {
  if (!h) return fail(IG_INVALID_ARGUMENT, "vcycle: null handle");
  return ig_vcycle_at(h, h->L - 1, r, x);
}

int ig_coarse_solve(ig_hier* h, const double* r, double* x) {
  if (!h) return fail(IG_INVALID_ARGUMENT, "coarse_solve: null handle");
  return ig_vcycle_at(h, 0, r, x);
}

int ig_smoother_apply(ig_hier* h, int32_t level, const double* r, double* x) {
  if (!h || !r || !x) return fail(IG_INVALID_ARGUMENT, "smoother_apply: null argument");
  if (level < 1 || level >= h->L) return fail(IG_INVALID_ARGUMENT, "smoother_apply: level has no smoother");
  std::lock_guard<std::mutex> lk(h->mu);
  OptScope os_(&h->opts);
  return guarded([&] {
    Level& L = h->lv[level];
    CK(cudaMemcpyAsync(L.r_in, r, sizeof(double) * L.n, cudaMemcpyHostToDevice, h->stream));
    h->smoother(L, L.r_in, h->hx, false, nullptr, nullptr);
    CK(cudaMemcpyAsync(x, h->hx, sizeof(double) * L.n, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return IG_OK;
  });
}

int ig_smoother_apply_dir(ig_hier* h, int32_t level, const double* r, double* x, int32_t dir) {
  if (!h || !r || !x) return fail(IG_INVALID_ARGUMENT, "smoother_apply: null argument");
  if (level < 1 || level >= h->L) return fail(IG_INVALID_ARGUMENT, "smoother_apply: level has no smoother");
  if (dir != 0 && dir != 1) return fail(IG_INVALID_ARGUMENT, "smoother_apply: dir must be 0 (Forward) or 1 (Reverse)");
  std::lock_guard<std::mutex> lk(h->mu);
  OptScope os_(&h->opts);
  return guarded([&] {
    Level& L = h->lv[level];
    CK(cudaMemcpyAsync(L.r_in, r, sizeof(double) * L.n, cudaMemcpyHostToDevice, h->stream));
    h->smoother(L, L.r_in, h->hx, false, nullptr, nullptr, dir);
    CK(cudaMemcpyAsync(x, h->hx, sizeof(double) * L.n, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return IG_OK;
  });
}

int ig_smoother_apply_symmetric(ig_hier* h, int32_t level, const double* r, double* x) {
  if (!h || !r || !x) return fail(IG_INVALID_ARGUMENT, "smoother_apply_symmetric: null argument");
  if (level < 1 || level >= h->L) return fail(IG_INVALID_ARGUMENT, "smoother_apply_symmetric: level has no smoother");
  std::lock_guard<std::mutex> lk(h->mu);
  OptScope os_(&h->opts);
  return guarded([&] {
    Level& L = h->lv[level];
    CK(cudaMemcpyAsync(L.r_in, r, sizeof(double) * L.n, cudaMemcpyHostToDevice, h->stream));
    h->smoother(L, L.r_in, h->hx, false, nullptr, nullptr, 0);   // x1 = S(r, Forward)
    h->spmv(L.A, 1, h->hx, L.cor, L.r_in, nullptr);            // r - A x1
    h->smoother(L, L.cor, h->hx, true, nullptr, nullptr, 1);    // x1 + S(., Reverse)
    CK(cudaMemcpyAsync(x, h->hx, sizeof(double) * L.n, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return IG_OK;
  });
}

int ig_level_spmv(ig_hier* h, int32_t level, const double* x, double* y, int32_t mode) {
  if (!h || !x || !y) return fail(IG_INVALID_ARGUMENT, "level_spmv: null argument");
  if (level < 0 || level >= h->L) return fail(IG_INVALID_ARGUMENT, "level_spmv: level out of range");
  if (mode < 0 || mode > 3) return fail(IG_INVALID_ARGUMENT, "level_spmv: bad mode");
  if (mode >= 2 && level == 0) return fail(IG_INVALID_ARGUMENT, "level_spmv: coarsest level has no R");
  std::lock_guard<std::mutex> lk(h->mu);
  OptScope os_(&h->opts);
  return guarded([&] {
    Level& L = h->lv[level];
    const DevSell* M = nullptr;
    if (mode <= 1) {
      if (level == 0 && h->L > 1) throw Error(IG_UNSUPPORTED, "level_spmv: coarsest A is not resident (dense factor only)");
      M = &L.A;
    } else {
      M = mode == 2 ? &L.R : &L.P;
    }
    const int32_t nin = M->s.n_cols, nout = M->s.n_rows;
    double* din = h->hb;   // finest-sized scratch (every level fits)
    double* dout = h->hx;
    CK(cudaMemcpyAsync(din, x, sizeof(double) * nin, cudaMemcpyHostToDevice, h->stream));
    if (mode == 1) CK(cudaMemcpyAsync(dout, y, sizeof(double) * nout, cudaMemcpyHostToDevice, h->stream));
    h->spmv(*M, mode == 1 ? 1 : 0, din, dout, dout);
    CK(cudaMemcpyAsync(y, dout, sizeof(double) * nout, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return IG_OK;
  });
}

int ig_level_spmv_device(ig_hier* h, int32_t level, const double* d_x, double* d_y, int32_t mode) {
  if (!h || !d_x || !d_y) return fail(IG_INVALID_ARGUMENT, "level_spmv_device: null argument");
  if (!aligned16(d_x) || !aligned16(d_y))
    return fail(IG_INVALID_ARGUMENT, "level_spmv_device: device vectors must be 16-byte aligned");
  if (level < 0 || level >= h->L || mode < 0 || mode > 3 || (mode >= 2 && level == 0))
    return fail(IG_INVALID_ARGUMENT, "level_spmv_device: bad level or mode");
  std::lock_guard<std::mutex> lk(h->mu);
  OptScope os_(&h->opts);
  return guarded([&] {
    Level& L = h->lv[level];
    if (mode <= 1 && level == 0 && h->L > 1)
      throw Error(IG_UNSUPPORTED, "level_spmv_device: coarsest A is not resident (dense factor only)");
    const DevSell& M = mode <= 1 ? L.A : (mode == 2 ? L.R : L.P);
    h->spmv(M, mode == 1 ? 1 : 0, d_x, d_y, d_y);
    return IG_OK;
  });
}

// Host-only: builds the pattern-SELL layout of a CSR operator (no device
// work) and reports its slice statistics (profiles/psell_stats.py), classes
// c = GENERAL, FAST, FAST2, FAST4, FAST2M: out[c] slices, out[5 + c] lanes
// used, out[10 + 4 c + b] slices by lanes used (1-8, 9-16, 17-24, 25-32),
// out[30] layout bytes, out[31] rows reading values from the constant-bank table.
int ig_debug_psell_stats(const ig_csr* a, int64_t* out, int32_t n_out) {
  if (!a || !out || n_out < 32) return fail(IG_INVALID_ARGUMENT, "debug_psell_stats: bad argument");
  return guarded([&] {
    OptScope os_(&g_defaults);
    HostPSell hp;
    for (int i = 0; i < n_out; ++i) out[i] = 0;
    if (!to_psell(a->n_rows, a->n_cols, a->row_ptr, a->col_idx, a->val, hp)) return IG_UNSUPPORTED;
    for (const PSliceMeta& m : hp.meta) {
      const int count = static_cast<int>((m.pk >> 11) & 0x3f);
      if (count == 0) continue;
      const bool fast = m.pk & (1u << 17);
      const int wv = static_cast<int>((m.pk >> 19) & 0x3f);
      const int cls = !fast ? ((m.pk >> 31) ? 1 : 0) : wv == 0 ? 1 : wv == 1 || wv == 4 ? 2 : wv == 2 || wv == 5 ? 3 : 4;  // (FASTE with FAST)  // (FASTAB counted with FAST2)
      ++out[cls];
      out[5 + cls] += count;
      ++out[10 + 4 * cls + (count - 1) / 8];
    }
    out[30] = hp.layout_bytes;
    out[31] = hp.tab_rows;
    return IG_OK;
  });
}

// Host-only: y = A x through the pattern-SELL layout the library would build
// for `a`, interpreted on the CPU with every index bounds-checked
// (psell_apply_host).  IG_UNSUPPORTED when the matrix does not fit the format.
int ig_debug_psell_apply(const ig_csr* a, const double* x, double* y) {
  if (!a || !x || !y) return fail(IG_INVALID_ARGUMENT, "debug_psell_apply: null argument");
  return guarded([&] {
    OptScope os_(&g_defaults);
    HostPSell hp;
    if (!to_psell(a->n_rows, a->n_cols, a->row_ptr, a->col_idx, a->val, hp)) return IG_UNSUPPORTED;
    std::string err;
    if (!psell_apply_host(hp, a->n_rows, a->n_cols, x, y, err)) throw Error(IG_INVALID_ARGUMENT, "debug_psell_apply: layout validation failed: " + err);
    return IG_OK;
  });
}

int ig_debug_vcycle_timeline(ig_hier* h, const double* d_r, double* d_x, int32_t max_steps, float* ms,
                             int32_t* levels, char* labels, int32_t label_len, int32_t* count) {
  if (!h || !d_r || !d_x || !ms || !count) return fail(IG_INVALID_ARGUMENT, "timeline: null argument");
  if (!aligned16(d_r) || !aligned16(d_x)) return fail(IG_INVALID_ARGUMENT, "timeline: device vectors must be 16-byte aligned");
  std::lock_guard<std::mutex> lk(h->mu);
  OptScope os_(&h->opts);
  return guarded([&] {
    std::vector<ig_hier::Mark> tl;
    cudaEvent_t start;
    CK(cudaEventCreate(&start));
    CK(cudaEventRecord(start, h->stream));
    h->timeline = &tl;
    try {
      h->vcycle(h->L - 1, d_r, d_x, nullptr, nullptr);
    } catch (...) {
      h->timeline = nullptr;
      throw;
    }
    h->timeline = nullptr;
    CK(cudaStreamSynchronize(h->stream));
    cudaEvent_t prev = start;
    int32_t k = 0;
    for (const auto& m : tl) {
      if (k < max_steps) {
        CK(cudaEventElapsedTime(&ms[k], prev, m.ev));
        if (levels) levels[k] = m.level;
        if (labels && label_len > 0) {
          std::strncpy(labels + static_cast<size_t>(k) * label_len, m.what, label_len - 1);
          labels[static_cast<size_t>(k) * label_len + label_len - 1] = 0;
        }
        ++k;
      }
      prev = m.ev;
    }
    *count = k;
    for (const auto& m : tl) cudaEventDestroy(m.ev);
    cudaEventDestroy(start);
    return IG_OK;
  });
}

int ig_vcycle_at_device(ig_hier* h, int32_t level, const double* d_r, double* d_x) {
  if (!h || !d_r || !d_x) return fail(IG_INVALID_ARGUMENT, "vcycle_device: null argument");
  if (level < 0 || level >= h->L) return fail(IG_INVALID_ARGUMENT, "vcycle_at_device: level out of range");
  if (!aligned16(d_r) || !aligned16(d_x))
    return fail(IG_INVALID_ARGUMENT, "vcycle_device: device vectors must be 16-byte aligned");
  std::lock_guard<std::mutex> lk(h->mu);
  OptScope os_(&h->opts);
  return guarded([&] {
    if (!opt().use_graph) {
      h->vcycle(level, d_r, d_x, nullptr, nullptr);
      return IG_OK;
    }
    cudaGraphExec_t ex = nullptr;
    for (auto& g : h->vc_graphs)
      if (g.level == level && g.r == d_r && g.x == d_x) ex = g.exec;
    if (!ex) {
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
      h->vcycle(level, d_r, d_x, nullptr, nullptr);
      CK(cudaStreamEndCapture(h->stream, &g));
      CK(cudaGraphInstantiate(&ex, g, 0));
      CK(cudaGraphDestroy(g));
      h->vc_graphs.push_back({level, d_r, d_x, ex});
    }
    CK(cudaGraphLaunch(ex, h->stream));
    return IG_OK;
  });
}

int ig_vcycle_device(ig_hier* h, const double* d_r, double* d_x) {
  if (!h) return fail(IG_INVALID_ARGUMENT, "vcycle_device: null argument");
  return ig_vcycle_at_device(h, h->L - 1, d_r, d_x);
}

int ig_pcg_device(ig_hier* h, const double* d_b, double tol, int32_t maxit, double* d_x) {
  if (!h || !d_b || !d_x) return fail(IG_INVALID_ARGUMENT, "pcg_device: null argument");
  if (!aligned16(d_b) || !aligned16(d_x))
    return fail(IG_INVALID_ARGUMENT, "pcg_device: device vectors must be 16-byte aligned");
  std::lock_guard<std::mutex> lk(h->mu);
  OptScope os_(&h->opts);
  return guarded([&] {
    h->pcg_launch(d_b, d_x, tol, maxit);
    return IG_OK;
  });
}

int ig_pcg_result(ig_hier* h, double* residuals, int32_t* iterations) {
  if (!h) return fail(IG_INVALID_ARGUMENT, "pcg_result: null handle");
  std::lock_guard<std::mutex> lk(h->mu);
  OptScope os_(&h->opts);
  return guarded([&] {
    const int s = h->pcg_collect(residuals, iterations);
    if (s == IG_NOT_CONVERGED) g_err = "pcg: no convergence within the iteration budget";
    if (s == IG_BREAKDOWN) g_err = "pcg: p^T A p <= 0 (operator not SPD)";
    return s;
  });
}

int ig_pcg(ig_hier* h, const double* b, double tol, int32_t maxit, double* x, double* residuals,
           int32_t* iterations, double* seconds) {
  if (!h || !b || !x || !residuals || !iterations) return fail(IG_INVALID_ARGUMENT, "pcg: null argument");
  if (maxit < 0) return fail(IG_INVALID_ARGUMENT, "pcg: maxit must be >= 0");
  std::lock_guard<std::mutex> lk(h->mu);
  OptScope os_(&h->opts);
  return guarded([&] {
    const int32_t n = h->lv[h->L - 1].n;
    CK(cudaMemcpyAsync(h->hb, b, sizeof(double) * n, cudaMemcpyHostToDevice, h->stream));
    CK(cudaEventRecord(h->ev0, h->stream));
    h->pcg_launch(h->hb, h->hx, tol, maxit);
    CK(cudaEventRecord(h->ev1, h->stream));
    CK(cudaMemcpyAsync(x, h->hx, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
    const int s = h->pcg_collect(residuals, iterations);
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    if (seconds) *seconds = 1e-3 * ms;
    if (s == IG_NOT_CONVERGED) g_err = "pcg: no convergence within " + std::to_string(maxit) + " iterations";
    if (s == IG_BREAKDOWN) g_err = "pcg: p^T A p <= 0 (operator not SPD)";
    return s;
  });
}

int ig_richardson(ig_hier* h, const double* b, double tol, int32_t maxit, double* x, double* residuals,
                  int32_t* iterations, double* seconds) {
  if (!h || !b || !x || !residuals || !iterations) return fail(IG_INVALID_ARGUMENT, "richardson: null argument");
  if (maxit < 0) return fail(IG_INVALID_ARGUMENT, "richardson: maxit must be >= 0");
  std::lock_guard<std::mutex> lk(h->mu);
  OptScope os_(&h->opts);
  return guarded([&] {
    const int32_t n = h->lv[h->L - 1].n;
    CK(cudaMemcpyAsync(h->hb, b, sizeof(double) * n, cudaMemcpyHostToDevice, h->stream));
    CK(cudaEventRecord(h->ev0, h->stream));
    h->rich_launch(h->hb, h->hx, tol, maxit);
    CK(cudaEventRecord(h->ev1, h->stream));
    CK(cudaMemcpyAsync(x, h->hx, sizeof(double) * n, cudaMemcpyDeviceToHost, h->stream));
    const int s = h->rich_collect(residuals, iterations);
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    if (seconds) *seconds = 1e-3 * ms;
    if (s == IG_NOT_CONVERGED) g_err = "richardson: no convergence within " + std::to_string(maxit) + " iterations";
    if (s == IG_DIVERGED) g_err = "richardson: residual grew for 10 consecutive steps";
    return s;
  });
}

}  // extern "C"

// ----------------------------------------------------- device Galerkin -----
namespace {

// Device CSR owned by the Galerkin driver (int64 row offsets while building).
struct GalMat {
  int32_t nr = 0, nc = 0;
  int64_t nnz = 0;
  int32_t* ptr = nullptr;  // int32 row offsets (kernels' input form)
  int32_t* col = nullptr;
  double* val = nullptr;
  GalCsr view() const { return GalCsr{nr, nc, ptr, col, val}; }
  void free_all() {
    cudaFree(ptr);
    cudaFree(col);
    cudaFree(val);
    ptr = nullptr;
    col = nullptr;
    val = nullptr;
  }
};

template <typename T>
T* dmalloc(size_t n) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

__global__ void k_i64_to_i32(int64_t n, const int64_t* a, int32_t* b) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) b[i] = static_cast<int32_t>(a[i]);
}

GalMat gal_upload(const ig_csr& a, cudaStream_t st) {
  GalMat m;
  m.nr = a.n_rows;
  m.nc = a.n_cols;
  m.nnz = a.nnz;
  m.ptr = dmalloc<int32_t>(static_cast<size_t>(a.n_rows) + 1);
  m.col = dmalloc<int32_t>(static_cast<size_t>(a.nnz));
  m.val = dmalloc<double>(static_cast<size_t>(a.nnz));
  CK(cudaMemcpyAsync(m.ptr, a.row_ptr, sizeof(int32_t) * (a.n_rows + 1), cudaMemcpyHostToDevice, st));
  if (a.nnz) {
    CK(cudaMemcpyAsync(m.col, a.col_idx, sizeof(int32_t) * a.nnz, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(m.val, a.val, sizeof(double) * a.nnz, cudaMemcpyHostToDevice, st));
  }
  return m;
}

// Offsets from per-row counts; returns the total (synchronises).
int64_t gal_offsets(int32_t n, const int32_t* cnt, int64_t* off64, int32_t* off32, cudaStream_t st) {
  k_scan_counts<<<1, 1024, 0, st>>>(n, cnt, off64);
  CK(cudaGetLastError());
  int64_t tot = 0;
  CK(cudaMemcpyAsync(&tot, off64 + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (tot > INT32_MAX) throw Error(IG_UNSUPPORTED, "galerkin: product has more than 2^31 nonzeros (int32 CSR)");
  const int64_t n1 = static_cast<int64_t>(n) + 1;
  k_i64_to_i32<<<static_cast<unsigned>((n1 + 255) / 256), 256, 0, st>>>(n1, off64, off32);
  CK(cudaGetLastError());
  return tot;
}

GalMat gal_transpose(const GalMat& m, cudaStream_t st) {
  GalMat t;
  t.nr = m.nc;
  t.nc = m.nr;
  t.nnz = m.nnz;
  int32_t* cnt = dmalloc<int32_t>(static_cast<size_t>(t.nr));
  int64_t* off = dmalloc<int64_t>(static_cast<size_t>(t.nr) + 1);
  t.ptr = dmalloc<int32_t>(static_cast<size_t>(t.nr) + 1);
  t.col = dmalloc<int32_t>(static_cast<size_t>(t.nnz));
  t.val = dmalloc<double>(static_cast<size_t>(t.nnz));
  CK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * t.nr, st));
  const unsigned g = static_cast<unsigned>((m.nr + 255) / 256);
  if (g) k_tr_count<<<g, 256, 0, st>>>(m.view(), cnt);
  CK(cudaGetLastError());
  gal_offsets(t.nr, cnt, off, t.ptr, st);
  CK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * t.nr, st));
  if (g) k_tr_scatter<<<g, 256, 0, st>>>(m.view(), off, cnt, t.col, t.val);
  const unsigned gt = static_cast<unsigned>((t.nr + 255) / 256);
  if (gt) k_tr_sort<<<gt, 256, 0, st>>>(t.nr, off, t.col, t.val);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  cudaFree(cnt);
  cudaFree(off);
  return t;
}

// C = A B with the host spgemm's summation order (galerkin.cuh).
GalMat gal_spgemm(const GalMat& a, const GalMat& b, cudaStream_t st) {
  if (a.nc != b.nr) throw Error(IG_INVALID_ARGUMENT, "galerkin: inner dimension mismatch");
  GalMat c;
  c.nr = a.nr;
  c.nc = b.nc;
  int32_t* cnt = dmalloc<int32_t>(static_cast<size_t>(c.nr));
  int64_t* off = dmalloc<int64_t>(static_cast<size_t>(c.nr) + 1);
  c.ptr = dmalloc<int32_t>(static_cast<size_t>(c.nr) + 1);
  const unsigned g = static_cast<unsigned>((c.nr + kGalWarps - 1) / kGalWarps);
  // B rows of at most 32 entries (R^T): the prefetching kernel.
  int32_t bmax = 0;
  {
    std::vector<int32_t> bp(static_cast<size_t>(b.nr) + 1);
    CK(cudaMemcpyAsync(bp.data(), b.ptr, sizeof(int32_t) * (b.nr + 1), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int32_t i = 0; i < b.nr; ++i) bmax = std::max(bmax, bp[i + 1] - bp[i]);
  }
  const bool shortb = bmax <= 32 && opt().gal_short;
  if (shortb) {
    CK(cudaFuncSetAttribute(k_gal_short<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kGalFillSmem)));
    CK(cudaFuncSetAttribute(k_gal_short<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kGalFillSmem)));
    if (g) k_gal_short<false><<<g, 32 * kGalWarps, kGalCountSmem, st>>>(a.view(), b.view(), cnt, nullptr, nullptr, nullptr);
  } else if (g) {
    k_gal_count<<<g, 32 * kGalWarps, kGalCountSmem, st>>>(a.view(), b.view(), cnt);
  }
  CK(cudaGetLastError());
  // Rows that do not fit the per-warp table: fail loudly.
  {
    int32_t mx = 0;
    std::vector<int32_t> hc(static_cast<size_t>(c.nr));
    if (c.nr) CK(cudaMemcpyAsync(hc.data(), cnt, sizeof(int32_t) * c.nr, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int32_t v : hc) mx = std::max(mx, v);
    if (mx > kGalLoad)
      throw Error(IG_UNSUPPORTED, "galerkin: a product row has more than " + std::to_string(kGalLoad) +
                                      " distinct columns (device table limit)");
  }
  c.nnz = gal_offsets(c.nr, cnt, off, c.ptr, st);
  c.col = dmalloc<int32_t>(static_cast<size_t>(c.nnz));
  c.val = dmalloc<double>(static_cast<size_t>(c.nnz));
  if (g && shortb)
    k_gal_short<true><<<g, 32 * kGalWarps, kGalFillSmem, st>>>(a.view(), b.view(), nullptr, off, c.col, c.val);
  else if (g)
    k_gal_fill<<<g, 32 * kGalWarps, kGalFillSmem, st>>>(a.view(), b.view(), off, c.col, c.val);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  cudaFree(cnt);
  cudaFree(off);
  return c;
}

}  // namespace

extern "C" {

int ig_galerkin_hierarchy(const ig_csr* A_fine, const ig_csr* R, int32_t n_levels, ig_csr* A_out, double* seconds) {
  if (!A_fine || !R || !A_out || n_levels < 1) return fail(IG_INVALID_ARGUMENT, "galerkin: null argument");
  for (int32_t l = 0; l + 1 < n_levels; ++l) A_out[l] = ig_csr{};
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  GalMat A, Rd, Rt, C;
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = guarded([&] {
    check_csr(*A_fine, "galerkin: A");
    for (int32_t l = 1; l < n_levels; ++l) check_csr(R[l], "galerkin: R");
    CK(cudaFuncSetAttribute(k_gal_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kGalFillSmem)));
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    A = gal_upload(*A_fine, st);
    float dev_ms = 0.f;
    for (int32_t l = n_levels - 1; l >= 1; --l) {
      const ig_csr& r = R[l];
      if (r.n_cols != A.nr || r.n_rows <= 0)
        throw Error(IG_INVALID_ARGUMENT, "galerkin: R[" + std::to_string(l) + "] does not match level " +
                                             std::to_string(l));
      Rd = gal_upload(r, st);
      CK(cudaStreamSynchronize(st));
      CK(cudaEventRecord(e0, st));
      Rt = gal_transpose(Rd, st);
      C = gal_spgemm(A, Rt, st);  // A R^T
      Rt.free_all();
      GalMat Ac = gal_spgemm(Rd, C, st);  // R (A R^T)
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      dev_ms += ms;
      C.free_all();
      Rd.free_all();
      A.free_all();
      A = Ac;
      ig_csr& o = A_out[l - 1];
      o.n_rows = A.nr;
      o.n_cols = A.nc;
      o.nnz = A.nnz;
      int32_t* hp = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (A.nr + 1)));
      int32_t* hc = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * std::max<int64_t>(A.nnz, 1)));
      double* hv = static_cast<double*>(std::malloc(sizeof(double) * std::max<int64_t>(A.nnz, 1)));
      o.row_ptr = hp;
      o.col_idx = hc;
      o.val = hv;
      if (!hp || !hc || !hv) throw Error(IG_CUDA_ERROR, "galerkin: host allocation failed");
      CK(cudaMemcpyAsync(hp, A.ptr, sizeof(int32_t) * (A.nr + 1), cudaMemcpyDeviceToHost, st));
      if (A.nnz) {
        CK(cudaMemcpyAsync(hc, A.col, sizeof(int32_t) * A.nnz, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hv, A.val, sizeof(double) * A.nnz, cudaMemcpyDeviceToHost, st));
      }
      CK(cudaStreamSynchronize(st));
    }
    if (seconds) {
      seconds[1] = 1e-3 * dev_ms;
    }
    return IG_OK;
  });
  A.free_all();
  Rd.free_all();
  Rt.free_all();
  C.free_all();
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st) cudaStreamDestroy(st);
  if (seconds) seconds[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (rc != IG_OK)
    for (int32_t l = 0; l + 1 < n_levels; ++l) ig_csr_free(&A_out[l]);
  return rc;
}

void ig_csr_free(ig_csr* m) {
  if (!m) return;
  std::free(const_cast<int32_t*>(m->row_ptr));
  std::free(const_cast<int32_t*>(m->col_idx));
  std::free(const_cast<double*>(m->val));
  *m = ig_csr{};
}

}  // extern "C"

namespace {

// Host-owned post-filter layout produced by the device factorisation.
struct HostBlocks {
  std::vector<int32_t> ptr, dofs;
  std::vector<int64_t> fptr;
  std::vector<double> fac;
  int64_t filtered = 0;
};

// factorize_blocks on a device-resident A (blockfac.cuh); synchronous on st.
// dev_ms accumulates the kernels' device time.
HostBlocks fac_blocks_dev(const GalMat& Ad, int32_t n_blocks, const int32_t* blk_ptr, const int32_t* blk_dofs,
                          double filter_ratio, cudaStream_t st, float* dev_ms) {
  HostBlocks hb;
  std::vector<void*> dev;
  struct Free {
    std::vector<void*>& v;
    ~Free() {
      for (void* p : v) cudaFree(p);
    }
  } fr{dev};
  auto dal = [&](size_t bytes) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(bytes, 8)));
    dev.push_back(p);
    return p;
  };
  if (blk_ptr[0] != 0) throw Error(IG_INVALID_ARGUMENT, "factorize_blocks: blk_ptr[0] != 0");
  std::vector<int64_t> soff(static_cast<size_t>(n_blocks) + 1, 0);
  std::vector<int32_t> big;
  for (int32_t b = 0; b < n_blocks; ++b) {
    const int64_t sb = blk_ptr[b + 1] - blk_ptr[b];
    if (sb < 1) throw Error(IG_INVALID_ARGUMENT, "factorize_blocks: empty block");
    for (int32_t i = blk_ptr[b]; i < blk_ptr[b + 1]; ++i)
      if (blk_dofs[i] < 0 || blk_dofs[i] >= Ad.nr) throw Error(IG_INVALID_ARGUMENT, "factorize_blocks: DOF out of range");
    soff[b + 1] = soff[b] + 3 * sb * sb;
    if (sb >= kBfWarpMin && sb <= 32) big.push_back(b);
  }
  const int64_t nd = n_blocks ? blk_ptr[n_blocks] : 0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  struct Ev {
    cudaEvent_t a, b;
    ~Ev() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  } ev{e0, e1};
  auto* dptr = static_cast<int32_t*>(dal(sizeof(int32_t) * (n_blocks + 1)));
  auto* ddofs = static_cast<int32_t*>(dal(sizeof(int32_t) * nd));
  auto* dsoff = static_cast<int64_t*>(dal(sizeof(int64_t) * (n_blocks + 1)));
  auto* scratch = static_cast<double*>(dal(sizeof(double) * soff[n_blocks]));
  auto* kdofs = static_cast<int32_t*>(dal(sizeof(int32_t) * nd));
  auto* ksize = static_cast<int32_t*>(dal(sizeof(int32_t) * n_blocks));
  auto* dbig = static_cast<int32_t*>(dal(sizeof(int32_t) * big.size()));
  CK(cudaMemcpyAsync(dptr, blk_ptr, sizeof(int32_t) * (n_blocks + 1), cudaMemcpyHostToDevice, st));
  if (nd) CK(cudaMemcpyAsync(ddofs, blk_dofs, sizeof(int32_t) * nd, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dsoff, soff.data(), sizeof(int64_t) * (n_blocks + 1), cudaMemcpyHostToDevice, st));
  if (!big.empty()) CK(cudaMemcpyAsync(dbig, big.data(), sizeof(int32_t) * big.size(), cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaEventRecord(e0, st));
  BlockFacArgs fa{Ad.view(), n_blocks, dptr, ddofs, dsoff, scratch, kdofs, ksize, filter_ratio, 1};
  const unsigned g = static_cast<unsigned>((n_blocks + 127) / 128);
  CK(cudaFuncSetAttribute(k_block_factor_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(kBfWarpSmem)));
  if (!big.empty())
    k_block_factor_warp<<<static_cast<unsigned>((big.size() + kBfWarps - 1) / kBfWarps), 32 * kBfWarps, kBfWarpSmem,
                          st>>>(fa, dbig, static_cast<int32_t>(big.size()));
  if (g) k_block_factor<<<g, 128, 0, st>>>(fa);
  CK(cudaGetLastError());
  std::vector<int32_t> hs(static_cast<size_t>(n_blocks));
  if (n_blocks) CK(cudaMemcpyAsync(hs.data(), ksize, sizeof(int32_t) * n_blocks, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<int64_t> optr(static_cast<size_t>(n_blocks) + 1, 0);
  hb.fptr.assign(static_cast<size_t>(n_blocks) + 1, 0);
  for (int32_t b = 0; b < n_blocks; ++b) {
    if (hs[b] < 0) throw Error(IG_INVALID_ARGUMENT, "factorize_blocks: all DOFs filtered from a block");
    optr[b + 1] = optr[b] + hs[b];
    hb.fptr[b + 1] = hb.fptr[b] + static_cast<int64_t>(hs[b]) * hs[b];
  }
  if (optr[n_blocks] > INT32_MAX) throw Error(IG_UNSUPPORTED, "factorize_blocks: more than 2^31 DOF entries");
  auto* doptr = static_cast<int64_t*>(dal(sizeof(int64_t) * (n_blocks + 1)));
  auto* dofptr = static_cast<int64_t*>(dal(sizeof(int64_t) * (n_blocks + 1)));
  auto* odofs = static_cast<int32_t*>(dal(sizeof(int32_t) * optr[n_blocks]));
  auto* ofac = static_cast<double*>(dal(sizeof(double) * hb.fptr[n_blocks]));
  CK(cudaMemcpyAsync(doptr, optr.data(), sizeof(int64_t) * (n_blocks + 1), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dofptr, hb.fptr.data(), sizeof(int64_t) * (n_blocks + 1), cudaMemcpyHostToDevice, st));
  if (g) k_block_compact<<<g, 128, 0, st>>>(n_blocks, dptr, kdofs, ksize, dsoff, scratch, doptr, dofptr, odofs, ofac);
  CK(cudaGetLastError());
  CK(cudaEventRecord(e1, st));
  hb.ptr.resize(static_cast<size_t>(n_blocks) + 1);
  for (int32_t b = 0; b <= n_blocks; ++b) hb.ptr[b] = static_cast<int32_t>(optr[b]);
  hb.dofs.resize(static_cast<size_t>(optr[n_blocks]));
  hb.fac.resize(static_cast<size_t>(hb.fptr[n_blocks]));
  if (!hb.dofs.empty())
    CK(cudaMemcpyAsync(hb.dofs.data(), odofs, sizeof(int32_t) * hb.dofs.size(), cudaMemcpyDeviceToHost, st));
  if (!hb.fac.empty())
    CK(cudaMemcpyAsync(hb.fac.data(), ofac, sizeof(double) * hb.fac.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  hb.filtered = nd - optr[n_blocks];
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  if (dev_ms) *dev_ms += ms;
  return hb;
}

}  // namespace

extern "C" {

int ig_factorize_blocks(const ig_csr* A, int32_t n_blocks, const int32_t* blk_ptr, const int32_t* blk_dofs,
                        double filter_ratio, ig_blocks* out, int64_t* filtered_dofs, double* seconds) {
  if (!A || !blk_ptr || (n_blocks > 0 && !blk_dofs) || !out || n_blocks < 0)
    return fail(IG_INVALID_ARGUMENT, "factorize_blocks: null argument");
  *out = ig_blocks{};
  cudaStream_t st = nullptr;
  GalMat Ad;
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = guarded([&] {
    check_csr(*A, "factorize_blocks: A");
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    Ad = gal_upload(*A, st);
    float ms = 0.f;
    HostBlocks hb = fac_blocks_dev(Ad, n_blocks, blk_ptr, blk_dofs, filter_ratio, st, &ms);
    auto* hp = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * hb.ptr.size()));
    auto* hd = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * std::max<size_t>(hb.dofs.size(), 1)));
    auto* hfp = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * hb.fptr.size()));
    auto* hf = static_cast<double*>(std::malloc(sizeof(double) * std::max<size_t>(hb.fac.size(), 1)));
    out->n_blocks = n_blocks;
    out->blk_ptr = hp;
    out->blk_dofs = hd;
    out->fac_ptr = hfp;
    out->fac = hf;
    if (!hp || !hd || !hfp || !hf) throw Error(IG_CUDA_ERROR, "factorize_blocks: host allocation failed");
    std::memcpy(hp, hb.ptr.data(), sizeof(int32_t) * hb.ptr.size());
    std::memcpy(hd, hb.dofs.data(), sizeof(int32_t) * hb.dofs.size());
    std::memcpy(hfp, hb.fptr.data(), sizeof(int64_t) * hb.fptr.size());
    std::memcpy(hf, hb.fac.data(), sizeof(double) * hb.fac.size());
    if (filtered_dofs) *filtered_dofs = hb.filtered;
    if (seconds) seconds[1] = 1e-3 * ms;
    return IG_OK;
  });
  Ad.free_all();
  if (st) cudaStreamDestroy(st);
  if (seconds) seconds[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (rc != IG_OK) ig_blocks_free(out);
  return rc;
}

void ig_blocks_free(ig_blocks* b) {
  if (!b) return;
  std::free(const_cast<int32_t*>(b->blk_ptr));
  std::free(const_cast<int32_t*>(b->blk_dofs));
  std::free(const_cast<int64_t*>(b->fac_ptr));
  std::free(const_cast<double*>(b->fac));
  *b = ig_blocks{};
}

}  // extern "C"

extern "C" {

int ig_pstrf(int32_t n, double* a, int32_t* piv, double tol, int32_t* rank) {
  if (n < 0 || (n > 0 && (!a || !piv)) || !rank) return fail(IG_INVALID_ARGUMENT, "pstrf: bad argument");
  double* da = nullptr;
  double* dw = nullptr;
  int32_t* dp = nullptr;
  int32_t* dr = nullptr;
  const int rc = guarded([&] {
    const size_t nn = static_cast<size_t>(n) * n;
    CK(cudaMalloc(&da, std::max<size_t>(nn, 1) * sizeof(double)));
    CK(cudaMalloc(&dw, std::max<size_t>(2 * static_cast<size_t>(n), 1) * sizeof(double)));
    CK(cudaMalloc(&dp, std::max<int32_t>(n, 1) * sizeof(int32_t)));
    CK(cudaMalloc(&dr, sizeof(int32_t)));
    if (nn) CK(cudaMemcpy(da, a, nn * sizeof(double), cudaMemcpyHostToDevice));
    const int threads = std::max(32, std::min(1024, ((n + 31) / 32) * 32));
    k_pstrf<<<1, threads>>>(n, da, dp, tol, dw, dr);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    if (nn) CK(cudaMemcpy(a, da, nn * sizeof(double), cudaMemcpyDeviceToHost));
    if (n) CK(cudaMemcpy(piv, dp, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(rank, dr, sizeof(int32_t), cudaMemcpyDeviceToHost));
    return IG_OK;
  });
  cudaFree(da);
  cudaFree(dw);
  cudaFree(dp);
  cudaFree(dr);
  return rc;
}

}  // extern "C"

extern "C" {

int ig_hier_build(const ig_csr* A_fine, const ig_csr* R, const ig_blocks* prefilter, const double* gamma,
                  int32_t smoother_kind, double filter_ratio, int32_t n_levels, ig_hier** out, double* seconds) {
  if (!A_fine || !R || !prefilter || !gamma || !out || n_levels < 1)
    return fail(IG_INVALID_ARGUMENT, "hier_build: null argument");
  *out = nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  std::vector<GalMat> Ad(static_cast<size_t>(n_levels));
  GalMat Rd, Rt, Cm;
  double t_create = 0.0;
  float dev_ms = 0.f;
  const int rc = guarded([&] {
    check_csr(*A_fine, "hier_build: A");
    for (int32_t l = 1; l < n_levels; ++l) check_csr(R[l], "hier_build: R");
    CK(cudaFuncSetAttribute(k_gal_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kGalFillSmem)));
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    // 1. Galerkin chain (multigrid.cpp:37-41), every level kept on the device.
    Ad[n_levels - 1] = gal_upload(*A_fine, st);
    for (int32_t l = n_levels - 1; l >= 1; --l) {
      if (R[l].n_cols != Ad[l].nr || R[l].n_rows <= 0)
        throw Error(IG_INVALID_ARGUMENT, "hier_build: R[" + std::to_string(l) + "] does not match level " +
                                             std::to_string(l));
      Rd = gal_upload(R[l], st);
      CK(cudaStreamSynchronize(st));
      CK(cudaEventRecord(e0, st));
      Rt = gal_transpose(Rd, st);
      Cm = gal_spgemm(Ad[l], Rt, st);
      Rt.free_all();
      Ad[l - 1] = gal_spgemm(Rd, Cm, st);
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      dev_ms += ms;
      Cm.free_all();
      Rd.free_all();
    }
    // 2. Schwarz blocks of levels >= 1 (make_smoother: factorize_blocks).
    std::vector<HostBlocks> hb(static_cast<size_t>(n_levels));
    for (int32_t l = 1; l < n_levels; ++l) {
      const ig_blocks& pb = prefilter[l];
      if (pb.n_blocks < 0 || (pb.n_blocks > 0 && (!pb.blk_ptr || !pb.blk_dofs)))
        throw Error(IG_INVALID_ARGUMENT, "hier_build: bad pre-filter layout");
      hb[l] = fac_blocks_dev(Ad[l], pb.n_blocks, pb.blk_ptr, pb.blk_dofs, filter_ratio, st, &dev_ms);
    }
    // 3. Coarse operators back to the host (the layouts are built there).
    std::vector<std::vector<int32_t>> hp(static_cast<size_t>(n_levels)), hc(static_cast<size_t>(n_levels));
    std::vector<std::vector<double>> hv(static_cast<size_t>(n_levels));
    for (int32_t l = 0; l + 1 < n_levels; ++l) {
      const GalMat& m = Ad[l];
      hp[l].resize(static_cast<size_t>(m.nr) + 1);
      hc[l].resize(static_cast<size_t>(m.nnz));
      hv[l].resize(static_cast<size_t>(m.nnz));
      CK(cudaMemcpyAsync(hp[l].data(), m.ptr, sizeof(int32_t) * (m.nr + 1), cudaMemcpyDeviceToHost, st));
      if (m.nnz) {
        CK(cudaMemcpyAsync(hc[l].data(), m.col, sizeof(int32_t) * m.nnz, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hv[l].data(), m.val, sizeof(double) * m.nnz, cudaMemcpyDeviceToHost, st));
      }
    }
    CK(cudaStreamSynchronize(st));
    for (auto& m : Ad) m.free_all();
    // 4. Coarsest pivoted Cholesky on the device (multigrid.cpp:57-73).
    const int32_t n0 = n_levels > 1 ? static_cast<int32_t>(hp[0].size()) - 1 : A_fine->n_rows;
    const int32_t* p0 = n_levels > 1 ? hp[0].data() : A_fine->row_ptr;
    const int32_t* c0 = n_levels > 1 ? hc[0].data() : A_fine->col_idx;
    const double* v0 = n_levels > 1 ? hv[0].data() : A_fine->val;
    std::vector<double> L(static_cast<size_t>(n0) * n0, 0.0);
    for (int32_t i = 0; i < n0; ++i)
      for (int32_t k = p0[i]; k < p0[i + 1]; ++k) L[static_cast<size_t>(c0[k]) * n0 + i] = v0[k];
    double max_diag = 0.0;
    for (int32_t i = 0; i < n0; ++i) max_diag = std::max(max_diag, L[static_cast<size_t>(i) * n0 + i]);
    std::vector<int32_t> piv(static_cast<size_t>(std::max(n0, 1)), 0);
    int32_t rank = 0;
    {
      double *da = nullptr, *dw = nullptr;
      int32_t *dp = nullptr, *dr = nullptr;
      struct F {
        double*& a;
        double*& w;
        int32_t*& p;
        int32_t*& r;
        ~F() {
          cudaFree(a);
          cudaFree(w);
          cudaFree(p);
          cudaFree(r);
        }
      } fr{da, dw, dp, dr};
      CK(cudaMalloc(&da, std::max<size_t>(L.size(), 1) * sizeof(double)));
      CK(cudaMalloc(&dw, std::max<size_t>(2 * static_cast<size_t>(n0), 1) * sizeof(double)));
      CK(cudaMalloc(&dp, piv.size() * sizeof(int32_t)));
      CK(cudaMalloc(&dr, sizeof(int32_t)));
      if (!L.empty()) CK(cudaMemcpyAsync(da, L.data(), L.size() * sizeof(double), cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(e0, st));
      k_pstrf<<<1, std::max(32, std::min(1024, ((n0 + 31) / 32) * 32)), 0, st>>>(n0, da, dp, 1e-14 * max_diag, dw, dr);
      CK(cudaGetLastError());
      CK(cudaEventRecord(e1, st));
      if (!L.empty()) CK(cudaMemcpyAsync(L.data(), da, L.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (n0) CK(cudaMemcpyAsync(piv.data(), dp, n0 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&rank, dr, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      dev_ms += ms;
    }
    // 5. The device hierarchy (layouts, upload): ig_hier_create.
    std::vector<ig_level> lv(static_cast<size_t>(n_levels));
    for (int32_t l = 0; l < n_levels; ++l) {
      ig_level& v = lv[l];
      if (l + 1 < n_levels) {
        v.A = ig_csr{static_cast<int32_t>(hp[l].size()) - 1, static_cast<int32_t>(hp[l].size()) - 1,
                     static_cast<int64_t>(hc[l].size()), hp[l].data(), hc[l].data(), hv[l].data()};
      } else {
        v.A = *A_fine;
      }
      v.R = l >= 1 ? R[l] : ig_csr{};
      v.smoother_kind = smoother_kind;
      v.gamma = gamma[l];
      if (l >= 1) {
        const HostBlocks& b = hb[l];
        v.blocks.n_blocks = prefilter[l].n_blocks;
        v.blocks.blk_ptr = b.ptr.data();
        v.blocks.blk_dofs = b.dofs.data();
        v.blocks.fac_ptr = b.fptr.data();
        v.blocks.fac = b.fac.data();
        v.blocks.n_colors = prefilter[l].n_colors;
        v.blocks.color_of = prefilter[l].color_of;
      }
    }
    ig_coarse co{n0, rank, L.data(), piv.data()};
    const auto tc = std::chrono::steady_clock::now();
    const int c = ig_hier_create(lv.data(), n_levels, &co, out);
    t_create = std::chrono::duration<double>(std::chrono::steady_clock::now() - tc).count();
    return c;
  });
  for (auto& m : Ad) m.free_all();
  Rd.free_all();
  Rt.free_all();
  Cm.free_all();
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st) cudaStreamDestroy(st);
  if (seconds) {
    seconds[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    seconds[1] = 1e-3 * dev_ms;
    seconds[2] = t_create;
  }
  return rc;
}

}  // extern "C"

namespace {
__global__ void k_set_unit(double* e, int32_t prev, int32_t j) {
  if (threadIdx.x == 0) {
    if (prev >= 0) e[prev] = 0.0;
    e[j] = 1.0;
  }
}
}  // namespace

extern "C" {

int ig_operator_columns(ig_hier* h, int32_t kind, int32_t j0, int32_t count, double* out) {
  if (!h || !out) return fail(IG_INVALID_ARGUMENT, "operator_columns: null argument");
  if (kind < IG_OP_A || kind > IG_OP_SMOOTHER_SYMMETRIC) return fail(IG_INVALID_ARGUMENT, "operator_columns: bad kind");
  std::lock_guard<std::mutex> lk(h->mu);
  OptScope os_(&h->opts);
  const int32_t top = h->L - 1;
  const int32_t n = h->lv[top].n;
  if (j0 < 0 || count < 0 || j0 + static_cast<int64_t>(count) > n)
    return fail(IG_INVALID_ARGUMENT, "operator_columns: column range outside the operator");
  if (kind == IG_OP_SMOOTHER_SYMMETRIC && top < 1)
    return fail(IG_INVALID_ARGUMENT, "operator_columns: a 1-level hierarchy has no smoother");
  double *e = nullptr, *u = nullptr, *cols = nullptr;
  const int rc = guarded([&] {
    if (count == 0) return IG_OK;
    CK(cudaMalloc(&e, sizeof(double) * n));
    CK(cudaMalloc(&u, sizeof(double) * n));
    CK(cudaMalloc(&cols, sizeof(double) * static_cast<size_t>(n) * count));
    CK(cudaMemsetAsync(e, 0, sizeof(double) * n, h->stream));
    Level& F = h->lv[top];
    for (int32_t c = 0; c < count; ++c) {
      const int32_t j = j0 + c;
      k_set_unit<<<1, 32, 0, h->stream>>>(e, c == 0 ? -1 : j - 1, j);
      CK(cudaGetLastError());
      double* col = cols + static_cast<size_t>(c) * n;
      if (kind == IG_OP_A) {
        h->spmv(F.A, 0, e, col, col);
        continue;
      }
      h->spmv(F.A, 0, e, u, u);  // A e_j
      if (kind == IG_OP_VCYCLE) {
        h->vcycle(top, u, col, nullptr, nullptr);  // MgHierarchy::apply(A e_j)
      } else {                                      // Smoother::apply_symmetric(A e_j)
        h->smoother(F, u, col, false, nullptr, nullptr, 0);
        h->spmv(F.A, 1, col, F.cor, u, nullptr);
        h->smoother(F, F.cor, col, true, nullptr, nullptr, 1);
      }
    }
    CK(cudaMemcpyAsync(out, cols, sizeof(double) * static_cast<size_t>(n) * count, cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return IG_OK;
  });
  cudaFree(e);
  cudaFree(u);
  cudaFree(cols);
  return rc;
}

}  // extern "C"

extern "C" {

int ig_assemble(const ig_assembly* a, ig_csr* A_out, double* b_out, double* seconds) {
  if (!a || !A_out || !b_out) return fail(IG_INVALID_ARGUMENT, "assemble: null argument");
  *A_out = ig_csr{};
  std::vector<void*> dev;
  auto dal = [&](size_t bytes) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(bytes, 8)));
    dev.push_back(p);
    return p;
  };
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = guarded([&] {
    if (a->dim != 2 && a->dim != 3) throw Error(IG_INVALID_ARGUMENT, "assemble: dim must be 2 or 3");
    if (a->p < 1 || a->n < 1 || a->n_elements < 1 || a->n_tables < 1)
      throw Error(IG_INVALID_ARGUMENT, "assemble: empty payload");
    if (!a->el_ix || !a->el_iy || (a->dim == 3 && !a->el_iz) || !a->el_table || !a->K || !a->F || !a->anchors ||
        !a->supp_ptr || !a->supp_el || !a->kept)
      throw Error(IG_INVALID_ARGUMENT, "assemble: null array");
    int nl = 1;
    for (int d = 0; d < a->dim; ++d) nl *= a->p + 1;
    const int W = 2 * a->p + 1;
    const int wsize = a->dim == 3 ? W * W * W : W * W;
    const int64_t nun = static_cast<int64_t>(a->nf[0]) * a->nf[1] * (a->dim == 3 ? a->nf[2] : 1);
    const int64_t nsupp = a->supp_ptr[a->n];
    const size_t smem = static_cast<size_t>(kAsmWarps) * wsize * (sizeof(double) + 1);
    if (smem > 200 * 1024) throw Error(IG_UNSUPPORTED, "assemble: window too large for shared memory");
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto up = [&](const void* src, size_t bytes) {
      void* d = dal(bytes);
      if (bytes) CK(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st));
      return d;
    };
    const size_t ne = static_cast<size_t>(a->n_elements);
    AsmArgs g{};
    g.dim = a->dim;
    g.p = a->p;
    g.family = a->family;
    g.n = a->n;
    g.nloc = nl;
    g.W = W;
    g.wsize = wsize;
    g.nf0 = a->nf[0];
    g.nf1 = a->nf[1];
    g.nf2 = a->dim == 3 ? a->nf[2] : 1;
    g.el_ix = static_cast<const int32_t*>(up(a->el_ix, 4 * ne));
    g.el_iy = static_cast<const int32_t*>(up(a->el_iy, 4 * ne));
    g.el_iz = a->dim == 3 ? static_cast<const int32_t*>(up(a->el_iz, 4 * ne)) : nullptr;
    g.el_table = static_cast<const int32_t*>(up(a->el_table, 4 * ne));
    g.K = static_cast<const double*>(up(a->K, sizeof(double) * static_cast<size_t>(a->n_tables) * nl * nl));
    g.F = static_cast<const double*>(up(a->F, sizeof(double) * static_cast<size_t>(a->n_tables) * nl));
    g.anchors = static_cast<const int64_t*>(up(a->anchors, 8 * static_cast<size_t>(a->n)));
    g.supp_ptr = static_cast<const int64_t*>(up(a->supp_ptr, 8 * (static_cast<size_t>(a->n) + 1)));
    g.supp_el = static_cast<const int32_t*>(up(a->supp_el, 4 * static_cast<size_t>(nsupp)));
    g.kept = static_cast<const int32_t*>(up(a->kept, 4 * static_cast<size_t>(nun)));
    auto* cnt = static_cast<int32_t*>(dal(4 * static_cast<size_t>(a->n)));
    auto* off = static_cast<int64_t*>(dal(8 * (static_cast<size_t>(a->n) + 1)));
    auto* ptr = static_cast<int32_t*>(dal(4 * (static_cast<size_t>(a->n) + 1)));
    auto* db = static_cast<double*>(dal(8 * static_cast<size_t>(a->n)));
    auto* bad = static_cast<int*>(dal(sizeof(int)));
    CK(cudaMemsetAsync(bad, 0, sizeof(int), st));
    CK(cudaFuncSetAttribute(k_asm_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    CK(cudaFuncSetAttribute(k_asm_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    CK(cudaStreamSynchronize(st));
    CK(cudaEventRecord(e0, st));
    const unsigned gr = static_cast<unsigned>((a->n + kAsmWarps - 1) / kAsmWarps);
    k_asm_rows<false><<<gr, 32 * kAsmWarps, smem, st>>>(g, cnt, nullptr, nullptr, nullptr, nullptr);
    CK(cudaGetLastError());
    const int64_t nnz = gal_offsets(a->n, cnt, off, ptr, st);
    auto* col = static_cast<int32_t*>(dal(4 * static_cast<size_t>(nnz)));
    auto* val = static_cast<double*>(dal(8 * static_cast<size_t>(nnz)));
    auto* sym = static_cast<double*>(dal(8 * static_cast<size_t>(nnz)));
    k_asm_rows<true><<<gr, 32 * kAsmWarps, smem, st>>>(g, nullptr, off, col, val, db);
    CK(cudaGetLastError());
    k_asm_sym<<<static_cast<unsigned>((a->n + 255) / 256), 256, 0, st>>>(a->n, ptr, col, val, sym, bad);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1, st));
    int hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hbad) throw Error(IG_INVALID_ARGUMENT, "assemble: unsymmetric pattern");
    auto* hp = static_cast<int32_t*>(std::malloc(4 * (static_cast<size_t>(a->n) + 1)));
    auto* hc = static_cast<int32_t*>(std::malloc(4 * std::max<size_t>(static_cast<size_t>(nnz), 1)));
    auto* hv = static_cast<double*>(std::malloc(8 * std::max<size_t>(static_cast<size_t>(nnz), 1)));
    A_out->n_rows = A_out->n_cols = a->n;
    A_out->nnz = nnz;
    A_out->row_ptr = hp;
    A_out->col_idx = hc;
    A_out->val = hv;
    if (!hp || !hc || !hv) throw Error(IG_CUDA_ERROR, "assemble: host allocation failed");
    CK(cudaMemcpyAsync(hp, ptr, 4 * (static_cast<size_t>(a->n) + 1), cudaMemcpyDeviceToHost, st));
    if (nnz) {
      CK(cudaMemcpyAsync(hc, col, 4 * static_cast<size_t>(nnz), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(hv, sym, 8 * static_cast<size_t>(nnz), cudaMemcpyDeviceToHost, st));
    }
    CK(cudaMemcpyAsync(b_out, db, 8 * static_cast<size_t>(a->n), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (seconds) seconds[1] = 1e-3 * ms;
    return IG_OK;
  });
  for (void* p : dev) cudaFree(p);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st) cudaStreamDestroy(st);
  if (seconds) seconds[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (rc != IG_OK) ig_csr_free(A_out);
  return rc;
}

}  // extern "C"

// ------------------------------------------------ cut-element quadrature --
extern "C" {

int ig_cut_quadrature3(const ig_cut3* in, double* K, double* F, double* vol, double* seconds) {
  if (!in || !K || !F) return fail(IG_INVALID_ARGUMENT, "cut_quadrature3: null argument");
  if (in->p < 1 || in->p > 2)
    return fail(IG_UNSUPPORTED, "cut_quadrature3: degrees 1 and 2 on the device (shared-memory basis tables)");
  if (in->depth < 0 || in->depth > 3 || in->classify_depth < 0 || in->classify_depth > 6)
    return fail(IG_INVALID_ARGUMENT, "cut_quadrature3: depth in 0..3, classify depth in 0..6");
  if (in->prog_len <= 0 || !in->prog) return fail(IG_UNSUPPORTED, "cut_quadrature3: no level-set program");
  if (in->n_cut == 0) return IG_OK;
  return guarded([&] {
    const int q = in->p + 1, nl = q * q * q;
    const int64_t n = in->n_cut;
    std::vector<void*> mem;
    auto up = [&](const void* src, size_t bytes) {
      void* d = nullptr;
      CK(cudaMalloc(&d, std::max<size_t>(bytes, 8)));
      mem.push_back(d);
      if (bytes && src) CK(cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice));
      return d;
    };
    struct Free {
      std::vector<void*>& m;
      ~Free() {
        for (void* p : m) cudaFree(p);
      }
    } free_{mem};
    ig_cut3 D = *in;
    D.lo = static_cast<const double*>(up(in->lo, sizeof(double) * 3 * n));
    D.cls = static_cast<const int32_t*>(up(in->cls, sizeof(int32_t) * 3 * n));
    for (int d = 0; d < 3; ++d)
      D.ext[d] = static_cast<const double*>(up(in->ext[d], sizeof(double) * in->n_cls[d] * q * q));
    D.prog = static_cast<const double*>(up(in->prog, sizeof(double) * in->prog_len));
    D.gauss_tet = static_cast<const double*>(up(in->gauss_tet, sizeof(double) * 4));
    D.gauss_tri = static_cast<const double*>(up(in->gauss_tri, sizeof(double) * 6));
    D.gauss_box = static_cast<const double*>(up(in->gauss_box, sizeof(double) * 2 * q));
    D.table = nullptr;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    // Every element's level-set program specialised to its cell (cutquad.cuh).
    double* eprog = static_cast<double*>(up(nullptr, sizeof(double) * n * in->prog_len));
    int* elen = static_cast<int*>(up(nullptr, sizeof(int) * n));
    double* dh = static_cast<double*>(up(in->h, sizeof(double) * 3));
    k_ls_specialize<<<static_cast<unsigned>((n + 127) / 128), 128>>>(D.prog, in->prog_len, static_cast<int>(n), 3, D.lo,
                                                                      nullptr, dh, eprog, elen);
    CK(cudaGetLastError());
    int64_t* dcount = static_cast<int64_t*>(up(nullptr, sizeof(int64_t) * (n + 1)));
    k_cq_prims<false><<<static_cast<unsigned>(n), kCqThreads>>>(D, nullptr, dcount, nullptr, eprog, elen);
    CK(cudaGetLastError());
    std::vector<int64_t> cnt(static_cast<size_t>(n)), offs(static_cast<size_t>(n) + 1, 0);
    CK(cudaMemcpy(cnt.data(), dcount, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
    for (int64_t e = 0; e < n; ++e) offs[e + 1] = offs[e] + cnt[e];
    int64_t* doff = static_cast<int64_t*>(up(offs.data(), sizeof(int64_t) * (n + 1)));
    double* prim = static_cast<double*>(up(nullptr, sizeof(double) * kCqPrim * std::max<int64_t>(offs[n], 1)));
    k_cq_prims<true><<<static_cast<unsigned>(n), kCqThreads>>>(D, doff, nullptr, prim, eprog, elen);
    CK(cudaGetLastError());
    double* dK = static_cast<double*>(up(nullptr, sizeof(double) * n * nl * nl));
    double* dF = static_cast<double*>(up(nullptr, sizeof(double) * n * nl));
    double* dv = static_cast<double*>(up(nullptr, sizeof(double) * n));
    if (nl == 27)
      k_cq_integrate<27><<<static_cast<unsigned>(n), kCqThreads>>>(D, doff, prim, dK, dF, dv);
    else
      k_cq_integrate<8><<<static_cast<unsigned>(n), kCqThreads>>>(D, doff, prim, dK, dF, dv);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CK(cudaMemcpy(K, dK, sizeof(double) * n * nl * nl, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(F, dF, sizeof(double) * n * nl, cudaMemcpyDeviceToHost));
    if (vol) CK(cudaMemcpy(vol, dv, sizeof(double) * n, cudaMemcpyDeviceToHost));
    if (seconds) *seconds = ms * 1e-3;
    return IG_OK;
  });
}

}  // extern "C"

extern "C" {

int ig_cut_quadrature2(const ig_cut2* in, double* K, double* F, double* vol, double* seconds) {
  if (!in || !K || !F) return fail(IG_INVALID_ARGUMENT, "cut_quadrature2: null argument");
  if (in->p < 1 || in->p > 4) return fail(IG_UNSUPPORTED, "cut_quadrature2: degrees 1..4");
  if (in->depth < 0 || in->depth > 6 || in->classify_depth < 0 || in->classify_depth > 8 || in->gauss_order < 1 ||
      in->gauss_order > 16)
    return fail(IG_INVALID_ARGUMENT, "cut_quadrature2: depth in 0..6, classify depth in 0..8, Gauss order 1..16");
  if (in->prog_len <= 0 || !in->prog) return fail(IG_UNSUPPORTED, "cut_quadrature2: no level-set program");
  if (in->n_elem == 0) return IG_OK;
  return guarded([&] {
    const int q = in->p + 1, nl = q * q, go = in->gauss_order;
    const int64_t n = in->n_elem;
    std::vector<void*> mem;
    auto up = [&](const void* src, size_t bytes) {
      void* d = nullptr;
      CK(cudaMalloc(&d, std::max<size_t>(bytes, 8)));
      mem.push_back(d);
      if (bytes && src) CK(cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice));
      return d;
    };
    struct Free {
      std::vector<void*>& m;
      ~Free() {
        for (void* p : m) cudaFree(p);
      }
    } free_{mem};
    ig_cut2 D = *in;
    D.lo = static_cast<const double*>(up(in->lo, sizeof(double) * 2 * n));
    D.hi = static_cast<const double*>(up(in->hi, sizeof(double) * 2 * n));
    D.cls = static_cast<const int32_t*>(up(in->cls, sizeof(int32_t) * 2 * n));
    D.cut = static_cast<const int32_t*>(up(in->cut, sizeof(int32_t) * n));
    D.sides = static_cast<const int32_t*>(up(in->sides, sizeof(int32_t) * n));
    for (int d = 0; d < 2; ++d)
      D.ext[d] = static_cast<const double*>(up(in->ext[d], sizeof(double) * in->n_cls[d] * q * q));
    D.prog = static_cast<const double*>(up(in->prog, sizeof(double) * in->prog_len));
    D.gauss_q = static_cast<const double*>(up(in->gauss_q, sizeof(double) * 2 * go));
    D.gauss_q1 = static_cast<const double*>(up(in->gauss_q1, sizeof(double) * 2 * (go + 1)));
    D.table = nullptr;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    double* eprog = static_cast<double*>(up(nullptr, sizeof(double) * n * in->prog_len));
    int* elen = static_cast<int*>(up(nullptr, sizeof(int) * n));
    k_ls_specialize<<<static_cast<unsigned>((n + 127) / 128), 128>>>(D.prog, in->prog_len, static_cast<int>(n), 2, D.lo,
                                                                      D.hi, nullptr, eprog, elen);
    CK(cudaGetLastError());
    int64_t* dn = static_cast<int64_t*>(up(nullptr, sizeof(int64_t) * 3 * n));
    k_cq2_points<false><<<static_cast<unsigned>(n), kCq2Threads>>>(D, nullptr, dn, nullptr, eprog, elen);
    CK(cudaGetLastError());
    std::vector<int64_t> cnt(static_cast<size_t>(3 * n)), offs(static_cast<size_t>(n) + 1, 0);
    CK(cudaMemcpy(cnt.data(), dn, sizeof(int64_t) * 3 * n, cudaMemcpyDeviceToHost));
    for (int64_t e = 0; e < n; ++e) offs[e + 1] = offs[e] + cnt[3 * e] + cnt[3 * e + 1] + cnt[3 * e + 2];
    int64_t* doff = static_cast<int64_t*>(up(offs.data(), sizeof(int64_t) * (n + 1)));
    double* pts = static_cast<double*>(up(nullptr, sizeof(double) * 4 * std::max<int64_t>(offs[n], 1)));
    k_cq2_points<true><<<static_cast<unsigned>(n), kCq2Threads>>>(D, doff, nullptr, pts, eprog, elen);
    CK(cudaGetLastError());
    double* dK = static_cast<double*>(up(nullptr, sizeof(double) * n * nl * nl));
    double* dF = static_cast<double*>(up(nullptr, sizeof(double) * n * nl));
    double* dv = static_cast<double*>(up(nullptr, sizeof(double) * n));
    switch (q) {
      case 2: k_cq2_integrate<4><<<static_cast<unsigned>(n), kCq2Threads>>>(D, doff, dn, pts, dK, dF, dv); break;
      case 3: k_cq2_integrate<9><<<static_cast<unsigned>(n), kCq2Threads>>>(D, doff, dn, pts, dK, dF, dv); break;
      case 4: k_cq2_integrate<16><<<static_cast<unsigned>(n), kCq2Threads>>>(D, doff, dn, pts, dK, dF, dv); break;
      default: k_cq2_integrate<25><<<static_cast<unsigned>(n), kCq2Threads>>>(D, doff, dn, pts, dK, dF, dv); break;
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CK(cudaMemcpy(K, dK, sizeof(double) * n * nl * nl, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(F, dF, sizeof(double) * n * nl, cudaMemcpyDeviceToHost));
    if (vol) CK(cudaMemcpy(vol, dv, sizeof(double) * n, cudaMemcpyDeviceToHost));
    if (seconds) *seconds = ms * 1e-3;
    return IG_OK;
  });
}

}  // extern "C"

extern "C" {

int ig_assemble_thb(const ig_thb_asm* in, ig_csr* A_out, double* b_out, double* seconds) {
  if (!in || !A_out || !b_out) return fail(IG_INVALID_ARGUMENT, "assemble_thb: null argument");
  *A_out = ig_csr{};
  if (in->p < 1 || in->p > 4) return fail(IG_UNSUPPORTED, "assemble_thb: degrees 1..4");
  if (in->prog_len <= 0 || !in->prog) return fail(IG_UNSUPPORTED, "assemble_thb: no level-set program");
  if (in->n <= 0 || in->n_elem <= 0) return fail(IG_INVALID_ARGUMENT, "assemble_thb: empty space");
  const auto tw0 = std::chrono::steady_clock::now();
  return guarded([&] {
    const int q = in->p + 1, nb = q * q, go = in->gauss_order;
    const int64_t ne = in->n_elem, n = in->n;
    std::vector<void*> mem;
    auto up = [&](const void* src, size_t bytes) {
      void* d = nullptr;
      CK(cudaMalloc(&d, std::max<size_t>(bytes, 8)));
      mem.push_back(d);
      if (bytes && src) CK(cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice));
      return d;
    };
    struct Free {
      std::vector<void*>& m;
      ~Free() {
        for (void* p : m) cudaFree(p);
      }
    } free_{mem};
    const int64_t nrows = in->erow_ptr[ne];
    std::vector<int64_t> koff(static_cast<size_t>(ne) + 1, 0);
    for (int64_t e = 0; e < ne; ++e) {
      const int64_t nl = in->erow_ptr[e + 1] - in->erow_ptr[e];
      koff[e + 1] = koff[e] + nl * nl;
    }
    ig_cut2 V{};
    V.p = in->p;
    V.n_elem = in->n_elem;
    V.lo = static_cast<const double*>(up(in->lo, sizeof(double) * 2 * ne));
    V.hi = static_cast<const double*>(up(in->hi, sizeof(double) * 2 * ne));
    V.cut = static_cast<const int32_t*>(up(in->cut, sizeof(int32_t) * ne));
    V.sides = static_cast<const int32_t*>(up(in->sides, sizeof(int32_t) * ne));
    V.beta = in->beta;
    V.f = in->f;
    V.depth = in->depth;
    V.classify_depth = in->classify_depth;
    V.gauss_order = go;
    V.edge_tol = in->edge_tol;
    V.prog_len = in->prog_len;
    V.prog = static_cast<const double*>(up(in->prog, sizeof(double) * in->prog_len));
    V.gauss_q = static_cast<const double*>(up(in->gauss_q, sizeof(double) * 2 * go));
    V.gauss_q1 = static_cast<const double*>(up(in->gauss_q1, sizeof(double) * 2 * (go + 1)));
    auto* erow = static_cast<int32_t*>(up(in->erow_ptr, sizeof(int32_t) * (ne + 1)));
    auto* anch = static_cast<int32_t*>(up(in->anchors, sizeof(int32_t) * nrows));
    auto* dE = static_cast<double*>(up(in->E, sizeof(double) * nrows * nb));
    auto* sptr = static_cast<int64_t*>(up(in->supp_ptr, sizeof(int64_t) * (n + 1)));
    auto* sel = static_cast<int32_t*>(up(in->supp_el, sizeof(int32_t) * in->supp_ptr[n]));
    auto* sli = static_cast<int32_t*>(up(in->supp_li, sizeof(int32_t) * in->supp_ptr[n]));
    auto* dkoff = static_cast<int64_t*>(up(koff.data(), sizeof(int64_t) * (ne + 1)));
    auto* bad = static_cast<int*>(up(nullptr, sizeof(int)));
    CK(cudaMemset(bad, 0, sizeof(int)));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    double* eprog = static_cast<double*>(up(nullptr, sizeof(double) * ne * in->prog_len));
    int* elen = static_cast<int*>(up(nullptr, sizeof(int) * ne));
    k_ls_specialize<<<static_cast<unsigned>((ne + 127) / 128), 128>>>(V.prog, in->prog_len, static_cast<int>(ne), 2, V.lo,
                                                                       V.hi, nullptr, eprog, elen);
    CK(cudaGetLastError());
    int64_t* dn = static_cast<int64_t*>(up(nullptr, sizeof(int64_t) * 3 * ne));
    k_cq2_points<false><<<static_cast<unsigned>(ne), kCq2Threads>>>(V, nullptr, dn, nullptr, eprog, elen);
    CK(cudaGetLastError());
    std::vector<int64_t> cnt(static_cast<size_t>(3 * ne)), offs(static_cast<size_t>(ne) + 1, 0);
    CK(cudaMemcpy(cnt.data(), dn, sizeof(int64_t) * 3 * ne, cudaMemcpyDeviceToHost));
    for (int64_t e = 0; e < ne; ++e) offs[e + 1] = offs[e] + cnt[3 * e] + cnt[3 * e + 1] + cnt[3 * e + 2];
    auto* doff = static_cast<int64_t*>(up(offs.data(), sizeof(int64_t) * (ne + 1)));
    auto* pts = static_cast<double*>(up(nullptr, sizeof(double) * 4 * std::max<int64_t>(offs[ne], 1)));
    k_cq2_points<true><<<static_cast<unsigned>(ne), kCq2Threads>>>(V, doff, nullptr, pts, eprog, elen);
    CK(cudaGetLastError());
    auto* dK = static_cast<double*>(up(nullptr, sizeof(double) * std::max<int64_t>(koff[ne], 1)));
    auto* dF = static_cast<double*>(up(nullptr, sizeof(double) * std::max<int64_t>(nrows, 1)));
    k_thb_integrate<<<static_cast<unsigned>(ne), kCq2Threads>>>(V, erow, dE, doff, dn, pts, dkoff, dK, dF, bad);
    CK(cudaGetLastError());
    auto* rc = static_cast<int32_t*>(up(nullptr, sizeof(int32_t) * n));
    const unsigned gr = static_cast<unsigned>((n + 127) / 128);
    k_thb_rows<false><<<gr, 128>>>(static_cast<int32_t>(n), sptr, sel, sli, erow, anch, dkoff, dK, dF, rc, nullptr,
                                   nullptr, nullptr, nullptr, bad);
    CK(cudaGetLastError());
    std::vector<int32_t> hc(static_cast<size_t>(n));
    CK(cudaMemcpy(hc.data(), rc, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    std::vector<int64_t> ro(static_cast<size_t>(n) + 1, 0);
    std::vector<int32_t> rp(static_cast<size_t>(n) + 1, 0);
    for (int64_t a = 0; a < n; ++a) ro[a + 1] = ro[a] + hc[a];
    const int64_t nnz = ro[n];
    if (nnz > INT32_MAX) throw Error(IG_UNSUPPORTED, "assemble_thb: more than 2^31 nonzeros");
    for (int64_t a = 0; a <= n; ++a) rp[a] = static_cast<int32_t>(ro[a]);
    auto* dro = static_cast<int64_t*>(up(ro.data(), sizeof(int64_t) * (n + 1)));
    auto* drp = static_cast<int32_t*>(up(rp.data(), sizeof(int32_t) * (n + 1)));
    auto* col = static_cast<int32_t*>(up(nullptr, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
    auto* val = static_cast<double*>(up(nullptr, sizeof(double) * std::max<int64_t>(nnz, 1)));
    auto* sym = static_cast<double*>(up(nullptr, sizeof(double) * std::max<int64_t>(nnz, 1)));
    auto* db = static_cast<double*>(up(nullptr, sizeof(double) * n));
    k_thb_rows<true><<<gr, 128>>>(static_cast<int32_t>(n), sptr, sel, sli, erow, anch, dkoff, dK, dF, nullptr, dro,
                                  col, val, db, bad);
    CK(cudaGetLastError());
    k_asm_sym<<<gr, 128>>>(static_cast<int32_t>(n), drp, col, val, sym, bad);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    int hbad = 0;
    CK(cudaMemcpy(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost));
    if (hbad) throw Error(IG_UNSUPPORTED, "assemble_thb: an element has more than 32 functions, a row more than "
                                          "160 columns, or the pattern is unsymmetric");
    auto* hp = static_cast<int32_t*>(std::malloc(4 * (static_cast<size_t>(n) + 1)));
    auto* hcol = static_cast<int32_t*>(std::malloc(4 * std::max<size_t>(static_cast<size_t>(nnz), 1)));
    auto* hv = static_cast<double*>(std::malloc(8 * std::max<size_t>(static_cast<size_t>(nnz), 1)));
    if (!hp || !hcol || !hv) {
      std::free(hp);
      std::free(hcol);
      std::free(hv);
      throw Error(IG_CUDA_ERROR, "assemble_thb: host allocation failed");
    }
    std::copy(rp.begin(), rp.end(), hp);
    CK(cudaMemcpy(hcol, col, 4 * static_cast<size_t>(nnz), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hv, sym, 8 * static_cast<size_t>(nnz), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b_out, db, 8 * static_cast<size_t>(n), cudaMemcpyDeviceToHost));
    A_out->n_rows = A_out->n_cols = static_cast<int32_t>(n);
    A_out->nnz = nnz;
    A_out->row_ptr = hp;
    A_out->col_idx = hcol;
    A_out->val = hv;
    if (seconds) {
      seconds[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - tw0).count();
      seconds[1] = ms * 1e-3;
    }
    return IG_OK;
  });
}

}  // extern "C"
