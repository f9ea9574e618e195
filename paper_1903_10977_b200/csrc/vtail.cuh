// vtail.cuh — the small levels of the V-cycle in ONE persistent kernel.
//
// Why: below ~40k rows a level's work is a few microseconds of memory
// traffic, but its V-cycle step is ~9 dependent kernels (smoother phases,
// residual, restriction, prolongation, residual update, smoother again), and
// at graph-launch latency every one of them costs more than its work: on C4
// the four coarsest levels took ~450 us of a 1.34 ms V-cycle, on C5 (THB)
// five of its six levels ~250 us of 300.  Here the whole descent, the coarse
// solve and the ascent of those levels run in one cooperative launch with
// grid-wide barriers between dependent phases.  Every phase calls the same
// device functions as the standalone kernels (kernels.cuh), in the same
// per-element operation order, so results are bit-identical.
//
// Phases for level l (vcycle_at, multigrid.cpp:90-108):
//   down: [AS blocks + simple DOFs] | [complex DOFs] | res = r - A x | rc = R res
//   coarse: CTA 0 runs the pivoted L11 solve (others wait at the barrier)
//   up:   x += P xc | res -= A cor | [AS blocks + simple, acc] | [complex, acc]
#pragma once

#include <cooperative_groups.h>

#include "kernels.cuh"

namespace igk {

constexpr int kTailThreads = 512;

struct TailLevel {
  int32_t n;
  Sell A, R, P;  // row-dictionary SELL (small levels)
  AsGroups G;
  AsGather S;
  int32_t n_items;  // G.n_groups + G.n_wblocks (warp work items of phase 1)
  double *r_in, *x, *res, *cor, *ybuf;
};

struct TailParams {
  const TailLevel* lv;  // [0 .. top]; lv[0] only supplies the coarse r_in / x
  int32_t top;
  const double* r_top;  // input residual / output of the top level
  double* x_top;
  int32_t n0, rank;
  const double* Lp;
  const int32_t* piv;
  unsigned long long* prof;  // optional: %globaltimer after every phase (CTA 0, thread 0)
  int32_t debug_mode;        // 1: only the descent residual SpMVs (profiling)
};

// Profiling layout: prof[k] = CTA 0's time after barrier k; prof[256 + k*gridDim + b]
// = CTA b's arrival time at barrier k (thread 0, after its own __syncthreads).
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void tail_arrive(const TailParams& T, int k) {
  if (T.prof) {
    __syncthreads();
    if (threadIdx.x == 0 && k < 64) T.prof[256 + k * gridDim.x + blockIdx.x] = gtimer();
  }
}
__device__ __forceinline__ void tail_stamp(const TailParams& T, int& k) {
  if (T.prof && blockIdx.x == 0 && threadIdx.x == 0) T.prof[k] = gtimer();
  ++k;
}

struct TailIdx {
  int gt, nt, gw, nw, lane;
};

template <bool ACC>
__device__ __forceinline__ void tail_smooth_p1(const TailLevel& L, const double* r, double* x, const TailIdx& ix) {
  for (int w = ix.gw; w < L.n_items; w += ix.nw) as_blocks_item(L.G, w, ix.lane, r, L.ybuf);
  for (int d = ix.gt; d < L.n; d += ix.nt) as_simple_item<ACC>(L.S, d, r, x);
}

template <bool ACC>
__device__ __forceinline__ void tail_smooth_p2(const TailLevel& L, const double* r, double* x, const TailIdx& ix) {
  for (int c = ix.gt; c < L.S.n_complex; c += ix.nt) as_complex_item<ACC>(L.S, c, r, L.ybuf, x);
}

template <int MODE>
__device__ __forceinline__ void tail_spmv_grp(const Sell& A, const double* x, double* y, const double* rsrc,
                                              const TailIdx& ix) {
  const int total = ((A.n_rows * 8) + 31) & ~31;  // whole warps (shuffles inside)
  for (int base = ix.gw * 32; base < total; base += ix.nw * 32) spmv_grp_item<MODE, 8>(A, base + ix.lane, x, y, rsrc);
}

// Thread-per-row row sum for latency: batches of 16 entries, the next
// batch's values/columns loaded before this batch's ordered adds.
__device__ __forceinline__ double sell_row_lat(const Sell& A, int row, const double* __restrict__ x) {
  constexpr int U = 16;
  const int64_t base = A.slice_ptr[row >> 5] + (row & 31);
  const int info = A.rowinfo[row];
  const int len = info & 0xffff;
  const int vd = (info >> 16) & 0xff;
  const int od = (info >> 24) & 0xff;
  const double* vp = A.val + base;
  const int32_t* cp = A.col + base;
  const double* dv = A.dval + (vd > 0 ? (vd - 1) * A.dict_w : 0);
  const int32_t* dc = A.doff + (od > 0 ? (od - 1) * A.dict_w : 0);
  auto val_at = [&](int k) { return vd ? __ldg(dv + k) : __ldg(vp + static_cast<int64_t>(k) * kSell); };
  auto col_at = [&](int k) { return od ? row + __ldg(dc + k) : __ldg(cp + static_cast<int64_t>(k) * kSell); };
  double v[U];
  int32_t c[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    v[u] = u < len ? val_at(u) : 0.0;
    c[u] = u < len ? col_at(u) : row;
  }
  double acc = 0.0;
  for (int k0 = 0; k0 < len; k0 += U) {
    double xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = __ldg(x + c[u]);
    double vn[U];
    int32_t cn[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + U + u;
      vn[u] = k < len ? val_at(k) : 0.0;
      cn[u] = k < len ? col_at(k) : row;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k0 + u < len) acc = acc + v[u] * xv[u];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = vn[u];
      c[u] = cn[u];
    }
  }
  return acc;
}

template <int MODE>
__device__ __forceinline__ void tail_spmv(const Sell& A, const double* x, double* y, const double* rsrc,
                                          const TailIdx& ix) {
  for (int row = ix.gt; row < A.n_rows; row += ix.nt) {
    const double acc = sell_row_lat(A, row, x);
    y[row] = (MODE == 0) ? acc : rsrc[row] - acc;
  }
}

// CL: launched as ONE thread-block cluster (kTailCluster CTAs; barriers are
// cluster barriers), else as a cooperative grid (grid barriers).
constexpr int kTailCluster = 16;

template <bool CL>
struct TailBarrier {
  __device__ __forceinline__ void sync() {
    namespace cg = cooperative_groups;
    if (CL)
      cg::this_cluster().sync();
    else
      cg::this_grid().sync();
  }
};

template <bool SM, bool CL>
__global__ void __launch_bounds__(kTailThreads, 1) k_vtail(TailParams T) {
  extern __shared__ __align__(16) double smem[];
  TailBarrier<CL> grid;
  TailIdx ix;
  ix.gt = blockIdx.x * blockDim.x + threadIdx.x;
  ix.nt = gridDim.x * blockDim.x;
  ix.gw = ix.gt >> 5;
  ix.nw = ix.nt >> 5;
  ix.lane = threadIdx.x & 31;
  int ks = 0;
  tail_stamp(T, ks);
  if (T.debug_mode == 1) {
    for (int l = T.top; l >= 1; --l) {
      const TailLevel& L = T.lv[l];
      for (int rep = 0; rep < 3; ++rep) {
        tail_spmv<1>(L.A, L.x, L.res, L.r_in, ix);
        tail_arrive(T, ks);
        grid.sync();
        tail_stamp(T, ks);
      }
    }
    return;
  }
  // ---- descent ----
  for (int l = T.top; l >= 1; --l) {
    const TailLevel& L = T.lv[l];
    const TailLevel& C = T.lv[l - 1];
    const double* r = (l == T.top) ? T.r_top : L.r_in;
    double* x = (l == T.top) ? T.x_top : L.x;
    tail_smooth_p1<false>(L, r, x, ix);  // x = S(r, Forward)
    tail_arrive(T, ks);
    grid.sync();
    tail_stamp(T, ks);
    if (L.S.n_complex > 0) {
      tail_smooth_p2<false>(L, r, x, ix);
      tail_arrive(T, ks);
    grid.sync();
    tail_stamp(T, ks);
    }
    tail_spmv<1>(L.A, x, L.res, r, ix);  // res = r - A x
    tail_arrive(T, ks);
    grid.sync();
    tail_stamp(T, ks);
    tail_spmv<0>(L.R, L.res, C.r_in, nullptr, ix);  // R res
    tail_arrive(T, ks);
    grid.sync();
    tail_stamp(T, ks);
  }
  // ---- coarse solve ----
  {
    const TailLevel& C = T.lv[0];
    const double* r = (T.top == 0) ? T.r_top : C.r_in;
    double* x = (T.top == 0) ? T.x_top : C.x;
    if (blockIdx.x == 0) coarse_solve_cta<SM>(T.n0, T.rank, T.Lp, T.piv, r, x, smem);
    tail_arrive(T, ks);
    if (T.top > 0) grid.sync();
    tail_stamp(T, ks);
  }
  // ---- ascent ----
  for (int l = 1; l <= T.top; ++l) {
    const TailLevel& L = T.lv[l];
    const TailLevel& C = T.lv[l - 1];
    double* x = (l == T.top) ? T.x_top : L.x;
    for (int row = ix.gt; row < L.P.n_rows; row += ix.nt) {  // cor = R^T xc; x += cor
      const double c = sell_row<false, 3>(L.P, row, C.x);
      L.cor[row] = c;
      x[row] = x[row] + c;
    }
    tail_arrive(T, ks);
    grid.sync();
    tail_stamp(T, ks);
    tail_spmv<1>(L.A, L.cor, L.res, L.res, ix);  // res -= A cor
    tail_arrive(T, ks);
    grid.sync();
    tail_stamp(T, ks);
    tail_smooth_p1<true>(L, L.res, x, ix);  // x += S(res, Reverse)
    if (L.S.n_complex > 0) {
      tail_arrive(T, ks);
    grid.sync();
    tail_stamp(T, ks);
      tail_smooth_p2<true>(L, L.res, x, ix);
    }
    tail_arrive(T, ks);
    if (l < T.top) grid.sync();
    tail_stamp(T, ks);
  }
}

}  // namespace igk
