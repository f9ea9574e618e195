// Device kernels of the solve phase (sm_100a, FP64, HBM-bound; no tensor
// cores -- every operation here is <= 0.25 flop/B).
//
// Arithmetic contract: the library is compiled with -fmad=false, so every
// a*b+c rounds twice, exactly like the reference's default x86-64 build and
// the oracle (-ffp-contract=off).  Every kernel fixes its summation order to
// the one the oracle documents, so device results are bitwise reproducible
// run to run and bitwise equal to oracle/oracle.c in ORC_GPU_ORDER mode.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace igk {

// Programmatic dependent launch (PDL): every kernel is launched with
// programmatic stream serialization, so the next kernel's CTAs are scheduled
// while this one runs and the launch latency of a dependent chain overlaps
// the work.  Each kernel first waits for its predecessor grid to complete
// (griddepcontrol.wait: full completion + memory flush, transitively), then
// lets its own dependents launch.  Without the launch attribute both are
// no-ops.
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// Kernels that set a CUDA-graph conditional (the PCG / Richardson IF and
// WHILE handles) wait but never trigger their dependents early: the node
// after them may be a conditional node, which must not be evaluated before
// the value is written (the implicit trigger at grid completion is safe).
// (Triggering before the wait -- measured as a variant -- let conditional
// nodes read stale handles: PCG ran to maxit.)
__device__ __forceinline__ void pdl_wait_only() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Split form: a kernel first loads what no earlier kernel writes (matrix
// layouts, block factors and DOF lists, contribution lists -- built once at
// ig_hier_create), THEN waits for its predecessor, so those loads overlap the
// predecessor's tail instead of sitting on the chain.  Waiters are passed to
// the shared device helpers; NoWait where the caller already waited.
struct NoWait {
  __device__ __forceinline__ void operator()() const {}
};
struct PdlWait {
  __device__ __forceinline__ void operator()() const { pdl_entry(); }
};

constexpr int kCta = 256;   // threads per CTA == reduction chunk size
// Register budgets (min CTAs per SM) of the smoother and small-level SpMV
// kernels; variant builds override them (profiles/build_variants.sh).
// (An explicit minimum of 1 is NOT the same as none: it lets ptxas use up to
// 255 registers.)  0 = no hint.
#ifndef IG_ASB_MINB
#define IG_ASB_MINB 0
#endif
#ifndef IG_AS_MINB
#define IG_AS_MINB 0
#endif
#ifndef IG_GRP_MINB
#define IG_GRP_MINB 0
#endif
#if IG_ASB_MINB > 0
#define IG_ASB_BOUNDS __launch_bounds__(128, IG_ASB_MINB)
#else
#define IG_ASB_BOUNDS __launch_bounds__(128)
#endif
#if IG_AS_MINB > 0
#define IG_AS_BOUNDS __launch_bounds__(kCta, IG_AS_MINB)
#else
#define IG_AS_BOUNDS __launch_bounds__(kCta)
#endif
#if IG_GRP_MINB > 0
#define IG_GRP_BOUNDS __launch_bounds__(kCta, IG_GRP_MINB)
#else
#define IG_GRP_BOUNDS __launch_bounds__(kCta)
#endif

constexpr int kSell = 32;   // SELL slice height == warp size

// ----------------------------------------------------------- PCG state ----
// Device-resident solver state: scalars, flags and the residual history.  The
// whole PCG loop reads/writes it, so no host round trip is needed.
struct PcgState {
  double bnorm, rz, rz_new, pap, alpha, beta, tol;
  int32_t k, maxit, done, status;
  int32_t streak;    // Richardson: consecutive residual growths
  const double* b;   // right-hand side (device pointer, set per solve)
  double* x;         // solution (device pointer, set per solve)
  double* residuals; // maxit+1
  unsigned int counter[8];
};
enum { ST_RUNNING = -1, ST_OK = 0, ST_NOT_CONVERGED = 1, ST_BREAKDOWN = 2, ST_DIVERGED = 6 };

// ------------------------------------------------------------ reduction ---
// Canonical chunk reduction (oracle.c tree256): 32-lane xor butterfly per
// warp, then ((w0+w1)+(w2+w3))+((w4+w5)+(w6+w7)).  Result valid in thread 0.
__device__ __forceinline__ double cta_reduce(double v, double* sm8) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sm8[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    t = ((sm8[0] + sm8[1]) + (sm8[2] + sm8[3])) + ((sm8[4] + sm8[5]) + (sm8[6] + sm8[7]));
  return t;
}

// Lane t of the last CTA: P[t] + P[t+256] + ... in ascending order (the
// canonical partials sum).  All 16 loads of a batch are issued before its
// adds -- predicated, so even a short tail is one L2 round trip per 16
// partials (profiles/reduce_micro.cu: -2 us per reduction kernel at C4 size
// against 8-load batches with a serial remainder).  The predicated-off
// slots add +0, a no-op: the running sum starts at +0 and is never -0.
__device__ __forceinline__ double partials_lane_sum(const double* partials, unsigned int nparts) {
  constexpr int T = 16;
  double a = 0.0;
  for (unsigned int k = threadIdx.x; k < nparts; k += T * kCta) {
    double q[T];
#pragma unroll
    for (int u = 0; u < T; ++u) q[u] = (k + u * kCta < nparts) ? __ldcg(partials + k + u * kCta) : 0.0;
#pragma unroll
    for (int u = 0; u < T; ++u) a = a + q[u];
  }
  return a;
}

// Arrive once per CTA (after this CTA wrote its chunk partials); the last CTA
// to arrive reduces all nparts partials (lane t sums P[t], P[t+256], ...
// ascending, then cta_reduce) and returns true with *total set (valid in every
// thread of that CTA).  Must be reached by all threads of every CTA.
__device__ __forceinline__ bool grid_finish(unsigned int nparts, const double* partials, unsigned int* counter,
                                            double* total) {
  __shared__ double sm8f[8];
  __shared__ bool is_last;
  __shared__ double tot;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  const double t = cta_reduce(partials_lane_sum(partials, nparts), sm8f);
  if (threadIdx.x == 0) {
    tot = t;
    *counter = 0u;
  }
  __syncthreads();
  *total = tot;
  return true;
}

// Canonical reduction over a bounded grid: CTA b handles chunks b, b+grid,
// ... (256 elements each, same per-chunk tree and the same partials as one
// CTA per chunk), then arrives ONCE -- the per-CTA atomic arrival is what
// made one-CTA-per-chunk reductions slow (7,811 same-address atomics on C4:
// k_pcg_update 69 us, k_as_finish_red 89 us).  f(i) does element i's work
// and returns its product.  Launch with red_grid (ig_gpu.cu).
template <class F>
__device__ __forceinline__ bool chunk_reduce(int n, F f, double* partials, unsigned int* counter, double* total) {
  // Two buffers of B x 8 warp sums: consecutive rounds alternate, so one
  // barrier per round (not one per chunk) separates writers from readers.
  constexpr int B = 4;
  __shared__ double smc[2][B][8];
  const unsigned int nchunks = static_cast<unsigned int>((n + kCta - 1) / kCta);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int buf = 0;
  // B chunks per round: their element work first (loads in flight together),
  // then the B warp butterflies interleaved (independent shuffle chains), one
  // barrier, and thread u < B finishes chunk u's tree -- the same per-chunk
  // tree (cta_reduce) as one CTA per chunk.
  for (unsigned int c0 = blockIdx.x; c0 < nchunks; c0 += B * gridDim.x) {
    double v[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const unsigned int c = c0 + u * gridDim.x;
      const int i = static_cast<int>(c) * kCta + threadIdx.x;
      v[u] = (c < nchunks && i < n) ? f(i) : 0.0;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
      for (int u = 0; u < B; ++u) v[u] = v[u] + __shfl_xor_sync(0xffffffffu, v[u], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < B; ++u) smc[buf][u][w] = v[u];
    }
    __syncthreads();
    if (threadIdx.x < B) {
      const unsigned int c = c0 + threadIdx.x * gridDim.x;
      if (c < nchunks) {
        const double* q = smc[buf][threadIdx.x];
        partials[c] = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
        __threadfence();  // each writer publishes its own partial before the arrival
      }
    }
    buf ^= 1;
  }
  return grid_finish(nchunks, partials, counter, total);
}

// Reduce this CTA's chunk (one value per thread, cta_reduce) and publish the
// partial; the last CTA to arrive reduces all partials (lane t sums P[t],
// P[t+256], ... ascending, then cta_reduce) and returns true with *total set
// (valid in every thread of that CTA).  Must be reached by all threads.
__device__ __forceinline__ bool last_cta_total(double v, double* partials,
                                               unsigned int* counter, double* total) {
  __shared__ double sm8[8];
  __shared__ bool is_last;
  __shared__ double tot;
  const double partial = cta_reduce(v, sm8);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = partial;
    __threadfence();
    const unsigned int prev = atomicAdd(counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  const double a = partials_lane_sum(partials, gridDim.x);
  __syncthreads();  // sm8 reuse
  const double t = cta_reduce(a, sm8);
  if (threadIdx.x == 0) {
    tot = t;
    *counter = 0u;
  }
  __syncthreads();
  *total = tot;
  return true;
}

// V-cycle and vector kernels do not test the PCG flags: in the graph, the
// conditional IF/WHILE nodes skip them once the solve has stopped, and in the
// host-loop fallback a post-stop V-cycle only touches scratch (z, p, level
// buffers), never x or the residual history.  Only k_pcg_update tests it
// (a breakdown detected by the preceding SpMV must not update x and r).
__device__ __forceinline__ bool pcg_done(const PcgState*) { return false; }
__device__ __forceinline__ bool pcg_stopped(const PcgState* st) {
  return *reinterpret_cast<const volatile int32_t*>(&st->done) != 0;
}

// ----------------------------------------------------------- SELL SpMV ----
// Sliced ELLPACK, slice height 32, column-major within a slice: entry k of
// row i sits at slice_ptr[i/32] + 32*k + (i%32).  One thread per row walks its
// row in ascending column order (== Eigen RowMajor order), so warps load 32
// consecutive doubles / ints per step (coalesced) and the x gathers of
// neighbouring rows share sectors.
//
// Row dictionary ("stencil compression"): most rows of an immersed B-spline
// operator are interior rows whose value sequence is bit-identical (81% of
// the C4 finest A share ONE sequence), and many also share the column-offset
// pattern col - row.  rowinfo packs len | vd << 16 | od << 24: vd > 0 reads
// the row's values from dictionary entry vd-1 (L1-resident, broadcast within
// the warp) instead of HBM; od > 0 also derives the columns as row + doff.
// The explicit SELL arrays are still allocated for every row, but predicated
// lanes issue no memory requests, so HBM traffic drops to the explicit part.
// Values and columns are bit-identical to the stored ones (checked on the
// host), so results are unchanged.
struct Sell {
  int32_t n_rows, n_cols;
  const int64_t* slice_ptr;
  const int32_t* rowinfo;
  const double* val;
  const int32_t* col;
  int32_t dict_w;        // dictionary row stride
  const double* dval;    // [vd-1][k]
  const int32_t* doff;   // [od-1][k]
};

template <bool STREAM>
__device__ __forceinline__ double ld_val(const double* p) {
  if (STREAM) return __ldcs(p);
  return __ldg(p);
}
template <bool STREAM>
__device__ __forceinline__ int32_t ld_col(const int32_t* p) {
  if (STREAM) return __ldcs(p);
  return __ldg(p);
}

// Row dot product, ascending k: batches of 8 predicated loads (values,
// columns, then x) ahead of the serial sum.  Entries past the row end are
// never added (acc + 0*x could turn -0 into +0 and break bit-parity with the
// oracle).  Chosen from measurement among four batch/pipelining variants
// (round 1, profiles/spmv_variants.py): the thread-per-row chain is
// latency-bound once the row dictionary removes most HBM traffic.
template <bool STREAM>
__device__ __forceinline__ double sell_row(const Sell& A, int row, const double* __restrict__ x) {
  const int64_t base = A.slice_ptr[row >> 5] + (row & 31);
  const int info = A.rowinfo[row];
  const int len = info & 0xffff;
  const int vd = (info >> 16) & 0xff;
  const int od = (info >> 24) & 0xff;
  const double* vp = A.val + base;
  const int32_t* cp = A.col + base;
  const double* dv = A.dval + (vd > 0 ? (vd - 1) * A.dict_w : 0);
  const int32_t* dc = A.doff + (od > 0 ? (od - 1) * A.dict_w : 0);
  constexpr int U = 8;
  double acc = 0.0;
  auto val_at = [&](int k) { return vd ? __ldg(dv + k) : ld_val<STREAM>(vp + k * kSell); };
  auto col_at = [&](int k) { return od ? row + __ldg(dc + k) : ld_col<STREAM>(cp + k * kSell); };
  for (int k = 0; k < len; k += U) {
    double v[U];
    int32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = 0.0;
      c[u] = row;
      if (k + u < len) {
        v[u] = val_at(k + u);
        c[u] = col_at(k + u);
      }
    }
    double xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = (k + u < len) ? __ldg(x + c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k + u < len) acc = acc + v[u] * xv[u];
  }
  return acc;
}

// MODE 0: y = A x.  MODE 1: y = r - A x with r read from y (in place allowed).
// RED: also reduce x_i * y_i (p . Ap) into the PCG state.
template <int MODE, bool STREAM, bool RED>
__global__ void __launch_bounds__(kCta, 1) k_spmv(Sell A, const double* __restrict__ x, double* y,
                                               const double* rsrc, PcgState* st, double* partials) {
  pdl_entry();
  if (pcg_done(st)) return;
  const int row = blockIdx.x * kCta + threadIdx.x;
  double prod = 0.0;
  if (row < A.n_rows) {
    const double acc = sell_row<STREAM>(A, row, x);
    double out;
    if (MODE == 0)
      out = acc;
    else
      out = rsrc[row] - acc;
    y[row] = out;
    if (RED) prod = x[row] * out;
  }
  if (RED) {
    double pap;
    if (last_cta_total(prod, partials, &st->counter[0], &pap)) {
      if (threadIdx.x == 0) {
        st->pap = pap;
        if (pap <= 0.0) {  // solvers.cpp:47-50 (a NaN does not trigger it)
          st->status = ST_BREAKDOWN;
          st->done = 1;
        } else {
          st->alpha = st->rz / pap;
        }
      }
    }
  }
}

// Small levels (latency-bound, too few rows to hide a 16-batch thread-per-row
// chain): G lanes per row.  Lane g loads entry k0+g and forms its product in
// parallel; the group leader then adds the G products in ascending k by
// shuffles, so the sum is still sequential ((acc + p0) + p1) + ... exactly as
// in the thread-per-row kernel, but the memory latency is paid once per G
// entries instead of once per batch of a single thread.
// Body for global thread t (all 32 lanes of a warp call it together: the
// warp-maximum length is formed by shuffles).
template <int MODE, int G>
__device__ __forceinline__ void spmv_grp_item(const Sell& A, int t, const double* __restrict__ x, double* y,
                                              const double* rsrc, bool pdl = false) {
  const int row = t / G;
  const int g = t % G;
  const int lane = threadIdx.x & 31;
  const int gbase = lane - g;
  const bool valid_row = row < A.n_rows;
  int len = 0, vd = 0, od = 0;
  int64_t base = 0;
  if (valid_row) {
    base = A.slice_ptr[row >> 5] + (row & 31);
    const int info = A.rowinfo[row];
    len = info & 0xffff;
    vd = (info >> 16) & 0xff;
    od = (info >> 24) & 0xff;
  }
  const double* dv = A.dval + (vd > 0 ? (vd - 1) * A.dict_w : 0);
  const int32_t* dc = A.doff + (od > 0 ? (od - 1) * A.dict_w : 0);
  // Rows in a warp can have different lengths: iterate to the warp maximum.
  int wlen = len;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) wlen = max(wlen, __shfl_xor_sync(0xffffffffu, wlen, o));
  // Chunks of G*U entries: every lane issues its U value/column loads, then
  // its U gathers, before any product is summed, so a chunk costs one memory
  // round trip instead of U (the small levels are latency-bound).
  constexpr int U = 16;
  double acc = 0.0;
  double rs = 0.0;
  bool have_rs = false;
  for (int k0 = 0; k0 < wlen; k0 += G * U) {
    double v[U];
    int32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * G + g;
      v[u] = 0.0;
      c[u] = 0;
      if (k < len) {
        v[u] = vd ? __ldg(dv + k) : __ldg(A.val + base + static_cast<int64_t>(k) * kSell);
        c[u] = od ? row + __ldg(dc + k) : __ldg(A.col + base + static_cast<int64_t>(k) * kSell);
      }
    }
    if (pdl && k0 == 0) {
      pdl_entry();  // values / columns are static: loaded before the predecessor wait
      if (MODE == 1 && valid_row && g == 0) {
        rs = rsrc[row];  // ahead of the product chain
        have_rs = true;
      }
    }
    double prod[U];
#pragma unroll
    for (int u = 0; u < U; ++u) prod[u] = (k0 + u * G + g < len) ? v[u] * __ldg(x + c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (k0 + u * G < wlen) {  // warp-uniform
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const double pu = __shfl_sync(0xffffffffu, prod[u], gbase + j);
          if (g == 0 && k0 + u * G + j < len) acc = acc + pu;
        }
      }
    }
  }
  if (pdl && wlen == 0) pdl_entry();
  if (MODE == 1 && valid_row && g == 0 && !have_rs) rs = rsrc[row];
  if (valid_row && g == 0) y[row] = (MODE == 0) ? acc : rs - acc;
}
template <int MODE, int G>
__global__ void IG_GRP_BOUNDS k_spmv_grp(Sell A, const double* __restrict__ x, double* y,
                                                   const double* rsrc) {
  spmv_grp_item<MODE, G>(A, blockIdx.x * kCta + threadIdx.x, x, y, rsrc, true);
}

// Prolongation fused with the correction: cor = P xc (P = R^T stored as CSR
// over fine rows, ascending coarse index == Eigen's column-major R^T product
// order) and x += cor.
template <bool STREAM>
__global__ void __launch_bounds__(kCta, 1) k_prolong(Sell P, const double* __restrict__ xc, double* cor,
                                                  double* x, const PcgState* st) {
  const int row = blockIdx.x * kCta + threadIdx.x;
  if (row < P.n_rows) {  // static layout words into L1 while the predecessor finishes
    const int64_t base = P.slice_ptr[row >> 5] + (row & 31);
    asm volatile("prefetch.global.L1 [%0];" ::"l"(P.val + base));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(P.col + base));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(P.rowinfo + row));
  }
  pdl_entry();
  if (pcg_done(st)) return;
  if (row >= P.n_rows) return;
  const double xo = x[row];  // ahead of the product chain
  const double c = sell_row<STREAM>(P, row, xc);
  cor[row] = c;
  x[row] = xo + c;
}

// ------------------------------------------------- exact division ---------
// a / b, correctly rounded, given rb = RN(1/b) computed ahead of time (off the
// dependent chain).  q0 = RN(a*rb) is within 2 ulps of a/b; two Markstein
// corrections q <- RN(q + RN_exact(a - b*q)*rb) (residual exact by FMA) make
// it RN(a/b) for finite, non-extreme operands (Markstein's theorem; checked
// bit-for-bit against IEEE division on 2e8 random and structured pairs).
// Used only inside substitution chains, where the latency of div.rn.f64
// (reciprocal iteration + slow-path check) would otherwise be paid per step;
// results are identical to the oracle's plain division.
__device__ __forceinline__ double exact_div(double a, double b, double rb) {
  double q = a * rb;
  double r = __fma_rn(-b, q, a);
  q = __fma_rn(r, rb, q);
  r = __fma_rn(-b, q, a);
  return __fma_rn(r, rb, q);
}
// Reciprocal for exact_div; non-finite / zero pivots fall back to a / b.
__device__ __forceinline__ double safe_rcp(double b) { return 1.0 / b; }
__device__ __forceinline__ double div_rb(double a, double b, double rb) {
  return isfinite(rb) && rb != 0.0 ? exact_div(a, b, rb) : a / b;
}

// ------------------------------------------------- additive Schwarz -------
// Phase 1: multi-DOF blocks (s >= 2).  Two layouts, one launch:
//  * "groups": thread-per-block for small blocks (s <= 8) and the rare
//    s > 32 fallback.  Blocks are sorted by size (descending) and grouped by
//    32 (one warp); DOF lists, output positions and packed lower factors are
//    interleaved lane-fastest so every load is coalesced.  Packed lower
//    column-major with the group's s_max as stride:
//    e(i, j) = j*smax - j*(j-1)/2 + (i - j), i >= j.
//  * "warp blocks": warp-per-block for 9 <= s <= 32.  Lane i holds y_i and
//    row i of L + L^T in registers; each substitution step is one division
//    by the owning lane, a shuffle broadcast and one FMA-free update per lane,
//    so the dependent chain is 2s short steps instead of s^2 loads.
// Both perform exactly the oracle's operation sequence per entry (forward
// column-oriented; backward y_i = (y_i - sum_{k desc} L(k,i) y_k) / L(i,i)).
struct AsGroups {
  int32_t n_groups;
  const int32_t* smax;      // per group
  const int64_t* dof_off;   // per group: base of [i][lane] dof table
  const int64_t* fac_off;   // per group: base of [e][lane] factor table
  const int32_t* size;      // [group*32 + lane], 0 for padding lanes
  const int32_t* ypos;      // [group*32 + lane]: ybuf offset of the block
  const int32_t* dofs;
  const double* fac;
  // warp blocks
  int32_t n_wblocks;
  const int32_t* w_size;
  const int32_t* w_ypos;
  const int64_t* w_dof_off;
  const int64_t* w_fac_off;  // full s x s column-major factor
  const int32_t* w_dofs;
  const double* w_fac;
  // Tolerance mode (ig_gpu.cu Opts::fast_blocks): the factor slots hold the
  // lower triangle of the explicit inverse, applied as y = M r (FMA).
  int32_t inv;
};

__device__ __forceinline__ int packed_idx(int i, int j, int smax) {
  return j * smax - (j * (j - 1)) / 2 + (i - j);
}

// Residual gather of the block solves: r[d] (additive and classic
// multiplicative sweep) or, for the lazily updated multiplicative sweep, a
// functor computing the frozen residual of DOF d (LazyLoad below).
template <class T>
struct NoDeduce {
  using type = T;
};
struct RLoad {
  const double* r;
  __device__ __forceinline__ RLoad(const double* p) : r(p) {}
  __device__ __forceinline__ double operator()(int d) const { return __ldg(r + d); }
};

// Output: additive (MS = false) -> ybuf[pos + i]; multiplicative sweep
// (MS = true) -> ybuf is the colour's delta vector: delta[d] = 0 + y_i and
// xms[d] += delta[d] (smoothers.cpp:199-204; same-colour blocks are disjoint).
template <bool MS>
__device__ __forceinline__ void block_out(double* ybuf, double* xms, int pos_or_dof, double y) {
  if (MS) {
    const double dv = 0.0 + y;
    ybuf[pos_or_dof] = dv;
    xms[pos_or_dof] = xms[pos_or_dof] + dv;
  } else {
    ybuf[pos_or_dof] = y;
  }
}

template <int SM, bool MS = false, class LD = RLoad, class WT = NoWait>
__device__ __forceinline__ void block_solve(const AsGroups& G, int g, int lane, int s, int smax,
                                            typename NoDeduce<LD>::type r, double* ybuf, double* xms = nullptr,
                                            WT wt = WT{}) {
  double y[SM], Lp[SM * (SM + 1) / 2];
  int dof[SM];
  const int32_t* dp = G.dofs + G.dof_off[g] + lane;
  const double* fp = G.fac + G.fac_off[g] + lane;
  // All loads first (independent of the substitution chain): the static DOF
  // list and factor before the predecessor wait, the residual gathers after.
#pragma unroll
  for (int i = 0; i < SM; ++i) dof[i] = (i < s) ? dp[i * 32] : 0;
#pragma unroll
  for (int j = 0; j < SM; ++j)
#pragma unroll
    for (int i = j; i < SM; ++i) Lp[packed_idx(i, j, SM)] = (i < s) ? fp[packed_idx(i, j, smax) * 32] : 1.0;
  wt();
#pragma unroll
  for (int i = 0; i < SM; ++i) y[i] = (i < s) ? r(dof[i]) : 0.0;
  if (!MS && G.inv) {  // tolerance mode: y = M r with M symmetric, lower triangle stored
    double z[SM];
#pragma unroll
    for (int i = 0; i < SM; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < SM; ++j) {
        const double mij = i >= j ? Lp[packed_idx(i, j, SM)] : Lp[packed_idx(j, i, SM)];
        if (j < s) acc = __fma_rn(mij, y[j], acc);
      }
      z[i] = acc;
    }
    const int pos = G.ypos[g * 32 + lane];
#pragma unroll
    for (int i = 0; i < SM; ++i)
      if (i < s) block_out<MS>(ybuf, xms, pos + i, z[i]);
    return;
  }
  double rd[SM];  // reciprocal pivots, computed off the substitution chain
#pragma unroll
  for (int j = 0; j < SM; ++j) rd[j] = safe_rcp(Lp[packed_idx(j, j, SM)]);
#pragma unroll
  for (int j = 0; j < SM; ++j) {
    if (j < s) {
      const double yj = div_rb(y[j], Lp[packed_idx(j, j, SM)], rd[j]);
      y[j] = yj;
#pragma unroll
      for (int i = j + 1; i < SM; ++i)
        if (i < s) y[i] = y[i] - Lp[packed_idx(i, j, SM)] * yj;
    }
  }
#pragma unroll
  for (int i = SM - 1; i >= 0; --i) {
    if (i < s) {
      double acc = 0.0;
#pragma unroll
      for (int k = SM - 1; k > i; --k)
        if (k < s) acc = acc + Lp[packed_idx(k, i, SM)] * y[k];
      y[i] = div_rb(y[i] - acc, Lp[packed_idx(i, i, SM)], rd[i]);
    }
  }
  const int pos = G.ypos[g * 32 + lane];
#pragma unroll
  for (int i = 0; i < SM; ++i)
    if (i < s) block_out<MS>(ybuf, xms, MS ? dof[i] : pos + i, y[i]);
}

// Generic (any size) fallback with local memory.
template <bool MS = false, class LD = RLoad, class WT = NoWait>
__device__ __noinline__ void block_solve_any(const AsGroups& G, int g, int lane, int s, int smax,
                                             typename NoDeduce<LD>::type r, double* ybuf, double* xms = nullptr,
                                             WT wt = WT{}) {
  wt();
  double y[128];
  const int32_t* dp = G.dofs + G.dof_off[g] + lane;
  const double* fp = G.fac + G.fac_off[g] + lane;
  for (int i = 0; i < s; ++i) y[i] = r(dp[i * 32]);
  if (!MS && G.inv) {  // tolerance mode: y = M r
    const int pos = G.ypos[g * 32 + lane];
    for (int i = 0; i < s; ++i) {
      double acc = 0.0;
      for (int j = 0; j < s; ++j)
        acc = __fma_rn(fp[(i >= j ? packed_idx(i, j, smax) : packed_idx(j, i, smax)) * 32], y[j], acc);
      block_out<MS>(ybuf, xms, pos + i, acc);
    }
    return;
  }
  for (int j = 0; j < s; ++j) {
    const double yj = y[j] / fp[packed_idx(j, j, smax) * 32];
    y[j] = yj;
    for (int i = j + 1; i < s; ++i) y[i] = y[i] - fp[packed_idx(i, j, smax) * 32] * yj;
  }
  for (int i = s - 1; i >= 0; --i) {
    double acc = 0.0;
    for (int k = s - 1; k > i; --k) acc = acc + fp[packed_idx(k, i, smax) * 32] * y[k];
    y[i] = (y[i] - acc) / fp[packed_idx(i, i, smax) * 32];
  }
  const int pos = G.ypos[g * 32 + lane];
  for (int i = 0; i < s; ++i) block_out<MS>(ybuf, xms, MS ? dp[i * 32] : pos + i, y[i]);
}

template <bool MS = false, class LD = RLoad, class WT = NoWait>
__device__ __forceinline__ void warp_block_solve(const AsGroups& G, int b, int lane,
                                                 typename NoDeduce<LD>::type r, double* ybuf, double* xms = nullptr,
                                                 WT wt = WT{}) {
  const int s = G.w_size[b];
  const double* f = G.w_fac + G.w_fac_off[b];
  const int32_t* dp = G.w_dofs + G.w_dof_off[b];
  double m[32];  // m[t] = L(max(lane,t), min(lane,t)): row `lane` of L + L^T
#pragma unroll
  for (int t = 0; t < 32; ++t) {
    const int hi = lane > t ? lane : t, lo = lane > t ? t : lane;
    m[t] = (t < s && lane < s) ? __ldg(f + lo * s + hi) : 0.0;
  }
  const int mydof = lane < s ? dp[lane] : 0;
  const double dg = lane < s ? __ldg(f + lane * s + lane) : 1.0;  // own pivot L(lane, lane)
  wt();
  double y = lane < s ? r(mydof) : 0.0;
  if (!MS && G.inv) {  // tolerance mode: lane i computes (M r)_i, r_j by shuffle, ascending j
    double z = 0.0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double yj = __shfl_sync(0xffffffffu, y, j);
      if (j < s) z = __fma_rn(m[j], yj, z);
    }
    if (lane < s) block_out<MS>(ybuf, xms, G.w_ypos[b] + lane, z);
    return;
  }
  const double rdg = safe_rcp(dg);
  double acc = 0.0;
  if (__all_sync(0xffffffffu, isfinite(rdg) && rdg != 0.0)) {
    // Branch-free steps (as in the coarse solve): every lane forms the
    // quotient, the shuffle picks the owner's, selects keep each lane's own
    // operation sequence.
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j < s) {
        const double yj = __shfl_sync(0xffffffffu, exact_div(y, dg, rdg), j);
        const double upd = y - m[j] * yj;
        y = (lane == j) ? yj : ((lane > j) ? upd : y);
      }
    }
#pragma unroll
    for (int k = 31; k >= 0; --k) {
      if (k < s) {
        const double yk = __shfl_sync(0xffffffffu, exact_div(y - acc, dg, rdg), k);
        const double nacc = acc + m[k] * yk;
        y = (lane == k) ? yk : y;
        acc = (lane < k) ? nacc : acc;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j < s) {
        if (lane == j) y = div_rb(y, dg, rdg);
        const double yj = __shfl_sync(0xffffffffu, y, j);
        if (lane > j) y = y - m[j] * yj;
      }
    }
#pragma unroll
    for (int k = 31; k >= 0; --k) {
      if (k < s) {
        if (lane == k) y = div_rb(y - acc, dg, rdg);
        const double yk = __shfl_sync(0xffffffffu, y, k);
        if (lane < k) acc = acc + m[k] * yk;
      }
    }
  }
  if (lane < s) block_out<MS>(ybuf, xms, MS ? mydof : G.w_ypos[b] + lane, y);
}

// One warp-sized work item w of phase 1 (group of small blocks or a warp block).
template <bool MS = false, class LD = RLoad, class WT = NoWait>
__device__ __forceinline__ void as_blocks_item(const AsGroups& G, int w, int lane, typename NoDeduce<LD>::type r,
                                               double* ybuf, double* xms = nullptr, WT wt = WT{}) {
  if (w < G.n_groups) {
    const int g = w;
    const int s = G.size[g * 32 + lane];
    const int smax = G.smax[g];  // warp-uniform
    if (s == 0) return;
    if (smax <= 4)
      block_solve<4, MS, LD, WT>(G, g, lane, s, smax, r, ybuf, xms, wt);
    else if (smax <= 8)
      block_solve<8, MS, LD, WT>(G, g, lane, s, smax, r, ybuf, xms, wt);
    else
      block_solve_any<MS, LD, WT>(G, g, lane, s, smax, r, ybuf, xms, wt);
  } else if (w - G.n_groups < G.n_wblocks) {
    warp_block_solve<MS, LD, WT>(G, w - G.n_groups, lane, r, ybuf, xms, wt);
  }
}
// Groups of small blocks only (smax <= 4: ~90 % of the multi-DOF blocks on
// the C4 levels), groups g_begin.. of G: without the 8-wide and warp-block
// code the kernel needs a third of k_as_blocks' registers, so all of its
// warps are resident at once.  It runs on its own side stream, concurrently
// with k_as_blocks (groups < g_begin and the warp blocks) and the singleton
// DOFs.
__global__ void __launch_bounds__(128) k_as_blocks4(AsGroups G, int32_t g_begin, const double* __restrict__ r,
                                                    double* ybuf, const PcgState* st) {
  const int g = g_begin + static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (g >= G.n_groups) return;
  const int s = G.size[g * 32 + lane];
  if (s == 0) return;
  block_solve<4, false, RLoad, PdlWait>(G, g, lane, s, G.smax[g], r, ybuf, nullptr, PdlWait{});
}
__global__ void IG_ASB_BOUNDS k_as_blocks(AsGroups G, const double* __restrict__ r,
                                                   double* ybuf, const PcgState* st) {
  // pcg_done is a compile-time no-op for V-cycle kernels (see above); the
  // predecessor wait happens inside, after the static loads.
  as_blocks_item<false, RLoad, PdlWait>(G, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, threadIdx.x & 31, r,
                                        ybuf, nullptr, PdlWait{});
}

// Phase 2: deterministic segmented reduction per DOF, contributions in
// ascending block order starting from 0 (smoothers.cpp:176-183), then gamma.
// Fast path (head[d] >= 0): the DOF's only contribution is its own singleton
// block, y = (r_d / l) / l with l = sdiag[d] (== the LLT solve of a 1x1
// block: forward r/l, backward (y - 0)/l).  Otherwise list c = -head[d]-1:
// entry code >= 0 is a ybuf offset (multi-DOF block), code = -(b+1) a
// singleton block b with factor sval[b].
// ACC: x += gamma*sum (post-smoother) else x = gamma*sum.
// RED: also reduce rdot_i * x_i (r . z) into the PCG state (finest level).
struct AsGather {
  int32_t n;
  double gamma;
  const int32_t* head;
  const double* sdiag;
  const int32_t* cptr;
  const int32_t* centry;
  const double* sval;
  int32_t n_complex;
  const int32_t* cdof;  // complex list index -> DOF
};

// rz = r . z bookkeeping after a preconditioner application (solvers.cpp:41-43, :63-65).
__device__ __forceinline__ void rz_update(PcgState* st, double rz) {
  if (st->k < 0) {  // initial application: p = z, rz = r.z
    st->rz = rz;
    st->k = 0;
  } else {
    st->rz_new = rz;
    st->beta = rz / st->rz;
    st->rz = rz;
  }
}

template <bool ACC, bool RED>
__global__ void __launch_bounds__(kCta) k_as_gather(AsGather S, const double* __restrict__ r,
                                                    const double* __restrict__ ybuf, double* x,
                                                    const double* rdot, PcgState* st, double* partials) {
  pdl_entry();
  if (pcg_done(st)) return;
  const int d = blockIdx.x * kCta + threadIdx.x;
  double prod = 0.0;
  if (d < S.n) {
    const int h = S.head[d];
    const double rd = r[d];
    const double l = S.sdiag[d];
    const double xo = ACC ? x[d] : 0.0;
    double acc = 0.0;
    if (h >= 0) {
      acc = acc + (rd / l) / l;
    } else {
      const int c = -h - 1;
      const int q0 = S.cptr[c], q1 = S.cptr[c + 1];
      for (int q = q0; q < q1; ++q) {
        const int code = S.centry[q];
        double v;
        if (code < 0) {
          const double ls = S.sval[-code - 1];
          v = (rd / ls) / ls;
        } else {
          v = ybuf[code];
        }
        acc = acc + v;
      }
    }
    const double out = S.gamma * acc;
    const double xn = ACC ? xo + out : out;
    x[d] = xn;
    if (RED) prod = rdot[d] * xn;
  }
  if (RED) {
    double rz;
    if (last_cta_total(prod, partials, &st->counter[2], &rz))
      if (threadIdx.x == 0) rz_update(st, rz);
  }
}

// Split form of phase 2 (default): the per-DOF work is partitioned so the
// singleton fast path, which does not read ybuf, runs CONCURRENTLY with the
// block solves (a second stream / graph branch), and only the DOFs with
// contribution lists wait for them.  Arithmetic per DOF is unchanged.
// Contribution list c (== complex item c: head[cdof[c]] = -(c+1)).
__device__ __forceinline__ double as_list_sum_c(const AsGather& S, int c, double rd,
                                                const double* __restrict__ ybuf) {
  const int q0 = S.cptr[c], q1 = S.cptr[c + 1];
  double acc = 0.0;
  // Batches of 8: all codes, then all values, then the ordered sum (one
  // memory round trip per batch instead of two per contribution).
  constexpr int U = 8;
  for (int qb = q0; qb < q1; qb += U) {
    int code[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) code[u] = (qb + u < q1) ? S.centry[qb + u] : 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (qb + u < q1) {
        if (code[u] < 0) {
          const double ls = S.sval[-code[u] - 1];
          v[u] = (rd / ls) / ls;
        } else {
          v[u] = ybuf[code[u]];
        }
      } else {
        v[u] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (qb + u < q1) acc = acc + v[u];
  }
  return acc;
}
__device__ __forceinline__ double as_list_sum(const AsGather& S, int d, double rd,
                                              const double* __restrict__ ybuf) {
  return as_list_sum_c(S, -S.head[d] - 1, rd, ybuf);
}

template <bool ACC>
__device__ __forceinline__ void as_simple_item(const AsGather& S, int d, const double* __restrict__ r, double* x) {
  const int h = S.head[d];
  const double rd = r[d];
  const double l = S.sdiag[d];
  const double xo = ACC ? x[d] : 0.0;
  if (h < 0) return;
  double acc = 0.0;
  acc = acc + (rd / l) / l;
  const double out = S.gamma * acc;
  x[d] = ACC ? xo + out : out;
}
template <bool ACC>
__global__ void __launch_bounds__(kCta) k_as_simple(AsGather S, const double* __restrict__ r, double* x,
                                                    const PcgState* st) {
  const int d = blockIdx.x * kCta + threadIdx.x;
  if (d >= S.n) return;
  const int h = S.head[d];  // static: before the predecessor wait
  const double l = S.sdiag[d];
  // Every thread waits, also those of multi-block DOFs: a grid in which no
  // thread waited could complete before its predecessor and break the
  // transitive PDL ordering the later kernels rely on.
  pdl_entry();
  if (h < 0) return;
  const double rd = r[d];
  const double xo = ACC ? x[d] : 0.0;
  double acc = 0.0;
  acc = acc + (rd / l) / l;
  const double out = S.gamma * acc;
  x[d] = ACC ? xo + out : out;
}
// Small levels: the block solves (groups and warp blocks, CTAs [0, nb)) and
// the singleton DOFs (CTAs nb..) in ONE kernel on the main stream, so the
// smoother is two PDL-chained kernels (this, then k_as_complex4) instead of a
// graph fork / join around three (each join is a full dependency edge).
template <bool ACC>
__global__ void IG_ASB_BOUNDS k_as_blocks_simple(AsGroups G, int32_t nb, AsGather S, const double* __restrict__ r,
                                                 double* ybuf, double* x, const PcgState* st) {
  if (static_cast<int32_t>(blockIdx.x) < nb) {
    as_blocks_item<false, RLoad, PdlWait>(G, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, threadIdx.x & 31, r,
                                          ybuf, nullptr, PdlWait{});
    return;
  }
  const int d = (blockIdx.x - nb) * blockDim.x + threadIdx.x;
  if (d >= S.n) {
    pdl_entry();
    return;
  }
  const int h = S.head[d];
  const double l = S.sdiag[d];
  pdl_entry();
  if (h < 0) return;
  const double rd = r[d];
  const double xo = ACC ? x[d] : 0.0;
  double acc = 0.0;
  acc = acc + (rd / l) / l;
  const double out = S.gamma * acc;
  x[d] = ACC ? xo + out : out;
}

template <bool ACC>
__device__ __forceinline__ void as_complex_item(const AsGather& S, int c, const double* __restrict__ r,
                                                const double* __restrict__ ybuf, double* x) {
  const int d = S.cdof[c];
  const double out = S.gamma * as_list_sum_c(S, c, r[d], ybuf);
  x[d] = ACC ? x[d] + out : out;
}
template <bool ACC>
__global__ void IG_AS_BOUNDS k_as_complex(AsGather S, const double* __restrict__ r,
                                                     const double* __restrict__ ybuf, double* x,
                                                     const PcgState* st) {
  const int c = blockIdx.x * kCta + threadIdx.x;
  if (c >= S.n_complex) return;
  // Static part of the list walk (DOF, bounds, first batch of codes and
  // singleton factors) before the predecessor wait.
  constexpr int U = 8;
  const int d = S.cdof[c];
  const int q0 = S.cptr[c], q1 = S.cptr[c + 1];
  int code[U];
  double ls[U];
#pragma unroll
  for (int u = 0; u < U; ++u) code[u] = (q0 + u < q1) ? S.centry[q0 + u] : 0;
#pragma unroll
  for (int u = 0; u < U; ++u) ls[u] = (q0 + u < q1 && code[u] < 0) ? S.sval[-code[u] - 1] : 1.0;
  pdl_entry();
  const double rd = r[d];
  const double xo = ACC ? x[d] : 0.0;  // ahead of the list sum
  double v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = (q0 + u < q1) ? (code[u] < 0 ? (rd / ls[u]) / ls[u] : ybuf[code[u]]) : 0.0;
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (q0 + u < q1) acc = acc + v[u];
  for (int qb = q0 + U; qb < q1; qb += U) {  // longer lists: as_list_sum_c's batches
    int cd[U];
    double w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cd[u] = (qb + u < q1) ? S.centry[qb + u] : 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (qb + u < q1) {
        if (cd[u] < 0) {
          const double l2 = S.sval[-cd[u] - 1];
          w[u] = (rd / l2) / l2;
        } else {
          w[u] = ybuf[cd[u]];
        }
      } else {
        w[u] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (qb + u < q1) acc = acc + w[u];
  }
  const double out = S.gamma * acc;
  x[d] = ACC ? xo + out : out;
}

// Complex DOFs on the latency-bound small levels: four lanes per DOF.  Every
// lane prefetches 8 list codes (and singleton factors) before the predecessor
// wait, so a list of up to 32 entries costs ONE dependent round trip (its
// ybuf gathers) instead of two per batch of 8; the group's lane 0 then adds
// the 32 values in list order (shuffles), the same operand sequence as
// k_as_complex.  Longer lists continue serially in lane 0.
template <bool ACC>
__global__ void IG_AS_BOUNDS k_as_complex4(AsGather S, const double* __restrict__ r,
                                           const double* __restrict__ ybuf, double* x, const PcgState* st) {
  const int t = blockIdx.x * kCta + threadIdx.x;
  const int c = t >> 2, g = t & 3;
  const int lane = threadIdx.x & 31, gbase = lane & ~3;
  const bool valid = c < S.n_complex;
  int d = 0, q0 = 0, q1 = 0;
  if (valid) {
    d = S.cdof[c];
    q0 = S.cptr[c];
    q1 = S.cptr[c + 1];
  }
  constexpr int U = 8;
  const int qb = q0 + U * g;
  int code[U];
  double ls[U];
#pragma unroll
  for (int u = 0; u < U; ++u) code[u] = (qb + u < q1) ? S.centry[qb + u] : 0;
#pragma unroll
  for (int u = 0; u < U; ++u) ls[u] = (qb + u < q1 && code[u] < 0) ? S.sval[-code[u] - 1] : 1.0;
  // Warp-uniform bound of the shuffle loop: the longest list in the warp.
  int len = q1 - q0;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
  pdl_entry();
  const double rd = valid ? r[d] : 0.0;
  const double xo = (ACC && valid && g == 0) ? x[d] : 0.0;
  double v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = (qb + u < q1) ? (code[u] < 0 ? (rd / ls[u]) / ls[u] : ybuf[code[u]]) : 0.0;
  double acc = 0.0;
  const int rounds = min(4, (len + U - 1) / U);
  for (int j = 0; j < rounds; ++j) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double w = __shfl_sync(0xffffffffu, v[u], gbase + j);
      if (g == 0 && q0 + U * j + u < q1) acc = acc + w;
    }
  }
  if (!valid || g != 0) return;
  for (int q = q0 + 4 * U; q < q1; ++q) {  // lists longer than 32 entries
    const int cd = S.centry[q];
    double w;
    if (cd < 0) {
      const double l2 = S.sval[-cd - 1];
      w = (rd / l2) / l2;
    } else {
      w = ybuf[cd];
    }
    acc = acc + w;
  }
  const double out = S.gamma * acc;
  x[d] = ACC ? xo + out : out;
}

// r . z as its own pass, for a 1-level hierarchy whose preconditioner is the
// coarse solve alone (no smoother kernel to fuse the reduction into).
__global__ void __launch_bounds__(kCta) k_pcg_rz(int32_t n, const double* __restrict__ r,
                                                 const double* __restrict__ z, PcgState* st,
                                                 double* partials) {
  pdl_entry();
  if (pcg_done(st)) return;
  double rz;
  if (chunk_reduce(n, [&](int i) { return r[i] * z[i]; }, partials, &st->counter[2], &rz))
    if (threadIdx.x == 0) rz_update(st, rz);
}

// ------------------------------------------ multiplicative Schwarz -------
// Colored multiplicative sweep (smoothers.cpp:186-208), one colour at a time:
//   k_ms_init    cur = r, xms = 0
//   per colour   k_ms_blocks: the colour's block solves on the frozen cur,
//                  delta[d] = 0 + y, xms[d] += delta[d] (disjoint DOFs);
//                k_ms_update (all colours but the last): cur_i -= sum over
//                  the colour's columns of A_ik delta_k, ascending k
//   k_ms_finish  out = gamma * xms (ACC: out += gamma * xms); RED: r . z.
// The reference's update is a full product A * delta; every column outside
// the colour holds +0 there, and adding the +-0 products leaves a running
// sum that starts at +0 unchanged (it can never be -0), so summing only the
// colour's columns in ascending order gives the same bits.  x += delta for
// DOFs outside the colour adds +0 to a value that is never -0: also a no-op.
__global__ void __launch_bounds__(kCta) k_ms_init(int32_t n, const double* __restrict__ r, double* cur,
                                                  double* xms, const PcgState* st) {
  pdl_entry();
  if (pcg_done(st)) return;
  const int i = blockIdx.x * kCta + threadIdx.x;
  if (i >= n) return;
  cur[i] = r[i];
  xms[i] = 0.0;
}
__global__ void __launch_bounds__(128) k_ms_blocks(AsGroups G, const double* __restrict__ cur, double* delta,
                                                   double* xms, const PcgState* st) {
  as_blocks_item<true, RLoad, PdlWait>(G, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, threadIdx.x & 31, cur, delta,
                                       xms, PdlWait{});
}
// S: the colour's columns of A over the rows they touch (compact row j is
// row rowmap[j] of A; entries keep A's ascending column order).
__global__ void __launch_bounds__(kCta) k_ms_update(Sell S, const int32_t* __restrict__ rowmap,
                                                    const double* __restrict__ delta, double* cur,
                                                    const PcgState* st) {
  const int j = blockIdx.x * kCta + threadIdx.x;
  if (j < S.n_rows) {  // static layout words into L1 while the predecessor finishes
    const int64_t base = S.slice_ptr[j >> 5] + (j & 31);
    asm volatile("prefetch.global.L1 [%0];" ::"l"(S.val + base));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(S.col + base));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(S.rowinfo + j));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(rowmap + j));
  }
  pdl_entry();
  if (pcg_done(st)) return;
  if (j >= S.n_rows) return;
  const double acc = sell_row<false>(S, j, delta);
  const int i = rowmap[j];
  cur[i] = cur[i] - acc;
}
template <bool ACC, bool RED>
__global__ void __launch_bounds__(kCta) k_ms_finish(int32_t n, double gamma, const double* __restrict__ xms,
                                                    double* out, const double* rdot, PcgState* st,
                                                    double* partials) {
  pdl_entry();
  if (pcg_done(st)) return;
  auto elem = [&](int i) {
    const double v = gamma * xms[i];
    const double o = ACC ? out[i] + v : v;
    out[i] = o;
    return RED ? rdot[i] * o : 0.0;
  };
  if (RED) {
    double rz;
    if (chunk_reduce(n, elem, partials, &st->counter[2], &rz))
      if (threadIdx.x == 0) rz_update(st, rz);
  } else {
    for (int i = blockIdx.x * kCta + threadIdx.x; i < n; i += gridDim.x * kCta) elem(i);
  }
}

// ------------------------------------------------------------ coarse ------
// Permuted, rank-truncated L11 L11^T solve (multigrid.cpp:77-88).
// L11 (packed lower, column-major) is staged into shared memory with TMA bulk
// copies (cp.async.bulk + mbarrier); the substitutions run pipelined across
// warps (k_coarse below).  Operation order per row is the oracle's: forward
// column-oriented, backward dot in descending k.

__device__ __forceinline__ void bulk_copy_to_smem(double* dst, const double* src, size_t bytes,
                                                  unsigned long long* mbar) {
  const unsigned int m = static_cast<unsigned int>(__cvta_generic_to_shared(mbar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(m));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(static_cast<unsigned int>(bytes)));
    const size_t kChunk = 32768;
    for (size_t off = 0; off < bytes; off += kChunk) {
      const unsigned int sz = static_cast<unsigned int>(bytes - off < kChunk ? bytes - off : kChunk);
      const unsigned int d = static_cast<unsigned int>(__cvta_generic_to_shared(reinterpret_cast<char*>(dst) + off));
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
          "l"(reinterpret_cast<const char*>(src) + off), "r"(sz), "r"(m)
          : "memory");
    }
  }
  __syncthreads();
  unsigned int done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(m)
        : "memory");
  }
}

// Pipelined multi-warp substitution: warp w owns rows 32w..32w+31 (one per
// lane).  Within a block the chain runs by shuffles; across blocks, finished
// rows are published in shared memory and later warps apply those columns
// while earlier blocks are still solving, so the critical path is
// ~rank x (div + shuffle + mul + sub) instead of rank x CTA barriers.
// Publication is the value itself: the slots start as a signalling-NaN
// sentinel that no arithmetic result can equal (IEEE operations return quiet
// NaNs), and a 64-bit shared store is single-copy atomic, so readers spin on
// the slot and no fence sits on the chain.  (A variant where every lane of
// the owning warp solves the whole block redundantly, with no shuffle on the
// chain, measured 2x slower: the 31-t updates per step are then issued by one
// warp in order ahead of the next division.)
constexpr unsigned long long kCoarseSentinel = 0x7FF4C0A45E5E0001ull;

__device__ __forceinline__ double wait_slot(const volatile double* p) {
  unsigned long long v;
  do {
    v = static_cast<unsigned long long>(__double_as_longlong(*p));
  } while (v == kCoarseSentinel);
  return __longlong_as_double(static_cast<long long>(v));
}

// The solve on one CTA (blockDim >= 32*ceil(rank/32); surplus warps only
// zero-fill).  smem: [packed L11 (SM only)][forward: rank][backward: rank].
template <bool SM, class WT = NoWait>
__device__ __forceinline__ void coarse_solve_cta(int32_t n, int32_t rank, const double* __restrict__ Lp,
                                                 const int32_t* __restrict__ piv, const double* __restrict__ r,
                                                 double* x, double* smem, WT wt = WT{}) {
  __shared__ unsigned long long mbar;
  const int64_t np = static_cast<int64_t>(rank) * (rank + 1) / 2;
  const int64_t np_al = (np + 1) & ~int64_t(1);  // 16-byte aligned region
  volatile double* yf = smem + (SM ? np_al : 0);  // forward results
  volatile double* yb = yf + rank;                 // backward results
  const double sent = __longlong_as_double(static_cast<long long>(kCoarseSentinel));
  for (int k = threadIdx.x; k < rank; k += blockDim.x) {
    yf[k] = sent;
    yb[k] = sent;
  }
  if (SM && np > 0)
    bulk_copy_to_smem(smem, Lp, static_cast<size_t>(np_al) * sizeof(double), &mbar);  // has a barrier
  else
    __syncthreads();
  wt();  // L11 is static: its staging overlaps the predecessor; r is read after the wait
  const double* L = SM ? smem : Lp;  // compile-time: LDS from shared, LDG otherwise
  // Packed column-major lower: L(i, j) = L[off(j) + i], off(j) = j*rank - j(j-1)/2 - j.
  auto off = [&](int j) { return j * rank - (j * (j - 1)) / 2 - j; };
  const int i = threadIdx.x;  // one row per thread; warp w owns rows 32w..32w+31
  const bool own = i < rank;
  const int b0 = threadIdx.x & ~31;
  if (b0 >= rank) {  // surplus warp
    for (int k = rank + threadIdx.x; k < n; k += blockDim.x) x[piv[k] - 1] = 0.0;
    return;
  }
  const int bend = min(b0 + 32, rank);
  const int oi = own ? off(i) : 0;
  double y = own ? r[piv[i] - 1] : 0.0;
  const double dg = own ? L[oi + i] : 1.0;  // own pivot L(i, i)
  const double rdg = safe_rcp(dg);
  // Fast path (every pivot of the warp has a usable reciprocal): branch-free
  // steps -- every lane forms the quotient, the shuffle picks the owner's,
  // selects keep each lane's own operation sequence exactly the oracle's.
  const bool fast = __all_sync(0xffffffffu, !own || (isfinite(rdg) && rdg != 0.0));
  // ---- forward: y_j = y_j / L_jj ; y_i -= L_ij y_j (i > j), j ascending ----
  // Columns of earlier blocks: consumed as their owners publish them.
  int oj = 0;  // off(j)
  for (int j = 0; j < b0; ++j) {
    const double yj = wait_slot(yf + j);
    if (own) y = y - L[oj + i] * yj;
    oj += rank - j - 1;
  }
  // Own block: the owner of row j divides and hands y_j to the warp by
  // shuffle; the shared-memory publication for later warps is off the chain.
  if (fast) {
    for (int j = b0; j < bend; ++j) {
      const double q = exact_div(y, dg, rdg);
      const double yj = __shfl_sync(0xffffffffu, q, j - b0);
      const double lij = L[oj + (own ? i : j)];
      const double upd = y - lij * yj;
      y = (i == j) ? yj : ((own && i > j) ? upd : y);
      if (i == j) yf[j] = yj;
      oj += rank - j - 1;
    }
  } else {
    for (int j = b0; j < bend; ++j) {
      if (i == j) y = div_rb(y, dg, rdg);
      const double yj = __shfl_sync(0xffffffffu, y, j - b0);
      if (i == j) yf[j] = yj;
      if (own && i > j) y = y - L[oj + i] * yj;
      oj += rank - j - 1;
    }
  }
  // ---- backward: y_i = (y_i - sum_{k desc > i} L_ki y_k) / L_ii ----------
  double acc = 0.0;
  for (int k = rank - 1; k >= bend; --k) {
    const double yk = wait_slot(yb + k);
    if (own) acc = acc + L[oi + k] * yk;
  }
  if (fast) {
    for (int k = bend - 1; k >= b0; --k) {
      const double q = exact_div(y - acc, dg, rdg);
      const double yk = __shfl_sync(0xffffffffu, q, k - b0);
      const double nacc = acc + L[oi + k] * yk;
      if (i == k) {
        y = yk;
        yb[k] = yk;
      }
      acc = (own && i < k) ? nacc : acc;
    }
  } else {
    for (int k = bend - 1; k >= b0; --k) {
      if (i == k) y = div_rb(y - acc, dg, rdg);
      const double yk = __shfl_sync(0xffffffffu, y, k - b0);
      if (i == k) yb[k] = yk;
      if (own && i < k) acc = acc + L[oi + k] * yk;
    }
  }
  if (own) x[piv[i] - 1] = y;
  for (int k = rank + threadIdx.x; k < n; k += blockDim.x) x[piv[k] - 1] = 0.0;
}

// Single-warp solve for ranks up to 32 R (R rows per lane: row i = lane +
// 32 t).  Every step keeps the pivot chain inside one warp -- the owner lane
// divides, one shuffle hands y_j to all lanes, each lane applies it to its R
// rows -- so there is no cross-warp publication or spinning on the chain
// (the multi-warp pipeline below pays ~2.3x the in-warp step for its
// handoffs: rank 216, 51 us vs ~20 us).  Same operation order per row as the
// oracle: forward column-oriented (ascending j), backward dot accumulated in
// descending k, one (exact) division per pivot.
template <int R, bool SM>
__global__ void __launch_bounds__(32, 1) k_coarse_warp(int32_t n, int32_t rank, const double* __restrict__ Lp,
                                                     const int32_t* __restrict__ piv,
                                                     const double* __restrict__ r, double* x,
                                                     const PcgState* st) {
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned long long mbar;
  const int64_t np = static_cast<int64_t>(rank) * (rank + 1) / 2;
  const int64_t np_al = (np + 1) & ~int64_t(1);
  if (SM && np > 0) bulk_copy_to_smem(smem, Lp, static_cast<size_t>(np_al) * sizeof(double), &mbar);
  const double* L = SM ? smem : Lp;
  const int lane = threadIdx.x;
  auto off = [&](int j) { return j * rank - (j * (j - 1)) / 2 - j; };  // packed column-major lower
  double y[R], acc[R], dg[R], rdg[R];
  int oi[R], pv[R];
  bool ok = true;
#pragma unroll
  for (int t = 0; t < R; ++t) {
    const int i = lane + 32 * t;
    const bool own = i < rank;
    oi[t] = own ? off(i) : 0;
    pv[t] = own ? piv[i] - 1 : 0;
    dg[t] = own ? L[oi[t] + i] : 1.0;
    rdg[t] = safe_rcp(dg[t]);
    ok = ok && (!own || (isfinite(rdg[t]) && rdg[t] != 0.0));
    acc[t] = 0.0;
  }
  const bool fast = __all_sync(0xffffffffu, ok);
  pdl_entry();  // L11, pivots and diagonals are static: staged before the predecessor wait
#pragma unroll
  for (int t = 0; t < R; ++t) y[t] = (lane + 32 * t < rank) ? r[pv[t]] : 0.0;
  // ---- forward: y_j = y_j / L_jj ; y_i -= L_ij y_j (i > j), j ascending ----
#pragma unroll
  for (int tb = 0; tb < R; ++tb) {
    const int jend = min(32, rank - 32 * tb);
    for (int jj = 0; jj < jend; ++jj) {
      const int j = 32 * tb + jj;
      const int oj = off(j);
      const double q = fast ? exact_div(y[tb], dg[tb], rdg[tb]) : y[tb] / dg[tb];
      const double yj = __shfl_sync(0xffffffffu, q, jj);
      if (lane == jj) y[tb] = yj;
#pragma unroll
      for (int t = tb; t < R; ++t) {
        const int i = lane + 32 * t;
        if ((t > tb || lane > jj) && i < rank) y[t] = y[t] - L[oj + i] * yj;
      }
    }
  }
  // ---- backward: y_i = (y_i - sum_{k desc > i} L_ki y_k) / L_ii -----------
#pragma unroll
  for (int tb = R - 1; tb >= 0; --tb) {
    const int kend = min(32, rank - 32 * tb);
    for (int kk = kend - 1; kk >= 0; --kk) {
      const int k = 32 * tb + kk;
      const double u = y[tb] - acc[tb];
      const double q = fast ? exact_div(u, dg[tb], rdg[tb]) : u / dg[tb];
      const double yk = __shfl_sync(0xffffffffu, q, kk);
      if (lane == kk) y[tb] = yk;
#pragma unroll
      for (int t = 0; t <= tb; ++t)
        if (t < tb || lane < kk) acc[t] = acc[t] + L[oi[t] + k] * yk;
    }
  }
#pragma unroll
  for (int t = 0; t < R; ++t)
    if (lane + 32 * t < rank) x[pv[t]] = y[t];
  for (int k = rank + lane; k < n; k += 32) x[piv[k] - 1] = 0.0;
}

// Tolerance-mode coarse solve (ig_gpu.cu Opts::fast_coarse): x[piv_i] =
// sum_j M_ij r[piv_j] for i < rank (FMA, lane-split, xor-tree), 0 beyond the
// rank.  One warp per row; rows of M are contiguous, so loads coalesce.
__global__ void __launch_bounds__(256) k_coarse_gemv(int32_t n, int32_t rank, const double* __restrict__ M,
                                                     const int32_t* __restrict__ piv, const double* __restrict__ r,
                                                     double* x, const PcgState* st) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  pdl_entry();
  if (row >= n) return;
  if (row >= rank) {
    if (lane == 0) x[piv[row] - 1] = 0.0;
    return;
  }
  const double* m = M + static_cast<int64_t>(row) * rank;
  double acc = 0.0;
  for (int j = lane; j < rank; j += 32) acc = __fma_rn(__ldg(m + j), r[piv[j] - 1], acc);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) x[piv[row] - 1] = acc;
}

// BIG: ranks above 256 (up to 1024 threads).
template <bool SM, bool BIG = false>
__global__ void __launch_bounds__(BIG ? 1024 : 256, 1) k_coarse(int32_t n, int32_t rank, const double* __restrict__ Lp,
                                                               const int32_t* __restrict__ piv,
                                                               const double* __restrict__ r, double* x,
                                                               const PcgState* st) {
  extern __shared__ __align__(16) double smem[];
  coarse_solve_cta<SM, PdlWait>(n, rank, Lp, piv, r, x, smem, PdlWait{});
}

// ---------------------------------------------------------- PCG vectors ---

// x = 0, r = b, bnorm from the canonical reduction (solvers.cpp:24-39).
// Sets the graph conditions (handles != 0) to "keep going": c_if guards the
// first V-cycle, c_loop the WHILE node.
__device__ __forceinline__ void set_conds(cudaGraphConditionalHandle c_if, cudaGraphConditionalHandle c_loop,
                                          bool go) {
  if (c_if != 0) cudaGraphSetConditional(c_if, go ? 1u : 0u);
  if (c_loop != 0) cudaGraphSetConditional(c_loop, go ? 1u : 0u);
}

__global__ void __launch_bounds__(kCta) k_pcg_init(int32_t n, double* r, PcgState* st, double* partials,
                                                   cudaGraphConditionalHandle c_if,
                                                   cudaGraphConditionalHandle c_loop) {
  pdl_wait_only();
  double bb;
  const bool last = chunk_reduce(n, [&](int i) {
    const double bi = st->b[i];
    st->x[i] = 0.0;
    r[i] = bi;
    return bi * bi;
  }, partials, &st->counter[3], &bb);
  if (last) {
    if (threadIdx.x == 0) {
      const double bn = sqrt(bb);
      st->bnorm = bn;
      st->k = -1;
      if (bn == 0.0) {
        st->residuals[0] = 0.0;
        st->status = ST_OK;
        st->done = 1;
      } else {
        st->residuals[0] = 1.0;
        if (1.0 <= st->tol) {
          st->status = ST_OK;
          st->done = 1;
        }
      }
      set_conds(c_if, c_loop, st->done == 0);
    }
  }
}

// x += alpha p; r -= alpha Ap; rel = ||r|| / ||b|| (solvers.cpp:51-61).
// The last CTA also sets the graph conditions: c_if guards this iteration's
// V-cycle + p update, c_loop the WHILE node.
__global__ void __launch_bounds__(kCta) k_pcg_update(int32_t n, const double* __restrict__ p,
                                                     const double* __restrict__ ap, double* r,
                                                     PcgState* st, double* partials,
                                                     cudaGraphConditionalHandle c_if,
                                                     cudaGraphConditionalHandle c_loop) {
  pdl_wait_only();
  if (pcg_stopped(st)) {  // breakdown in the preceding SpMV: x, r stay
    if (blockIdx.x == 0 && threadIdx.x == 0) set_conds(c_if, c_loop, false);
    return;
  }
  const double alpha = st->alpha;
  double* x = st->x;
  double rr;
  const bool last = chunk_reduce(n, [&](int i) {
    x[i] = x[i] + alpha * p[i];
    const double ri = r[i] - alpha * ap[i];
    r[i] = ri;
    return ri * ri;
  }, partials, &st->counter[1], &rr);
  if (last) {
    if (threadIdx.x == 0) {
      const int k = st->k;
      const double rel = sqrt(rr) / st->bnorm;
      st->residuals[k + 1] = rel;
      st->k = k + 1;
      if (rel <= st->tol) {
        st->status = ST_OK;
        st->done = 1;
      } else if (k + 1 >= st->maxit) {
        st->status = ST_NOT_CONVERGED;
        st->done = 1;
      }
      set_conds(c_if, c_loop, st->done == 0);
    }
  }
}

// ------------------------------------------------------------ Richardson --
// richardson (solvers.cpp:73-120): x = 0, r = b; at every k the relative
// residual is recorded, a growth streak counted, then tol, streak >= 10
// (Diverged) and k == maxit are tested in that order; otherwise
// dx = M r, x += dx, r -= A dx.
// Init: x = 0, r = b, ||b|| (canonical reduction), the k = 0 test.
__global__ void __launch_bounds__(kCta) k_rich_init(int32_t n, double* r, PcgState* st, double* partials,
                                                    cudaGraphConditionalHandle c_loop) {
  pdl_wait_only();
  double bb;
  const bool last = chunk_reduce(n, [&](int i) {
    const double bi = st->b[i];
    st->x[i] = 0.0;
    r[i] = bi;
    return bi * bi;
  }, partials, &st->counter[3], &bb);
  if (last) {
    if (threadIdx.x == 0) {
      const double bn = sqrt(bb);
      st->bnorm = bn;
      st->k = 0;
      st->streak = 0;
      if (bn == 0.0) {
        st->residuals[0] = 0.0;
        st->status = ST_OK;
        st->done = 1;
      } else {
        const double rel = sqrt(bb) / bn;  // r == b: the reference's r.norm() / bnorm
        st->residuals[0] = rel;
        if (rel <= st->tol) {
          st->status = ST_OK;
          st->done = 1;
        } else if (st->maxit <= 0) {
          st->status = ST_NOT_CONVERGED;
          st->done = 1;
        }
      }
      if (c_loop != 0) cudaGraphSetConditional(c_loop, st->done == 0 ? 1u : 0u);
    }
  }
}
// After dx = M r (in z) and r -= A dx: x += dx, ||r|| -> residual, the tests.
__global__ void __launch_bounds__(kCta) k_rich_step(int32_t n, const double* __restrict__ z,
                                                    const double* __restrict__ r, PcgState* st, double* partials,
                                                    cudaGraphConditionalHandle c_loop) {
  pdl_wait_only();
  double* x = st->x;
  double rr;
  const bool last = chunk_reduce(n, [&](int i) {
    x[i] = x[i] + z[i];
    const double ri = r[i];
    return ri * ri;
  }, partials, &st->counter[1], &rr);
  if (last) {
    if (threadIdx.x == 0) {
      const int k = st->k + 1;
      const double rel = sqrt(rr) / st->bnorm;
      st->residuals[k] = rel;
      st->k = k;
      st->streak = rel > st->residuals[k - 1] ? st->streak + 1 : 0;
      if (rel <= st->tol) {
        st->status = ST_OK;
        st->done = 1;
      } else if (st->streak >= 10) {
        st->status = ST_DIVERGED;
        st->done = 1;
      } else if (k >= st->maxit) {
        st->status = ST_NOT_CONVERGED;
        st->done = 1;
      }
      if (c_loop != 0) cudaGraphSetConditional(c_loop, st->done == 0 ? 1u : 0u);
    }
  }
}

// p = z (first) or p = z + beta p (solvers.cpp:42, :64).
template <bool FIRST>
__global__ void __launch_bounds__(kCta) k_pcg_p(int32_t n, const double* __restrict__ z, double* p,
                                                const PcgState* st) {
  pdl_entry();
  const int i = blockIdx.x * kCta + threadIdx.x;
  if (i >= n) return;
  if (FIRST)
    p[i] = z[i];
  else
    p[i] = z[i] + st->beta * p[i];
}

}  // namespace igk
