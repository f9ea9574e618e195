// galerkin.cuh — device-side Galerkin coarse operators A_c = R (A R^T)
// (MgHierarchy::build, proj/src/multigrid.cpp:37-41: `SpMat rt = r.transpose();
// SpMat coarse_a = r * (down.back().A * rt);`), SURVEY.md §8(f) row 2.
//
// Result contract: bit-identical to the host restatement of Eigen's sparse
// product (paper_1903_10977_b200/host/spline_linalg.cpp spgemm): entry (i, j)
// of C = A B is the sum over the nonzeros k of row i of A, in ASCENDING k,
// of a_ik * b_kj, the first product assigned (not added to 0), rows sorted by
// column.  Every product and every partial sum is formed by one thread in
// exactly that order, so the bits cannot depend on scheduling.
//
// Shape: one warp per output row, a per-warp open-addressing hash table in
// shared memory (HS slots: column keys + values).  The warp walks row i of A
// in ascending k; for each k its lanes take the entries of row k of B (distinct
// columns, so no two lanes touch one slot's value in the same step; slot
// claiming is an atomicCAS on the key, whose order only decides WHERE a column
// lives, never its sum).  Two passes: symbolic (count distinct columns per
// row), exclusive scan (host side: CUB), numeric (accumulate, compact, rank
// sort by column, write).  Rows whose distinct count exceeds the table's load
// limit are reported to the host, which fails loudly (no such row in any
// immersed B-spline / THB hierarchy here: at most a 7^d coarse stencil).
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace igk {

constexpr int kGalHS = 1024;     // hash slots per warp (power of two)
constexpr int kGalLoad = 768;    // maximum distinct columns per row
constexpr int kGalWarps = 4;     // warps (rows) per CTA
constexpr uint32_t kGalEmpty = 0xffffffffu;

struct GalCsr {
  int32_t n_rows, n_cols;
  const int32_t* ptr;
  const int32_t* col;
  const double* val;
};

__device__ __forceinline__ uint32_t gal_hash(uint32_t j) { return (j * 2654435761u) >> (32 - 10); }

// Insert column j; returns the slot (fresh: newly claimed), or -1 when the
// table is full (at most kGalHS probes: never spins).
__device__ __forceinline__ int gal_insert(uint32_t* keys, uint32_t j, bool& fresh) {
  uint32_t s = gal_hash(j);
  fresh = false;
  for (int probe = 0; probe < kGalHS; ++probe) {
    const uint32_t k = *reinterpret_cast<volatile uint32_t*>(&keys[s]);
    if (k == j) return static_cast<int>(s);
    if (k == kGalEmpty) {
      const uint32_t prev = atomicCAS(&keys[s], kGalEmpty, j);
      if (prev == kGalEmpty) {
        fresh = true;
        return static_cast<int>(s);
      }
      if (prev == j) return static_cast<int>(s);
    }
    s = (s + 1) & (kGalHS - 1);
  }
  return -1;
}

// Pass 1: distinct columns of every row of C = A B (kGalLoad + 1 = too many).
__global__ void __launch_bounds__(32 * kGalWarps) k_gal_count(GalCsr A, GalCsr B, int32_t* cnt) {
  extern __shared__ uint32_t gsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* keys = gsm + w * kGalHS;
  const int row = blockIdx.x * kGalWarps + w;
  if (row >= A.n_rows) return;
  for (int s = lane; s < kGalHS; s += 32) keys[s] = kGalEmpty;
  __syncwarp();
  int n = 0;
  bool full = false;
  for (int32_t t = A.ptr[row]; t < A.ptr[row + 1]; ++t) {
    const int32_t k = A.col[t];
    for (int32_t q = B.ptr[k] + lane; q < B.ptr[k + 1]; q += 32) {
      bool fresh;
      full |= gal_insert(keys, static_cast<uint32_t>(B.col[q]), fresh) < 0;
      n += fresh ? 1 : 0;
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  full = __any_sync(0xffffffffu, full);
  if (lane == 0) cnt[row] = (full || n > kGalLoad) ? kGalLoad + 1 : n;
}

// Pass 2: values.  cptr = exclusive scan of the counts (n_rows + 1 entries).
__global__ void __launch_bounds__(32 * kGalWarps) k_gal_fill(GalCsr A, GalCsr B, const int64_t* cptr,
                                                            int32_t* ccol, double* cval) {
  extern __shared__ uint32_t gsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* keys = gsm + w * kGalHS;
  double* vals = reinterpret_cast<double*>(gsm + kGalWarps * kGalHS) + w * kGalHS;
  // Compacted (column, value) pairs reuse the front of the value table's
  // shadow: ck / cv below live past all tables.
  uint32_t* ck = gsm + kGalWarps * kGalHS * 3 + w * kGalLoad;
  double* cv = reinterpret_cast<double*>(gsm + kGalWarps * kGalHS * 3 + kGalWarps * kGalLoad) + w * kGalLoad;
  const int row = blockIdx.x * kGalWarps + w;
  if (row >= A.n_rows) return;
  for (int s = lane; s < kGalHS; s += 32) keys[s] = kGalEmpty;
  __syncwarp();
  for (int32_t t = A.ptr[row]; t < A.ptr[row + 1]; ++t) {
    const int32_t k = A.col[t];
    const double av = A.val[t];
    for (int32_t q = B.ptr[k] + lane; q < B.ptr[k + 1]; q += 32) {
      bool fresh;
      const int s = gal_insert(keys, static_cast<uint32_t>(B.col[q]), fresh);  // >= 0: count pass bounded the row
      const double prod = av * B.val[q];
      vals[s] = fresh ? prod : vals[s] + prod;  // spline_linalg.cpp spgemm: first product assigned
    }
    __syncwarp();  // step k complete before step k' > k touches the same slots
  }
  // Compact the used slots (slot order), then rank-sort by column.
  int base = 0;
  for (int s0 = 0; s0 < kGalHS; s0 += 32) {
    const uint32_t k = keys[s0 + lane];
    const bool used = k != kGalEmpty;
    const unsigned m = __ballot_sync(0xffffffffu, used);
    if (used) {
      const int pos = base + __popc(m & ((1u << lane) - 1u));
      ck[pos] = k;
      cv[pos] = vals[s0 + lane];
    }
    base += __popc(m);
  }
  __syncwarp();
  const int n = base;
  const int64_t o = cptr[row];
  for (int e = lane; e < n; e += 32) {
    const uint32_t key = ck[e];
    int rank = 0;
    for (int f = 0; f < n; ++f) rank += ck[f] < key ? 1 : 0;
    ccol[o + rank] = static_cast<int32_t>(key);
    cval[o + rank] = cv[e];
  }
}

// Short-B-row variant (every row of B has <= 32 entries: B = R^T in A R^T,
// a fine DOF's coarse parents).  The warp first loads 32 entries of row i of
// A and their B-row bounds in parallel (one lane each), then walks them in
// ascending order with B row t+1's columns / values already in flight while
// row t is inserted -- the per-step chain is the shared-memory insert only,
// not three dependent global loads.  Same per-entry order (k ascending,
// first product assigned): same bits as k_gal_fill / k_gal_count.
template <bool FILL>
__global__ void __launch_bounds__(32 * kGalWarps) k_gal_short(GalCsr A, GalCsr B, int32_t* cnt, const int64_t* cptr,
                                                             int32_t* ccol, double* cval) {
  extern __shared__ uint32_t gsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* keys = gsm + w * kGalHS;
  double* vals = reinterpret_cast<double*>(gsm + kGalWarps * kGalHS) + w * kGalHS;
  uint32_t* ck = gsm + kGalWarps * kGalHS * 3 + w * kGalLoad;
  double* cv = reinterpret_cast<double*>(gsm + kGalWarps * kGalHS * 3 + kGalWarps * kGalLoad) + w * kGalLoad;
  const int row = blockIdx.x * kGalWarps + w;
  if (row >= A.n_rows) return;
  for (int s = lane; s < kGalHS; s += 32) keys[s] = kGalEmpty;
  __syncwarp();
  const int32_t a0 = A.ptr[row], a1 = A.ptr[row + 1];
  int n = 0;
  bool full = false;
  for (int32_t c0 = a0; c0 < a1; c0 += 32) {
    const int32_t t = c0 + lane;
    const int32_t k = t < a1 ? A.col[t] : 0;
    const double av = (FILL && t < a1) ? A.val[t] : 0.0;
    const int32_t q0 = t < a1 ? B.ptr[k] : 0;
    const int32_t q1 = t < a1 ? B.ptr[k + 1] : 0;
    const int steps = min(32, a1 - c0);
    // Step j's B entries, one per lane: prefetched one step ahead.
    int32_t nb0 = __shfl_sync(0xffffffffu, q0, 0), ne0 = __shfl_sync(0xffffffffu, q1, 0);
    int32_t bc = nb0 + lane < ne0 ? B.col[nb0 + lane] : 0;
    double bv = (FILL && nb0 + lane < ne0) ? B.val[nb0 + lane] : 0.0;
    for (int j = 0; j < steps; ++j) {
      const int32_t b0 = nb0, b1 = ne0;
      const int32_t cc = bc;
      const double cvv = bv;
      const double a = __shfl_sync(0xffffffffu, av, j);
      if (j + 1 < steps) {
        nb0 = __shfl_sync(0xffffffffu, q0, j + 1);
        ne0 = __shfl_sync(0xffffffffu, q1, j + 1);
        bc = nb0 + lane < ne0 ? B.col[nb0 + lane] : 0;
        if (FILL) bv = nb0 + lane < ne0 ? B.val[nb0 + lane] : 0.0;
      }
      if (b0 + lane < b1) {
        bool fresh;
        const int s = gal_insert(keys, static_cast<uint32_t>(cc), fresh);
        if (s < 0) {
          full = true;
        } else {
          n += fresh ? 1 : 0;
          if (FILL) {
            const double prod = a * cvv;
            vals[s] = fresh ? prod : vals[s] + prod;
          }
        }
      }
      __syncwarp();
    }
  }
  if (!FILL) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    full = __any_sync(0xffffffffu, full);
    if (lane == 0) cnt[row] = (full || n > kGalLoad) ? kGalLoad + 1 : n;
    return;
  }
  int base = 0;
  for (int s0 = 0; s0 < kGalHS; s0 += 32) {
    const uint32_t kk = keys[s0 + lane];
    const bool used = kk != kGalEmpty;
    const unsigned m = __ballot_sync(0xffffffffu, used);
    if (used) {
      const int pos = base + __popc(m & ((1u << lane) - 1u));
      ck[pos] = kk;
      cv[pos] = vals[s0 + lane];
    }
    base += __popc(m);
  }
  __syncwarp();
  const int64_t o = cptr[row];
  for (int e = lane; e < base; e += 32) {
    const uint32_t key = ck[e];
    int rank = 0;
    for (int f = 0; f < base; ++f) rank += ck[f] < key ? 1 : 0;
    ccol[o + rank] = static_cast<int32_t>(key);
    cval[o + rank] = cv[e];
  }
}

constexpr size_t kGalFillSmem =
    static_cast<size_t>(kGalWarps) * (kGalHS * (4 + 8) + kGalLoad * (4 + 8));
constexpr size_t kGalCountSmem = static_cast<size_t>(kGalWarps) * kGalHS * 4;

// Transpose with the host transpose's entry order (rows of M visited
// ascending, so each row of T lists its source rows ascending): column counts
// and scatter use integer atomics (positions within a row of T arbitrary),
// then each row of T is sorted by its unique source-row index, which restores
// exactly that order.
// Pass 1 (k_tr_count): column counts.
__global__ void k_tr_count(GalCsr M, int32_t* ccount) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M.n_rows) return;
  for (int32_t t = M.ptr[i]; t < M.ptr[i + 1]; ++t) atomicAdd(&ccount[M.col[t]], 1);
}
// Pass 2: scatter with an atomic cursor (positions arbitrary within a row of T) ...
__global__ void k_tr_scatter(GalCsr M, const int64_t* tptr, int32_t* cursor, int32_t* tcol, double* tval) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M.n_rows) return;
  for (int32_t t = M.ptr[i]; t < M.ptr[i + 1]; ++t) {
    const int32_t c = M.col[t];
    const int64_t p = tptr[c] + atomicAdd(&cursor[c], 1);
    tcol[p] = i;
    tval[p] = M.val[t];
  }
}
// ... pass 3: sort each row of T by its (unique) source-row index, which
// restores exactly the ascending-i order (one thread per row of T; rows of a
// restriction's transpose are short).
__global__ void k_tr_sort(int32_t n, const int64_t* tptr, int32_t* tcol, double* tval) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t a = tptr[r], b = tptr[r + 1];
  for (int64_t p = a + 1; p < b; ++p) {  // insertion sort
    const int32_t c = tcol[p];
    const double v = tval[p];
    int64_t q = p - 1;
    while (q >= a && tcol[q] > c) {
      tcol[q + 1] = tcol[q];
      tval[q + 1] = tval[q];
      --q;
    }
    tcol[q + 1] = c;
    tval[q + 1] = v;
  }
}

// Exclusive scan of n int32 counts into int64 offsets (n + 1 entries), one
// CTA of 1024 threads: thread t owns a contiguous chunk; chunk totals are
// scanned in shared memory.  Setup-time only (a few 10 us at 2M rows).
__global__ void __launch_bounds__(1024) k_scan_counts(int32_t n, const int32_t* __restrict__ cnt, int64_t* out) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t chunk = (static_cast<int64_t>(n) + 1023) / 1024;
  const int64_t a = min(static_cast<int64_t>(n), t * chunk), b = min(static_cast<int64_t>(n), a + chunk);
  int64_t s = 0;
  for (int64_t i = a; i < b; ++i) s += cnt[i];
  part[t] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // Hillis-Steele inclusive scan
    const int64_t v = t >= off ? part[t - off] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = part[t] - s;  // exclusive prefix of this chunk
  for (int64_t i = a; i < b; ++i) {
    out[i] = run;
    run += cnt[i];
  }
  if (t == 1023) out[n] = part[1023];
}

}  // namespace igk
