// spmv_psell.cuh — pattern-SELL: the SpMV layout of the large levels.
//
// Why: the row-dictionary SELL (kernels.cuh: Sell) removed most value bytes
// but the finest C4 SpMV stayed at ~300 us, 57 % issue-busy at 26 SASS
// instructions per matrix slot (per-lane selects between dictionary and
// explicit streams, predicated batches) with 4 B of column index per slot
// still streamed for 56 % of the rows.  The operators of an immersed
// B-spline discretisation are far more regular than that: 61 % of the 32-row
// slices of C4's finest level have ONE value sequence, ONE column-offset
// sequence (col - row) and one length for all 32 rows, and most of the rest
// have a handful of distinct offset sequences (slices crossing an x-line end).
//
// Layout, per slice of 32 consecutive rows (one warp):
//   * FAST slices (all rows: same length, same values, same offsets): the warp
//     reads one value sequence V[vbase + k] and one offset sequence
//     O[obase + k] with warp-uniform addresses (one L1 wavefront each, the
//     sequences deduplicated across the matrix, the most frequent value
//     sequences shared through the global dictionary at the start of V), and
//     gathers x[row + o_k] coalesced: 6 instructions per slot, no predication;
//   * general slices: per-slice column-major tables of the DISTINCT offset
//     sequences (width wo) and of the distinct non-dictionary value sequences
//     (width wv); rowinfo[row] selects the row's columns and its value source
//     (dictionary entry or table column).  Table entries past a row's length
//     are zero (offset 0 keeps the gather in bounds; the product is never
//     added).
// The sum is the same serial ascending-k chain as every other SpMV here
// (Eigen RowMajor order), and values/offsets are stored bit-exactly, so the
// results are identical to kernels.cuh's k_spmv and to the oracle.
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace igk {

constexpr uint32_t kPFast = 1u;  // slice: one length/value/offset sequence for all rows
constexpr uint32_t kPUlen = 2u;  // slice: all 32 rows have length lmax

struct PSliceMeta {
  uint32_t vbase;  // FAST: start of the value sequence; general: value table
  uint32_t obase;  // FAST: start of the offset sequence; general: offset table
  uint16_t lmax;
  uint8_t wv, wo;  // general: table widths (column-major strides)
  uint32_t flags;
};

// rowinfo (general slices): len | vsel << 11 | vi << 17 | oi << 22;
// vsel > 0: values = dictionary entry vsel-1 (V[(vsel-1)*dict_w + k]),
// vsel = 0: values = table column vi.  oi: offset-table column.
constexpr int kPLenBits = 11;
constexpr int kPMaxLen = (1 << kPLenBits) - 1;
constexpr int kPMaxDict = 63;

struct PSell {
  int32_t n_rows, n_cols;
  const PSliceMeta* meta;
  const uint32_t* rowinfo;
  const double* V;
  const int32_t* O;
  int32_t dict_w;
};

__device__ __forceinline__ PSliceMeta load_meta(const PSliceMeta* p) {
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  PSliceMeta m;
  m.vbase = u.x;
  m.obase = u.y;
  m.lmax = static_cast<uint16_t>(u.z & 0xffffu);
  m.wv = static_cast<uint8_t>((u.z >> 16) & 0xffu);
  m.wo = static_cast<uint8_t>(u.z >> 24);
  m.flags = u.w;
  return m;
}

template <bool STREAM>
__device__ __forceinline__ int32_t ld_off(const int32_t* p) {
  if (STREAM) return __ldcs(p);
  return __ldg(p);
}

// Row sum of one row of a pattern-SELL matrix (warp = slice; `row` < n_rows
// for every lane that calls it with a valid row, others pass valid=false and
// still follow the warp-uniform branches).
template <bool STREAM>
__device__ __forceinline__ double psell_row(const PSell& A, int row, bool valid, const double* __restrict__ x) {
  const PSliceMeta m = load_meta(A.meta + (row >> 5));
  const double* xr = x + row;
  double acc = 0.0;
  constexpr int U = 8;
  if (m.flags & kPFast) {  // warp-uniform branch
    const double* vp = A.V + m.vbase;
    const int32_t* op = A.O + m.obase;
    const int L = m.lmax;
    int k = 0;
    for (; k + U <= L; k += U) {
      double v[U], xv[U];
      int32_t o[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        v[u] = __ldg(vp + k + u);
        o[u] = __ldg(op + k + u);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = __ldg(xr + o[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) acc = acc + v[u] * xv[u];
    }
    for (; k < L; ++k) acc = acc + __ldg(vp + k) * __ldg(xr + __ldg(op + k));
    return acc;
  }
  const uint32_t info = valid ? __ldg(A.rowinfo + row) : 0u;
  const int len = static_cast<int>(info & kPMaxLen);
  const int vsel = static_cast<int>((info >> 11) & 0x3f);
  const int vi = static_cast<int>((info >> 17) & 0x1f);
  const int oi = static_cast<int>((info >> 22) & 0x1f);
  const double* vp = vsel ? A.V + static_cast<int64_t>(vsel - 1) * A.dict_w : A.V + m.vbase + vi;
  const int vs = vsel ? 1 : m.wv;
  const int32_t* op = A.O + m.obase + oi;
  const int os = m.wo;
  const int L = m.lmax;
  // Out-of-range lanes of the last slice read table column 0 (the slice's
  // first row): relative to that row, the discarded gathers stay in bounds.
  if (!valid) xr = x + (row & ~31);
  if (m.flags & kPUlen) {  // warp-uniform branch: every row has length L
    int k = 0;
    for (; k + U <= L; k += U) {
      double v[U], xv[U];
      int32_t o[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        v[u] = __ldg(vp + (k + u) * vs);
        o[u] = ld_off<STREAM>(op + (k + u) * os);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = __ldg(xr + o[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) acc = acc + v[u] * xv[u];
    }
    for (; k < L; ++k) acc = acc + __ldg(vp + k * vs) * __ldg(xr + ld_off<STREAM>(op + k * os));
    return acc;
  }
  // Mixed lengths: run to the slice maximum, add only k < len.  Entries past
  // len are zero in the tables; dictionary rows past their length read the
  // zero padding after the dictionary (V is padded by the host).
  int k = 0;
  for (; k + U <= L; k += U) {
    double v[U], xv[U];
    int32_t o[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = __ldg(vp + (k + u) * vs);
      o[u] = ld_off<STREAM>(op + (k + u) * os);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = __ldg(xr + o[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double t = acc + v[u] * xv[u];
      acc = (k + u < len) ? t : acc;
    }
  }
  for (; k < L; ++k) {
    const double t = acc + __ldg(vp + k * vs) * __ldg(xr + ld_off<STREAM>(op + k * os));
    acc = (k < len) ? t : acc;
  }
  return acc;
}

// MODE 0: y = A x.  MODE 1: y = r - A x (r read from rsrc; in place allowed).
// RED: p . Ap chunk partials, last CTA -> alpha / Breakdown (as k_spmv).
template <int MODE, bool STREAM, bool RED>
__global__ void __launch_bounds__(kCta) k_pspmv(PSell A, const double* __restrict__ x, double* y,
                                               const double* rsrc, PcgState* st, double* partials) {
  if (pcg_done(st)) return;
  const int row = blockIdx.x * kCta + threadIdx.x;
  const bool valid = row < A.n_rows;
  double prod = 0.0;
  const double acc = psell_row<STREAM>(A, row, valid, x);
  if (valid) {
    const double out = (MODE == 0) ? acc : rsrc[row] - acc;
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

// Prolongation fused with the correction (k_prolong on the pattern layout).
template <bool STREAM>
__global__ void __launch_bounds__(kCta) k_pprolong(PSell P, const double* __restrict__ xc, double* cor, double* x,
                                                  const PcgState* st) {
  if (pcg_done(st)) return;
  const int row = blockIdx.x * kCta + threadIdx.x;
  const bool valid = row < P.n_rows;
  const double c = psell_row<STREAM>(P, row, valid, xc);
  if (!valid) return;
  cor[row] = c;
  x[row] = x[row] + c;
}

}  // namespace igk
