// assemble.cuh — the global assembly on the device:
// the reference's assemble() after the element loop (proj/src/assembly.cpp:
// 164-180): triplets (i, j, K_e[li][lj]) of every element summed by
// setFromTriplets, then A = 0.5 (A + A^T); b_i = sum of F_e[li].
//
// Result contract: bit-identical to the host row gather
// (paper_1903_10977_b200/host/assembly.cpp): every entry starts from its first
// nonzero element contribution and adds the others in ascending element order
// (the order setFromTriplets meets the duplicates in), exact zeros dropped,
// columns in window order (= ascending, the anchor numbering is monotone).
//
// Shape: one warp per row (DOF).  The row's window of (2p+1)^dim candidate
// columns lives in shared memory; the warp walks the DOF's physical support
// (elements ascending) and its lanes add the element row's nloc entries (one
// lane per local function: distinct columns, so no two lanes touch one slot
// in a step).  Count pass, scan, fill pass; then the symmetrisation looks up
// each transposed entry by binary search.
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace igk {

struct AsmArgs {
  int32_t dim, p, family, n, nloc, W, wsize;
  int32_t nf0, nf1, nf2;
  const int32_t *el_ix, *el_iy, *el_iz, *el_table;
  const double *K, *F;
  const int64_t *anchors, *supp_ptr;
  const int32_t *supp_el, *kept;
};

constexpr int kAsmWarps = 4;

// FILL = false: cnt[row] = number of touched window slots.  FILL = true: the
// row's columns / values at rowptr[row], b[row].
template <bool FILL>
__global__ void __launch_bounds__(32 * kAsmWarps) k_asm_rows(AsmArgs a, int32_t* cnt, const int64_t* rowptr,
                                                            int32_t* col, double* val, double* b) {
  extern __shared__ double asm_sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* acc = asm_sm + static_cast<size_t>(w) * a.wsize;
  unsigned char* touched =
      reinterpret_cast<unsigned char*>(asm_sm + static_cast<size_t>(kAsmWarps) * a.wsize) + w * a.wsize;
  const int row = blockIdx.x * kAsmWarps + w;
  if (row >= a.n) return;
  const int64_t u = a.anchors[row];
  const int ax = static_cast<int>(u % a.nf0);
  const int ay = static_cast<int>((u / a.nf0) % a.nf1);
  const int az = static_cast<int>(u / (static_cast<int64_t>(a.nf0) * a.nf1));
  for (int s = lane; s < a.wsize; s += 32) touched[s] = 0;
  __syncwarp();
  const int p = a.p, q = p + 1, W = a.W, nl = a.nloc;
  double bsum = 0.0;
  for (int64_t k = a.supp_ptr[row]; k < a.supp_ptr[row + 1]; ++k) {
    const int e = a.supp_el[k];
    const int t = a.el_table[e];
    const int x0 = a.family ? a.el_ix[e] : p * a.el_ix[e];
    const int y0 = a.family ? a.el_iy[e] : p * a.el_iy[e];
    const int z0 = a.dim == 3 ? (a.family ? a.el_iz[e] : p * a.el_iz[e]) : 0;
    const int li = a.dim == 3 ? ((az - z0) * q + (ay - y0)) * q + (ax - x0) : (ay - y0) * q + (ax - x0);
    if (FILL && lane == 0) bsum = bsum + a.F[static_cast<int64_t>(t) * nl + li];
    const double* Krow = a.K + (static_cast<int64_t>(t) * nl + li) * nl;
    for (int lj = lane; lj < nl; lj += 32) {
      const double v = Krow[lj];
      if (v == 0.0) continue;
      const int jx = x0 + lj % q, jy = y0 + (lj / q) % q, jz = a.dim == 3 ? z0 + lj / (q * q) : 0;
      const int s = ((a.dim == 3 ? (jz - az + p) : 0) * W + (jy - ay + p)) * W + (jx - ax + p);
      if (!touched[s]) {
        touched[s] = 1;
        acc[s] = v;  // 0 + v == v
      } else {
        acc[s] = acc[s] + v;
      }
    }
    __syncwarp();  // element k complete before element k+1 (ascending order per slot)
  }
  int base = 0;
  const int64_t o = FILL ? rowptr[row] : 0;
  for (int s0 = 0; s0 < a.wsize; s0 += 32) {
    const int s = s0 + lane;
    const bool used = s < a.wsize && touched[s];
    const unsigned m = __ballot_sync(0xffffffffu, used);
    if (FILL && used) {
      const int pos = base + __popc(m & ((1u << lane) - 1u));
      const int dx = s % W - p, dy = (s / W) % W - p, dz = a.dim == 3 ? s / (W * W) - p : 0;
      const int64_t un = (static_cast<int64_t>(az + dz) * a.nf1 + (ay + dy)) * a.nf0 + (ax + dx);
      col[o + pos] = a.kept[un];
      val[o + pos] = acc[s];
    }
    base += __popc(m);
  }
  if (lane == 0) {
    if (FILL)
      b[row] = bsum;
    else
      cnt[row] = base;
  }
}

// A = 0.5 (A + A^T) entry by entry (assembly.cpp:177-180); *bad counts entries
// whose transpose is missing (unsymmetric pattern).
__global__ void k_asm_sym(int32_t n, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                          const double* __restrict__ val, double* sym, int* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int32_t k = ptr[i]; k < ptr[i + 1]; ++k) {
    const int32_t j = col[k];
    int32_t lo = ptr[j], hi = ptr[j + 1];
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (col[mid] < i)
        lo = mid + 1;
      else
        hi = mid;
    }
    if (lo == ptr[j + 1] || col[lo] != i) {
      atomicAdd(bad, 1);
      continue;
    }
    sym[k] = 0.5 * (val[k] + val[lo]);
  }
}

}  // namespace igk
