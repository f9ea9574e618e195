// spmv_psell.cuh — pattern-SELL: the SpMV layout of the large levels.
//
// Why: the row-dictionary SELL (kernels.cuh: Sell) removed most value bytes
// but the finest C4 SpMV stayed at ~300 us, 57 % issue-busy at 26 SASS
// instructions per matrix slot, with 4 B of column index per slot still
// streamed for 56 % of the rows.  The operators of an immersed B-spline
// discretisation are far more regular than a general sparse matrix: on C4's
// finest level 91 % of the rows lie in RUNS of consecutive rows with the same
// value sequence and the same column-offset sequence (an x-line interior: the
// typical run is 124 rows); the rest are single rows (line ends, cut cells).
//
// Layout: a list of warp-sized slices, each one warp:
//   * FAST slice = up to 32 consecutive rows of one run: the warp reads ONE
//     value sequence V[vbase + k] and ONE offset sequence O[obase + k] with
//     warp-uniform 16-byte loads (one L1 wavefront per 2 values / 4 offsets;
//     sequences deduplicated over the matrix) and gathers x[base(row) + o_k]
//     coalesced -- no per-row matrix bytes at all;
//   * GENERAL slice = up to 32 leftover rows (in row order): per-slice tables
//     of their DISTINCT offset sequences (wo columns) and distinct
//     non-dictionary value sequences (wv columns), k-blocked for vector loads
//     (offsets [k/4][col][k%4], values [k/2][col][k%2]); ginfo selects each
//     row's offset column and value source (global dictionary entry at the
//     start of V, or table column).  Entries past a row's length are never
//     added; their offsets repeat the row's first one (an empty row gets its
//     own column pointing at x[0]), so every gather stays inside x whatever
//     base(row) is.
// Offsets are taken against base(row) = (row * smul) >> sshift, chosen per
// matrix (A: row; restriction R: 2 row -- coarse x-lines map to every other
// fine column; prolongation P: row / 2) so that runs and tables repeat.
//
// The sum is the same serial ascending-k chain as every other SpMV here
// (Eigen RowMajor order), and values/offsets are stored bit-exactly, so the
// results are identical to kernels.cuh's k_spmv and to the oracle.  Slices
// are not aligned to the 256-row reduction chunks, so p . Ap is reduced by
// k_pap (same canonical chunk tree) after the product.
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace igk {

// pk: lmax (11 bits) | count << 11 (6) | fast << 17 | ulen << 18 | wv << 19 (6) | wo << 25 (6)
//     | FAST2 values in the constant-bank table << 31 (vbase = table offset)
struct PSliceMeta {
  uint32_t a;      // FAST: first row; GENERAL: index of the slice's entries in rlist/ginfo
  uint32_t vbase;  // FAST: value sequence; GENERAL: value table
  uint32_t obase;  // FAST: offset sequence; GENERAL: offset table
  uint32_t pk;
};

constexpr int kPLenBits = 11;
constexpr int kPMaxLen = (1 << kPLenBits) - 1;

// ginfo (GENERAL rows): len | vsel << 11 | vi << 17 | oi << 22; vsel > 0:
// values = dictionary entry vsel-1 (V[(vsel-1)*dict_w + k]); vsel = 0: table column vi.
struct PSell {
  int32_t n_rows, n_cols, n_slices;
  const PSliceMeta* meta;
  const int32_t* rlist;
  const uint32_t* ginfo;
  const double* V;
  const int32_t* O;
  int32_t dict_w;
  int32_t smul, sshift;  // base(row) = (row * smul) >> sshift
  const int2* seg;       // FAST2 segment lists (first offset, length); length 0 ends a list
  const int4* useg;      // FAST4 union lists: header {D, n}, then {offset, length, value index A | -1, B | -1}
  const double* xe;      // FASTE: edge-compacted copy of x (k_xgather), else null
};

// GENERAL-slice values: a row's own table column is read once per product
// (streamed, evict-first: 90 MB of unique cut-cell values per launch that
// would otherwise push the x lines and the solver's vectors out of L1 / L2 --
// C4 finest A p 76.7 -> 71.8 us, solve 85.6 -> 84.6 ms); dictionary sequences
// are shared between slices and stay cached.
__device__ __forceinline__ double2 ld_val2(const double2* p, int dict) {
  if (!dict) return __ldcs(p);
  return __ldg(p);
}
template <bool STREAM>
__device__ __forceinline__ int4 ld_off4(const int4* p) {
  if (STREAM) return __ldcs(p);
  return __ldg(p);
}

// FAST2: one segment (m consecutive offsets starting at o) for the two rows
// ra = r0 + 2 lane and ra + 1 (base(row) = row).  Both rows need the m+1
// values x[ra+o .. ra+o+m]; they are loaded once, as 16-byte pairs from the
// even index below (P = parity of r0 + o, warp-uniform), and each row adds
// its m products in ascending order.  Loads are 16-byte aligned (x is).
template <int P, int M>
__device__ __forceinline__ void fast2_segment(const double* __restrict__ x, int a, const double* __restrict__ vp,
                                              double& acc0, double& acc1) {
  constexpr int C = M + 1 + P;  // values needed from base = a - P
  const double* xb = x + (a - P);
  const double2* xb2 = reinterpret_cast<const double2*>(xb);
  double X[C + 1], v[M];
#pragma unroll
  for (int q = 0; 2 * q < C; ++q) {
    if (2 * q + 1 < C) {
      const double2 t = __ldg(xb2 + q);
      X[2 * q] = t.x;
      X[2 * q + 1] = t.y;
    } else {
      X[2 * q] = __ldg(xb + 2 * q);  // last value only: never read past x[a+M]
    }
  }
#pragma unroll
  for (int j = 0; j < M; ++j) v[j] = __ldg(vp + j);
#pragma unroll
  for (int j = 0; j < M; ++j) {
    acc0 = acc0 + v[j] * X[P + j];
    acc1 = acc1 + v[j] * X[P + j + 1];
  }
}
// Constant-bank value table (a __grid_constant__ kernel parameter): the most
// frequent FAST2 value sequences of the matrix (the interior stencils).  A
// warp-uniform indexed read of a kernel parameter is a constant-cache load
// (LDC / uniform datapath), not an L1TEX request -- and the L1 data pipe is
// what bounds this kernel (the per-run value loads were ~1/4 of its
// wavefronts).  FAST2 slices whose sequence is in the table carry pk bit 31
// and vbase = table offset.
constexpr int kPValTab = 1024;  // doubles (8 KB of kernel parameters; 32 KB measured: same graph time, but a direct launch then costs ~20 us)
struct PValTab {
  double v[kPValTab];
};
template <int P, int M>
__device__ __forceinline__ void fast2_segment_tab(const double* __restrict__ x, int a, const PValTab& tab, int vo,
                                                  double& acc0, double& acc1) {
  constexpr int C = M + 1 + P;
  const double* xb = x + (a - P);
  const double2* xb2 = reinterpret_cast<const double2*>(xb);
  double X[C + 1], v[M];
#pragma unroll
  for (int q = 0; 2 * q < C; ++q) {
    if (2 * q + 1 < C) {
      const double2 t = __ldg(xb2 + q);
      X[2 * q] = t.x;
      X[2 * q + 1] = t.y;
    } else {
      X[2 * q] = __ldg(xb + 2 * q);
    }
  }
#pragma unroll
  for (int j = 0; j < M; ++j) v[j] = tab.v[vo + j];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    acc0 = acc0 + v[j] * X[P + j];
    acc1 = acc1 + v[j] * X[P + j + 1];
  }
}
template <int P>
__device__ __forceinline__ void fast2_dispatch_tab(const double* __restrict__ x, int a, int m, const PValTab& tab,
                                                   int vo, double& acc0, double& acc1) {
  switch (m) {  // warp-uniform
    case 1: fast2_segment_tab<P, 1>(x, a, tab, vo, acc0, acc1); break;
    case 2: fast2_segment_tab<P, 2>(x, a, tab, vo, acc0, acc1); break;
    case 3: fast2_segment_tab<P, 3>(x, a, tab, vo, acc0, acc1); break;
    case 4: fast2_segment_tab<P, 4>(x, a, tab, vo, acc0, acc1); break;
    case 5: fast2_segment_tab<P, 5>(x, a, tab, vo, acc0, acc1); break;
    case 6: fast2_segment_tab<P, 6>(x, a, tab, vo, acc0, acc1); break;
    case 7: fast2_segment_tab<P, 7>(x, a, tab, vo, acc0, acc1); break;
    default: fast2_segment_tab<P, 8>(x, a, tab, vo, acc0, acc1); break;
  }
}

template <int P>
__device__ __forceinline__ void fast2_dispatch(const double* __restrict__ x, int a, int m,
                                               const double* __restrict__ vp, double& acc0, double& acc1) {
  switch (m) {  // warp-uniform
    case 1: fast2_segment<P, 1>(x, a, vp, acc0, acc1); break;
    case 2: fast2_segment<P, 2>(x, a, vp, acc0, acc1); break;
    case 3: fast2_segment<P, 3>(x, a, vp, acc0, acc1); break;
    case 4: fast2_segment<P, 4>(x, a, vp, acc0, acc1); break;
    case 5: fast2_segment<P, 5>(x, a, vp, acc0, acc1); break;
    case 6: fast2_segment<P, 6>(x, a, vp, acc0, acc1); break;
    case 7: fast2_segment<P, 7>(x, a, vp, acc0, acc1); break;
    default: fast2_segment<P, 8>(x, a, vp, acc0, acc1); break;
  }
}

// FAST2M (row pairs of up to four pieces per slice; table layout in
// ig_gpu.cu: to_psell).  The lane's first row; pid = its piece; odd = its
// second row does not exist (odd tail of the piece).
__device__ __forceinline__ int fast2m_lane(const int4* __restrict__ tb, int cl, int count, int& odd, int* pid_out = nullptr) {
  const int4 hd = __ldg(tb + 1);
  const int s1 = hd.x & 0xff, s2 = (hd.x >> 8) & 0xff, s3 = (hd.x >> 16) & 0xff;
  const int pid = (cl >= s1 ? 1 : 0) + (cl >= s2 ? 1 : 0) + (cl >= s3 ? 1 : 0);
  const int st = pid == 0 ? 0 : pid == 1 ? s1 : pid == 2 ? s2 : s3;
  const int en = min(count, pid == 0 ? s1 : pid == 1 ? s2 : pid == 2 ? s3 : 64);
  const int r0 = __ldg(reinterpret_cast<const int*>(tb) + pid);
  odd = ((hd.y >> pid) & 1) && cl == en - 1;
  if (pid_out) *pid_out = pid;
  return r0 + 2 * (cl - st);
}
// One column run (M consecutive columns from a = lane's first row + the
// piece's offset) for the lane's rows ra and ra + 1.  The parity of a differs
// from lane to lane here, so the aligned 16-byte loads start at a - (a & 1) and
// the M + 1 operands are selected per lane; each row still adds its M products
// in ascending order.  Never reads past x[a + M].
template <int M, class VS>
__device__ __forceinline__ void fast2m_segment(const double* __restrict__ x, int a, const VS& vs, int vo, double& acc0,
                                               double& acc1) {
  const int p = a & 1;
  const double* xb = x + (a - p);
  const double2* xb2 = reinterpret_cast<const double2*>(xb);
  constexpr int C0 = M + 1;  // operands when p = 0 (W[0..M]); p = 1 uses W[1..M+1]
  double W[C0 + 2];
#pragma unroll
  for (int q = 0; 2 * q <= C0; ++q) {
    if (2 * q + 1 < C0) {
      const double2 t = __ldg(xb2 + q);
      W[2 * q] = t.x;
      W[2 * q + 1] = t.y;
    } else if (2 * q + 1 == C0) {  // W[M] always, W[M + 1] only when p = 1
      if (p) {
        const double2 t = __ldg(xb2 + q);
        W[2 * q] = t.x;
        W[2 * q + 1] = t.y;
      } else {
        W[2 * q] = __ldg(xb + 2 * q);
        W[2 * q + 1] = 0.0;
      }
    } else {  // 2 q == C0: W[M + 1], only when p = 1
      W[2 * q] = p ? __ldg(xb + 2 * q) : 0.0;
    }
  }
  double S[C0];
#pragma unroll
  for (int j = 0; j < C0; ++j) S[j] = p ? W[j + 1] : W[j];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const double v = vs(vo + j);
    acc0 = acc0 + v * S[j];
    acc1 = acc1 + v * S[j + 1];
  }
}
template <class VS>
__device__ __forceinline__ void fast2m_slice(const double* __restrict__ x, const int4* __restrict__ tb, const int2* __restrict__ sg,
                                            int n, int ra, int pid, const VS& vs, double& acc0, double& acc1) {
  const int* ob = reinterpret_cast<const int*>(tb + 2) + pid;
  int vo = 0;
  // (The next run's length and offset are loaded a run ahead: the offset
  // table is per slice -- an L2 round trip that would otherwise sit in front
  // of every run's window loads.)
  int mn = n > 0 ? __ldg(sg).y : 0, on = n > 0 ? __ldg(ob) : 0;
  for (int u = 0; u < n; ++u) {
    const int m = mn;  // warp-uniform
    const int a = ra + on;
    if (u + 1 < n) {
      mn = __ldg(sg + u + 1).y;
      on = __ldg(ob + 4 * (u + 1));
    }
    switch (m) {
      case 1: fast2m_segment<1>(x, a, vs, vo, acc0, acc1); break;
      case 2: fast2m_segment<2>(x, a, vs, vo, acc0, acc1); break;
      case 3: fast2m_segment<3>(x, a, vs, vo, acc0, acc1); break;
      case 4: fast2m_segment<4>(x, a, vs, vo, acc0, acc1); break;
      case 5: fast2m_segment<5>(x, a, vs, vo, acc0, acc1); break;
      case 6: fast2m_segment<6>(x, a, vs, vo, acc0, acc1); break;
      case 7: fast2m_segment<7>(x, a, vs, vo, acc0, acc1); break;
      default: fast2m_segment<8>(x, a, vs, vo, acc0, acc1); break;
    }
    vo += m;
  }
}

// The rows this lane will own in a slice (psell_slice's mapping), from the
// static metadata: lets a kernel issue its per-row loads (residual source,
// the x being corrected) ahead of the slice's product chain.  GENERAL slices:
// gen = {row, ginfo} of the lane's (clamped) entry, loaded here together --
// both depend on the slice metadata only, so psell_slice's chain is meta ->
// {row, info} -> offsets -> x instead of meta -> row -> info -> offsets -> x
// (profiles: the prolongation's ginfo wait was 8 % of its stall samples).
template <bool F4 = true>
__device__ __forceinline__ void psell_rows(const PSell& A, const uint4 mu, int* rows, uint2& gen) {
  const int lane = threadIdx.x & 31;
  const uint32_t pk = mu.w;
  const int count = static_cast<int>((pk >> 11) & 0x3f);
  int& row = rows[0];
  int& row2 = rows[1];
  row = row2 = rows[2] = rows[3] = -1;
  gen = make_uint2(0u, 0u);
  if (count > 0 && !(pk & (1u << 17))) {
    const int idx = static_cast<int>(mu.x) + min(lane, count - 1);
    gen.x = static_cast<uint32_t>(__ldg(A.rlist + idx));
    gen.y = __ldg(A.ginfo + idx);
  }
  if (count == 0 || lane >= count) return;
  const int wv = static_cast<int>((pk >> 19) & 0x3f);
  if (F4 && (pk & (1u << 17)) && wv == 3) {  // FAST2M: row pairs of up to four pieces
    int odd;
    row = fast2m_lane(A.useg + mu.z, lane, count, odd);
    row2 = odd ? -1 : row + 1;
  } else if (F4 && (pk & (1u << 17)) && wv == 2) {  // FAST4: B rows at + D
    const int D = __ldg(A.useg + mu.z).x;
    row = static_cast<int>(mu.x) + 2 * lane;
    row2 = row + 1;
    rows[2] = row + D;
    rows[3] = row + D + 1;
  } else if ((pk & (1u << 17)) && (wv == 1 || wv == 4)) {  // FAST2 / FASTAB: row pairs
    row = static_cast<int>(mu.x) + 2 * lane;
    row2 = row + 1;
  } else if (pk & (1u << 17)) {
    row = static_cast<int>(mu.x) + lane;
  } else {
    row = static_cast<int>(gen.x);
  }
}

// FAST4: one union column run (offset o from the lane's A row, length M) for
// the lane's rows ra, ra+1 (line A) and ra+D, ra+D+1 (line B): the x values
// are loaded once; A's rows add their products if vA >= 0, B's if vB >= 0.
template <int P, int M, class VS>
__device__ __forceinline__ void fast4_segment(const double* __restrict__ x, int a, const VS& vs, int vA, int vB,
                                              double& acc0, double& acc1, double& acc2, double& acc3) {
  constexpr int C = M + 1 + P;
  const double* xb = x + (a - P);
  const double2* xb2 = reinterpret_cast<const double2*>(xb);
  double X[C + 1];
#pragma unroll
  for (int q = 0; 2 * q < C; ++q) {
    if (2 * q + 1 < C) {
      const double2 t = __ldg(xb2 + q);
      X[2 * q] = t.x;
      X[2 * q + 1] = t.y;
    } else {
      X[2 * q] = __ldg(xb + 2 * q);
    }
  }
  if (vA >= 0) {  // warp-uniform
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const double v = vs(vA + j);
      acc0 = acc0 + v * X[P + j];
      acc1 = acc1 + v * X[P + j + 1];
    }
  }
  if (vB >= 0) {
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const double v = vs(vB + j);
      acc2 = acc2 + v * X[P + j];
      acc3 = acc3 + v * X[P + j + 1];
    }
  }
}
struct VGlob {
  const double* p;
  __device__ __forceinline__ double operator()(int j) const { return __ldg(p + j); }
};
struct VTabl {
  const PValTab* t;
  int o;  // the sequence's offset in the table
  __device__ __forceinline__ double operator()(int j) const { return t->v[o + j]; }
};
template <int P, class VS>
__device__ __forceinline__ void fast4_dispatch(const double* __restrict__ x, int a, int m, const VS& vs, int vA, int vB,
                                               double& acc0, double& acc1, double& acc2, double& acc3) {
  switch (m) {  // warp-uniform
    case 1: fast4_segment<P, 1>(x, a, vs, vA, vB, acc0, acc1, acc2, acc3); break;
    case 2: fast4_segment<P, 2>(x, a, vs, vA, vB, acc0, acc1, acc2, acc3); break;
    case 3: fast4_segment<P, 3>(x, a, vs, vA, vB, acc0, acc1, acc2, acc3); break;
    case 4: fast4_segment<P, 4>(x, a, vs, vA, vB, acc0, acc1, acc2, acc3); break;
    case 5: fast4_segment<P, 5>(x, a, vs, vA, vB, acc0, acc1, acc2, acc3); break;
    case 6: fast4_segment<P, 6>(x, a, vs, vA, vB, acc0, acc1, acc2, acc3); break;
    case 7: fast4_segment<P, 7>(x, a, vs, vA, vB, acc0, acc1, acc2, acc3); break;
    default: fast4_segment<P, 8>(x, a, vs, vA, vB, acc0, acc1, acc2, acc3); break;
  }
}
template <class VS>
__device__ __forceinline__ void fast4_slice(const double* __restrict__ x, const int4* __restrict__ ug, int n, int ra,
                                           int p0, const VS& vs, double* acc) {
  int4 en = __ldg(ug);
  for (int u = 0; u < n; ++u) {
    const int4 e = en;
    if (u + 1 < n) en = __ldg(ug + u + 1);  // a run ahead
    if (((p0 + e.x) & 1) == 0)
      fast4_dispatch<0>(x, ra + e.x, e.y, vs, e.z, e.w, acc[0], acc[1], acc[2], acc[3]);
    else
      fast4_dispatch<1>(x, ra + e.x, e.y, vs, e.z, e.w, acc[0], acc[1], acc[2], acc[3]);
  }
}

// FAST8: as FAST4 with FOUR rows of each of the two x-lines per lane (rows
// ra .. ra + 3 and ra + D .. ra + D + 3): one window of M + 3 values feeds 4 M
// products per line -- 1.6 B of x per product through the L1 data pipe (the
// unit that bounds this kernel) instead of FAST4's 2.8 B, and one warp per
// 124-row line pair instead of two.
template <int P, int M, class VS>
__device__ __forceinline__ void fast8_segment(const double* __restrict__ x, int a, const VS& vs, int vA, int vB,
                                              double* acc) {
  constexpr int C = M + 3 + P;  // values needed from base = a - P
  const double* xb = x + (a - P);
  const double2* xb2 = reinterpret_cast<const double2*>(xb);
  double X[C + 1];
#pragma unroll
  for (int q = 0; 2 * q < C; ++q) {
    if (2 * q + 1 < C) {
      const double2 t = __ldg(xb2 + q);
      X[2 * q] = t.x;
      X[2 * q + 1] = t.y;
    } else {
      X[2 * q] = __ldg(xb + 2 * q);  // last value only: never read past x[a + M + 2]
    }
  }
  if (vA >= 0) {  // warp-uniform
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const double v = vs(vA + j);
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = acc[r] + v * X[P + j + r];
    }
  }
  if (vB >= 0) {
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const double v = vs(vB + j);
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[4 + r] = acc[4 + r] + v * X[P + j + r];
    }
  }
}
// FAST8, column runs of 5 (the 3D p = 2 stencil): lanes are 32 bytes apart,
// so the window is read with 32-byte loads (sm_100 LDG.256: a warp request is
// 1 KB of consecutive bytes) from the 32-byte boundary below -- 2 requests
// when the run starts on it, else 2 + the 1-3 remaining values -- instead of
// 4-5 16-byte requests that each touch all of the warp's 8-9 cache lines.
// Q = the run's first element modulo 4 (warp-uniform).  Never reads past
// x[a + 7], the last operand.
#ifndef IG_F8_LD256
#define IG_F8_LD256 1
#endif
__device__ __forceinline__ void ldg256(const double* p, double* v) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
template <int Q, class VS>
__device__ __forceinline__ void fast8_segment5(const double* __restrict__ x, int a, const VS& vs, int vA, int vB,
                                               double* acc) {
  const double* xb = x + (a - Q);
  double X[12];
  ldg256(xb, X);
  ldg256(xb + 4, X + 4);
  if (Q == 1) {
    X[8] = __ldg(xb + 8);
  } else if (Q == 2) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(xb + 8));
    X[8] = t.x;
    X[9] = t.y;
  } else if (Q == 3) {
    const double2 t = __ldg(reinterpret_cast<const double2*>(xb + 8));
    X[8] = t.x;
    X[9] = t.y;
    X[10] = __ldg(xb + 10);
  }
  if (vA >= 0) {  // warp-uniform
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const double v = vs(vA + j);
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = acc[r] + v * X[Q + j + r];
    }
  }
  if (vB >= 0) {
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const double v = vs(vB + j);
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[4 + r] = acc[4 + r] + v * X[Q + j + r];
    }
  }
}
template <int P, class VS>
__device__ __forceinline__ void fast8_dispatch(const double* __restrict__ x, int a, int m, const VS& vs, int vA, int vB,
                                               double* acc) {
  switch (m) {  // warp-uniform
    case 1: fast8_segment<P, 1>(x, a, vs, vA, vB, acc); break;
    case 2: fast8_segment<P, 2>(x, a, vs, vA, vB, acc); break;
    case 3: fast8_segment<P, 3>(x, a, vs, vA, vB, acc); break;
    case 4: fast8_segment<P, 4>(x, a, vs, vA, vB, acc); break;
    case 5: fast8_segment<P, 5>(x, a, vs, vA, vB, acc); break;
    case 6: fast8_segment<P, 6>(x, a, vs, vA, vB, acc); break;
    case 7: fast8_segment<P, 7>(x, a, vs, vA, vB, acc); break;
    default: fast8_segment<P, 8>(x, a, vs, vA, vB, acc); break;
  }
}
template <class VS>
__device__ __forceinline__ void fast8_slice(const double* __restrict__ x, const int4* __restrict__ ug, int n, int ra,
                                           int a0, const VS& vs, double* acc) {
  const int p0 = a0 & 1;
  int4 en = __ldg(ug);
  const int q0 = static_cast<int>((reinterpret_cast<uintptr_t>(x) >> 3) & 3) + a0;  // warp-uniform
  for (int u = 0; u < n; ++u) {
    const int4 e = en;
    if (u + 1 < n) en = __ldg(ug + u + 1);  // a run ahead
    if (IG_F8_LD256 && e.y == 5) {
      // (from the address of the slice's first row, so any 8-byte aligned x works; lanes differ by 32 bytes)
      switch ((q0 + e.x) & 3) {
        case 0: fast8_segment5<0>(x, ra + e.x, vs, e.z, e.w, acc); break;
        case 1: fast8_segment5<1>(x, ra + e.x, vs, e.z, e.w, acc); break;
        case 2: fast8_segment5<2>(x, ra + e.x, vs, e.z, e.w, acc); break;
        default: fast8_segment5<3>(x, ra + e.x, vs, e.z, e.w, acc); break;
      }
    } else if (((p0 + e.x) & 1) == 0) {
      fast8_dispatch<0>(x, ra + e.x, e.y, vs, e.z, e.w, acc);
    } else {
      fast8_dispatch<1>(x, ra + e.x, e.y, vs, e.z, e.w, acc);
    }
  }
}

// One warp, one slice.  Returns the row this lane owns (-1: none) and its
// sum; FAST2 slices give each lane a second row (row2 / acc2, else -1).
// gen: psell_rows' {row, ginfo} (GENERAL slices).
template <bool STREAM, bool F4 = true>
__device__ __forceinline__ int psell_slice(const PSell& A, const uint4 mu, const uint2 gen, const double* __restrict__ x,
                                           double& acc, int& row2, double& acc2, const PValTab* tab, int* rowx,
                                           double* accx) {
  acc = 0.0;
  acc2 = 0.0;
  row2 = -1;
  rowx[0] = rowx[1] = -1;
  const int lane = threadIdx.x & 31;
  const uint32_t pk = mu.w;
  const int count = static_cast<int>((pk >> 11) & 0x3f);
  if (count == 0) return -1;  // padding slice (warp-uniform)
  const int L = static_cast<int>(pk & kPMaxLen);
  const int cl = min(lane, count - 1);  // surplus lanes recompute the last row, store nothing
  if (F4 && (pk & (1u << 17)) && ((pk >> 19) & 0x3f) == 3) {  // FAST2M: row pairs of several pieces (warp-uniform)
    const int4* tb = A.useg + mu.z;
    int odd, pid;
    const int ra = fast2m_lane(tb, cl, count, odd, &pid);
    const int4 hd = __ldg(tb + 1);
    if (tab != nullptr && (pk >> 31))
      fast2m_slice(x, tb, A.seg + hd.z, hd.w, ra, pid, VTabl{tab, static_cast<int>(mu.y)}, acc, acc2);
    else
      fast2m_slice(x, tb, A.seg + hd.z, hd.w, ra, pid, VGlob{A.V + mu.y}, acc, acc2);
    if (lane >= count) return -1;
    row2 = odd ? -1 : ra + 1;
    return ra;
  }
  if (F4 && (pk & (1u << 17)) && ((pk >> 19) & 0x3f) == 2) {  // FAST4: rows of two x-lines (warp-uniform)
    const int ra = static_cast<int>(mu.x) + 2 * cl;
    const int p0 = static_cast<int>(mu.x) & 1;
    const int4 hd = __ldg(A.useg + mu.z);
    double a4[4] = {0.0, 0.0, 0.0, 0.0};
    if (tab != nullptr && (pk >> 31))
      fast4_slice(x, A.useg + mu.z + 1, hd.y, ra, p0, VTabl{tab, static_cast<int>(mu.y)}, a4);
    else
      fast4_slice(x, A.useg + mu.z + 1, hd.y, ra, p0, VGlob{A.V + mu.y}, a4);
    acc = a4[0];
    acc2 = a4[1];
    if (lane >= count) return -1;
    row2 = ra + 1;
    rowx[0] = ra + hd.x;
    rowx[1] = ra + hd.x + 1;
    accx[0] = a4[2];
    accx[1] = a4[3];
    return ra;
  }
  if ((pk & (1u << 17)) && ((pk >> 19) & 0x3f) == 1) {  // FAST2: `count` row pairs (warp-uniform)
    const int ra = static_cast<int>(mu.x) + 2 * cl;
    const double* vp = A.V + mu.y;
    const int p0 = static_cast<int>(mu.x) & 1;
    if (tab != nullptr && (pk >> 31)) {  // values from the constant-bank table (warp-uniform branch)
      int vo = static_cast<int>(mu.y);
      for (const int2* sg = A.seg + mu.z;; ++sg) {
        const int2 e = __ldg(sg);
        if (e.y == 0) break;
        if (((p0 + e.x) & 1) == 0)
          fast2_dispatch_tab<0>(x, ra + e.x, e.y, *tab, vo, acc, acc2);
        else
          fast2_dispatch_tab<1>(x, ra + e.x, e.y, *tab, vo, acc, acc2);
        vo += e.y;
      }
      if (lane >= count) return -1;
      row2 = ra + 1;
      return ra;
    }
    for (const int2* sg = A.seg + mu.z;; ++sg) {
      const int2 e = __ldg(sg);
      if (e.y == 0) break;
      if (((p0 + e.x) & 1) == 0)
        fast2_dispatch<0>(x, ra + e.x, e.y, vp, acc, acc2);
      else
        fast2_dispatch<1>(x, ra + e.x, e.y, vp, acc, acc2);
      vp += e.y;
    }
    if (lane >= count) return -1;
    row2 = ra + 1;
    return ra;
  }
  if ((pk & (1u << 17)) && ((pk >> 19) & 0x3f) == 4) {  // FASTAB: row pairs sharing their columns (warp-uniform)
    // Rows ra and ra + 1 have the same column list (a prolongation's two
    // fine rows under one coarse stencil) and their own value sequences,
    // stored interleaved {A_k, B_k}; each x is gathered once for both.
    const int ra = static_cast<int>(mu.x) + 2 * cl;
    const double* xr = x + ((ra * A.smul) >> A.sshift);
    const int4* op4 = reinterpret_cast<const int4*>(A.O + mu.z);
    const bool tb = tab != nullptr && (pk >> 31);
    const double2* vp2 = reinterpret_cast<const double2*>(A.V + mu.y);
    const int vo = static_cast<int>(mu.y);
    int k = 0;
    for (; k + 4 <= L; k += 4) {
      const int4 b = __ldg(op4 + (k >> 2));
      const double x0 = __ldg(xr + b.x), x1 = __ldg(xr + b.y), x2 = __ldg(xr + b.z), x3 = __ldg(xr + b.w);
      double2 v0, v1, v2, v3;
      if (tb) {
        v0 = make_double2(tab->v[vo + 2 * k], tab->v[vo + 2 * k + 1]);
        v1 = make_double2(tab->v[vo + 2 * k + 2], tab->v[vo + 2 * k + 3]);
        v2 = make_double2(tab->v[vo + 2 * k + 4], tab->v[vo + 2 * k + 5]);
        v3 = make_double2(tab->v[vo + 2 * k + 6], tab->v[vo + 2 * k + 7]);
      } else {
        v0 = __ldg(vp2 + k);
        v1 = __ldg(vp2 + k + 1);
        v2 = __ldg(vp2 + k + 2);
        v3 = __ldg(vp2 + k + 3);
      }
      acc = acc + v0.x * x0;
      acc2 = acc2 + v0.y * x0;
      acc = acc + v1.x * x1;
      acc2 = acc2 + v1.y * x1;
      acc = acc + v2.x * x2;
      acc2 = acc2 + v2.y * x2;
      acc = acc + v3.x * x3;
      acc2 = acc2 + v3.y * x3;
    }
    for (; k < L; ++k) {
      const double xk = __ldg(xr + __ldg(A.O + mu.z + k));
      const double2 v = tb ? make_double2(tab->v[vo + 2 * k], tab->v[vo + 2 * k + 1]) : __ldg(vp2 + k);
      acc = acc + v.x * xk;
      acc2 = acc2 + v.y * xk;
    }
    if (lane >= count) return -1;
    row2 = ra + 1;
    return ra;
  }
  if ((pk & (1u << 17)) && tab != nullptr && (pk >> 31)) {  // FAST, values from the constant-bank table
    const int row = static_cast<int>(mu.x) + cl;
    const double* xr = x + ((row * A.smul) >> A.sshift);
    const int vo = static_cast<int>(mu.y);
    const int4* op4 = reinterpret_cast<const int4*>(A.O + mu.z);
    int k = 0;
    for (; k + 8 <= L; k += 8) {
      const int4 b0 = __ldg(op4 + (k >> 2)), b1 = __ldg(op4 + (k >> 2) + 1);
      const double x0 = __ldg(xr + b0.x), x1 = __ldg(xr + b0.y), x2 = __ldg(xr + b0.z), x3 = __ldg(xr + b0.w);
      const double x4 = __ldg(xr + b1.x), x5 = __ldg(xr + b1.y), x6 = __ldg(xr + b1.z), x7 = __ldg(xr + b1.w);
      acc = acc + tab->v[vo + k] * x0;
      acc = acc + tab->v[vo + k + 1] * x1;
      acc = acc + tab->v[vo + k + 2] * x2;
      acc = acc + tab->v[vo + k + 3] * x3;
      acc = acc + tab->v[vo + k + 4] * x4;
      acc = acc + tab->v[vo + k + 5] * x5;
      acc = acc + tab->v[vo + k + 6] * x6;
      acc = acc + tab->v[vo + k + 7] * x7;
    }
    for (; k < L; ++k) acc = acc + tab->v[vo + k] * __ldg(xr + __ldg(A.O + mu.z + k));
    return lane < count ? row : -1;
  }
  if (pk & (1u << 17)) {                // FAST (warp-uniform branch)
    const int row = static_cast<int>(mu.x) + cl;
    const double* xr = x + ((row * A.smul) >> A.sshift);
    const double* vp = A.V + mu.y;
    const int32_t* op = A.O + mu.z;
    const double2* vp2 = reinterpret_cast<const double2*>(vp);
    const int4* op4 = reinterpret_cast<const int4*>(op);
    int k = 0;
    for (; k + 8 <= L; k += 8) {
      const double2 a0 = __ldg(vp2 + (k >> 1)), a1 = __ldg(vp2 + (k >> 1) + 1);
      const double2 a2 = __ldg(vp2 + (k >> 1) + 2), a3 = __ldg(vp2 + (k >> 1) + 3);
      const int4 b0 = __ldg(op4 + (k >> 2)), b1 = __ldg(op4 + (k >> 2) + 1);
      const double x0 = __ldg(xr + b0.x), x1 = __ldg(xr + b0.y), x2 = __ldg(xr + b0.z), x3 = __ldg(xr + b0.w);
      const double x4 = __ldg(xr + b1.x), x5 = __ldg(xr + b1.y), x6 = __ldg(xr + b1.z), x7 = __ldg(xr + b1.w);
      acc = acc + a0.x * x0;
      acc = acc + a0.y * x1;
      acc = acc + a1.x * x2;
      acc = acc + a1.y * x3;
      acc = acc + a2.x * x4;
      acc = acc + a2.y * x5;
      acc = acc + a3.x * x6;
      acc = acc + a3.y * x7;
    }
    for (; k < L; ++k) acc = acc + __ldg(vp + k) * __ldg(xr + __ldg(op + k));
    return lane < count ? row : -1;
  }
  if (pk >> 31) {  // FASTE (warp-uniform): lane's row gen.x, anchor gen.y in xe; one value / offset sequence
    const int row = static_cast<int>(gen.x);
    const double* xr = A.xe + gen.y;
    const bool tb = tab != nullptr && (pk & (1u << 18));
    const int vo = static_cast<int>(mu.y);
    const double2* vp2 = reinterpret_cast<const double2*>(A.V + mu.y);
    const int4* op4 = reinterpret_cast<const int4*>(A.O + mu.z);
    int k = 0;
    for (; k + 8 <= L; k += 8) {
      const int4 b0 = __ldg(op4 + (k >> 2)), b1 = __ldg(op4 + (k >> 2) + 1);
      const double x0 = __ldg(xr + b0.x), x1 = __ldg(xr + b0.y), x2 = __ldg(xr + b0.z), x3 = __ldg(xr + b0.w);
      const double x4 = __ldg(xr + b1.x), x5 = __ldg(xr + b1.y), x6 = __ldg(xr + b1.z), x7 = __ldg(xr + b1.w);
      double v[8];
      if (tb) {
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = tab->v[vo + k + u];
      } else {
        const double2 a0 = __ldg(vp2 + (k >> 1)), a1 = __ldg(vp2 + (k >> 1) + 1);
        const double2 a2 = __ldg(vp2 + (k >> 1) + 2), a3 = __ldg(vp2 + (k >> 1) + 3);
        v[0] = a0.x, v[1] = a0.y, v[2] = a1.x, v[3] = a1.y, v[4] = a2.x, v[5] = a2.y, v[6] = a3.x, v[7] = a3.y;
      }
      acc = acc + v[0] * x0;
      acc = acc + v[1] * x1;
      acc = acc + v[2] * x2;
      acc = acc + v[3] * x3;
      acc = acc + v[4] * x4;
      acc = acc + v[5] * x5;
      acc = acc + v[6] * x6;
      acc = acc + v[7] * x7;
    }
    for (; k < L; ++k)
      acc = acc + (tb ? tab->v[vo + k] : __ldg(A.V + mu.y + k)) * __ldg(xr + __ldg(A.O + mu.z + k));
    return lane < count ? row : -1;
  }
  const int row = static_cast<int>(gen.x);
  const uint32_t info = gen.y;
  const int len = static_cast<int>(info & kPMaxLen);
  const int vsel = static_cast<int>((info >> 11) & 0x3f);
  const int vi = static_cast<int>((info >> 17) & 0x1f);
  const int oi = static_cast<int>((info >> 22) & 0x1f);
  const int wv = static_cast<int>((pk >> 19) & 0x3f), wo = static_cast<int>((pk >> 25) & 0x3f);
  const double* xr = x + ((row * A.smul) >> A.sshift);
  const double2* vp2 = reinterpret_cast<const double2*>(
      vsel ? A.V + static_cast<int64_t>(vsel - 1) * A.dict_w : A.V + mu.y + 2 * vi);
  const int vs = vsel ? 1 : wv;  // double2 stride per 2 k
  const int4* op4 = reinterpret_cast<const int4*>(A.O + mu.z + 4 * oi);
  const int L8 = (L + 7) & ~7;
  const int lfull = (pk & (1u << 18)) ? (L & ~7) : 0;  // blocks every row fills
  int k = 0;
  // (Each block's offsets are loaded a block ahead: offsets -> gathers is two
  // dependent round trips per block otherwise, and on the levels that are a
  // fraction of a wave of warps the slice's chain is the product's time.)
  int4 nb0 = make_int4(0, 0, 0, 0), nb1 = nb0;
  if (L8 > 0) {
    nb0 = ld_off4<STREAM>(op4);
    nb1 = ld_off4<STREAM>(op4 + wo);
  }
  for (; k < lfull; k += 8) {
    const double2 a0 = ld_val2(vp2 + (k >> 1) * vs, vsel), a1 = ld_val2(vp2 + ((k >> 1) + 1) * vs, vsel);
    const double2 a2 = ld_val2(vp2 + ((k >> 1) + 2) * vs, vsel), a3 = ld_val2(vp2 + ((k >> 1) + 3) * vs, vsel);
    const int4 b0 = nb0, b1 = nb1;
    if (k + 8 < L8) {
      nb0 = ld_off4<STREAM>(op4 + ((k + 8) >> 2) * wo);
      nb1 = ld_off4<STREAM>(op4 + (((k + 8) >> 2) + 1) * wo);
    }
    const double x0 = __ldg(xr + b0.x), x1 = __ldg(xr + b0.y), x2 = __ldg(xr + b0.z), x3 = __ldg(xr + b0.w);
    const double x4 = __ldg(xr + b1.x), x5 = __ldg(xr + b1.y), x6 = __ldg(xr + b1.z), x7 = __ldg(xr + b1.w);
    acc = acc + a0.x * x0;
    acc = acc + a0.y * x1;
    acc = acc + a1.x * x2;
    acc = acc + a1.y * x3;
    acc = acc + a2.x * x4;
    acc = acc + a2.y * x5;
    acc = acc + a3.x * x6;
    acc = acc + a3.y * x7;
  }
  for (; k < L8; k += 8) {
    const double2 a0 = ld_val2(vp2 + (k >> 1) * vs, vsel), a1 = ld_val2(vp2 + ((k >> 1) + 1) * vs, vsel);
    const double2 a2 = ld_val2(vp2 + ((k >> 1) + 2) * vs, vsel), a3 = ld_val2(vp2 + ((k >> 1) + 3) * vs, vsel);
    const int4 b0 = nb0, b1 = nb1;
    if (k + 8 < L8) {
      nb0 = ld_off4<STREAM>(op4 + ((k + 8) >> 2) * wo);
      nb1 = ld_off4<STREAM>(op4 + (((k + 8) >> 2) + 1) * wo);
    }
    const double xv[8] = {__ldg(xr + b0.x), __ldg(xr + b0.y), __ldg(xr + b0.z), __ldg(xr + b0.w),
                          __ldg(xr + b1.x), __ldg(xr + b1.y), __ldg(xr + b1.z), __ldg(xr + b1.w)};
    const double av[8] = {a0.x, a0.y, a1.x, a1.y, a2.x, a2.y, a3.x, a3.y};
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double t = acc + av[u] * xv[u];
      acc = (k + u < len) ? t : acc;
    }
  }
  return lane < count ? row : -1;
}

// MODE 0: y = A x.  MODE 1: y = r - A x (r read from rsrc; in place allowed:
// every row is read and written by its own lane only).
// Register budget: 256 threads x 4 CTAs per SM (<= 64 registers).  Measured
// on C4 (profiles/psell_sweep.py, variant builds): the compiler's default
// (40 registers, 6 CTAs) 172 us for the finest A p and 1036 us per V-cycle;
// with this bound 161 us and 904 us -- the extra registers hoist more gathers
// ahead of each serial chain, and 32 resident warps keep their x lines in L1.
#ifndef IG_PSPMV_MINB
#define IG_PSPMV_MINB 4
#endif
#ifndef IG_PPROLONG_MINB
#define IG_PPROLONG_MINB 4
#endif
#ifndef IG_PSPMV_CTA
#define IG_PSPMV_CTA 64  // threads per k_pspmv CTA: slices differ in cost (a FAST4 warp does 4x the products of a FAST one), small CTAs keep a slow warp from holding seven finished ones resident (C4 finest A p 134.4 -> 122.4 us vs 256; slices are padded to multiples of 8 per matrix)
#endif
constexpr int kPCta = IG_PSPMV_CTA;
template <int MODE, bool STREAM, bool F4 = true>
__global__ void __launch_bounds__(kPCta, IG_PSPMV_MINB * (256 / kPCta)) k_pspmv(PSell A, const double* __restrict__ x, double* y,
                                               const double* rsrc, const PcgState* st,
                                               const __grid_constant__ PValTab tab) {
  const int slice = blockIdx.x * (kPCta / 32) + (threadIdx.x >> 5);
  const uint4 mu = __ldg(reinterpret_cast<const uint4*>(A.meta + slice));  // static: before the wait
#ifdef IG_DBG_SKIP  // timing experiments only (profiles/build_variants.sh): drop one slice class
  {
    const bool fast = mu.w & (1u << 17);
    const int wv = static_cast<int>((mu.w >> 19) & 0x3f);
    if ((IG_DBG_SKIP == 1 && !fast) || (IG_DBG_SKIP == 2 && fast && wv != 2) || (IG_DBG_SKIP == 3 && fast && (wv == 2 || wv == 5)) ||
        (IG_DBG_SKIP == 4 && fast) || (IG_DBG_SKIP == 5 && fast && wv == 3) || (IG_DBG_SKIP == 6 && !(fast && wv == 3)) ||
        (IG_DBG_SKIP == 7 && !(fast && (wv == 2 || wv == 5))))
      return;
  }
#endif
  if (F4 && (mu.w & (1u << 17)) && ((mu.w >> 19) & 0x3f) == 5) {  // FAST8 (warp-uniform): own epilogue, 8 rows per lane
    const int lane = threadIdx.x & 31;
    const int count = static_cast<int>((mu.w >> 11) & 0x3f);
    const int4 hd = __ldg(A.useg + mu.z);
    pdl_entry();
    if (pcg_done(st)) return;
    const int ra = static_cast<int>(mu.x) + 4 * min(lane, count - 1);
    double a8[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (mu.w >> 31)
      fast8_slice(x, A.useg + mu.z + 1, hd.y, ra, static_cast<int>(mu.x), VTabl{&tab, static_cast<int>(mu.y)}, a8);
    else
      fast8_slice(x, A.useg + mu.z + 1, hd.y, ra, static_cast<int>(mu.x), VGlob{A.V + mu.y}, a8);
    if (lane >= count) return;
    if (MODE == 1) {  // (the eight residual sources together, after the chain: no registers held across it)
      double rs8[8];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        rs8[r] = rsrc[ra + r];
        rs8[4 + r] = rsrc[ra + hd.x + r];
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) a8[r] = rs8[r] - a8[r];
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      y[ra + r] = a8[r];
      y[ra + hd.x + r] = a8[4 + r];
    }
    return;
  }
  int pr[4];
  uint2 gen;
  psell_rows<F4>(A, mu, pr, gen);
  pdl_entry();
  if (pcg_done(st)) return;
  // The residual source is loaded before the product chain, not after it.
  double rs[4];
#pragma unroll
  for (int k = 0; k < (F4 ? 4 : 2); ++k) rs[k] = (MODE == 1 && pr[k] >= 0) ? rsrc[pr[k]] : 0.0;
  double acc, acc2, accx[2];
  int row2, rowx[2];
  const int row = psell_slice<STREAM, F4>(A, mu, gen, x, acc, row2, acc2, &tab, rowx, accx);
  if (row < 0) return;
  y[row] = (MODE == 0) ? acc : rs[0] - acc;
  if (row2 >= 0) y[row2] = (MODE == 0) ? acc2 : rs[1] - acc2;
  if (F4 && rowx[0] >= 0) {
    y[rowx[0]] = (MODE == 0) ? accx[0] : rs[2] - accx[0];
    y[rowx[1]] = (MODE == 0) ? accx[1] : rs[3] - accx[1];
  }
}

// FASTE: the edge-compacted copy of the input vector, xe[i] = x[G[i]]
// (ig_gpu.cu: to_psell), gathered ahead of the product that reads it.
__global__ void __launch_bounds__(kCta) k_xgather(int n, const int32_t* __restrict__ G, const double* __restrict__ x,
                                                 double* __restrict__ xe) {
  const int i = blockIdx.x * kCta + threadIdx.x;
  const int g = i < n ? __ldg(G + i) : 0;  // static: before the wait
  pdl_entry();
  if (i < n) xe[i] = x[g];
}

// p . Ap over the canonical 256-row chunks (kernels.cuh: last_cta_total), then
// alpha / Breakdown exactly as the fused k_spmv<...,RED> does.
__global__ void __launch_bounds__(kCta) k_pap(int n, const double* __restrict__ p, const double* __restrict__ ap,
                                             PcgState* st, double* partials) {
  pdl_entry();
  if (pcg_done(st)) return;
  double pap;
  if (chunk_reduce(n, [&](int row) { return p[row] * ap[row]; }, partials, &st->counter[0], &pap)) {
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

// Prolongation fused with the correction (k_prolong on the pattern layout).
template <bool STREAM>
__global__ void __launch_bounds__(kPCta, IG_PPROLONG_MINB * (256 / kPCta)) k_pprolong(PSell P, const double* __restrict__ xc, double* cor, double* x,
                                                  const PcgState* st, const __grid_constant__ PValTab tab) {
  const int slice = blockIdx.x * (kPCta / 32) + (threadIdx.x >> 5);
  const uint4 mu = __ldg(reinterpret_cast<const uint4*>(P.meta + slice));  // static: before the wait
  // (Two-line slices exist only in square matrices: never in P.)
  int pr[4];
  uint2 gen;
  psell_rows<false>(P, mu, pr, gen);
  pdl_entry();
  if (pcg_done(st)) return;
  // The x being corrected is loaded before the product chain, not after it.
  const double x1 = pr[0] >= 0 ? x[pr[0]] : 0.0;
  const double x2 = pr[1] >= 0 ? x[pr[1]] : 0.0;
  double c, c2, cx[2];
  int row2, rowx[2];
  const int row = psell_slice<STREAM, false>(P, mu, gen, xc, c, row2, c2, &tab, rowx, cx);
  if (row < 0) return;
  cor[row] = c;
  x[row] = x1 + c;
  if (row2 >= 0) {
    cor[row2] = c2;
    x[row2] = x2 + c2;
  }
}

}  // namespace igk
