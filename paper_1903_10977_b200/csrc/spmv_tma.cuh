// TMA-staged, compacted SELL SpMV for the large levels (sm_100a).
//
// Layout ("TSell"): rows in SELL-32 slices; per slice only the matrix words
// the row dictionary does not supply are stored, compacted over the lanes
// that need them (cmask: lanes with explicit columns, vmask: lanes with
// explicit values), in k-chunks of kKC entries:  cols [chunk][kk][jc] int32,
// vals [chunk][kk][jv] double.  A chunk is one contiguous run of bytes, so a
// warp streams its slice with cp.async.bulk (TMA bulk copies, completion on
// an mbarrier) into a double-buffered shared-memory stage, two tasks ahead of
// the compute; no register prefetch, no partially used sectors.  Each lane
// still sums its own row sequentially in ascending column order (the parity
// contract), reading values / columns from shared memory or the dictionary
// and gathering x.
//
// CTA = 8 warps = 256 consecutive rows = one reduction chunk; the grid is
// persistent over chunks, so p.Ap partials are written per chunk and reduced
// by the last CTA exactly as in k_spmv.
#pragma once

#include "kernels.cuh"

namespace igk {

constexpr int kKC = 16;  // k-entries per TMA chunk
constexpr int kTColB = kKC * 32 * 4;
constexpr int kTValB = kKC * 32 * 8;
constexpr int kTStageB = kTColB + kTValB;
constexpr int kTSmem = 8 * 2 * kTStageB;  // 8 warps x 2 stages

struct TSliceMeta {
  int64_t col_off;  // int32 index into cols
  int64_t val_off;  // double index into vals
  uint32_t cmask, vmask;
  int32_t nch, pad;
};

struct TSell {
  int32_t n_rows, n_slices, n_chunks;  // n_chunks = ceil(n_rows / 256)
  const TSliceMeta* meta;
  const int32_t* rowinfo;
  const int32_t* cols;
  const double* vals;
  int32_t dict_w;
  const double* dval;
  const int32_t* doff;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(smem_u32(b)), "r"(parity)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

template <int MODE, bool RED>
__global__ void __launch_bounds__(kCta) k_spmv_tma(TSell A, const double* __restrict__ x, double* y,
                                                   const double* rsrc, PcgState* st, double* partials) {
  pdl_entry();
  extern __shared__ __align__(128) unsigned char tsm[];
  __shared__ unsigned long long mbar[8][2];
  __shared__ double sm8[8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = tsm + w * 2 * kTStageB;
  if (lane == 0) {
    mbar_init(&mbar[w][0]);
    mbar_init(&mbar[w][1]);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const int G = gridDim.x, NC = A.n_chunks;
  auto nch_of = [&](int chunk) {
    const int s = chunk * 8 + w;
    return (chunk < NC && s < A.n_slices) ? A.meta[s].nch : 0;
  };
  // Prefetch iterator over this warp's (chunk, k-chunk) tasks (lane 0).
  int pc = blockIdx.x, pk = 0, pn = nch_of(blockIdx.x), issued = 0;
  auto skip_empty = [&]() {
    while (pc < NC && pk >= pn) {
      pc += G;
      pk = 0;
      pn = nch_of(pc);
    }
  };
  auto issue = [&]() {
    if (pc >= NC) return;
    const TSliceMeta m = A.meta[pc * 8 + w];
    const int st_i = issued & 1;
    unsigned long long* bar = &mbar[w][st_i];
    unsigned char* dst = wbase + st_i * kTStageB;
    const unsigned ec = __popc(m.cmask), ev = __popc(m.vmask);
    const unsigned cb = kKC * ec * 4, vb = kKC * ev * 8;
    mbar_expect(bar, cb + vb);
    if (cb) bulk_g2s(dst, A.cols + m.col_off + static_cast<int64_t>(pk) * kKC * ec, cb, bar);
    if (vb) bulk_g2s(dst + kTColB, A.vals + m.val_off + static_cast<int64_t>(pk) * kKC * ev, vb, bar);
    ++issued;
    ++pk;
    skip_empty();
  };
  if (lane == 0) {
    skip_empty();
    issue();
    issue();
  }
  const unsigned lt = (1u << lane) - 1u;
  int consumed = 0;
  for (int chunk = blockIdx.x; chunk < NC; chunk += G) {
    const int s = chunk * 8 + w;
    const int row = s * 32 + lane;
    int nch = 0, len = 0, vd = 0, od = 0;
    unsigned cmask = 0, vmask = 0;
    if (s < A.n_slices) {
      const TSliceMeta m = A.meta[s];
      nch = m.nch;
      cmask = m.cmask;
      vmask = m.vmask;
    }
    if (row < A.n_rows) {
      const int info = A.rowinfo[row];
      len = info & 0xffff;
      vd = (info >> 16) & 0xff;
      od = (info >> 24) & 0xff;
    }
    const int ec = __popc(cmask), ev = __popc(vmask);
    const int jc = __popc(cmask & lt), jv = __popc(vmask & lt);
    const double* dv = A.dval + (vd > 0 ? (vd - 1) * A.dict_w : 0);
    const int32_t* dc = A.doff + (od > 0 ? (od - 1) * A.dict_w : 0);
    double acc = 0.0;
    for (int kc = 0; kc < nch; ++kc) {
      const int st_i = consumed & 1;
      mbar_wait(&mbar[w][st_i], (consumed >> 1) & 1);
      const int32_t* scol = reinterpret_cast<const int32_t*>(wbase + st_i * kTStageB);
      const double* sval = reinterpret_cast<const double*>(wbase + st_i * kTStageB + kTColB);
#pragma unroll
      for (int h = 0; h < kKC; h += 8) {
        double v[8], xv[8];
        int32_t c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int kk = h + u, k = kc * kKC + kk;
          v[u] = 0.0;
          c[u] = row;
          if (k < len) {
            v[u] = vd ? __ldg(dv + k) : sval[kk * ev + jv];
            c[u] = od ? row + __ldg(dc + k) : scol[kk * ec + jc];
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = (kc * kKC + h + u < len) ? __ldg(x + c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (kc * kKC + h + u < len) acc = acc + v[u] * xv[u];
      }
      __syncwarp();
      if (lane == 0) issue();
      ++consumed;
    }
    double prod = 0.0;
    if (row < A.n_rows) {
      const double out = (MODE == 0) ? acc : rsrc[row] - acc;
      y[row] = out;
      if (RED) prod = x[row] * out;
    }
    if (RED) {
      const double part = cta_reduce(prod, sm8);
      if (threadIdx.x == 0) partials[chunk] = part;
      __syncthreads();
    }
  }
  if (RED) {
    double pap;
    if (grid_finish(static_cast<unsigned>(NC), partials, &st->counter[0], &pap)) {
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

// Same compact layout, read directly (no TMA staging): the chunked layout
// [chunk][kk][j] is simply [k][j] per slice, so at step k the lanes that need
// explicit words read a contiguous run of ec ints / ev doubles -- every
// fetched sector is fully used -- while the thread-per-row structure keeps
// the high occupancy of k_spmv.  One 256-row chunk per CTA.
template <int MODE, bool RED>
__global__ void __launch_bounds__(kCta) k_spmv_cmp(TSell A, const double* __restrict__ x, double* y,
                                                   const double* rsrc, PcgState* st, double* partials) {
  pdl_entry();
  const int row = blockIdx.x * kCta + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int s = row >> 5;
  double prod = 0.0;
  if (row < A.n_rows) {
    const TSliceMeta m = A.meta[s];
    const int info = A.rowinfo[row];
    const int len = info & 0xffff;
    const int vd = (info >> 16) & 0xff;
    const int od = (info >> 24) & 0xff;
    const unsigned lt = (1u << lane) - 1u;
    const int ec = __popc(m.cmask), ev = __popc(m.vmask);
    const int32_t* cp = A.cols + m.col_off + __popc(m.cmask & lt);
    const double* vp = A.vals + m.val_off + __popc(m.vmask & lt);
    const double* dv = A.dval + (vd > 0 ? (vd - 1) * A.dict_w : 0);
    const int32_t* dc = A.doff + (od > 0 ? (od - 1) * A.dict_w : 0);
    double acc = 0.0;
    int k = 0;
    for (; k + 8 <= len; k += 8) {
      double v[8], xv[8];
      int32_t c[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        v[u] = vd ? __ldg(dv + k + u) : __ldcs(vp + static_cast<int64_t>(k + u) * ev);
        c[u] = od ? row + __ldg(dc + k + u) : __ldcs(cp + static_cast<int64_t>(k + u) * ec);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = __ldg(x + c[u]);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = acc + v[u] * xv[u];
    }
    for (; k < len; ++k) {
      const double v = vd ? __ldg(dv + k) : __ldcs(vp + static_cast<int64_t>(k) * ev);
      const int32_t c = od ? row + __ldg(dc + k) : __ldcs(cp + static_cast<int64_t>(k) * ec);
      acc = acc + v * __ldg(x + c);
    }
    const double out = (MODE == 0) ? acc : rsrc[row] - acc;
    y[row] = out;
    if (RED) prod = x[row] * out;
  }
  if (RED) {
    double pap;
    if (last_cta_total(prod, partials, &st->counter[0], &pap)) {
      if (threadIdx.x == 0) {
        st->pap = pap;
        if (pap <= 0.0) {
          st->status = ST_BREAKDOWN;
          st->done = 1;
        } else {
          st->alpha = st->rz / pap;
        }
      }
    }
  }
}

}  // namespace igk
