// blockfac.cuh — batched Schwarz block factorisation on the device
// (make_smoother's factorize_blocks, proj/src/smoothers.cpp:131-162; SURVEY.md
// §8(f) row 2): per pre-filter block, gather A_b from the level's CSR, drop
// DOFs while lambda_min(A_b) < filter_ratio * max diag(A_b) (the DOF with the
// largest |component| of the lowest eigenvector; smoothers.cpp:144-156), then
// the in-place lower Cholesky factor (Eigen::LLT, unblocked).
//
// Result contract: bit-identical to the host restatement
// (paper_1903_10977_b200/host/hierarchy.cpp: factorize_blocks, sym_eig_min,
// llt_lower): the same cyclic Jacobi sweeps, the same serial sums, the same
// IEEE divisions and square roots (-fmad=false: no contraction), so every
// block's kept DOFs and factor bits match.
//
// Shape: one thread per block (blocks are small: 87 % singletons on C4, at
// most a few dozen DOFs), working in a private slice of a global scratch arena
// (3 s_b^2 doubles: the block matrix, and for the eigen filter its Jacobi copy
// and the rotation accumulator), which stays in L1/L2.  Pass 1 factorises
// and records each block's post-filter size; the host scans the sizes; pass 2
// compacts DOF lists and factors into the output layout.
#pragma once

#include <cstdint>

#include "galerkin.cuh"

namespace igk {

__device__ __forceinline__ double csr_coeff(const GalCsr& A, int32_t i, int32_t j) {
  int32_t lo = A.ptr[i], hi = A.ptr[i + 1];
  while (lo < hi) {  // lower_bound
    const int32_t mid = (lo + hi) >> 1;
    if (A.col[mid] < j)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < A.ptr[i + 1] && A.col[lo] == j) ? A.val[lo] : 0.0;
}

// Blocks of kBfWarpMin..32 DOFs take the warp-per-block kernel.
constexpr int kBfWarpMin = 5;
constexpr int kBfWarps = 2;  // warps per CTA
constexpr size_t kBfWarpSmem = static_cast<size_t>(kBfWarps) * 3 * 32 * 32 * sizeof(double);

struct BlockFacArgs {
  GalCsr A;
  int32_t n_blocks;
  const int32_t* ptr;   // pre-filter block pointers
  const int32_t* dofs;  // pre-filter DOFs
  const int64_t* soff;  // scratch offset of block b (3 * sum of s^2 before b)
  double* scratch;
  int32_t* kdofs;       // kept DOFs, written at ptr[b] (pre-filter positions)
  int32_t* ksize;       // post-filter size; -1: every DOF filtered (error)
  double filter_ratio;
  int warp_big;         // blocks with kBfWarpMin <= s0 <= 32 go to k_block_factor_warp
};

// Column-major s x s block: a(i, j) = M[j * s + i].
__device__ void bf_gather(const GalCsr& A, const int32_t* d, int s, double* M) {
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < s; ++j) M[j * s + i] = csr_coeff(A, d[i], d[j]);
}

// sym_eig_min: cyclic Jacobi on a copy (A0 stays), V accumulates rotations.
__device__ void bf_eig_min(const double* A0, double* A, double* V, int s, double& lmin, int& imin,
                           double& maxdiag) {
  for (int k = 0; k < s * s; ++k) {
    A[k] = A0[k];
    V[k] = 0.0;
  }
  for (int i = 0; i < s; ++i) V[i * s + i] = 1.0;
  maxdiag = -INFINITY;
  for (int i = 0; i < s; ++i) {
    const double v = A0[i * s + i];
    maxdiag = (maxdiag < v) ? v : maxdiag;  // std::max(maxdiag, v)
  }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) {
        const double x = A[j * s + i] * A[j * s + i];
        tot = tot + x;
        if (i != j) off = off + x;
      }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int pp = 0; pp < s - 1; ++pp)
      for (int q = pp + 1; q < s; ++q) {
        const double apq = A[q * s + pp];
        if (apq == 0.0) continue;
        const double theta = (A[q * s + q] - A[pp * s + pp]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
        for (int k = 0; k < s; ++k) {
          const double akp = A[pp * s + k], akq = A[q * s + k];
          A[pp * s + k] = c * akp - sn * akq;
          A[q * s + k] = sn * akp + c * akq;
        }
        for (int k = 0; k < s; ++k) {
          const double apk = A[k * s + pp], aqk = A[k * s + q];
          A[k * s + pp] = c * apk - sn * aqk;
          A[k * s + q] = sn * apk + c * aqk;
        }
        for (int k = 0; k < s; ++k) {
          const double vkp = V[pp * s + k], vkq = V[q * s + k];
          V[pp * s + k] = c * vkp - sn * vkq;
          V[q * s + k] = sn * vkp + c * vkq;
        }
      }
  }
  imin = 0;
  for (int i = 1; i < s; ++i)
    if (A[i * s + i] < A[imin * s + imin]) imin = i;
  lmin = A[imin * s + imin];
}

// llt_lower (Eigen::LLT unblocked, in place; stops at a non-positive pivot
// leaving the rest as is, like Eigen's NumericalIssue return).
__device__ void bf_llt(double* M, int n) {
  for (int k = 0; k < n; ++k) {
    double x = M[k * n + k];
    double sq = 0.0;
    for (int j = 0; j < k; ++j) sq = sq + M[j * n + k] * M[j * n + k];
    x = x - sq;
    if (x <= 0.0) return;
    x = sqrt(x);
    M[k * n + k] = x;
    for (int i = k + 1; i < n; ++i) {
      double acc = 0.0;
      for (int j = 0; j < k; ++j) acc = acc + M[j * n + i] * M[j * n + k];
      M[k * n + i] = (M[k * n + i] - acc) / x;
    }
  }
  for (int j = 1; j < n; ++j)
    for (int i = 0; i < j; ++i) M[j * n + i] = 0.0;
}

__global__ void __launch_bounds__(128) k_block_factor(BlockFacArgs a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.n_blocks) return;
  const int32_t p0 = a.ptr[b];
  const int s0 = a.ptr[b + 1] - p0;
  if (a.warp_big && s0 >= kBfWarpMin && s0 <= 32) return;  // k_block_factor_warp
  int32_t* d = a.kdofs + p0;
  for (int i = 0; i < s0; ++i) d[i] = a.dofs[p0 + i];
  double* M = a.scratch + a.soff[b];  // s0^2: the block (then its factor)
  double* W = M + s0 * s0;            // 2 s0^2: Jacobi work
  int s = s0;
  bf_gather(a.A, d, s, M);
  bool err = false;
  if (a.filter_ratio > 0.0 && s > 1) {
    while (true) {
      if (s == 0) {
        err = true;
        break;
      }
      double lmin, maxdiag;
      int imin = 0;
      double* V = nullptr;
      if (s == 1) {
        lmin = M[0];
        maxdiag = M[0];
      } else {
        V = W + s0 * s0;  // Jacobi copy in W, rotations in V (slice: 3 s0^2)
        bf_eig_min(M, W, V, s, lmin, imin, maxdiag);
      }
      if (lmin >= a.filter_ratio * maxdiag) break;
      int worst = 0;
      if (s > 1) {
        const double* v0 = V + imin * s;
        for (int i = 1; i < s; ++i)
          if (fabs(v0[i]) > fabs(v0[worst])) worst = i;
      }
      for (int i = worst; i + 1 < s; ++i) d[i] = d[i + 1];  // erase (order kept)
      --s;
      bf_gather(a.A, d, s, M);
    }
  } else if (a.filter_ratio > 0.0 && s == 1 && !(M[0] >= a.filter_ratio * M[0])) {
    err = true;  // 1x1: a < ratio*a only for a < 0 (or NaN)
  }
  if (s == 0) err = true;
  if (err) {
    a.ksize[b] = -1;
    return;
  }
  bf_llt(M, s);
  a.ksize[b] = s;
}

// Warp-per-block variant for the larger blocks (kBfWarpMin <= s0 <= 32; the
// thread kernel skips them): the block, the Jacobi copy and the rotations sit
// in shared memory; entry-independent work (gathers, the three rotation
// loops, the LLT column updates) is spread over the lanes, every serial sum
// stays in one lane in the host's order, so the bits are the thread kernel's.

__device__ __forceinline__ void bf_gather_w(const GalCsr& A, const int32_t* d, int s, double* M, int lane) {
  for (int e = lane; e < s * s; e += 32) {
    const int i = e % s, j = e / s;
    M[j * s + i] = csr_coeff(A, d[i], d[j]);
  }
  __syncwarp();
}

__global__ void __launch_bounds__(32 * kBfWarps) k_block_factor_warp(BlockFacArgs a, const int32_t* __restrict__ big,
                                                                    int32_t n_big) {
  extern __shared__ double bsm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * kBfWarps + w;
  if (idx >= n_big) return;
  const int b = big[idx];
  const int32_t p0 = a.ptr[b];
  const int s0 = a.ptr[b + 1] - p0;
  double* M = bsm + w * 3 * 1024;
  double* Aw = M + 1024;
  double* V = Aw + 1024;
  int32_t* d = a.kdofs + p0;
  for (int i = lane; i < s0; i += 32) d[i] = a.dofs[p0 + i];
  __syncwarp();
  int s = s0;
  bf_gather_w(a.A, d, s, M, lane);
  bool err = false;
  if (a.filter_ratio > 0.0) {  // s0 > 1 here
    while (true) {
      if (s == 0) {
        err = true;
        break;
      }
      double lmin = 0.0, maxdiag = 0.0;
      int imin = 0;
      if (s == 1) {
        lmin = M[0];
        maxdiag = M[0];
      } else {
        for (int k = lane; k < s * s; k += 32) {
          Aw[k] = M[k];
          V[k] = 0.0;
        }
        __syncwarp();
        if (lane < s) V[lane * s + lane] = 1.0;
        maxdiag = -INFINITY;
        for (int i = 0; i < s; ++i) {
          const double v = M[i * s + i];
          maxdiag = (maxdiag < v) ? v : maxdiag;
        }
        __syncwarp();
        for (int sweep = 0; sweep < 100; ++sweep) {
          int stop = 0;
          if (lane == 0) {
            double off = 0.0, tot = 0.0;
            for (int i = 0; i < s; ++i)
              for (int j = 0; j < s; ++j) {
                const double x = Aw[j * s + i] * Aw[j * s + i];
                tot = tot + x;
                if (i != j) off = off + x;
              }
            stop = (off <= 1e-32 * tot || off == 0.0) ? 1 : 0;
          }
          if (__shfl_sync(0xffffffffu, stop, 0)) break;
          for (int pp = 0; pp < s - 1; ++pp)
            for (int q = pp + 1; q < s; ++q) {
              const double apq = Aw[q * s + pp];
              if (apq == 0.0) continue;  // warp-uniform (same smem value)
              const double theta = (Aw[q * s + q] - Aw[pp * s + pp]) / (2.0 * apq);
              const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
              const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
              __syncwarp();
              if (lane < s) {
                const int k = lane;
                const double akp = Aw[pp * s + k], akq = Aw[q * s + k];
                Aw[pp * s + k] = c * akp - sn * akq;
                Aw[q * s + k] = sn * akp + c * akq;
              }
              __syncwarp();
              if (lane < s) {
                const int k = lane;
                const double apk = Aw[k * s + pp], aqk = Aw[k * s + q];
                Aw[k * s + pp] = c * apk - sn * aqk;
                Aw[k * s + q] = sn * apk + c * aqk;
                const double vkp = V[pp * s + k], vkq = V[q * s + k];
                V[pp * s + k] = c * vkp - sn * vkq;
                V[q * s + k] = sn * vkp + c * vkq;
              }
              __syncwarp();
            }
        }
        for (int i = 1; i < s; ++i)
          if (Aw[i * s + i] < Aw[imin * s + imin]) imin = i;
        lmin = Aw[imin * s + imin];
      }
      if (lmin >= a.filter_ratio * maxdiag) break;
      int worst = 0;
      if (s > 1) {
        const double* v0 = V + imin * s;
        for (int i = 1; i < s; ++i)
          if (fabs(v0[i]) > fabs(v0[worst])) worst = i;
      }
      __syncwarp();
      if (lane == 0)
        for (int i = worst; i + 1 < s; ++i) d[i] = d[i + 1];
      __syncwarp();
      --s;
      bf_gather_w(a.A, d, s, M, lane);
    }
  }
  if (s == 0) err = true;
  if (err) {
    if (lane == 0) a.ksize[b] = -1;
    return;
  }
  // LLT (bf_llt), column k: the pivot by lane 0, rows i > k by lane i.
  bool stopped = false;
  for (int k = 0; k < s && !stopped; ++k) {
    double x = M[k * s + k];
    double sq = 0.0;
    for (int j = 0; j < k; ++j) sq = sq + M[j * s + k] * M[j * s + k];
    x = x - sq;
    if (x <= 0.0) {  // warp-uniform
      stopped = true;
      break;
    }
    x = sqrt(x);
    __syncwarp();
    if (lane == 0) M[k * s + k] = x;
    for (int i = k + 1 + lane; i < s; i += 32) {
      double acc = 0.0;
      for (int j = 0; j < k; ++j) acc = acc + M[j * s + i] * M[j * s + k];
      M[k * s + i] = (M[k * s + i] - acc) / x;
    }
    __syncwarp();
  }
  if (!stopped)
    for (int e = lane; e < s * s; e += 32) {
      const int i = e % s, j = e / s;
      if (i < j) M[j * s + i] = 0.0;
    }
  __syncwarp();
  double* out = a.scratch + a.soff[b];
  for (int e = lane; e < s * s; e += 32) out[e] = M[e];
  if (lane == 0) a.ksize[b] = s;
}

// Pass 2: compact kept DOFs and s x s factors into the post-filter layout.
__global__ void __launch_bounds__(128) k_block_compact(int32_t n_blocks, const int32_t* __restrict__ ptr,
                                                      const int32_t* __restrict__ kdofs,
                                                      const int32_t* __restrict__ ksize,
                                                      const int64_t* __restrict__ soff,
                                                      const double* __restrict__ scratch,
                                                      const int64_t* __restrict__ optr,
                                                      const int64_t* __restrict__ ofptr, int32_t* odofs,
                                                      double* ofac) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_blocks) return;
  const int s = ksize[b];
  const int32_t p0 = ptr[b];
  for (int i = 0; i < s; ++i) odofs[optr[b] + i] = kdofs[p0 + i];
  const double* M = scratch + soff[b];
  for (int k = 0; k < s * s; ++k) ofac[ofptr[b] + k] = M[k];
}

}  // namespace igk

namespace igk {

// Coarsest-level pivoted Cholesky on the device: LAPACK dpstf2 with
// UPLO = 'L' (MgHierarchy::build, proj/src/multigrid.cpp:57-73), restated
// step for step as the host's pstrf_lower (host/hierarchy.cpp): one CTA,
// row-parallel updates of WORK, the swaps and the DGEMV column update (each
// entry accumulates over k ascending, reference-BLAS column order), the
// MAXLOC pivot search (first maximum) by thread 0.  a: n x n column-major in
// global memory (in place); piv 1-based; *rank_out = returned rank.
__global__ void __launch_bounds__(1024) k_pstrf(int32_t n, double* a, int32_t* piv, double tol, double* work,
                                               int32_t* rank_out) {
  __shared__ int s_pvt;
  __shared__ double s_ajj;
  __shared__ int s_ret;
  auto A = [&](int i, int j) -> double& { return a[static_cast<size_t>(j) * n + i]; };
  const int t = threadIdx.x, nt = blockDim.x;
  for (int i = t; i < n; i += nt) piv[i] = i + 1;
  if (n == 0) {
    if (t == 0) *rank_out = 0;
    return;
  }
  if (t == 0) {
    int pvt = 0;
    double ajj = A(0, 0);
    for (int i = 1; i < n; ++i)
      if (A(i, i) > ajj) {
        pvt = i;
        ajj = A(pvt, pvt);
      }
    s_pvt = pvt;
    s_ajj = ajj;
    s_ret = (ajj <= 0.0 || isnan(ajj)) ? 0 : -1;
  }
  for (int i = t; i < 2 * n; i += nt) work[i] = 0.0;
  __syncthreads();
  if (s_ret == 0) {
    if (t == 0) *rank_out = 0;
    return;
  }
  const double dstop = tol >= 0.0 ? tol : n * 2.220446049250313e-16 * s_ajj;
  for (int j = 0; j < n; ++j) {
    for (int i = j + t; i < n; i += nt) {
      if (j > 0) work[i] = work[i] + A(i, j - 1) * A(i, j - 1);
      work[n + i] = A(i, i) - work[i];
    }
    __syncthreads();
    if (j > 0) {
      if (t == 0) {
        int pvt = j;
        for (int i = j + 1; i < n; ++i)
          if (work[n + i] > work[n + pvt]) pvt = i;
        s_pvt = pvt;
        s_ajj = work[n + pvt];
        if (s_ajj <= dstop || isnan(s_ajj)) {
          A(j, j) = s_ajj;
          s_ret = j;
        }
      }
      __syncthreads();
      if (s_ret >= 0) {
        if (t == 0) *rank_out = s_ret;
        return;
      }
    }
    const int pvt = s_pvt;
    if (j != pvt) {
      // Same entries as the host's serial swaps: the three index sets are
      // disjoint, so their order does not matter.
      if (t == 0) {
        A(pvt, pvt) = A(j, j);
        const double w = work[j];
        work[j] = work[pvt];
        work[pvt] = w;
        const int p = piv[j];
        piv[j] = piv[pvt];
        piv[pvt] = p;
      }
      for (int k = t; k < j; k += nt) {
        const double x = A(j, k);
        A(j, k) = A(pvt, k);
        A(pvt, k) = x;
      }
      for (int k = pvt + 1 + t; k < n; k += nt) {
        const double x = A(k, j);
        A(k, j) = A(k, pvt);
        A(k, pvt) = x;
      }
      for (int k = t; k < pvt - j - 1; k += nt) {
        const double x = A(j + 1 + k, j);
        A(j + 1 + k, j) = A(pvt, j + 1 + k);
        A(pvt, j + 1 + k) = x;
      }
    }
    __syncthreads();
    const double ajj = sqrt(s_ajj);
    if (t == 0) A(j, j) = ajj;
    if (j < n - 1) {
      const double r = 1.0 / ajj;
      for (int i = j + 1 + t; i < n; i += nt) {
        double v = A(i, j);
        for (int k = 0; k < j; ++k) v = v + (-A(j, k)) * A(i, k);
        A(i, j) = v * r;
      }
    }
    __syncthreads();
  }
  if (t == 0) *rank_out = n;
}

}  // namespace igk
