// Latency of one warp running kernels.cuh spmv_grp_item (4 rows x 125
// entries, 8 lanes per row) and of sell_row (thread-per-row), cycles from
// clock64 -- the small-level SpMV is latency-bound, this is its floor.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false \
//        -I paper_1903_10977_b200/csrc profiles/grp_micro.cu -o /tmp/gm && /tmp/gm
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "kernels.cuh"

using namespace igk;

// Thread-per-row, SELL column-major, chunks of U entries with all loads of a
// chunk issued before its ordered adds; PIPE: next chunk's loads issued before
// this chunk's adds.
template <int U, bool PIPE>
__device__ __forceinline__ double row_lat(const Sell& A, int row, const double* __restrict__ x) {
  const int64_t base = A.slice_ptr[row >> 5] + (row & 31);
  const int len = A.rowinfo[row] & 0xffff;
  const double* vp = A.val + base;
  const int32_t* cp = A.col + base;
  double acc = 0.0;
  double v[U];
  int32_t c[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    v[u] = u < len ? __ldg(vp + u * 32) : 0.0;
    c[u] = u < len ? __ldg(cp + u * 32) : row;
  }
  for (int k0 = 0; k0 < len; k0 += U) {
    double xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = __ldg(x + c[u]);
    double vn[U];
    int32_t cn[U];
    if (PIPE) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + U + u;
        vn[u] = k < len ? __ldg(vp + k * 32) : 0.0;
        cn[u] = k < len ? __ldg(cp + k * 32) : row;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k0 + u < len) acc = acc + v[u] * xv[u];
    if (PIPE) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        v[u] = vn[u];
        c[u] = cn[u];
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = k0 + U + u;
        v[u] = k < len ? __ldg(vp + k * 32) : 0.0;
        c[u] = k < len ? __ldg(cp + k * 32) : row;
      }
    }
  }
  return acc;
}

__global__ void k_row_lat(Sell A, const double* x, double* y, long long* out) {
  double a = 0.0;
  long long t0 = clock64();
  if (threadIdx.x < 4) a = row_lat<16, false>(A, threadIdx.x, x);
  __syncwarp();
  long long t1 = clock64();
  if (threadIdx.x < 4) a += row_lat<16, false>(A, threadIdx.x, x);
  __syncwarp();
  long long t2 = clock64();
  if (threadIdx.x < 4) a += row_lat<16, true>(A, threadIdx.x, x);
  __syncwarp();
  long long t3 = clock64();
  if (threadIdx.x < 4) a += row_lat<32, true>(A, threadIdx.x, x);
  __syncwarp();
  long long t4 = clock64();
  if (threadIdx.x < 4) y[8 + threadIdx.x] = a;
  if (threadIdx.x == 0) {
    out[3] = t1 - t0;
    out[4] = t2 - t1;
    out[5] = t3 - t2;
    out[6] = t4 - t3;
  }
}

__global__ void k_grp_lat(Sell A, const double* x, double* y, long long* out) {
  long long t0 = clock64();
  spmv_grp_item<0, 8>(A, threadIdx.x, x, y, nullptr);
  __syncwarp();
  long long t1 = clock64();
  spmv_grp_item<0, 8>(A, threadIdx.x, x, y, nullptr);  // warm (L1/L2 hot)
  __syncwarp();
  long long t2 = clock64();
  double acc = 0.0;
  if (threadIdx.x < 4) acc = sell_row<false, 3>(A, threadIdx.x, x);
  __syncwarp();
  long long t3 = clock64();
  if (threadIdx.x < 4) y[4 + threadIdx.x] = acc;
  if (threadIdx.x == 0) {
    out[0] = t1 - t0;
    out[1] = t2 - t1;
    out[2] = t3 - t2;
  }
}

int main() {
  const int nr = 32, len = 125;  // one SELL slice
  std::vector<int64_t> sp = {0, int64_t(len) * 32};
  std::vector<int32_t> info(nr, len), col(len * 32);
  std::vector<double> val(len * 32), x(4096, 1.0);
  for (int r = 0; r < nr; ++r)
    for (int k = 0; k < len; ++k) {
      col[k * 32 + r] = (r * 37 + k * 13) % 4096;
      val[k * 32 + r] = 1.0 + 1e-3 * k;
    }
  Sell A{};
  A.n_rows = 4;
  A.n_cols = 4096;
  int64_t* dsp;
  int32_t *dinfo, *dcol;
  double *dval, *dx, *dy, *dd;
  int32_t* doff;
  long long* dout;
  cudaMalloc(&dsp, 16);
  cudaMalloc(&dinfo, nr * 4);
  cudaMalloc(&dcol, len * 32 * 4);
  cudaMalloc(&dval, len * 32 * 8);
  cudaMalloc(&dx, 4096 * 8);
  cudaMalloc(&dy, 64 * 8);
  cudaMalloc(&dd, 8);
  cudaMalloc(&doff, 4);
  cudaMalloc(&dout, 64);
  cudaMemcpy(dsp, sp.data(), 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dinfo, info.data(), nr * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dcol, col.data(), len * 32 * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dval, val.data(), len * 32 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, x.data(), 4096 * 8, cudaMemcpyHostToDevice);
  A.slice_ptr = dsp;
  A.rowinfo = dinfo;
  A.col = dcol;
  A.val = dval;
  A.dict_w = 1;
  A.dval = dd;
  A.doff = doff;
  for (int rep = 0; rep < 3; ++rep) {
    k_grp_lat<<<1, 32>>>(A, dx, dy, dout);
    k_row_lat<<<1, 32>>>(A, dx, dy, dout);
    cudaDeviceSynchronize();
    long long h[7];
    cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost);
    printf("grp item cold %lld cycles, warm %lld cycles; sell_row warm %lld cycles (%s)\n", h[0], h[1], h[2],
           cudaGetErrorString(cudaGetLastError()));
    printf("row_lat U16 cold %lld warm %lld; U16 pipelined %lld; U32 pipelined %lld\n", h[3], h[4], h[5], h[6]);
  }
  return 0;
}
