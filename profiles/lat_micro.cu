// Dependent-chain latencies on the device (cycles per op, one warp):
// DADD, DMUL, DFMA, the exact division (kernels.cuh exact_div), div.rn.f64,
// SHFL of a double, LDS->DMUL->DADD, and the coarse-solve step pattern.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false \
//        -I paper_1903_10977_b200/csrc profiles/lat_micro.cu -o /tmp/lat && /tmp/lat
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels.cuh"

using namespace igk;

constexpr int N = 1024;

__global__ void lat(double a, double b, long long* out, double* sink) {
  __shared__ double sh[64];
  for (int i = threadIdx.x; i < 64; i += 32) sh[i] = 1.0 + 1e-3 * i;
  __syncwarp();
  double x = a;
  const double rb = 1.0 / b;
  long long t0, t1;
  // DADD
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x + b;
  t1 = clock64();
  out[0] = t1 - t0;
  // DMUL
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x * b;
  t1 = clock64();
  out[1] = t1 - t0;
  // DFMA
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __fma_rn(x, b, a);
  t1 = clock64();
  out[2] = t1 - t0;
  // exact_div
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = exact_div(x, b, rb) + a;
  t1 = clock64();
  out[3] = t1 - t0;
  // IEEE division
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = x / b + a;
  t1 = clock64();
  out[4] = t1 - t0;
  // SHFL of a double (value-dependent chain)
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + a;
  t1 = clock64();
  out[5] = t1 - t0;
  // LDS + DMUL + DADD with the LDS address independent of the chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = x - sh[i & 63] * b;
  t1 = clock64();
  out[6] = t1 - t0;
  // coarse step: exact_div -> shfl -> mul/sub
  t0 = clock64();
  for (int i = 0; i < N; ++i) {
    double y = exact_div(x, b, rb);
    y = __shfl_sync(0xffffffffu, y, i & 31);
    x = x - sh[i & 63] * y;
  }
  t1 = clock64();
  out[7] = t1 - t0;
  // coarse step as in k_coarse: selects + volatile publication
  {
    volatile double* pub = sh;
    const int i = threadIdx.x;
    double y = x;
    t0 = clock64();
    for (int j = 0; j < N; ++j) {
      const double q = exact_div(y, b, rb);
      const double yj = __shfl_sync(0xffffffffu, q, j & 31);
      const double upd = y - sh[(j + i) & 63] * yj;
      y = (i == (j & 31)) ? yj : ((i > (j & 31)) ? upd : y);
      if (i == (j & 31)) pub[32 + (j & 31)] = yj;
    }
    t1 = clock64();
    out[8] = t1 - t0;
    x = y;
  }
  // same without the publication
  {
    const int i = threadIdx.x;
    double y = x;
    t0 = clock64();
    for (int j = 0; j < N; ++j) {
      const double q = exact_div(y, b, rb);
      const double yj = __shfl_sync(0xffffffffu, q, j & 31);
      const double upd = y - sh[(j + i) & 63] * yj;
      y = (i == (j & 31)) ? yj : ((i > (j & 31)) ? upd : y);
    }
    t1 = clock64();
    out[9] = t1 - t0;
    x = y;
  }
  sink[threadIdx.x] = x;
}

int main() {
  long long* d;
  double* s;
  cudaMalloc(&d, 16 * sizeof(long long));
  cudaMalloc(&s, 64 * sizeof(double));
  for (int rep = 0; rep < 2; ++rep) lat<<<1, 32>>>(1.0000001, 0.9999999, d, s);
  long long h[16];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"DADD", "DMUL", "DFMA", "exact_div+DADD", "div.rn+DADD", "SHFL.f64+DADD", "LDS+DMUL+DADD",
                         "coarse step (div,shfl,mul,sub)", "k_coarse step (selects+STS)", "k_coarse step (selects)"};
  for (int i = 0; i < 10; ++i) printf("%-32s %7.1f cycles/iter\n", names[i], double(h[i]) / N);
  return 0;
}
