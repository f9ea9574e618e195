// Micro-benchmark of the coarse solve (kernels.cuh: k_coarse) in isolation:
// device time per launch vs rank, with and without the shared-memory staging.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false \
//        -I paper_1903_10977_b200/csrc profiles/coarse_micro.cu -o /tmp/cm && /tmp/cm
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "kernels.cuh"

using namespace igk;

int main() {
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaFuncSetAttribute(k_coarse<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_optin - 1024);
  for (int rank : {32, 64, 128, 216, 256}) {
    const int n = rank;
    const int64_t np = int64_t(rank) * (rank + 1) / 2, np_al = (np + 1) & ~int64_t(1);
    std::vector<double> Lp(np_al, 0.0);
    for (int j = 0; j < rank; ++j)
      for (int i = j; i < rank; ++i) Lp[j * rank - (j * (j - 1)) / 2 + (i - j)] = (i == j) ? 2.0 + j : 0.01 * ((i * 7 + j) % 13);
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) piv[k] = k + 1;
    std::vector<double> r(n, 1.0);
    double *dL, *dr, *dx;
    int* dp;
    cudaMalloc(&dL, np_al * 8);
    cudaMalloc(&dr, n * 8);
    cudaMalloc(&dx, n * 8);
    cudaMalloc(&dp, n * 4);
    cudaMemcpy(dL, Lp.data(), np_al * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dr, r.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, piv.data(), n * 4, cudaMemcpyHostToDevice);
    const int threads = (rank + 31) / 32 * 32;
    for (int smv = 0; smv < 2; ++smv) {
      const size_t smem = smv ? 8 * size_t(np_al + 2 * rank + 2) : 8 * size_t(2 * rank + 2);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto launch = [&] {
        if (smv)
          k_coarse<true><<<1, threads, smem>>>(n, rank, dL, dp, dr, dx, nullptr);
        else
          k_coarse<false><<<1, threads, smem>>>(n, rank, dL, dp, dr, dx, nullptr);
      };
      for (int w = 0; w < 5; ++w) launch();
      cudaEventRecord(e0);
      const int N = 200;
      for (int w = 0; w < N; ++w) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("rank %4d smem=%d: %8.2f us per launch (%s)\n", rank, smv, ms * 1e3 / N,
             cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(dL);
    cudaFree(dr);
    cudaFree(dx);
    cudaFree(dp);
  }
  return 0;
}
