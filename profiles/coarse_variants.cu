// Coarse-solve kernels in isolation (kernels.cuh): the multi-warp pipeline
// k_coarse and the single-warp k_coarse_warp, bit-compared on random pivoted
// factors and timed per launch (CUDA events, 200 back-to-back launches).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false \
//        -I paper_1903_10977_b200/csrc profiles/coarse_variants.cu -o /tmp/cv && /tmp/cv
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "kernels.cuh"

using namespace igk;

template <int R>
float run_warp(int n, int rank, const double* dL, const int* dp, const double* dr, double* dx, size_t smem, int reps) {
  cudaFuncSetAttribute(k_coarse_warp<R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_coarse_warp<R, true><<<1, 32, smem>>>(n, rank, dL, dp, dr, dx, nullptr);
  cudaEventRecord(e0);
  for (int w = 0; w < reps; ++w) k_coarse_warp<R, true><<<1, 32, smem>>>(n, rank, dL, dp, dr, dx, nullptr);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / reps;
}

int main() {
  cudaFuncSetAttribute(k_coarse<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  for (int rank : {36, 155, 216, 256}) {
    const int n = rank + 3;
    const int64_t np = int64_t(rank) * (rank + 1) / 2, np_al = (np + 1) & ~int64_t(1);
    std::vector<double> Lp(np_al, 0.0);
    for (int j = 0; j < rank; ++j)
      for (int i = j; i < rank; ++i) Lp[j * rank - (j * (j - 1)) / 2 + (i - j)] = (i == j) ? 1.5 + U(rng) : 0.3 * U(rng);
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) piv[k] = (k * 37 + 11) % n + 1;  // a permutation when gcd(37, n) == 1
    std::vector<double> r(n);
    for (auto& v : r) v = U(rng);
    double *dL, *dr, *dx0, *dx1;
    int* dp;
    cudaMalloc(&dL, np_al * 8);
    cudaMalloc(&dr, n * 8);
    cudaMalloc(&dx0, n * 8);
    cudaMalloc(&dx1, n * 8);
    cudaMalloc(&dp, n * 4);
    cudaMemcpy(dL, Lp.data(), np_al * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dr, r.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, piv.data(), n * 4, cudaMemcpyHostToDevice);
    const int threads = (rank + 31) / 32 * 32;
    const size_t smem0 = 8 * size_t(np_al + 2 * rank + 2), smem1 = 8 * size_t(np_al);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 200;
    k_coarse<true, false><<<1, threads, smem0>>>(n, rank, dL, dp, dr, dx0, nullptr);
    cudaEventRecord(e0);
    for (int w = 0; w < reps; ++w) k_coarse<true, false><<<1, threads, smem0>>>(n, rank, dL, dp, dr, dx0, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms0 = 0;
    cudaEventElapsedTime(&ms0, e0, e1);
    float us1 = 0;
    switch ((rank + 31) / 32) {
      case 2: us1 = run_warp<2>(n, rank, dL, dp, dr, dx1, smem1, reps); break;
      case 5: us1 = run_warp<5>(n, rank, dL, dp, dr, dx1, smem1, reps); break;
      case 7: us1 = run_warp<7>(n, rank, dL, dp, dr, dx1, smem1, reps); break;
      case 8: us1 = run_warp<8>(n, rank, dL, dp, dr, dx1, smem1, reps); break;
    }
    std::vector<double> x0(n), x1(n);
    cudaMemcpy(x0.data(), dx0, n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(x1.data(), dx1, n * 8, cudaMemcpyDeviceToHost);
    const bool same = std::memcmp(x0.data(), x1.data(), n * 8) == 0;
    std::printf("rank %4d: multi-warp %7.2f us, single-warp %7.2f us, bit-identical %s (%s)\n", rank,
                ms0 * 1e3f / reps, us1, same ? "yes" : "NO", cudaGetErrorString(cudaGetLastError()));
    cudaFree(dL);
    cudaFree(dr);
    cudaFree(dx0);
    cudaFree(dx1);
    cudaFree(dp);
  }
  return 0;
}
