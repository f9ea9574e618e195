// Canonical chunk reduction (kernels.cuh chunk_reduce) in isolation: the
// PCG vector kernels' cost at C4 size (n = 2.0 M) for variants of the
// writer fence, the last-CTA tail batch, the round width B and the grid.
// Every variant produces the same partials and the same total (checked
// bitwise against variant 0).  Timed per launch with CUDA events over 200
// back-to-back launches, L2 flushed (a 256 MB write) or warm.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false \
//        -I paper_1903_10977_b200/csrc profiles/reduce_micro.cu -o /tmp/rm && /tmp/rm
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

#include "kernels.cuh"

using namespace igk;

// TB < 0: predicated tail, all -TB loads in flight at once (+0 adds are
// no-ops: the running sum starts at +0 and is never -0).  TB == 0: no tail.
template <int B, bool FENCE_EACH, int TB>
__device__ __forceinline__ bool chunk_reduce_v(int n, const double* __restrict__ a, const double* __restrict__ b,
                                               double* partials, unsigned int* counter, double* total) {
  __shared__ double smc[2][B][8];
  const unsigned int nchunks = static_cast<unsigned int>((n + kCta - 1) / kCta);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int buf = 0;
  bool wrote = false;
  for (unsigned int c0 = blockIdx.x; c0 < nchunks; c0 += B * gridDim.x) {
    double v[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const unsigned int c = c0 + u * gridDim.x;
      const int i = static_cast<int>(c) * kCta + threadIdx.x;
      v[u] = (c < nchunks && i < n) ? a[i] * b[i] : 0.0;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
      for (int u = 0; u < B; ++u) v[u] = v[u] + __shfl_xor_sync(0xffffffffu, v[u], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < B; ++u) smc[buf][u][w] = v[u];
    }
    __syncthreads();
    if (threadIdx.x < B) {
      const unsigned int c = c0 + threadIdx.x * gridDim.x;
      if (c < nchunks) {
        const double* q = smc[buf][threadIdx.x];
        partials[c] = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
        if (FENCE_EACH) __threadfence();
        wrote = true;
      }
    }
    buf ^= 1;
  }
  if (!FENCE_EACH && wrote) __threadfence();
  __shared__ double sm8f[8];
  __shared__ bool is_last;
  __shared__ double tot;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int prev = atomicAdd(counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (TB == 0 || !is_last) return false;
  __threadfence();
  double acc = 0.0;
  unsigned int k = threadIdx.x;
  if (TB < 0) {
    constexpr int T = TB < 0 ? -TB : 1;
    for (; k < nchunks; k += T * kCta) {
      double q[T];
#pragma unroll
      for (int u = 0; u < T; ++u) q[u] = (k + u * kCta < nchunks) ? __ldcg(partials + k + u * kCta) : 0.0;
#pragma unroll
      for (int u = 0; u < T; ++u) acc = acc + q[u];
    }
  }
  for (; TB > 0 && k + (TB - 1) * kCta < nchunks; k += TB * kCta) {
    constexpr int T = TB > 0 ? TB : 1;
    double q[T];
#pragma unroll
    for (int u = 0; u < T; ++u) q[u] = __ldcg(partials + k + u * kCta);
#pragma unroll
    for (int u = 0; u < T; ++u) acc = acc + q[u];
  }
  for (; k < nchunks; k += kCta) acc = acc + __ldcg(partials + k);
  const double t = cta_reduce(acc, sm8f);
  if (threadIdx.x == 0) {
    tot = t;
    *counter = 0u;
  }
  __syncthreads();
  *total = tot;
  return true;
}

template <int B, bool FE, int TB>
__global__ void __launch_bounds__(kCta) k_dot(int n, const double* a, const double* b, double* partials,
                                              unsigned int* counter, double* out) {
  double t;
  if (chunk_reduce_v<B, FE, TB>(n, a, b, partials, counter, &t))
    if (threadIdx.x == 0) *out = t;
}
// Streaming floor: the same bytes, a per-CTA sum only (no partials, no tail).
__global__ void __launch_bounds__(kCta) k_stream(int n, const double* a, const double* b, double* out) {
  double s = 0.0;
  for (int i = blockIdx.x * kCta + threadIdx.x; i < n; i += gridDim.x * kCta) s = s + a[i] * b[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void k_flush(double* f, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) f[i] = 1.0;
}

int main() {
  const int n = 2000000;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::vector<double> ha(n), hb(n);
  for (int i = 0; i < n; ++i) {
    ha[i] = 1.0 / (1.0 + (i % 977));
    hb[i] = ((static_cast<long long>(i) * 7919) % 1013) * 1e-3 - 0.5;
  }
  double *a, *b, *part, *out, *fl;
  unsigned int* cnt;
  const size_t nfl = size_t(256) << 17;  // 256 MB
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMalloc(&part, 65536 * 8);
  cudaMalloc(&out, 64);
  cudaMalloc(&cnt, 64);
  cudaMalloc(&fl, nfl * 8);
  cudaMemset(cnt, 0, 64);
  cudaMemcpy(a, ha.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(b, hb.data(), n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double ref = 0.0;
  auto run = [&](const char* name, auto launch) {
    for (int flush = 0; flush < 2; ++flush) {
      const int reps = flush ? 50 : 200;
      float tot = 0.f;
      if (!flush) {  // back-to-back launches
        launch();
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&tot, e0, e1);
      } else {  // one launch after each flush (includes its launch latency)
        for (int r = 0; r < reps; ++r) {
          k_flush<<<4 * sms, 512>>>(fl, nfl);
          cudaEventRecord(e0);
          launch();
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          tot += ms;
        }
      }
      double o;
      cudaMemcpy(&o, out, 8, cudaMemcpyDeviceToHost);
      if (ref == 0.0) ref = o;
      std::printf("%-34s %s %7.2f us  %s\n", name, flush ? "cold" : "warm", tot * 1e3f / reps,
                  (std::memcmp(&o, &ref, 8) == 0) ? "same" : "DIFF");
    }
  };
  const unsigned g4 = 4 * sms;
  run("cur B4 fence-each tail8 g4", [&] { k_dot<4, true, 8><<<g4, kCta>>>(n, a, b, part, cnt, out); });
  run("B4 fence-once tail8 g4", [&] { k_dot<4, false, 8><<<g4, kCta>>>(n, a, b, part, cnt, out); });
  run("B4 fence-once tail32 g4", [&] { k_dot<4, false, 32><<<g4, kCta>>>(n, a, b, part, cnt, out); });
  run("B4 fence-each tail32 g4", [&] { k_dot<4, true, 32><<<g4, kCta>>>(n, a, b, part, cnt, out); });
  run("B8 fence-once tail32 g4", [&] { k_dot<8, false, 32><<<g4, kCta>>>(n, a, b, part, cnt, out); });
  run("B2 fence-once tail32 g4", [&] { k_dot<2, false, 32><<<g4, kCta>>>(n, a, b, part, cnt, out); });
  run("B4 fence-once tail32 g2", [&] { k_dot<4, false, 32><<<2 * sms, kCta>>>(n, a, b, part, cnt, out); });
  run("B4 fence-once tail32 g8", [&] { k_dot<4, false, 32><<<8 * sms, kCta>>>(n, a, b, part, cnt, out); });
  run("B2 fence-once tail32 g8", [&] { k_dot<2, false, 32><<<8 * sms, kCta>>>(n, a, b, part, cnt, out); });
  const unsigned nch = (n + kCta - 1) / kCta;
  run("B1 fence-once tail32 1/chunk", [&] { k_dot<1, false, 32><<<nch, kCta>>>(n, a, b, part, cnt, out); });
  run("B4 fence-once ptail32 g4", [&] { k_dot<4, false, -32><<<g4, kCta>>>(n, a, b, part, cnt, out); });
  run("B4 fence-once ptail16 g4", [&] { k_dot<4, false, -16><<<g4, kCta>>>(n, a, b, part, cnt, out); });
  run("B2 fence-once ptail32 g8", [&] { k_dot<2, false, -32><<<8 * sms, kCta>>>(n, a, b, part, cnt, out); });
  run("B4 fence-once tail32 balanced", [&] {
    const unsigned rounds = (nch + 4 * g4 - 1) / (4 * g4);
    k_dot<4, false, 32><<<(nch + 4 * rounds - 1) / (4 * rounds), kCta>>>(n, a, b, part, cnt, out);
  });
  run("B4 fence-once NO tail g4", [&] { k_dot<4, false, 0><<<g4, kCta>>>(n, a, b, part, cnt, out); });
  ref = -1.0;  // streaming floor: no value check
  run("stream floor g4", [&] { k_stream<<<g4, kCta>>>(n, a, b, out); });
  run("stream floor g8", [&] { k_stream<<<8 * sms, kCta>>>(n, a, b, out); });
  std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
