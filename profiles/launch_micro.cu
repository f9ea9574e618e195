// Floor of a dependent kernel chain on the device: a CUDA graph of K kernels
// launched with programmatic dependent launch (as the library launches every
// kernel), each reading what its predecessor wrote (one dependent L2 round
// trip) -- time per kernel vs grid size; and the same chain as ONE persistent
// kernel whose phases are separated by (a) a grid-wide arrival barrier and (b)
// __syncthreads in a single CTA.  The gap between these is the budget a fused
// small-level V-cycle can win.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        profiles/launch_micro.cu -o /tmp/lm && /tmp/lm
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__global__ void step(const double* __restrict__ in, double* out, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[(i * 7) % n] + 1.0;
}

__device__ unsigned int g_bar;

__global__ void persistent(double* a, double* b, int n, int phases) {
  // grid barrier by a monotone arrival counter
  unsigned int target = 0;
  for (int p = 0; p < phases; ++p) {
    const double* in = (p & 1) ? b : a;
    double* out = (p & 1) ? a : b;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
      out[i] = __ldcg(in + (i * 7) % n) + 1.0;
    target += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&g_bar, 1u);
      while (atomicAdd(&g_bar, 0u) < target) {
      }
      __threadfence();
    }
    __syncthreads();
  }
}

__global__ void single_cta(double* a, double* b, int n, int phases) {
  for (int p = 0; p < phases; ++p) {
    const double* in = (p & 1) ? b : a;
    double* out = (p & 1) ? a : b;
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = __ldcg(in + (i * 7) % n) + 1.0;
    __syncthreads();
  }
}

int main() {
  const int K = 200;
  double *a, *b;
  cudaMalloc(&a, sizeof(double) * (1 << 22));
  cudaMalloc(&b, sizeof(double) * (1 << 22));
  cudaMemset(a, 0, sizeof(double) * (1 << 22));
  cudaMemset(b, 0, sizeof(double) * (1 << 22));
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int n : {256, 4096, 37703, 267238, 2000000}) {
    for (int pdl = 0; pdl <= 1; ++pdl) {
      cudaGraph_t g;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
      for (int k = 0; k < K; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((n + 255) / 256);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, step, (const double*)((k & 1) ? b : a), (k & 1) ? a : b, n);
      }
      cudaStreamEndCapture(st, &g);
      cudaGraphExec_t ex;
      cudaGraphInstantiate(&ex, g, 0);
      for (int w = 0; w < 3; ++w) cudaGraphLaunch(ex, st);
      cudaEventRecord(e0, st);
      for (int w = 0; w < 5; ++w) cudaGraphLaunch(ex, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      std::printf("graph chain n=%8d pdl=%d: %.2f us per kernel\n", n, pdl, ms * 1e3 / (5 * K));
      std::fflush(stdout);
      cudaGraphExecDestroy(ex);
      cudaGraphDestroy(g);
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int grid : {sms, 2 * sms}) {
      unsigned int zero = 0;
      cudaDeviceSynchronize();
      cudaMemcpyToSymbol(g_bar, &zero, sizeof(zero));
      cudaDeviceSynchronize();
      persistent<<<grid, 256, 0, st>>>(a, b, n, 10);
      cudaDeviceSynchronize();
      cudaMemcpyToSymbol(g_bar, &zero, sizeof(zero));
      cudaDeviceSynchronize();
      cudaEventRecord(e0, st);
      persistent<<<grid, 256, 0, st>>>(a, b, n, K);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      std::printf("persistent grid=%d n=%8d: %.2f us per phase\n", grid, n, ms * 1e3 / K);
    }
    if (n <= 37703) {
      for (int th : {256, 1024}) {
        single_cta<<<1, th, 0, st>>>(a, b, n, 10);
        cudaEventRecord(e0, st);
        single_cta<<<1, th, 0, st>>>(a, b, n, K);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        std::printf("single CTA (%d threads) n=%8d: %.2f us per phase\n", th, n, ms * 1e3 / K);
      }
    }
  }
  std::printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
