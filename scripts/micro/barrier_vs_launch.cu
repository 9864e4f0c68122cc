// Micro-benchmark: the cost of a pass-phase boundary on B200.
//   (1) graph of N dependent launches of a near-empty persistent kernel
//       (296 CTAs x 256 threads, each CTA copies a 2 KB control block into
//       shared memory first, as every pass kernel does);
//   (2) one cooperative kernel with N grid barriers (atomic arrive + spin on a
//       generation word), same grid and the same per-phase control-block copy;
//   (3) the same without the per-phase copy.
// Prints microseconds per boundary.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kCtlWords = 256;  // 2 KB

__device__ __forceinline__ void copy_ctl(const unsigned long long* g, unsigned long long* s) {
  for (int i = threadIdx.x; i < kCtlWords; i += blockDim.x) s[i] = __ldcg(g + i);
  __syncthreads();
}

__global__ void __launch_bounds__(256, 2) phase_kernel(const unsigned long long* ctl, unsigned long long* sink) {
  __shared__ unsigned long long s[kCtlWords];
  copy_ctl(ctl, s);
  if (s[threadIdx.x & 7] == 12345ull) sink[blockIdx.x] = 1;
}

__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = *gen;
    __threadfence();
    const unsigned arrived = atomicAdd(count, 1u);
    if (arrived == nblocks - 1) {
      *count = 0u;
      __threadfence();
      atomicExch((unsigned*)gen, g + 1u);
    } else {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
      } while (v == g);
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256, 2) barrier_kernel(const unsigned long long* ctl, unsigned long long* sink,
                                                         unsigned* count, unsigned* gen, int n, int copy) {
  __shared__ unsigned long long s[kCtlWords];
  for (int k = 0; k < n; ++k) {
    if (copy) copy_ctl(ctl, s);
    if (s[threadIdx.x & 7] == 12345ull) sink[blockIdx.x] = 1;
    grid_barrier(count, gen, gridDim.x);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 2, N = 2000;
  unsigned long long *ctl, *sink;
  unsigned *count, *gen;
  cudaMalloc(&ctl, kCtlWords * 8);
  cudaMemset(ctl, 0, kCtlWords * 8);
  cudaMalloc(&sink, grid * 8);
  cudaMalloc(&count, 4);
  cudaMalloc(&gen, 4);
  cudaMemset(count, 0, 4);
  cudaMemset(gen, 0, 4);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  // (1) graph of N launches
  const int per_graph = 100;
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int k = 0; k < per_graph; ++k) phase_kernel<<<grid, 256, 0, st>>>(ctl, sink);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
  cudaEventRecord(a, st);
  for (int k = 0; k < N / per_graph; ++k) cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"graph_launch_us\": %.3f, ", 1000.0 * ms / N);
  // (2), (3) cooperative kernel with N barriers
  for (int copy = 1; copy >= 0; --copy) {
    int n = N;
    void* args[] = {&ctl, &sink, &count, &gen, &n, &copy};
    cudaLaunchCooperativeKernel((void*)barrier_kernel, grid, 256, args, 0, st);  // warm-up
    cudaEventRecord(a, st);
    cudaLaunchCooperativeKernel((void*)barrier_kernel, grid, 256, args, 0, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("\"grid_barrier%s_us\": %.3f%s", copy ? "_with_ctl_copy" : "", 1000.0 * ms / N, copy ? ", " : "");
  }
  const cudaError_t e = cudaDeviceSynchronize();
  printf(", \"grid\": %d, \"status\": \"%s\"}\n", grid, cudaGetErrorString(e));
  return 0;
}
