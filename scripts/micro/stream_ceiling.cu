// Memory ceiling of the STEP access pattern on B200: read 3 streams, write 2
// (fp64, 16384^2), no arithmetic.  Variants: (a) plain 128-bit loads, grid-stride;
// (b) CUDA's cudaMemcpy D2D for reference.  Reports GB/s counting 40 B/elem.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rw5(const double2* __restrict__ a, const double2* __restrict__ b, const double2* __restrict__ c,
                    double2* __restrict__ x, double2* __restrict__ y, long n2) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  for (; i < n2; i += stride * 4) {
    double2 va[4], vb[4], vc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) if (i + k * stride < n2) { va[k] = __ldcs(a + i + k * stride); vb[k] = __ldcs(b + i + k * stride); vc[k] = __ldcs(c + i + k * stride); }
#pragma unroll
    for (int k = 0; k < 4; ++k) if (i + k * stride < n2) {
      double2 r; r.x = va[k].x + vb[k].x; r.y = va[k].y + vc[k].y;
      __stcs(x + i + k * stride, r); __stcs(y + i + k * stride, vc[k]); }
  }
}
int main() {
  const long n = 16384L * 16384L, n2 = n / 2;
  double *a, *b, *c, *x, *y;
  for (double** p : {&a, &b, &c, &x, &y}) { cudaMalloc(p, n * 8); cudaMemset(*p, 0, n * 8); }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocks : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) for (int th : {256, 512}) {
    for (int w = 0; w < 2; ++w) rw5<<<blocks, th>>>((double2*)a, (double2*)b, (double2*)c, (double2*)x, (double2*)y, n2);
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) rw5<<<blocks, th>>>((double2*)a, (double2*)b, (double2*)c, (double2*)x, (double2*)y, n2);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
    printf("rw5 blocks=%d th=%d: %.3f ms  %.0f GB/s\n", blocks, th, ms, 40.0 * n / (ms * 1e-3) / 1e9);
  }
  cudaEventRecord(e0);
  for (int it = 0; it < 10; ++it) cudaMemcpyAsync(x, a, n * 8, cudaMemcpyDeviceToDevice);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
  printf("memcpy D2D 2.15 GB: %.3f ms  %.0f GB/s (read+write)\n", ms, 16.0 * n / (ms * 1e-3) / 1e9);
  return 0;
}
