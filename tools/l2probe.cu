// L2-resident vs HBM read bandwidth probe: every CTA streams its slice of a
// buffer `reps` times with 256-bit loads (one launch), B200 sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double* __restrict__ a, size_t n, int reps, double* out) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)(blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += (size_t)gridDim.x * blockDim.x * 4) {
      double v0, v1, v2, v3;
      asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v0), "=d"(v1), "=d"(v2), "=d"(v3) : "l"(a + i));
      acc += v0 + v1 + v2 + v3;
    }
  if (acc == 12345.0) out[0] = acc;
}
int main() {
  size_t sizes[] = {8u << 20, 16u << 20, 32u << 20, 48u << 20, 64u << 20, 96u << 20, 2048u << 20};
  for (size_t bytes : sizes) {
    size_t n = bytes / 8;
    double *a, *o;
    cudaMalloc(&a, bytes); cudaMalloc(&o, 8); cudaMemset(a, 0, bytes);
    int reps = bytes < (1u << 30) ? 64 : 4;
    rd<<<148 * 8, 256>>>(a, n, 1, o);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    rd<<<148 * 8, 256>>>(a, n, reps, o);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%6zu MB x %2d: %8.0f GB/s\n", bytes >> 20, reps, (double)bytes * reps / (ms * 1e-3) / 1e9);
    cudaFree(a); cudaFree(o);
  }
}
