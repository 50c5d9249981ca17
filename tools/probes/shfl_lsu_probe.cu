// Do warp shuffles compete with shared-memory accesses for the LSU data pipe?
// Kernels over an SM-filling grid (8 CTAs x 256 threads per SM), CUDA-event timed:
//   smem : per round 4 independent (LDS.128 + STS.128) per thread, conflict-free
//   shfl : per round NS independent SHFL.IDX.b32 per thread
//   both : the two interleaved in one loop (no data dependence between them)
// both ~ max(smem, shfl): separate resources; both ~ smem + shfl: one shared pipe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o shfl_lsu_probe shfl_lsu_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void lds128(unsigned a, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
__device__ __forceinline__ void sts128(unsigned a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1,%2};" ::"r"(a), "d"(x), "d"(y));
}
__device__ __forceinline__ unsigned shfl(unsigned v, int src) {
  unsigned r;
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(r) : "r"(v), "r"(src));
  return r;
}

template <int MODE, int NS>
__global__ void __launch_bounds__(256) k(double* out, int rounds) {
  extern __shared__ double2 sm[];
  const int t = threadIdx.x, lane = t & 31;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
  for (int i = t; i < 2048; i += 256) sm[i] = make_double2(i, 1);
  __syncthreads();
  double ax[4] = {0, 0, 0, 0}, ay[4] = {0, 0, 0, 0};
  unsigned u[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) u[s] = t * 8 + s;
  for (int r = 0; r < rounds; ++r) {
    if (MODE & 1) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double x, y;
        lds128(base + 16 * ((t + 256 * q) & 2047), x, y);
        ax[q] += x; ay[q] += y;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) sts128(base + 16 * ((t + 256 * q + 1024) & 2047), ax[q], ay[q]);
    }
    if (MODE & 2) {
#pragma unroll
      for (int s = 0; s < NS; ++s) u[s & 7] = shfl(u[s & 7], (lane + 1 + s) & 31);
    }
  }
  double z = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) z += ax[q] + ay[q];
  unsigned w = 0;
#pragma unroll
  for (int s = 0; s < 8; ++s) w ^= u[s];
  if (z == 1.2345 || w == 0xdeadbeefu) out[0] = z + w;
}

template <int MODE, int NS>
float run(double* out, int rounds) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<MODE, NS><<<148 * 8, 256, 32768>>>(out, 16);
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  k<MODE, NS><<<148 * 8, 256, 32768>>>(out, rounds);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  double* out; cudaMalloc(&out, 8);
  const int R = 4000;
  for (int rep = 0; rep < 2; ++rep) {
    printf("smem only (32 wavefronts/round/warp) %.3f ms\n", run<1, 8>(out, R));
    printf("shfl only  8/round   %.3f ms\n", run<2, 8>(out, R));
    printf("both       8/round   %.3f ms\n", run<3, 8>(out, R));
    printf("shfl only 16/round   %.3f ms\n", run<2, 16>(out, R));
    printf("both      16/round   %.3f ms\n", run<3, 16>(out, R));
    printf("shfl only 32/round   %.3f ms\n", run<2, 32>(out, R));
    printf("both      32/round   %.3f ms\n", run<3, 32>(out, R));
  }
  return 0;
}
