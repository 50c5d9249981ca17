// Access-pattern probe for the middle pass (n = 128, G = 2): in-place copy of
// column tiles.  (a) rows of W complex at stride NR*H (current slab layout),
// (b) tile-major contiguous layout.  Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 128, G = 2, NR = 64, H = 65, ROW = NR * H;
template <int W, int NB>
__global__ void __launch_bounds__(128) strided(double2* S, int tiles) {
  const int bg = blockIdx.x / tiles, tile = blockIdx.x % tiles;
  for (int j = 0; j < NB; ++j) {
    double2* base = S + (size_t)(bg * NB + j) * N * G * ROW + tile * W;
    constexpr int PER = N * G * W / 128;
    double2 v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = threadIdx.x + k * 128, w = i % W, r = i / W;
      v[k] = base[(size_t)r * ROW + w];
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int i = threadIdx.x + k * 128, w = i % W, r = i / W;
      v[k].x += 1.0;
      base[(size_t)r * ROW + w] = v[k];
    }
  }
}
template <int W, int NB>
__global__ void __launch_bounds__(128) contiguous(double2* S, int tiles) {
  const int bg = blockIdx.x / tiles, tile = blockIdx.x % tiles;
  for (int j = 0; j < NB; ++j) {
    double2* base = S + ((size_t)(bg * NB + j) * tiles + tile) * N * G * W;
    constexpr int PER = N * G * W / 128;
    double2 v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) v[k] = base[threadIdx.x + k * 128];
#pragma unroll
    for (int k = 0; k < PER; ++k) { v[k].x += 1.0; base[threadIdx.x + k * 128] = v[k]; }
  }
}
int main() {
  const int B = 64;
  size_t elems = (size_t)B * N * G * ROW;
  double2* S; cudaMalloc(&S, elems * 16); cudaMemset(S, 0, elems * 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
    printf("%-28s %.3f ms %6.0f GB/s %s\n", name, ms, 2.0 * elems * 16 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  run("strided W=8 NB=8", [&] { strided<8, 8><<<(B / 8) * (ROW / 8), 128>>>(S, ROW / 8); });
  run("strided W=16 NB=8", [&] { strided<16, 8><<<(B / 8) * (ROW / 16), 128>>>(S, ROW / 16); });
  run("strided W=8 NB=1", [&] { strided<8, 1><<<B * (ROW / 8), 128>>>(S, ROW / 8); });
  run("contiguous W=8 NB=8", [&] { contiguous<8, 8><<<(B / 8) * (ROW / 8), 128>>>(S, ROW / 8); });
  run("contiguous W=8 NB=1", [&] { contiguous<8, 1><<<B * (ROW / 8), 128>>>(S, ROW / 8); });
}
