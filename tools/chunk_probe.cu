// Access-pattern probe for the spectrum layout at n >= 256 (not part of the
// product).  (1) middle-pass tile pattern: each CTA reads and rewrites rows of
// C bytes at a large stride (C = G*W*16 for the interleaved layout, W*16 for the
// current one).  (2) plane-pass pattern: G consecutive CTAs each own a P-byte
// piece of every 256-byte row of a plane chunk (interleaved layout) versus a
// contiguous region each (current layout).
#include <cstdio>
#include <cuda_runtime.h>

// (1) tile copy: rows of C bytes (C/16 double2), TB bytes per tile, row stride `stride` double2
template <int C, int TB>
__global__ void __launch_bounds__(256) tile_rw(double2* S, long long stride, int tiles_per_row) {
  constexpr int PIECE = C / 16;            // double2 per row
  constexpr int ROWS = TB / C;
  constexpr int PER = ROWS * PIECE / 256;  // double2 per thread
  const int t = blockIdx.x;
  const long long row0 = (long long)(t / tiles_per_row) * ROWS;
  const int col0 = (t % tiles_per_row) * PIECE;
  double2 v[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = threadIdx.x + k * 256, w = i % PIECE, r = i / PIECE;
    v[k] = S[(row0 + r) * stride + col0 + w];
  }
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = threadIdx.x + k * 256, w = i % PIECE, r = i / PIECE;
    v[k].x += 1.0;
    S[(row0 + r) * stride + col0 + w] = v[k];
  }
}

// (2) plane pass: G CTAs per plane, each writes (MODE 0) or reads (MODE 1) its
// share of a plane of PB bytes; interleaved: P-byte pieces of 256-byte rows.
template <int G, int MODE, bool INTERLEAVED>
__global__ void __launch_bounds__(256) plane_io(double2* S, double* sink, int PB) {
  const int plane = blockIdx.x / G, g = blockIdx.x % G;
  const long long base = (long long)plane * (PB / 16);
  const int share = PB / 16 / G;  // double2 per CTA
  constexpr int P = 256 / G / 16;  // double2 per piece (interleaved)
  double acc = 0.0;
  for (int i = threadIdx.x; i < share; i += 256) {
    long long idx;
    if (INTERLEAVED) {
      const int row = i / P, w = i % P;
      idx = base + (long long)row * (256 / 16) + g * P + w;
    } else {
      idx = base + (long long)g * share + i;
    }
    if (MODE == 0) {
      S[idx] = make_double2(i, g);
    } else {
      const double2 v = __ldcg(S + idx);
      acc += v.x + v.y;
    }
  }
  if (MODE == 1 && acc == 12345.678) sink[0] = acc;
}

int main() {
  const size_t bytes = (size_t)4 << 30;
  double2* S;
  double* sink;
  cudaMalloc(&S, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(S, 0, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, double moved, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 10;
    printf("%-44s %.3f ms %6.0f GB/s %s\n", name, ms, moved / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  const long long total2 = bytes / 16;
  // (1) the tile is 64 KB: rows of C bytes; row stride = a slab row (ROWB bytes)
  {
    constexpr int TB = 65536;
    const long long stride = 4128 * 8;  // 8 groups x 4128 columns (n = 256 plane row chunk)
#define TILE(C)                                                                              \
    {                                                                                        \
      const int tpr = (int)(stride * 16 / C);                                                \
      const long long rows = total2 / stride;                                                \
      const int grid = (int)(rows / (TB / C)) * tpr;                                         \
      run("tile rw C=" #C, 2.0 * grid * TB, [&] { tile_rw<C, TB><<<grid, 256>>>(S, stride, tpr); }); \
    }
    TILE(16) TILE(32) TILE(64) TILE(128) TILE(256) TILE(512)
  }
  // (2) plane passes, plane chunk of 528 KB (n = 256) / 2.1 MB (n = 512)
  {
    const int PB256 = 256 * 129 * 16 * 16 / 16;  // 256 rows x 129 x 16 B  (528384)
    const int PB512 = 512 * 257 * 16;            // 2105344
    const int np256 = (int)(bytes / PB256), np512 = (int)(bytes / PB512);
    run("write n256 G8 contiguous", (double)np256 * PB256, [&] { plane_io<8, 0, false><<<np256 * 8, 256>>>(S, sink, PB256); });
    run("write n256 G8 interleaved(32B)", (double)np256 * PB256, [&] { plane_io<8, 0, true><<<np256 * 8, 256>>>(S, sink, PB256); });
    run("read  n256 G8 contiguous", (double)np256 * PB256, [&] { plane_io<8, 1, false><<<np256 * 8, 256>>>(S, sink, PB256); });
    run("read  n256 G8 interleaved(32B)", (double)np256 * PB256, [&] { plane_io<8, 1, true><<<np256 * 8, 256>>>(S, sink, PB256); });
    run("write n512 G16 contiguous", (double)np512 * PB512, [&] { plane_io<16, 0, false><<<np512 * 16, 256>>>(S, sink, PB512); });
    run("write n512 G16 interleaved(16B)", (double)np512 * PB512, [&] { plane_io<16, 0, true><<<np512 * 16, 256>>>(S, sink, PB512); });
    run("read  n512 G16 contiguous", (double)np512 * PB512, [&] { plane_io<16, 1, false><<<np512 * 16, 256>>>(S, sink, PB512); });
    run("read  n512 G16 interleaved(16B)", (double)np512 * PB512, [&] { plane_io<16, 1, true><<<np512 * 16, 256>>>(S, sink, PB512); });
  }
  return 0;
}
