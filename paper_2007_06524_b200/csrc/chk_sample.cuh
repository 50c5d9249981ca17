// chk_sample.cuh -- checkerboard realizations drawn on the device.
//
// sample_realization (lattice.py:284-311) draws, per realization seed, a
// Generator(Philox(SeedSequence(seed))) stream (lattice.py:279-281) and takes
// one uniform per cell in C order for coverage (u < coverage_prob) and, for
// the two_value contrast, a second block of one uniform per cell for the
// amplitude choice (u < 1/2 -> betas[0]).  The SeedSequence hash stays on the
// host (a few microseconds per seed; it yields the 128-bit Philox key,
// SeedSequence.generate_state(2, uint64)); everything per cell runs here.
//
// numpy's Philox bit generator is Philox4x64-10 (Salmon et al., SC'11) with a
// 256-bit counter starting at 0 that is incremented BEFORE each block of four
// 64-bit outputs, so 64-bit output i is word i % 4 of the block at counter
// i / 4 + 1.  random() maps a 64-bit output w to (w >> 11) * 2^-53.  Every cell
// is independent: one thread per block of four cells, no sequential state.
#pragma once
#include <cstdint>

namespace chk {

struct Philox4x64 {
  uint64_t v[4];
};

__device__ __forceinline__ Philox4x64 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                                    uint64_t k0, uint64_t k1) {
  constexpr uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  constexpr uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += W0;
      k1 += W1;
    }
    const uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    const uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return Philox4x64{{c0, c1, c2, c3}};
}

// 64-bit output `i` of the stream keyed by (k0, k1)
__device__ __forceinline__ uint64_t philox_word(uint64_t i, uint64_t k0, uint64_t k1) {
  const uint64_t blk = (i >> 2) + 1;  // counter incremented before the first block
  const Philox4x64 o = philox4x64_10(blk, 0, 0, 0, k0, k1);
  return o.v[i & 3];
}

__device__ __forceinline__ double philox_uniform(uint64_t w) {
  return (double)(w >> 11) * (1.0 / 9007199254740992.0);  // Generator.random()
}

enum : int { CONTRAST_FIXED = 0, CONTRAST_TWO_VALUE = 1 };

// beta[b][c] for c < ncell: coverage u_c < p; amplitude beta0 (fixed) or
// beta0 / beta1 by the second-block uniform (two_value).  grid (x: cell
// quads, y: realization).
__global__ void __launch_bounds__(256) sample_cells_kernel(const uint64_t* __restrict__ keys, int ncell, double p,
                                                           int kind, double beta0, double beta1,
                                                           double* __restrict__ beta) {
  const int b = blockIdx.y;
  const uint64_t k0 = keys[2 * b], k1 = keys[2 * b + 1];
  double* out = beta + (size_t)b * ncell;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; 4 * q < ncell; q += gridDim.x * blockDim.x) {
    const Philox4x64 o = philox4x64_10((uint64_t)q + 1, 0, 0, 0, k0, k1);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int c = 4 * q + e;
      if (c >= ncell) break;
      const bool cov = philox_uniform(o.v[e]) < p;
      double v = beta0;
      if (kind == CONTRAST_TWO_VALUE)
        v = philox_uniform(philox_word((uint64_t)ncell + c, k0, k1)) < 0.5 ? beta0 : beta1;
      out[c] = cov ? v : 0.0;
    }
  }
}

}  // namespace chk
