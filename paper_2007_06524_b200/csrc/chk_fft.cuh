// chk_fft.cuh -- fp64 complex helpers and shared-memory FFT stages (sm_100a).
//
// All transforms are in-place mixed-radix (8, then 4/2) on pencils that live in
// shared memory.  The forward transform is decimation-in-frequency and leaves
// frequency k at the digit-reversed position pos(k); the inverse is the exact
// reverse (decimation-in-time, conjugate twiddles) and consumes that order, so a
// forward -> pointwise scale -> inverse chain never permutes data.  Twiddles come
// from one table w[k] = exp(-2 pi i k / ntab), k < ntab, computed on the host in
// fp64 (the reference uses numpy's pocketfft, lowrank.py:190-192).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace chk {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 cmul_mi(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// Twiddle sources.  A plan's table w[k] = exp(-2 pi i k / n) lives in global memory
// (read-only path); for the plane passes, whose shared-memory stages saturate the
// LSU data pipe, the same values come from constant memory instead (c_tw512, the
// n = 512 table: every power-of-two table is a stride of it, bit for bit), which
// takes the warp-uniform twiddle loads off the LSU.
__constant__ double2 c_tw512[512];
struct CTw {
  int mul;  // 512 / (length of the table being emulated)
};
__device__ __forceinline__ double2 tw_at(const double2* tw, int i) { return __ldg(tw + i); }
__device__ __forceinline__ double2 tw_at(CTw t, int i) { return c_tw512[i * t.mul]; }

template <bool INV>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
  double2 s0 = cadd(x0, x2), d0 = csub(x0, x2);
  double2 s1 = cadd(x1, x3), d1 = cmul_mi<INV>(csub(x1, x3));
  x0 = cadd(s0, s1);
  x2 = csub(s0, s1);
  x1 = cadd(d0, d1);
  x3 = csub(d0, d1);
}

// y_m = sum_t v_t w8^{tm}, natural order in and out.
template <bool INV>
__device__ __forceinline__ void dft8(double2 (&v)[8]) {
  constexpr double c = 0.70710678118654752440084436210485;
  double2 a0 = v[0], a1 = v[2], a2 = v[4], a3 = v[6];
  double2 b0 = v[1], b1 = v[3], b2 = v[5], b3 = v[7];
  dft4<INV>(a0, a1, a2, a3);
  dft4<INV>(b0, b1, b2, b3);
  // b_m *= w8^m
  if (!INV) {
    b1 = make_double2(c * (b1.x + b1.y), c * (b1.y - b1.x));
    b2 = make_double2(b2.y, -b2.x);
    b3 = make_double2(c * (b3.y - b3.x), -c * (b3.x + b3.y));
  } else {
    b1 = make_double2(c * (b1.x - b1.y), c * (b1.y + b1.x));
    b2 = make_double2(-b2.y, b2.x);
    b3 = make_double2(-c * (b3.x + b3.y), c * (b3.x - b3.y));
  }
  v[0] = cadd(a0, b0); v[4] = csub(a0, b0);
  v[1] = cadd(a1, b1); v[5] = csub(a1, b1);
  v[2] = cadd(a2, b2); v[6] = csub(a2, b2);
  v[3] = cadd(a3, b3); v[7] = csub(a3, b3);
}

// y_k = sum_t v_t w16^{tk}, natural order in and out: 16 = 4 x 4 (t = 4a + b, k = m + 4n),
// y[m + 4n] = sum_b w4^{bn} w16^{bm} sum_a w4^{am} v[4a + b].
template <bool INV>
__device__ __forceinline__ void dft16(double2 (&v)[16]) {
  constexpr double c1 = 0.92387953251128675612818318939679;  // cos(pi/8)
  constexpr double s1 = 0.38268343236508977172845998403040;  // sin(pi/8)
  constexpr double c2 = 0.70710678118654752440084436210485;
#pragma unroll
  for (int b = 0; b < 4; ++b) dft4<INV>(v[b], v[4 + b], v[8 + b], v[12 + b]);  // v[4m + b] = u_b[m]
  // u_b[m] *= w16^{bm} (conjugated for the inverse)
  auto tw = [](double2 a, double wr, double wi) {
    const double si = INV ? -wi : wi;
    return make_double2(a.x * wr - a.y * si, a.x * si + a.y * wr);
  };
  v[4 * 1 + 1] = tw(v[4 * 1 + 1], c1, -s1);   // w^1
  v[4 * 1 + 2] = tw(v[4 * 1 + 2], c2, -c2);   // w^2
  v[4 * 1 + 3] = tw(v[4 * 1 + 3], s1, -c1);   // w^3
  v[4 * 2 + 1] = tw(v[4 * 2 + 1], c2, -c2);   // w^2
  v[4 * 2 + 2] = cmul_mi<INV>(v[4 * 2 + 2]);  // w^4 = -i
  v[4 * 2 + 3] = tw(v[4 * 2 + 3], -c2, -c2);  // w^6
  v[4 * 3 + 1] = tw(v[4 * 3 + 1], s1, -c1);   // w^3
  v[4 * 3 + 2] = tw(v[4 * 3 + 2], -c2, -c2);  // w^6
  v[4 * 3 + 3] = tw(v[4 * 3 + 3], -c1, s1);   // w^9
#pragma unroll
  for (int m = 0; m < 4; ++m) dft4<INV>(v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3]);  // v[4m + n] = y[m + 4n]
  double2 y[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) y[k] = v[4 * (k % 4) + k / 4];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = y[k];
}

template <int R, bool INV>
__device__ __forceinline__ void dftR(double2 (&v)[R]) {
  if constexpr (R == 16) {
    dft16<INV>(v);
  } else if constexpr (R == 8) {
    dft8<INV>(v);
  } else if constexpr (R == 4) {
    dft4<INV>(v[0], v[1], v[2], v[3]);
  } else {
    dft2<INV>(v[0], v[1]);
  }
}

// Radix of the stage at sub-length M.  RULE 0: 8, then 4 / 2.  RULE 1: 16 while it divides
// (the x2 transforms of the n >= 256 plane passes: 128 = 16 x 8, 256 = 16 x 16 -- one
// shared-memory pass fewer than 8 x 4 x 4 / 8 x 8 x 4).
__host__ __device__ constexpr int radix_rule(int M, int rule) {
  return (rule == 1 && M % 16 == 0) ? 16 : ((M % 8 == 0) ? 8 : ((M % 4 == 0) ? 4 : 2));
}
template <int M, int RULE = 0>
struct Radix {
  static constexpr int value = radix_rule(M, RULE);
};

// One in-place stage at sub-length M of a length-N transform over `npencil`
// pencils; element e of pencil p is at buf[addr(p, e)].  Consecutive threads
// take consecutive pencils (callers lay pencils out bank-conflict free).
template <int N, int M, bool INV, int NP, int RULE, class Addr, class TW>
__device__ __forceinline__ void fft_stage_r(double2* buf, const Addr& addr, TW tw, int twstride) {
  constexpr int R = Radix<M, RULE>::value;
  constexpr int S = M / R;
  constexpr int NBF = N / R;
  constexpr int total = NP * NBF;
  for (int w = threadIdx.x; w < total; w += blockDim.x) {
    const int p = w % NP;
    const int bf = w / NP;
    const int blk = bf / S, j = bf - (bf / S) * S;
    const int base = blk * M + j;
    double2 v[R];
#pragma unroll
    for (int t = 0; t < R; ++t) v[t] = buf[addr(p, base + t * S)];
    if (!INV) {
      dftR<R, false>(v);
      if (S > 1) {
#pragma unroll
        for (int m = 1; m < R; ++m) v[m] = cmul(v[m], tw_at(tw, (j * m * (N / M)) * twstride));
      }
    } else {
      if (S > 1) {
#pragma unroll
        for (int m = 1; m < R; ++m) v[m] = cmulc(v[m], tw_at(tw, (j * m * (N / M)) * twstride));
      }
      dftR<R, true>(v);
    }
#pragma unroll
    for (int t = 0; t < R; ++t) buf[addr(p, base + t * S)] = v[t];
  }
}

template <int N, int M, bool INV, int NP, class Addr, class TW>
__device__ __forceinline__ void fft_stage(double2* buf, const Addr& addr, TW tw, int twstride) {
  fft_stage_r<N, M, INV, NP, 0>(buf, addr, tw, twstride);
}

template <int N, int M, bool INV, int NP, int RULE = 0>
struct FftRec {
  template <class Addr, class TW>
  __device__ __forceinline__ static void run(double2* buf, const Addr& addr, TW tw, int twstride) {
    constexpr int R = Radix<M, RULE>::value;
    if constexpr (!INV) {
      fft_stage_r<N, M, false, NP, RULE>(buf, addr, tw, twstride);
      __syncthreads();
      if constexpr (M / R > 1) FftRec<N, M / R, false, NP, RULE>::run(buf, addr, tw, twstride);
    } else {
      if constexpr (M / R > 1) FftRec<N, M / R, true, NP, RULE>::run(buf, addr, tw, twstride);
      fft_stage_r<N, M, true, NP, RULE>(buf, addr, tw, twstride);
      __syncthreads();
    }
  }
};

// All stages but the last one (the last stage is the M == R stage: contiguous
// groups of R, no twiddles), so a caller can fuse it with pointwise work.
template <int N, int M, bool INV, int NP>
struct FftRecButLast {
  template <class Addr, class TW>
  __device__ __forceinline__ static void run(double2* buf, const Addr& addr, TW tw, int twstride) {
    constexpr int R = Radix<M>::value;
    if constexpr (M / R > 1) {
      if constexpr (!INV) {
        fft_stage<N, M, false, NP>(buf, addr, tw, twstride);
        __syncthreads();
        FftRecButLast<N, M / R, false, NP>::run(buf, addr, tw, twstride);
      } else {
        FftRecButLast<N, M / R, true, NP>::run(buf, addr, tw, twstride);
        fft_stage<N, M, true, NP>(buf, addr, tw, twstride);
        __syncthreads();
      }
    }
  }
};

// radix of the last stage of fft_smem<N>
template <int M>
struct LastRadix {
  static constexpr int R = Radix<M>::value;
  static constexpr int value = (M / R > 1) ? LastRadix<M / R>::value : R;
};
template <>
struct LastRadix<1> {
  static constexpr int value = 1;
};

// Full length-N transform; the caller must __syncthreads() before (data in
// smem); returns after a __syncthreads().  Forward: natural -> digit-reversed.
// Inverse (unnormalised): digit-reversed -> natural, result scaled by N.
template <int N, bool INV, int NP, class Addr, class TW>
__device__ __forceinline__ void fft_smem(double2* buf, const Addr& addr, TW tw, int ntab) {
  if constexpr (N > 1) FftRec<N, N, INV, NP>::run(buf, addr, tw, ntab / N);
}
template <int N, bool INV, int NP, int RULE, class Addr, class TW>
__device__ __forceinline__ void fft_smem_r(double2* buf, const Addr& addr, TW tw, int ntab) {
  if constexpr (N > 1) FftRec<N, N, INV, NP, RULE>::run(buf, addr, tw, ntab / N);
}

// In-register in-place DIF / inverse DIT of length L on v[0..L): identical
// index semantics to fft_smem<L> (digit-reversed output), all loops unrolled.
template <int L, int M, bool INV>
struct RegFft {
  template <class TW>
  __device__ __forceinline__ static void run(double2 (&v)[L], TW tw, int ntab) {
    constexpr int R = Radix<M>::value, S = M / R;
    if constexpr (INV && S > 1) RegFft<L, S, true>::run(v, tw, ntab);
#pragma unroll
    for (int blk = 0; blk < L / M; ++blk) {
#pragma unroll
      for (int j = 0; j < S; ++j) {
        double2 a[R];
#pragma unroll
        for (int t = 0; t < R; ++t) a[t] = v[blk * M + j + t * S];
        if constexpr (!INV) {
          dftR<R, false>(a);
          if (j > 0) {
#pragma unroll
            for (int m = 1; m < R; ++m) a[m] = cmul(a[m], tw_at(tw, (j * m) * (ntab / M)));
          }
        } else {
          if (j > 0) {
#pragma unroll
            for (int m = 1; m < R; ++m) a[m] = cmulc(a[m], tw_at(tw, (j * m) * (ntab / M)));
          }
          dftR<R, true>(a);
        }
#pragma unroll
        for (int t = 0; t < R; ++t) v[blk * M + j + t * S] = a[t];
      }
    }
    if constexpr (!INV && S > 1) RegFft<L, S, false>::run(v, tw, ntab);
  }
};
template <int L, bool INV, class TW>
__device__ __forceinline__ void reg_fft(double2 (&v)[L], TW tw, int ntab) {
  if constexpr (L > 1) RegFft<L, L, INV>::run(v, tw, ntab);
}

// Stages of a length-N transform down to (forward) / up from (inverse) sub-length
// BL, the block of the last two stages; FftStop<N, N, INV, NP, BL> runs them in smem.
template <int M>
struct LastTwo {  // sub-length at which the last two stages start
  static constexpr int R = Radix<M>::value;
  static constexpr int value = ((M / R) > 1 && (M / R) / Radix<M / R>::value > 1) ? LastTwo<M / R>::value : M;
};
template <>
struct LastTwo<1> {
  static constexpr int value = 1;
};
template <int N, int M, bool INV, int NP, int BL>
struct FftStop {
  template <class Addr, class TW>
  __device__ __forceinline__ static void run(double2* buf, const Addr& addr, TW tw, int twstride) {
    if constexpr (M > BL) {
      constexpr int R = Radix<M>::value;
      if constexpr (!INV) {
        fft_stage<N, M, false, NP>(buf, addr, tw, twstride);
        __syncthreads();
        FftStop<N, M / R, false, NP, BL>::run(buf, addr, tw, twstride);
      } else {
        FftStop<N, M / R, true, NP, BL>::run(buf, addr, tw, twstride);
        fft_stage<N, M, true, NP>(buf, addr, tw, twstride);
        __syncthreads();
      }
    }
  }
};

// ----------------------------------------------------------------------------
// reductions (deterministic: fixed shuffle tree, fixed warp order)
// ----------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sum; result valid in every thread.  `scratch` >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double t = (threadIdx.x < nw) ? scratch[threadIdx.x] : 0.0;
  if (wid == 0) t = warp_sum(t);
  if (threadIdx.x == 0) scratch[0] = t;
  __syncthreads();
  double r = scratch[0];
  __syncthreads();
  return r;
}

// Two block sums in one pass (results valid in every thread). scratch >= 64 doubles.
__device__ __forceinline__ void block_sum2(double& a, double& b, double* scratch) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    scratch[wid] = a;
    scratch[32 + wid] = b;
  }
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double ta = (threadIdx.x < nw) ? scratch[threadIdx.x] : 0.0;
  double tb = (threadIdx.x < nw) ? scratch[32 + threadIdx.x] : 0.0;
  if (wid == 0) {
    ta = warp_sum(ta);
    tb = warp_sum(tb);
  }
  if (threadIdx.x == 0) {
    scratch[0] = ta;
    scratch[32] = tb;
  }
  __syncthreads();
  a = scratch[0];
  b = scratch[32];
  __syncthreads();
}

}  // namespace chk
