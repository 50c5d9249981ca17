// chk_kernels.cuh -- sm_100a kernels of the batched PCG hot path.
//
// One PCG iteration k >= 1 (pcg_solve loop, solver.py:161-185) is three
// kernels over all B realizations of the batch:
//
//   fwd_plane<FWD_Q>   q = A p (matrix-free 7-point stencil from the L^3 cell
//                      array), <p, q> -> alpha; R2C along x2 and C2C along the
//                      x1 group of q in shared memory        (solver.py:162-166)
//   mid_column*        group combine + x0 transform of Q, R -= alpha Q (the
//                      residual is kept as its spectrum), ||r||^2 (stop test),
//                      z = D R with D[i,j,l] = sum_k U0[k,i]U1[k,j]U2[k,l]
//                      evaluated per column tile (never materialised), r.z,
//                      inverse x0 / group combine            (solver.py:168-183)
//   inv_plane<INV_ITER> inverse x1-group C2C + C2R -> z; u += alpha p;
//                      p = z + beta p                         (solver.py:167,184)
//
// CTA = one (realization, x0-plane, x1-group) slab or one spectral column tile.
// Reductions are deterministic: every CTA writes a partial, the last CTA of the
// realization (atomic ticket) sums them in a fixed order and takes the scalar
// decisions (alpha, breakdown, stop, beta) -- or, when one grid is
// slab-decomposed over GPUs, publishes rank-local sums for an allreduce.
#pragma once
#include <type_traits>

#include "chk_fft.cuh"
#include "chk_tma.cuh"

#ifndef CHK_MARCH  // marching stencil in the plane passes (n = 64, 128)
#define CHK_MARCH 1
#endif
#ifndef CHK_FWD_PF  // L2 prefetch of the CTA's own p rows at the start of the forward pass
#define CHK_FWD_PF 1
#endif
#ifndef CHK_FWD_CS  // n = 256 plane passes: CTA-uniform cell-row de-duplication + half-row halo shuffles
#define CHK_FWD_CS 1
#endif
#ifndef CHK_INV_PF_LATE  // n >= CHK_INV_PF_LATE_MIN: the same prefetch just before the last inverse FFT stage
#define CHK_INV_PF_LATE 1
#endif
#ifndef CHK_INV_PF_LATE_MIN
#define CHK_INV_PF_LATE_MIN 256
#endif
#ifndef CHK_INV_PF  // L2 prefetch of the p / u rows at the start of the inverse pass (n <= 128;
#define CHK_INV_PF 1    // at n >= 256 the prefetched rows are evicted before use: +38 % DRAM reads)
#endif
#ifndef CHK_MARCH_S0  // marching stencil: specialised body for planes whose x0 - 1 is in the same cell
#define CHK_MARCH_S0 1
#endif
#ifndef CHK_MID_RPF
#define CHK_MID_RPF 1
#endif
#ifndef CHK_FUSED_PF  // n = 512 middle pass: L2 prefetch of the residual / diagonal tile at the
#define CHK_FUSED_PF 1  // start of each realization
#endif
#ifndef CHK_SC_FENCE
#define CHK_SC_FENCE 0
#endif
#ifndef CHK_U_TMA  // n = 128 inverse pass: u += alpha p as a TMA bulk reduce-add from shared memory
#define CHK_U_TMA 1
#endif

namespace chk {

enum : int { ST_CONVERGED = 0, ST_NOT_CONVERGED = 1, ST_BREAKDOWN = 2, ST_ACTIVE = 3 };
enum : int { KIND_FOURIER = 0, KIND_LKR = 1, KIND_REGULARIZED = 2 };

// Per-realization solver state (device).
struct RState {
  int status;
  int iters;
  int rhs_projected;
  int pad0;
  double normf;      // ||f|| after the optional mean projection (solver.py:132,142)
  double norm_pf;    // sqrt|r0.z0| (solver.py:156)
  double mean_f;     // mean removed from f when projected
  double rz[2];      // r.z of the last two iterations (parity-indexed)
  double pq;         // p.Ap of the current iteration
  double alpha;      // rz_{k-1} / pq_k
  double beta;       // rz_k / rz_{k-1}
  double final_rel;  // last relative residual
  double mean_u;     // final projection (solver.py:169)
  unsigned cnt;      // last-block ticket
  unsigned pad1;
};

struct Geo {
  int n;
  int L;
  int sh;    // log2 n0
  int mask;  // n0 - 1
  int k;     // sub-cell width
  int off;   // sub-cell offset
  double lam;
};

// Ownership of a rank when one grid is slab-decomposed over P GPUs (SURVEY
// §8e): planes x0 in [x0_off, x0_off + nloc), spectral column chunk `rank`
// (ncols = NR*(n/2+1)/P columns, tiles [tile_off, tile_off + tiles) of the
// middle pass).  Exchange buffers are laid out [chunk s][b][x0 local][g][ncols]
// so one all_to_all moves x0 slabs <-> column chunks.  P = 1 is the
// single-GPU layout (nloc = n, one chunk, periodic halo inside p).
struct SlabGeo {
  int nloc;
  int x0_off;
  int P;
  int ncols;
  int tile_off;
  int tiles;
  const double* halo_lo;  // [B][n*n] plane x0_off-1, null -> periodic inside p
  const double* halo_hi;  // [B][n*n] plane x0_off+nloc, null -> periodic inside p
  int run0;               // plane passes: launch covers local planes [run0, run0 + nrun)
  int nrun;               // (a slab phase split into plane chunks overlapped with the exchange)
};

// Interleaved spectrum layout (n >= 256): a plane chunk is stored [ncols/W][G][W]
// instead of [G][ncols], so that one x0 row of a middle-pass tile (W columns of
// all G groups) is G*W*16 = 256 contiguous bytes, while the plane passes move
// pieces of W*16 = 32 bytes (whole DRAM sectors; the G CTAs of a plane run
// together).  n = 256: W = 2, each CTA moves its own pieces.  Measured access patterns
// (tools/chunk_probe.cu): tile rows of 16 B 2.3 TB/s, 32 B 3.5 TB/s, 256 B
// 6.3 TB/s; 32 B plane pieces 6.0 (write) / 5.6 (read) TB/s vs 7.4 contiguous,
// 16 B pieces 1.1 / 3.5 TB/s.  IlW = 0: the contiguous [G][ncols] layout.
// n = 512: contiguous layout.  (A 2-CTA-cluster interleaved variant exchanging the
// 16-byte pieces through DSMEM measured 8 % slower on config 5 and was removed.)
#ifndef CHK_NT512
#define CHK_NT512 512
#endif
// pieces per tensor-map box of the interleaved layout: ncols/W = 2064/P at n = 256,
// boxes of 172 pieces (5.5 KB, 128-byte aligned in shared memory) for P = 1, 2, 4;
// P = 8 keeps the cp.async path
template <int N>
struct TmapBox {
  static constexpr int value = 172;
};
template <int N>
struct IlW {
  static constexpr int value = (N == 256) ? 2 : 0;
};
// threads per CTA of the plane passes and the fused middle pass: n = 512 runs one
// CTA per SM (131 KB slab), so it takes more warps per CTA
// (n = 256: 512-thread CTAs measured slower -- 64 registers spill -- for both.)
// The fused middle pass states its 2 CTAs per SM at n <= 256 (<= 128 registers):
// an explicit minimum of 1 lets nvcc take 164 registers and halves occupancy.
#ifndef CHK_NT128
#define CHK_NT128 256
#endif
template <int N>
struct PlaneNT {
  static constexpr int value = (N == 512) ? CHK_NT512 : ((N == 128) ? CHK_NT128 : 256);
  // 256 threads: <= 80 registers, 3 CTAs per SM (66.5 KB slabs); 512 threads at n = 128: 2 CTAs
  static constexpr int minb = (N == 512) ? 1 : (value == 512 ? 2 : 3);
};
template <int N>
struct MidNT {
  static constexpr int value = (N == 512) ? CHK_NT512 : 256;
  static constexpr int minb = (N == 512) ? 1 : 2;
  static constexpr int minb_dg = (N == 512) ? 1 : 3;  // diagonal read from L2: tile-only smem
};

// start of the (s, b, x0l, g) row chunk of an exchange buffer (complex units)
__host__ __device__ __forceinline__ size_t slab_row(const SlabGeo& sg, int B, int G, int s, int b, int x0l,
                                                    int g) {
  return ((((size_t)s * B + b) * sg.nloc + x0l) * G + g) * (size_t)sg.ncols;
}

struct SolveCtl {
  RState* st;        // [B]
  double2* Rh;       // [B][TILES][N][G*W] residual spectrum, tile-major (PCG)
  double* part;      // [B][maxblk][2]
  double* hist;      // [B][max_iter] or null
  int maxblk;
  int max_iter;
  double tol;
  int prs;           // precond_residual_stopping
  double* red;       // [B][4] rank-local sums (slab mode), null otherwise
  int red_only;      // slab mode: last CTAs publish rank-local sums, decisions after allreduce
};

struct PlanDev {
  const double2* tw;  // [n] exp(-2 pi i k / n)
  const double* U;    // [3][r1][n] (LKR)
  const double* Up;   // [r1][n] U0 with columns in digit-reversed order (LKR)
  const double* lam;  // [n] eigenvalues (FOURIER / REGULARIZED)
  int r1;
  int kind;
  double delta;
  const double* D;    // [tiles][n][G*W] precomputed diagonal tiles (chk_dtile_kernel), or null
};

// ----------------------------------------------------------------------------
// digit-reversed position <-> frequency for the radix sequence of fft_smem
// ----------------------------------------------------------------------------
template <int N, int RULE = 0>
__device__ __forceinline__ int dig_pos(int k) {
  int p = 0;
  int M = N;
#pragma unroll
  for (int s = 0; s < 12; ++s) {
    if (M <= 1) break;
    const int R = radix_rule(M, RULE);
    const int m = k % R;
    k /= R;
    p += m * (M / R);
    M /= R;
  }
  return p;
}
template <int N, int RULE = 0>
__device__ __forceinline__ int dig_freq(int p) {
  int k = 0, mul = 1;
  int M = N;
#pragma unroll
  for (int s = 0; s < 12; ++s) {
    if (M <= 1) break;
    const int R = radix_rule(M, RULE);
    const int Mn = M / R;
    const int m = p / Mn;
    p -= m * Mn;
    k += m * mul;
    mul *= R;
    M = Mn;
  }
  return k;
}

// x0-axis radix policy of the middle pass.  n = 256 (CHK_R256): 2, 8, 8, 2 -- a
// radix-2 first stage lets the group combine and that stage share registers
// (mid_column_r256_kernel); every other length uses the generic 8, 4, 2 rule.
#ifndef CHK_R256
#define CHK_R256 1
#endif
__host__ __device__ constexpr int x0_radix(int N, int M) {
  return (N == 256 && CHK_R256)   ? ((M == 256 || M == 2) ? 2 : 8)
                                  : ((M % 8 == 0) ? 8 : ((M % 4 == 0) ? 4 : 2));
}
// frequency held at position p after the forward x0 transform (x0_radix order)
template <int N>
__device__ __forceinline__ int dig_freq0(int p) {
  int k = 0, mul = 1;
  int M = N;
#pragma unroll
  for (int s = 0; s < 12; ++s) {
    if (M <= 1) break;
    const int R = x0_radix(N, M);
    const int Mn = M / R;
    const int m = p / Mn;
    p -= m * Mn;
    k += m * mul;
    mul *= R;
    M = Mn;
  }
  return k;
}

// Radix rule of the x2 (real-FFT) transforms of the plane passes: radix 16 first at
// n >= CHK_X2R16_MIN (half length 128 = 16 x 8, 256 = 16 x 16).
#ifndef CHK_X2R16_MIN
#define CHK_X2R16_MIN 256
#endif
template <int N>
struct X2Rule {
  static constexpr int value = (N >= CHK_X2R16_MIN) ? 1 : 0;
};

// ----------------------------------------------------------------------------
// last-block reduction of two scalars per realization
// ----------------------------------------------------------------------------
// Release / acquire fences of the last-CTA ticket (message passing through
// the partials); lighter than the sequentially consistent __threadfence().
__device__ __forceinline__ void fence_release_gpu() {
#if CHK_SC_FENCE
  __threadfence();
#else
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Sum of the nblk partial pairs of a realization by its last CTA (after the
// ticket): fixed order, result valid in every thread.  scratch >= 64 doubles.
__device__ __forceinline__ void last_sum2(const double* part, int nblk, double* scratch, double& t0,
                                          double& t1) {
  fence_release_gpu();
  double a = 0.0, c = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    a += __ldcg(part + 2 * i);
    c += __ldcg(part + 2 * i + 1);
  }
  block_sum2(a, c, scratch);
  t0 = a;
  t1 = c;
}

// Per-CTA partial (v0, v1) of a realization -> part[blk]; true in the CTA that
// took the last ticket, with the totals in t0 / t1 (every thread).
// scratch >= 64 doubles.
__device__ __forceinline__ bool reduce2_last(double v0, double v1, double* part, unsigned* cnt,
                                             int blk, int nblk, double* scratch, double& t0,
                                             double& t1) {
  __shared__ int s_last;
  block_sum2(v0, v1, scratch);
  if (threadIdx.x == 0) {
    part[2 * blk] = v0;
    part[2 * blk + 1] = v1;
    fence_release_gpu();
    const unsigned prev = atomicAdd(cnt, 1u);
    s_last = (prev == (unsigned)(nblk - 1));
  }
  __syncthreads();
  if (!s_last) return false;
  last_sum2(part, nblk, scratch, t0, t1);
  if (threadIdx.x == 0) *cnt = 0u;
  return true;
}

// Deferred form for CTAs that process several realizations: per realization j
// each warp leaves its shuffle sums in wsum[j][warp][2] (warp_partials, no
// barrier); after the last realization (and a __syncthreads) mid_tickets folds
// them in the fixed order of block_sum2, publishes the partials, takes one
// ticket per realization (one fence per writer instead of one per
// realization) and runs the decisions of the realizations whose last CTA this
// is.  Same sums, same order as reduce2_last.
// wsum: [NB][warps per CTA][2]
__device__ __forceinline__ void warp_partials(double v0, double v1, double* wsum, int j) {
  v0 = warp_sum(v0);
  v1 = warp_sum(v1);
  if ((threadIdx.x & 31) == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    wsum[2 * (j * nw + (threadIdx.x >> 5))] = v0;
    wsum[2 * (j * nw + (threadIdx.x >> 5)) + 1] = v1;
  }
}
template <int NB, class Decide>
__device__ __forceinline__ void mid_tickets(const double* wsum, const int* act, int b0, int blk,
                                            int nblk, const SolveCtl& ctl, double* scratch, Decide decide) {
  __shared__ int s_last[NB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  for (int j = wid; j < NB; j += nw) {
    int last = 0;
    if (act[j]) {
      double a = (lane < nw) ? wsum[2 * (j * nw + lane)] : 0.0;
      double c = (lane < nw) ? wsum[2 * (j * nw + lane) + 1] : 0.0;
      a = warp_sum(a);
      c = warp_sum(c);
      if (lane == 0) {
        const int b = b0 + j;
        double* part = ctl.part + (size_t)b * 2 * ctl.maxblk;
        part[2 * blk] = a;
        part[2 * blk + 1] = c;
        fence_release_gpu();
        const unsigned prev = atomicAdd(&ctl.st[b].cnt, 1u);
        last = (prev == (unsigned)(nblk - 1));
      }
    }
    if (lane == 0) s_last[j] = last;
  }
  __syncthreads();
  for (int j = 0; j < NB; ++j) {
    if (!s_last[j]) continue;
    const int b = b0 + j;
    double t0, t1;
    last_sum2(ctl.part + (size_t)b * 2 * ctl.maxblk, nblk, scratch, t0, t1);
    if (threadIdx.x == 0) {
      ctl.st[b].cnt = 0u;
      decide(b, t0, t1);
    }
  }
}

// ----------------------------------------------------------------------------
// stiffness: 7-point stencil with on-the-fly edge conductivities
// ----------------------------------------------------------------------------
// F of h-cell (j0, j1, j2): beta(cell) if the h-cell lies inside the sub-cell
// on every axis (lattice.py:314-317,326-332), else 0.
__device__ __forceinline__ double fcell(const double* __restrict__ beta, const Geo& g, int j0,
                                        int j1, int j2) {
  const bool in = ((unsigned)((j0 & g.mask) - g.off) < (unsigned)g.k) &&
                  ((unsigned)((j1 & g.mask) - g.off) < (unsigned)g.k) &&
                  ((unsigned)((j2 & g.mask) - g.off) < (unsigned)g.k);
  return in ? __ldg(beta + ((j0 >> g.sh) * g.L + (j1 >> g.sh)) * g.L + (j2 >> g.sh)) : 0.0;
}

// Per-row context of the stencil for row (x0, x1) of one realization.
struct RowCtx {
  const double* pc;      // p(x0,   x1,   :)
  const double* pxm;     // p(x0-1, x1,   :)
  const double* pxp;     // p(x0+1, x1,   :)
  const double* pym;     // p(x0,   x1-1, :)
  const double* pyp;     // p(x0,   x1+1, :)
  const double* bab[4];  // beta row of cells (c(j0), c(j1), :) for (j0, j1) in
                         // {(x0-1,x1-1), (x0-1,x1), (x0,x1-1), (x0,x1)}; null = outside sub-cell
};

// Base pointers of planes x0-1, x0, x0+1 of one realization (slab halos or
// the periodic wrap inside p).
struct Planes {
  const double* m;
  const double* c;
  const double* p;
};

__device__ __forceinline__ Planes periodic_planes(const double* pb, int x0, int n) {
  const size_t nn = (size_t)n * n;
  return Planes{pb + (size_t)((x0 - 1) & (n - 1)) * nn, pb + (size_t)x0 * nn, pb + (size_t)((x0 + 1) & (n - 1)) * nn};
}

__device__ __forceinline__ RowCtx make_row(const Planes& pl, const double* __restrict__ beta,
                                           const Geo& g, int x0, int x1) {
  const int n = g.n, nm = n - 1;
  const int a0 = (x0 - 1) & nm, a1 = (x1 - 1) & nm, p1 = (x1 + 1) & nm;
  RowCtx rc;
  rc.pc = pl.c + (size_t)x1 * n;
  rc.pxm = pl.m + (size_t)x1 * n;
  rc.pxp = pl.p + (size_t)x1 * n;
  rc.pym = pl.c + (size_t)a1 * n;
  rc.pyp = pl.c + (size_t)p1 * n;
  const int j0[2] = {a0, x0}, j1[2] = {a1, x1};
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const bool in = ((unsigned)((j0[a] & g.mask) - g.off) < (unsigned)g.k) &&
                      ((unsigned)((j1[b] & g.mask) - g.off) < (unsigned)g.k);
      rc.bab[a * 2 + b] = in ? beta + ((size_t)(j0[a] >> g.sh) * g.L + (j1[b] >> g.sh)) * g.L : nullptr;
    }
  return rc;
}

__device__ __forceinline__ void ld4(const double* __restrict__ p, double (&v)[4]) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

// (A p)_x for the 4 nodes x2 = x2s .. x2s+3 (x2s % 4 == 0) of one row:
//   g_a(x) = lam + 1/4 sum_{delta} F[h-cell x_a, transverse x_b - delta_b]
//   (A p)_x = sum_a g_a(x)(p_x - p_{x+e_a}) + g_a(x-e_a)(p_x - p_{x-e_a})
// (tests/oracles.py:52-75; transverse delta order of the reference loop).
// n0 >= 4 and x2s % 4 == 0 put x2s..x2s+3 in one cell, so each of the four
// (j0, j1) cell rows needs two beta loads for the five h-cells x2s-1..x2s+3.
__device__ __forceinline__ void stencil4(const Geo& g, const RowCtx& rc, int x2s, double (&pc)[4],
                                         double (&q)[4]) {
  const int nm = g.n - 1;
  double xm[4], xp[4], ym[4], yp[4];
  ld4(rc.pc + x2s, pc);
  ld4(rc.pxm + x2s, xm);
  ld4(rc.pxp + x2s, xp);
  ld4(rc.pym + x2s, ym);
  ld4(rc.pyp + x2s, yp);
  const double pl = __ldg(rc.pc + ((x2s - 1) & nm));
  const double pr = __ldg(rc.pc + ((x2s + 4) & nm));
  const int jm = (x2s - 1) & nm;
  const bool inm = (unsigned)((jm & g.mask) - g.off) < (unsigned)g.k;
  bool in[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) in[i] = (unsigned)(((x2s + i) & g.mask) - g.off) < (unsigned)g.k;
  double f[4][5];
#pragma unroll
  for (int ab = 0; ab < 4; ++ab) {
    const double* br = rc.bab[ab];
    const double bm = (br && inm) ? __ldg(br + (jm >> g.sh)) : 0.0;
    const double b0 = br ? __ldg(br + (x2s >> g.sh)) : 0.0;
    f[ab][0] = bm;
#pragma unroll
    for (int i = 0; i < 4; ++i) f[ab][i + 1] = in[i] ? b0 : 0.0;
  }
  const double lam = g.lam;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // F_{abc}: a in {x0-1, x0}, b in {x1-1, x1}, c in {x2-1, x2}
    const double f000 = f[0][i], f001 = f[0][i + 1], f010 = f[1][i], f011 = f[1][i + 1];
    const double f100 = f[2][i], f101 = f[2][i + 1], f110 = f[3][i], f111 = f[3][i + 1];
    const double g0p = lam + (((f111 + f110) + f101) + f100) * 0.25;
    const double g0m = lam + (((f011 + f010) + f001) + f000) * 0.25;
    const double g1p = lam + (((f111 + f110) + f011) + f010) * 0.25;
    const double g1m = lam + (((f101 + f100) + f001) + f000) * 0.25;
    const double g2p = lam + (((f111 + f101) + f011) + f001) * 0.25;
    const double g2m = lam + (((f110 + f100) + f010) + f000) * 0.25;
    const double c = pc[i];
    const double left = (i == 0) ? pl : pc[i - 1];
    const double right = (i == 3) ? pr : pc[i + 1];
    const double q0 = g0p * (c - xp[i]) + g0m * (c - xm[i]);
    const double q1 = g1p * (c - yp[i]) + g1m * (c - ym[i]);
    const double q2 = g2p * (c - right) + g2m * (c - left);
    q[i] = (q0 + q1) + q2;
  }
}

// Fast path when every h-cell lies inside its sub-cell (k == n0, offset 0, i.e.
// alpha = 1/2, the BASELINE configurations): F = beta(cell) everywhere, the
// quad x2s..x2s+3 shares one cell column, and nodes 1..3 of the quad share
// their six edge weights.  Same formulas and summation order as stencil4.
// Rows are read with 256-bit loads; when one warp (segment) covers whole rows
// (n = 64, 128) the x2 halo comes from the neighbouring lane by shuffle.
__device__ __forceinline__ void ldg4v(const double* p, double (&v)[4]) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}

// Arithmetic of the all-inside quad: p rows (center, x0 -+ 1, x1 -+ 1), the x2
// halo (pl, prr) and the eight cell values m.. (cells of x2s - 1) / z.. (cells
// of x2s) for the (x0-1|x0, x1-1|x1) cell rows.
__device__ __forceinline__ void stencil4_allin_q(double lam, const double (&pc)[4], const double (&xm)[4],
                                                 const double (&xp)[4], const double (&ym)[4],
                                                 const double (&yp)[4], double pl, double prr, double m00,
                                                 double m01, double m10, double m11, double z00, double z01,
                                                 double z10, double z11, double (&q)[4]) {
  auto wsum = [lam](double a, double b, double c, double d) { return lam + (((a + b) + c) + d) * 0.25; };
  // node 0: h-cells x2-1 -> m.., x2 -> z..
  const double A0p = wsum(z11, m11, z10, m10), A0m = wsum(z01, m01, z00, m00);
  const double A1p = wsum(z11, m11, z01, m01), A1m = wsum(z10, m10, z00, m00);
  const double A2p = wsum(z11, z10, z01, z00), A2m = wsum(m11, m10, m01, m00);
  // nodes 1..3: both h-cells in the quad's cell
  const double B0p = wsum(z11, z11, z10, z10), B0m = wsum(z01, z01, z00, z00);
  const double B1p = wsum(z11, z11, z01, z01), B1m = wsum(z10, z10, z00, z00);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double g0p = i ? B0p : A0p, g0m = i ? B0m : A0m;
    const double g1p = i ? B1p : A1p, g1m = i ? B1m : A1m;
    const double g2p = A2p, g2m = i ? A2p : A2m;
    const double c = pc[i];
    const double left = (i == 0) ? pl : pc[i - 1];
    const double right = (i == 3) ? prr : pc[i + 1];
    const double q0 = g0p * (c - xp[i]) + g0m * (c - xm[i]);
    const double q1 = g1p * (c - yp[i]) + g1m * (c - ym[i]);
    const double q2 = g2p * (c - right) + g2m * (c - left);
    q[i] = (q0 + q1) + q2;
  }
}

// Cell values of the four cell rows (c0m|c00) x (c1m|c10) at cell column c: rows
// coincide when x0 - 1 (x1 - 1) lies in the same cell as x0 (x1) -- 3 of 4 node
// planes / rows at n0 = 4 -- and are then loaded once (same values, same bits).
__device__ __forceinline__ void cell4(const double* b00, const double* b01, const double* b10, const double* b11,
                                      bool s0, bool s1, int c, double& v00, double& v01, double& v10,
                                      double& v11) {
  v11 = __ldg(b11 + c);
  v10 = s1 ? v11 : __ldg(b10 + c);
  v01 = s0 ? v11 : __ldg(b01 + c);
  v00 = s0 ? v10 : (s1 ? v01 : __ldg(b00 + c));
}

// CS (compile-time, n >= 256 plane passes): the caller knows per CTA that the x0 - 1
// and x0 cell planes coincide (bit 0) / the x1 - 1 and x1 cell rows coincide
// (bit 1), so those cell rows are loaded once (same values, same bits); CS = -1:
// decide at run time (DEDUP) or not at all.  HALF: the 32 lanes of a warp hold 32
// consecutive quads of one row (n >= 256), so the x2 halo comes from the
// neighbouring lane by shuffle except at the two ends of the warp.
template <int N, bool DEDUP = false, int CS = -1, bool HALF = false>
__device__ __forceinline__ void stencil4_allin(const Geo& g, const Planes& P3,
                                               const double* __restrict__ beta, int x0, int x1,
                                               int x2s, double (&pc)[4], double (&q)[4]) {
  constexpr int nm = N - 1;
  constexpr int Q4 = N / 4;
  constexpr bool SHFL = (Q4 == 16 || Q4 == 32);
  const long long row = (long long)x1 * N;
  const long long d1m = (x1 == 0) ? (long long)nm * N : -(long long)N;
  const long long d1p = (x1 == nm) ? -(long long)nm * N : (long long)N;
  const double* pr = P3.c + row + x2s;
  double xm[4], xp[4], ym[4], yp[4];
  ldg4v(pr, pc);
  ldg4v(P3.m + row + x2s, xm);
  ldg4v(P3.p + row + x2s, xp);
  ldg4v(pr + d1m, ym);
  ldg4v(pr + d1p, yp);
  double pl, prr;
  if constexpr (SHFL) {
    pl = __shfl_sync(0xffffffffu, pc[3], (threadIdx.x - 1) & (Q4 - 1), Q4);
    prr = __shfl_sync(0xffffffffu, pc[0], (threadIdx.x + 1) & (Q4 - 1), Q4);
  } else if constexpr (HALF) {
    const int lane = threadIdx.x & 31;
    pl = __shfl_sync(0xffffffffu, pc[3], (lane - 1) & 31);
    prr = __shfl_sync(0xffffffffu, pc[0], (lane + 1) & 31);
    if (lane == 0) pl = __ldg(P3.c + row + ((x2s - 1) & nm));
    if (lane == 31) prr = __ldg(P3.c + row + ((x2s + 4) & nm));
  } else {
    pl = __ldg(P3.c + row + ((x2s - 1) & nm));
    prr = __ldg(P3.c + row + ((x2s + 4) & nm));
  }
  // cell rows (c(j0), c(j1), :) for j0 in {x0-1, x0}, j1 in {x1-1, x1}
  const int L = g.L, sh = g.sh;
  const int c0m = ((x0 - 1) & nm) >> sh, c00 = x0 >> sh;
  const int c1m = ((x1 - 1) & nm) >> sh, c10 = x1 >> sh;
  const int cm = ((x2s - 1) & nm) >> sh, cc = x2s >> sh;
  const double* b00 = beta + ((size_t)c0m * L + c1m) * L;  // (x0-1, x1-1)
  const double* b01 = beta + ((size_t)c0m * L + c10) * L;  // (x0-1, x1)
  const double* b10 = beta + ((size_t)c00 * L + c1m) * L;  // (x0,   x1-1)
  const double* b11 = beta + ((size_t)c00 * L + c10) * L;  // (x0,   x1)
  // DEDUP: coinciding cell rows loaded once (fewer loads, more live registers:
  // pays in the stand-alone stencil, not inside the register-bound plane passes)
  const bool s0 = (CS >= 0) ? (CS & 1) != 0 : (DEDUP && (c0m == c00));
  const bool s1 = (CS >= 0) ? (CS & 2) != 0 : (DEDUP && (c1m == c10));
  double m00, m01, m10, m11, z00, z01, z10, z11;
  cell4(b00, b01, b10, b11, s0, s1, cm, m00, m01, m10, m11);
  cell4(b00, b01, b10, b11, s0, s1, cc, z00, z01, z10, z11);
  stencil4_allin_q(g.lam, pc, xm, xp, ym, yp, pl, prr, m00, m01, m10, m11, z00, z01, z10, z11, q);
}

__device__ __forceinline__ void ldv4(const double* p, double (&v)[4]) {
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p)
               : "memory");
}
__device__ __forceinline__ void stv4(double* p, const double (&v)[4]) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
               : "memory");
}

// Quad (4 consecutive doubles of a smem row, x2s % 4 == 0) as two 16-byte
// accesses in a swizzled order: quads 4i..4i+3 start with their low half, quads
// 4i+4..4i+7 with their high half, so a warp's 32 consecutive quads (32-byte
// lane stride) hit every bank exactly 4 times per instruction (the plain order
// is a 2-way bank conflict).
__device__ __forceinline__ void st_quad_smem(double* rowp, int x2s, const double (&q)[4]) {
  double2* s2 = reinterpret_cast<double2*>(rowp + x2s);
  const int h = (x2s >> 4) & 1;
  const double2 lo = make_double2(q[0], q[1]), hi = make_double2(q[2], q[3]);
  s2[h] = h ? hi : lo;
  s2[h ^ 1] = h ? lo : hi;
}
__device__ __forceinline__ void ld_quad_smem(const double* rowp, int x2s, double (&q)[4]) {
  const double2* s2 = reinterpret_cast<const double2*>(rowp + x2s);
  const int h = (x2s >> 4) & 1;
  const double2 a = s2[h];
  const double2 b = s2[h ^ 1];
  const double2 lo = h ? b : a, hi = h ? a : b;
  q[0] = lo.x; q[1] = lo.y; q[2] = hi.x; q[3] = hi.y;
}

// Marching form of the all-inside stencil for the plane passes (n = 64, 128:
// Q4 lanes cover one row, G <= 2): the lanes of a row group walk RPS
// consecutive group rows t, x1 = gg + G t, so the x1 - 1 row of a step is the
// x1 + 1 row of the previous one (G = 2; G = 1 also reuses the centre row):
// 4 (3) row loads per step instead of 5.  The cell values of x2s - 1 come from
// lane - 1 by shuffle (the quad is one aligned 4-node run inside a cell, n0 >= 4).
// Same formulas as stencil4_allin; q goes to the smem row of t, <p, q> into acc.
// out: shared rows (pitch rowpitch, row index t) or, with OUTG, the global plane
// x0 of the result (row x1, 32-byte stores).
// S0 / S1 (compile-time): the x0 - 1 and x0 cell planes coincide / the x1 - 1 and x1
// cell rows coincide on every row of this CTA (caller checked), so those cell rows are
// loaded once.
template <int N, int G, int NR, bool OUTG = false, bool DEDUP = false, bool S0 = false, bool S1 = false>
__device__ __forceinline__ void stencil_march(const Geo& g, const Planes& P3, const double* __restrict__ beta,
                                              int x0, int gg, double* sm, int rowpitch, double& acc) {
  constexpr int nm = N - 1;
  constexpr int Q4 = N / 4;
  static_assert(Q4 == 16 || Q4 == 32, "one row per 16/32 lanes");
  static_assert(G == 1 || G == 2, "row reuse along x1 needs G <= 2");
  const int nsub = blockDim.x / Q4;
  const int RPS = NR / nsub;  // rows per lane group
  const int sub = threadIdx.x / Q4, lane = threadIdx.x % Q4;
  const int x2s = 4 * lane;
  const int L = g.L, sh = g.sh;
  const int c0m = ((x0 - 1) & nm) >> sh, c00 = x0 >> sh;
  const int cc = x2s >> sh;
  const int t0 = sub * RPS;
  double ym[4], pc[4];
  {
    const int x1 = gg + G * t0;
    ldg4v(P3.c + (long long)((x1 - 1) & nm) * N + x2s, ym);
    if (G == 1) ldg4v(P3.c + (long long)x1 * N + x2s, pc);
  }
  for (int k = 0; k < RPS; ++k) {
    const int t = t0 + k;
    const int x1 = gg + G * t;
    const long long row = (long long)x1 * N + x2s;
    double xm[4], xp[4], yp[4];
    if (G == 2) ldg4v(P3.c + row, pc);
    ldg4v(P3.c + (long long)((x1 + 1) & nm) * N + x2s, yp);
    ldg4v(P3.m + row, xm);
    ldg4v(P3.p + row, xp);
    const int c1m = ((x1 - 1) & nm) >> sh, c10 = x1 >> sh;
    const double* b00 = beta + ((size_t)c0m * L + c1m) * L;
    const double* b01 = beta + ((size_t)c0m * L + c10) * L;
    const double* b10 = beta + ((size_t)c00 * L + c1m) * L;
    const double* b11 = beta + ((size_t)c00 * L + c10) * L;
    double z00, z01, z10, z11;
    if constexpr (S0 && S1) {
      z11 = __ldg(b11 + cc);
      z10 = z11;
      z01 = z11;
      z00 = z11;
    } else if constexpr (S0) {
      z11 = __ldg(b11 + cc);
      z10 = __ldg(b10 + cc);
      z01 = z11;
      z00 = z10;
    } else if constexpr (S1) {
      z11 = __ldg(b11 + cc);
      z01 = __ldg(b01 + cc);
      z10 = z11;
      z00 = z01;
    } else {
      cell4(b00, b01, b10, b11, DEDUP && c0m == c00, DEDUP && c1m == c10, cc, z00, z01, z10, z11);
    }
    const int src = (lane - 1) & (Q4 - 1);
    const double m00 = __shfl_sync(0xffffffffu, z00, src, Q4), m01 = __shfl_sync(0xffffffffu, z01, src, Q4);
    const double m10 = __shfl_sync(0xffffffffu, z10, src, Q4), m11 = __shfl_sync(0xffffffffu, z11, src, Q4);
    const double pl = __shfl_sync(0xffffffffu, pc[3], src, Q4);
    const double prr = __shfl_sync(0xffffffffu, pc[0], (lane + 1) & (Q4 - 1), Q4);
    double q[4];
    stencil4_allin_q(g.lam, pc, xm, xp, ym, yp, pl, prr, m00, m01, m10, m11, z00, z01, z10, z11, q);
    if constexpr (OUTG) {
      stv4(sm + (size_t)x1 * N + x2s, q);
    } else {
      st_quad_smem(sm + t * rowpitch, x2s, q);
    }
    acc += ((pc[0] * q[0] + pc[1] * q[1]) + pc[2] * q[2]) + pc[3] * q[3];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (G == 1) {
        ym[e] = pc[e];
        pc[e] = yp[e];
      } else {
        ym[e] = yp[e];
      }
    }
  }
}

template <int N, bool ALLIN, bool DEDUP = false>
__device__ __forceinline__ void stencil_quad(const Geo& g, const Planes& P3,
                                             const double* __restrict__ beta, int x0, int x1,
                                             int x2s, double (&pc)[4], double (&q)[4]) {
  if constexpr (ALLIN) {
    stencil4_allin<N, DEDUP>(g, P3, beta, x0, x1, x2s, pc, q);
  } else {
    const RowCtx rc = make_row(P3, beta, g, x0, x1);
    stencil4(g, rc, x2s, pc, q);
  }
}

// Standalone matvec y = A x (+ optional <x, y>), CTA per (realization, x0, group).
template <int N, int G, bool ALLIN>
__global__ void __launch_bounds__(256) stencil_apply_kernel(Geo g, const double* __restrict__ beta,
                                                            const double* __restrict__ x,
                                                            double* __restrict__ y, double* xy,
                                                            double* part, unsigned* cnt) {
  constexpr int NR = N / G;
  __shared__ double scratch[64];
  const int b = blockIdx.x / (N * G);
  const int rem = blockIdx.x - b * (N * G);
  const int x0 = rem / G, gg = rem - (rem / G) * G;
  const size_t nb = (size_t)N * N * N;
  const double* xb = x + b * nb;
  const double* bb = beta + (size_t)b * g.L * g.L * g.L;
  const Planes P3 = periodic_planes(xb, x0, N);
  double acc = 0.0;
  constexpr int Q4 = N / 4;
  if (CHK_FWD_PF && threadIdx.x < NR)  // this CTA's rows of x: start the DRAM reads now
    bulk_prefetch_l2(P3.c + (size_t)(gg + G * threadIdx.x) * N, N * sizeof(double));
  if constexpr (ALLIN && CHK_MARCH && (Q4 == 16 || Q4 == 32) && G <= 2) {
    stencil_march<N, G, NR, true, true>(g, P3, bb, x0, gg, y + b * nb + (size_t)x0 * N * N, 0, acc);
  } else {
    for (int i = threadIdx.x; i < NR * Q4; i += blockDim.x) {
      const int t = i / Q4, x2 = 4 * (i - (i / Q4) * Q4);
      const int x1 = gg + G * t;
      double pc[4], q[4];
      stencil_quad<N, ALLIN, (N == 512)>(g, P3, bb, x0, x1, x2, pc, q);  // (n = 256: -8 % with dedup)
      stv4(y + b * nb + ((size_t)x0 * N + x1) * N + x2, q);
      acc += ((pc[0] * q[0] + pc[1] * q[1]) + pc[2] * q[2]) + pc[3] * q[3];
    }
  }
  if (xy != nullptr) {
    double t0, t1;
    if (reduce2_last(acc, 0.0, part + (size_t)b * 2 * N * G, cnt + b, rem, N * G, scratch, t0, t1)) {
      if (threadIdx.x == 0) xy[b] = t0;
    }
  }
}

// ----------------------------------------------------------------------------
// corrector right-hand side (homogenize.py:75-89 with lattice.py:335-345)
// ----------------------------------------------------------------------------
__device__ __forceinline__ double nodal_coef(const double* __restrict__ beta, const Geo& g, int x0,
                                             int x1, int x2) {
  // c[x] = 1/8 sum_{delta in {0,1}^3} F[x - delta]: lattice.py:342-345 applies
  // 0.5*(v + roll(v,1)) axis by axis; replicate that order.
  const int nm = g.n - 1;
  const int a0 = (x0 - 1) & nm, a1 = (x1 - 1) & nm, a2 = (x2 - 1) & nm;
  // axis 0 first
  auto c0 = [&](int j1, int j2) { return 0.5 * (fcell(beta, g, x0, j1, j2) + fcell(beta, g, a0, j1, j2)); };
  auto c1 = [&](int j2) { return 0.5 * (c0(x1, j2) + c0(a1, j2)); };
  return 0.5 * (c1(x2) + c1(a2));
}

template <int N>
__global__ void __launch_bounds__(256) corrector_rhs_kernel(Geo g, const double* __restrict__ beta,
                                                            double* __restrict__ f, int axis,
                                                            double scale) {
  const size_t nb = (size_t)N * N * N;
  const int b = blockIdx.y;
  const double* bb = beta + (size_t)b * g.L * g.L * g.L;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
       i += (size_t)gridDim.x * blockDim.x) {
    const int x2 = (int)(i % N), x1 = (int)((i / N) % N), x0 = (int)(i / ((size_t)N * N));
    int xp[3] = {x0, x1, x2}, xm[3] = {x0, x1, x2};
    xp[axis] = (xp[axis] + 1) & (N - 1);
    xm[axis] = (xm[axis] - 1) & (N - 1);
    const double cp = nodal_coef(bb, g, xp[0], xp[1], xp[2]);
    const double cm = nodal_coef(bb, g, xm[0], xm[1], xm[2]);
    f[b * nb + i] = scale * (0.5 * (cp - cm));
  }
}

// ----------------------------------------------------------------------------
// shared-memory addressing of the plane and column tiles
// ----------------------------------------------------------------------------
struct RowAddr {  // pencil = row t (stride HP), element along k2
  int hp;
  __device__ __forceinline__ int operator()(int p, int e) const { return p * hp + e; }
};
struct ColAddr {  // pencil = k2 column, element along rows
  int hp;
  __device__ __forceinline__ int operator()(int p, int e) const { return e * hp + p; }
};
struct X0Addr {  // middle tile: pencil = slot s, element along x0 rows (stride rs)
  int rs;
  __device__ __forceinline__ int operator()(int p, int e) const { return e * rs + p; }
};
template <int W>
struct GAddr {  // middle tile: pencil = (x0, w), element = group slot g
  int rs;
  __device__ __forceinline__ int operator()(int p, int e) const {
    return (p / W) * rs + e * W + (p % W);
  }
};

// Half-length real FFT post-processing, in place at digit-reversed positions of
// each row (length N/2 complex + slot N/2 for the Nyquist term).
template <int N, class TW>
__device__ __forceinline__ void r2c_post(double2* buf, int nrows, int hp, TW tw) {
  constexpr int N2 = N / 2;
  constexpr int NP = N2 / 2 + 1;
  for (int i = threadIdx.x; i < nrows * NP; i += blockDim.x) {
    const int t = i % nrows, k = i / nrows;
    double2* row = buf + t * hp;
    const int kc = (N2 - k) & (N2 - 1);
    const int q = dig_pos<N2, X2Rule<N>::value>(k), qc = dig_pos<N2, X2Rule<N>::value>(kc);
    const double2 zk = row[q];
    const double2 zc = cconj(row[qc]);
    const double2 s = cadd(zk, zc), d = csub(zk, zc);
    const double2 E = make_double2(0.5 * s.x, 0.5 * s.y);
    const double2 O = make_double2(0.5 * d.y, -0.5 * d.x);  // -i d / 2
    if (k == 0) {
      row[q] = make_double2(E.x + O.x, 0.0);
      row[N2] = make_double2(E.x - O.x, 0.0);
    } else {
      const double2 a = cadd(E, cmul(tw_at(tw, k), O));
      const double2 c = cadd(cconj(E), cmul(tw_at(tw, N2 - k), cconj(O)));
      row[q] = a;
      row[qc] = c;
    }
  }
}

// Inverse of r2c_post: X (permuted + Nyquist slot) -> Z at digit-reversed positions.
template <int N, class TW>
__device__ __forceinline__ void c2r_pre(double2* buf, int nrows, int hp, TW tw) {
  constexpr int N2 = N / 2;
  constexpr int NP = N2 / 2 + 1;
  for (int i = threadIdx.x; i < nrows * NP; i += blockDim.x) {
    const int t = i % nrows, k = i / nrows;
    double2* row = buf + t * hp;
    const int kc = (N2 - k) & (N2 - 1);
    const int q = dig_pos<N2, X2Rule<N>::value>(k), qc = dig_pos<N2, X2Rule<N>::value>(kc);
    const double2 xk = row[q];
    const double2 xc = (k == 0) ? row[N2] : row[qc];
    {
      const double2 s = cadd(xk, cconj(xc));
      const double2 d = cmulc(csub(xk, cconj(xc)), tw_at(tw, k));
      // Z = E + i O with E = s/2, O = d/2
      row[q] = make_double2(0.5 * (s.x - d.y), 0.5 * (s.y + d.x));
    }
    if (k != 0 && kc != k) {
      const double2 s = cadd(xc, cconj(xk));
      const double2 d = cmulc(csub(xc, cconj(xk)), tw_at(tw, kc));
      row[qc] = make_double2(0.5 * (s.x - d.y), 0.5 * (s.y + d.x));
    }
  }
}

// Twiddle source of the plane passes: constant memory (CHK_CTW, default) or the
// plan's global table.
#ifndef CHK_CTW
#define CHK_CTW 1
#endif
// Measured (same box A/B): pair pass n = 128 -3.5 %, fwd / inv n = 256 -3.8 % / -3.6 %;
// n = 512 (one CTA per SM, latency-bound, not LSU-bound) +1.4 %, so it keeps the table.
template <int N, bool C>
struct TwSel {
  using type = const double2*;
  __device__ __forceinline__ static type get(const PlanDev& pl) { return pl.tw; }
};
template <int N>
struct TwSel<N, true> {
  using type = CTw;
  __device__ __forceinline__ static type get(const PlanDev&) { return CTw{512 / N}; }
};
template <int N>
using PlaneTw = typename TwSel<N, (CHK_CTW != 0 && N <= 256)>::type;
template <int N>
__device__ __forceinline__ PlaneTw<N> plane_tw(const PlanDev& pl) { return TwSel<N, (CHK_CTW != 0 && N <= 256)>::get(pl); }
// middle passes: register FFTs (reg_fft) index the table with compile-time constants,
// which become constant-bank operands of the multiplies (no load instruction at all):
// reg_tw (n = 128 middle pass -3.7 %, n = 256 -6 %; n = 512, register-capped at 128 and
// latency-bound, +8 %, so it keeps the table).  Stages whose twiddle index varies inside a warp keep the global table
// (divergent constant loads replay: n = 128 middle pass +30 %, n = 512 +12 % when tried),
// except in the n = 256 register-phase kernel, where every twiddle from constant memory
// measured -6 % (mid_tw).
#ifndef CHK_CTW_MID
#define CHK_CTW_MID 1
#endif
template <int N>
using RegTw = typename TwSel<N, (CHK_CTW_MID != 0 && N <= 256)>::type;
template <int N>
__device__ __forceinline__ RegTw<N> reg_tw(const PlanDev& pl) { return TwSel<N, (CHK_CTW_MID != 0 && N <= 256)>::get(pl); }
template <int N>
using MidTw = typename TwSel<N, (CHK_CTW_MID != 0 && N == 256)>::type;
template <int N>
__device__ __forceinline__ MidTw<N> mid_tw(const PlanDev& pl) { return TwSel<N, (CHK_CTW_MID != 0 && N == 256)>::get(pl); }

// ----------------------------------------------------------------------------
// kernel 1: stencil + forward plane transform
// ----------------------------------------------------------------------------
// FWD_APPLY: x rows -> smem.  FWD_INIT: u = 0, f (mean-projected) rows -> smem.
// FWD_Q: q = A p for the slab's rows (the only stencil of the iteration),
// <p, q> partials (the last CTA forms alpha = r.z / p.Aq, solver.py:163-166);
// then R2C along x2 and the x1-group C2C of the smem rows -> spectrum slab S.
enum : int { FWD_APPLY = 0, FWD_INIT = 1, FWD_Q = 2 };

__device__ __forceinline__ void ld4v(const double* p, double (&v)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}

// CTA body, `bid` = plane block index (blockIdx.x of the stand-alone kernel)
template <int N, int G, int MODE, bool ALLIN>
__device__ __forceinline__ void fwd_plane_body(const Geo& g, const double* __restrict__ beta,
                                               const double* __restrict__ src,  // x (APPLY) / f (INIT) / p (Q)
                                               double* __restrict__ u, double2* __restrict__ S,
                                               const PlanDev& pl, const SolveCtl& ctl, const SlabGeo& sg,
                                               int B, int it, int bid, const CUtensorMap* tmap = nullptr) {
  constexpr int NR = N / G;
  constexpr int N2 = N / 2;
  constexpr int H = N2 + 1;
  constexpr int HP = H;
  extern __shared__ __align__(128) double2 buf[];
  __shared__ double scratch[64];
  const int nlg = sg.nloc * G;                        // CTAs per realization (all planes)
  const int b = bid / (sg.nrun * G);
  const int rrun = bid - b * (sg.nrun * G);
  const int x0l = sg.run0 + rrun / G, gg = rrun - (rrun / G) * G;  // local plane, x1 group
  const int rem = x0l * G + gg;                       // partial slot of this CTA
  const int x0 = sg.x0_off + x0l;                     // global plane
  const size_t nn = (size_t)N * N;
  const size_t nb = (size_t)sg.nloc * nn;             // local DOF per realization
  double* sm = reinterpret_cast<double*>(buf);
  RState* st = (MODE == FWD_APPLY) ? nullptr : ctl.st + b;
  constexpr int Q4 = N / 4;

  if (MODE == FWD_APPLY) {
    // rows of x -> smem rows, 32 bytes per thread
    for (int i = threadIdx.x; i < NR * Q4; i += blockDim.x) {
      const int t = i / Q4, x2 = 4 * (i - (i / Q4) * Q4);
      double v[4];
      ldg4v(src + b * nb + ((size_t)x0l * N + gg + G * t) * N + x2, v);
      st_quad_smem(sm + t * 2 * HP, x2, v);
    }
  } else if (MODE == FWD_INIT) {
    const int status = st->status;
    const double shift = st->rhs_projected ? st->mean_f : 0.0;  // solver.py:139-143
    for (int i = threadIdx.x; i < NR * Q4; i += blockDim.x) {
      const int t = i / Q4, x2 = 4 * (i - (i / Q4) * Q4);
      const size_t idx = b * nb + ((size_t)x0l * N + gg + G * t) * N + x2;
      double v[4];
      ldg4v(src + idx, v);
      const double zero[4] = {0.0, 0.0, 0.0, 0.0};
      stv4(u + idx, zero);
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] -= shift;
      st_quad_smem(sm + t * 2 * HP, x2, v);
    }
    if (status != ST_ACTIVE) return;
  } else {  // FWD_Q
    if (st->status != ST_ACTIVE) return;
    const double* pb = src + b * nb;
    const double* bb = beta + (size_t)b * g.L * g.L * g.L;
    Planes P3;
    P3.c = pb + (size_t)x0l * nn;
    P3.m = (x0l > 0) ? P3.c - nn : (sg.halo_lo ? sg.halo_lo + b * nn : pb + (size_t)(N - 1) * nn);
    P3.p = (x0l < sg.nloc - 1) ? P3.c + nn : (sg.halo_hi ? sg.halo_hi + b * nn : pb);
    if (CHK_FWD_PF && threadIdx.x < NR)  // this CTA's rows of p: start the DRAM reads now
      bulk_prefetch_l2(P3.c + (size_t)(gg + G * threadIdx.x) * N, N * sizeof(double));
    double acc = 0.0;
    if constexpr (ALLIN && CHK_MARCH && (Q4 == 16 || Q4 == 32) && G <= 2) {
      // s0: cell planes of x0 - 1 and x0 coincide; s1: every row x1 = gg + G t of this CTA
      // shares its cell row with x1 - 1 (G = 2, odd gg, n0 >= 2)
      const bool s0 = CHK_MARCH_S0 && ((((x0 - 1) & (N - 1)) >> g.sh) == (x0 >> g.sh));
      const bool s1 = CHK_MARCH_S0 && G == 2 && (gg & 1) && g.sh >= 1;
      if (s0 && s1)
        stencil_march<N, G, NR, false, false, true, true>(g, P3, bb, x0, gg, sm, 2 * HP, acc);
      else if (s0)
        stencil_march<N, G, NR, false, false, true, false>(g, P3, bb, x0, gg, sm, 2 * HP, acc);
      else if (s1)
        stencil_march<N, G, NR, false, false, false, true>(g, P3, bb, x0, gg, sm, 2 * HP, acc);
      else
        stencil_march<N, G, NR, false, false>(g, P3, bb, x0, gg, sm, 2 * HP, acc);
    } else if constexpr (ALLIN && Q4 == 64 && CHK_FWD_CS) {
      // G >= n0: every row x1 = gg + G t of this CTA has the same x1 mod n0, so whether
      // the x1 - 1 cell row coincides is CTA-uniform, as is the x0 - 1 cell plane
      // (x0 fixed): four compile-time variants with the coinciding rows loaded once
      const bool u0 = ((((x0 - 1) & (N - 1)) >> g.sh) == (x0 >> g.sh));
      const bool u1 = (G >= g.mask + 1) && ((gg & g.mask) != 0);
      auto body = [&](auto cs_tag) {
        constexpr int CS = decltype(cs_tag)::value;
        for (int i = threadIdx.x; i < NR * Q4; i += blockDim.x) {
          const int t = i / Q4, x2 = 4 * (i - (i / Q4) * Q4);
          double pc[4], q[4];
          stencil4_allin<N, false, CS, true>(g, P3, bb, x0, gg + G * t, x2, pc, q);
          st_quad_smem(sm + t * 2 * HP, x2, q);
          acc += ((pc[0] * q[0] + pc[1] * q[1]) + pc[2] * q[2]) + pc[3] * q[3];
        }
      };
      if (u0 && u1) body(std::integral_constant<int, 3>{});
      else if (u0) body(std::integral_constant<int, 1>{});
      else if (u1) body(std::integral_constant<int, 2>{});
      else body(std::integral_constant<int, 0>{});
    } else {
      for (int i = threadIdx.x; i < NR * Q4; i += blockDim.x) {
        const int t = i / Q4, x2 = 4 * (i - (i / Q4) * Q4);
        double pc[4], q[4];
        stencil_quad<N, ALLIN, (N == 512)>(g, P3, bb, x0, gg + G * t, x2, pc, q);
        st_quad_smem(sm + t * 2 * HP, x2, q);
        acc += ((pc[0] * q[0] + pc[1] * q[1]) + pc[2] * q[2]) + pc[3] * q[3];
      }
    }
    double t0, t1;
    if (reduce2_last(acc, 0.0, ctl.part + (size_t)b * 2 * ctl.maxblk, &st->cnt, rem, nlg,
                     scratch, t0, t1)) {
      if (threadIdx.x == 0) {
        if (ctl.red_only) {
          ctl.red[4 * b] = t0;  // rank-local p.Ap, decided after the allreduce
        } else {
          if ((!(t0 > 0.0) || !isfinite(t0))) {  // solver.py:164-165
            st->status = ST_BREAKDOWN;
            st->iters = it;
          }
          st->pq = t0;
          st->alpha = st->rz[(it - 1) & 1] / t0;  // solver.py:166
        }
      }
    }
  }
  __syncthreads();
  // R2C along x2: rows of N reals viewed as N/2 complex (z_m = x_2m + i x_2m+1)
  const PlaneTw<N> ptw = plane_tw<N>(pl);
  fft_smem_r<N2, false, NR, X2Rule<N>::value>(buf, RowAddr{HP}, ptw, N);
  r2c_post<N>(buf, NR, HP, ptw);
  __syncthreads();
  // C2C along the x1 group (length NR)
  fft_smem<NR, false, H>(buf, ColAddr{HP}, ptw, N);
  // the slab row is contiguous in smem (HP == H); it leaves in P column chunks
  // (one bulk store each; a single chunk when the grid is not slab-decomposed)
  fence_proxy_async_smem();
  __syncthreads();
  if constexpr (IlW<N>::value > 0) {
    // interleaved layout: 32-byte pieces at a stride of G*W complex
    constexpr int IW = IlW<N>::value;
    static_assert(IW == 2, "pieces are two complex values");
    if (tmap) {
      // tensor-map TMA store: box {4 doubles, 1 group, TPB pieces, 1 row} from the dense
      // smem row to the 32-byte pieces at a stride of G*W complex (chk_plane_tmap)
      if (threadIdx.x == 0) {
        const int npc = sg.ncols / IW;
        for (int c = 0; c < sg.P; ++c) {
          const int row = (c * B + b) * sg.nloc + x0l;
          for (int i0 = 0; i0 < npc; i0 += TmapBox<N>::value)
            tma_store_4d(tmap, buf + (size_t)c * sg.ncols + (size_t)i0 * IW, 0, gg, i0, row);
        }
        bulk_commit();
        bulk_wait_read0();
      }
    } else {
      const int npc = sg.ncols / IW;
      for (int c = 0; c < sg.P; ++c) {
        double* dst = reinterpret_cast<double*>(S + slab_row(sg, B, G, c, b, x0l, 0) + gg * IW);
        const double* src = reinterpret_cast<const double*>(buf + (size_t)c * sg.ncols);
        for (int i = threadIdx.x; i < npc; i += blockDim.x) {
          const double2 a = *reinterpret_cast<const double2*>(src + 4 * i);
          const double2 d = *reinterpret_cast<const double2*>(src + 4 * i + 2);
          const double v[4] = {a.x, a.y, d.x, d.y};
          stv4(dst + (size_t)i * 2 * G * IW, v);
        }
      }
    }
    return;
  }
  if (threadIdx.x < sg.P) {
    const int c = threadIdx.x;
    bulk_s2g(S + slab_row(sg, B, G, c, b, x0l, gg), buf + (size_t)c * sg.ncols,
             (uint32_t)(sg.ncols * sizeof(double2)));
    bulk_commit();
    bulk_wait_read0();
  }
}

// ----------------------------------------------------------------------------
// kernel 2: spectral column pass (x1 group combine + x0), diagonal scaling
// ----------------------------------------------------------------------------
// MID_APPLY: z = D * X (standalone preconditioner, DC term kept).
// MID_INIT:  R = X (the spectrum of r0 = f), ||r0||^2 and r0.z0 by Parseval.
// MID_ITER:  R -= alpha * Q (Q = FFT of q = A p; solver.py:168 in the Fourier
//            domain -- r is only ever consumed through its spectrum), then
//            ||r||^2 (stop test, solver.py:171-177), z = D * R with the mean
//            projection (solver.py:179) and r.z (solver.py:180-183).
// The residual spectrum R lives in HBM tile-major (one contiguous N x G*W block
// per column tile), so each CTA streams its own slice.
enum : int { MID_APPLY = 0, MID_INIT = 1, MID_ITER = 2 };

__host__ __device__ __forceinline__ int mid_dsm_offset(int tile_elems, int gw, int r1) {
  const int a = tile_elems * 16, c = r1 * gw * 8;
  return ((a > c ? a : c) + 15) & ~15;
}

// Scalar decisions of one iteration, taken by the last CTA of a realization
// (rr = ||r||^2, rz = r.z, both already divided by N^3).
__device__ __forceinline__ void mid_decide(RState* st, const SolveCtl& ctl, int b, int it, double rr,
                                           double rz) {
  if (ctl.red_only) {  // slab mode: rank-local sums, decided after the allreduce
    ctl.red[4 * b + 1] = rr;
    ctl.red[4 * b + 2] = rz;
    return;
  }
  if (it == 0) {
    st->normf = sqrt(rr);  // solver.py:132 (after the optional projection, :142)
    if (!(rr > 0.0)) {     // projected RHS vanished (solver.py:144-148)
      st->status = ST_CONVERGED;
      st->iters = 0;
      st->final_rel = 0.0;
      return;
    }
    st->rz[0] = rz;
    st->norm_pf = sqrt(fabs(rz));  // solver.py:156
    st->beta = 0.0;
    return;
  }
  const double rel = sqrt(rr) / st->normf;  // solver.py:171
  if (ctl.hist) ctl.hist[(size_t)b * ctl.max_iter + (it - 1)] = rel;
  st->final_rel = rel;
  if (!isfinite(rel)) {  // solver.py:172-173
    st->status = ST_BREAKDOWN;
    st->iters = it;
    return;
  }
  if (!ctl.prs && rel <= ctl.tol) {  // solver.py:175-177
    st->status = ST_CONVERGED;
    st->iters = it;
    return;
  }
  st->beta = rz / st->rz[(it - 1) & 1];  // solver.py:184
  st->rz[it & 1] = rz;
  if (ctl.prs && sqrt(fabs(rz)) / st->norm_pf <= ctl.tol) {  // solver.py:181-183
    st->status = ST_CONVERGED;
    st->iters = it;
    return;
  }
  if (it >= ctl.max_iter) {
    st->status = ST_NOT_CONVERGED;
    st->iters = it;
  }
}

// Slot bookkeeping of a middle-pass tile starting at global column c0.
template <int N, int G, int W>
__device__ __forceinline__ void mid_slots(int c0, const PlanDev& pl, int* s_k1, int* s_k2, double* s_wgt,
                                          double2* s_tw) {
  constexpr int NR = N / G, N2 = N / 2, H = N2 + 1, GW = G * W;
  for (int s = threadIdx.x; s < GW; s += blockDim.x) {
    const int m = dig_freq<G>(s / W), w = s % W;
    const int c = c0 + w;
    const int q1 = c / H, q2 = c - (c / H) * H;
    const int kp = dig_freq<NR>(q1);
    s_k1[s] = kp + m * NR;
    const int k2 = (q2 == N2) ? N2 : dig_freq<N2, X2Rule<N>::value>(q2);
    s_k2[s] = k2;
    s_wgt[s] = (k2 == 0 || k2 == N2) ? 1.0 : 2.0;
    if (s_tw) s_tw[s] = __ldg(pl.tw + (s / W) * kp);  // as a load slot (group s/W, column w)
  }
}

// The diagonal tile D[pos0][slot] (x0 in digit-reversed order) of the
// preconditioner, evaluated from its factors (slots from mid_slots, synced).
// `coef` is scratch of r1 * G*W doubles.
template <int N, int G, int W>
__device__ __forceinline__ void mid_dtile(double* coef, double* Dsm, const PlanDev& pl, const int* s_k1,
                                          const int* s_k2) {
  constexpr int GW = G * W;
  if (pl.kind == KIND_LKR) {
    // D = U0p^T C, C[r][slot] = U1[r][k1] U2[r][k2]: rank-r1 contraction
    const double* U1 = pl.U + (size_t)pl.r1 * N;
    const double* U2 = pl.U + (size_t)2 * pl.r1 * N;
    for (int i = threadIdx.x; i < pl.r1 * GW; i += blockDim.x) {
      const int s = i % GW, rr = i / GW;
      coef[rr * GW + s] = __ldg(U1 + rr * N + s_k1[s]) * __ldg(U2 + rr * N + s_k2[s]);
    }
    __syncthreads();
    // 4 positions x 4 slots per thread: 2 x 256-bit U0p loads + 2 smem loads per 16 FMA
    constexpr int PQ = N / 4, SQ = GW / 4;
    static_assert(GW % 4 == 0, "slots per tile must be a multiple of 4");
    for (int i = threadIdx.x; i < PQ * SQ; i += blockDim.x) {
      const int sq = i % SQ, pq = i / SQ;
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
      const double* up = pl.Up + 4 * pq;
      const double* cp = coef + 4 * sq;
#pragma unroll 2
      for (int rr = 0; rr < pl.r1; ++rr) {
        double u4[4];
        ldg4v(up + (size_t)rr * N, u4);
        const double2 c01 = *reinterpret_cast<const double2*>(cp + rr * GW);
        const double2 c23 = *reinterpret_cast<const double2*>(cp + rr * GW + 2);
        const double cc[4] = {c01.x, c01.y, c23.x, c23.y};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][c] = fma(u4[a], cc[c], acc[a][c]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) Dsm[(4 * pq + a) * GW + 4 * sq + c] = acc[a][c];
    }
  } else {
    for (int i = threadIdx.x; i < N * GW; i += blockDim.x) {
      const int s = i % GW, pos0 = i / GW;
      const int k0 = dig_freq0<N>(pos0);
      // eigensum order of spectral.py:47-52: (lam_i + lam_j) + lam_k
      const double gsum = (__ldg(pl.lam + k0) + __ldg(pl.lam + s_k1[s])) + __ldg(pl.lam + s_k2[s]);
      double D;
      if (pl.kind == KIND_REGULARIZED && pl.delta > 0.0) {
        D = 1.0 / (gsum + pl.delta);
      } else {
        D = (gsum > 0.0) ? 1.0 / gsum : 0.0;
      }
      Dsm[pos0 * GW + s] = D;
    }
  }
}

// Precompute of every diagonal tile of a plan (once per plan; the middle
// passes then stream their tile from HBM instead of re-evaluating the rank-r1
// contraction per CTA).  CTA = tile; smem: r1 * GW + N * GW doubles.
template <int N, int G, int W>
__global__ void __launch_bounds__(256) dtile_kernel(PlanDev pl, double* __restrict__ Dout) {
  constexpr int GW = G * W;
  extern __shared__ __align__(128) double dsh[];
  __shared__ int s_k1[GW], s_k2[GW];
  __shared__ double s_wgt[GW];
  const int r1 = pl.kind == KIND_LKR ? pl.r1 : 0;
  double* coef = dsh;
  double* Dsm = dsh + ((r1 * GW + 1) & ~1);
  mid_slots<N, G, W>(blockIdx.x * W, pl, s_k1, s_k2, s_wgt, nullptr);
  __syncthreads();
  mid_dtile<N, G, W>(coef, Dsm, pl, s_k1, s_k2);
  __syncthreads();
  double* out = Dout + (size_t)blockIdx.x * N * GW;
  for (int i = threadIdx.x; i < N * GW; i += blockDim.x) out[i] = Dsm[i];
}

// Shared prologue of both middle kernels: slot bookkeeping and the diagonal
// tile (16-byte async copies of the precomputed tile, or evaluated in place).
template <int N, int G, int W, int MODE>
__device__ __forceinline__ void mid_prologue(double2* buf, double* Dsm, int c0, const PlanDev& pl,
                                             int* s_k1, int* s_k2, double* s_wgt, double2* s_tw) {
  constexpr int GW = G * W;
  mid_slots<N, G, W>(c0, pl, s_k1, s_k2, s_wgt, s_tw);
  if (pl.D) {
    const double* src = pl.D + (size_t)(c0 / W) * N * GW;
    for (int i = threadIdx.x; i < N * GW / 2; i += blockDim.x) cp_async16(Dsm + 2 * i, src + 2 * i);
    cp_async_commit();
    cp_async_wait_all();
  }
  __syncthreads();
  if (!pl.D) {
    mid_dtile<N, G, W>(reinterpret_cast<double*>(buf), Dsm, pl, s_k1, s_k2);
  }
  __syncthreads();
  if (MODE != MID_APPLY && threadIdx.x < GW) {
    // mean projection of z (solver.py:153,179): the zero-frequency coefficient is 0
    if (s_k1[threadIdx.x] == 0 && s_k2[threadIdx.x] == 0) Dsm[threadIdx.x] = 0.0;
  }
  __syncthreads();
}

// Residual update + scaling of one spectral element (pos0, slot s).
template <int MODE>
__device__ __forceinline__ double2 mid_point(double2 v, double D, double wgt, double scale,
                                             double alpha, double2* rptr, double& rr, double& rz) {
  if (MODE == MID_APPLY) return cscale(v, D * scale);
  double2 R = v;
  if (MODE == MID_ITER) {
    const double2 Ro = *rptr;
    R = make_double2(fma(-alpha, v.x, Ro.x), fma(-alpha, v.y, Ro.y));
  }
  *rptr = R;
  const double m2 = R.x * R.x + R.y * R.y;
  rr = fma(wgt, m2, rr);
  rz = fma(wgt * D, m2, rz);
  return cscale(R, D * scale);
}


// Fused shared-memory kernel for large n (n >= 256: the plane slab forces G >= 8):
// load + group combine in registers, the x0 stages but the last through shared
// memory, [last forward stage + residual update + scaling + Parseval + first
// inverse stage] in registers, remaining inverse stages, inverse group combine
// + store in registers: 12 shared-memory passes per element instead of 20.
// DG: the diagonal tile is read from the plan's precomputed table (L2) in the
// fused last stage instead of being staged in shared memory -- the tile alone
// then fits 3 CTAs per SM at n = 256 (2 with the staged diagonal).
template <int N, int G, int W, int NB, int MODE, bool DG = false>
__global__ void __launch_bounds__(MidNT<N>::value, DG ? MidNT<N>::minb_dg : MidNT<N>::minb)
    mid_column_fused_kernel(double2* __restrict__ S, PlanDev pl, SolveCtl ctl, SlabGeo sg, int it, int B) {
  constexpr int NR = N / G;
  constexpr int N2 = N / 2;
  constexpr int H = N2 + 1;
  constexpr int GW = G * W;
  constexpr int RS = GW + 1;
  constexpr int RL = LastRadix<N>::value;  // radix of the fused last x0 stage
  constexpr bool IL = IlW<N>::value > 0;
  static_assert(!IL || IlW<N>::value == W, "interleaved pieces are one tile wide");
  const size_t GSTR = IL ? (size_t)W : (size_t)sg.ncols;  // stride between the groups of a column
  const int TILES = sg.tiles;
  const int nsh = __ffs(sg.nloc) - 1;
  extern __shared__ __align__(128) double2 buf[];
  const int doff = mid_dsm_offset(N * RS, GW, pl.kind == KIND_LKR ? pl.r1 : 0);
  double* Dsm = reinterpret_cast<double*>(reinterpret_cast<char*>(buf) + doff);  // [N][GW]
  __shared__ double scratch[64];
  __shared__ int s_k1[GW], s_k2[GW];
  __shared__ double s_wgt[GW];
  __shared__ double2 s_tw[GW];
  __shared__ int s_act[NB];
  __shared__ double s_alpha[NB];
  __shared__ double s_wsum[NB * (MidNT<N>::value / 32) * 2];  // per-warp Parseval partials (warp_partials)
  const int bg = blockIdx.x / TILES;
  const int tile = blockIdx.x - bg * TILES;
  const int c0 = tile * W;
  const int cg0 = (sg.tile_off + tile) * W;
  const int b0 = bg * NB;
  if (threadIdx.x == 0) {
    int any = 0;
    for (int j = 0; j < NB; ++j) {
      const int b = b0 + j;
      int a = (b < B);
      if (a && MODE != MID_APPLY) a = (ctl.st[b].status == ST_ACTIVE);
      s_act[j] = a;
      s_alpha[j] = (a && MODE == MID_ITER) ? ctl.st[b].alpha : 0.0;
      any |= a;
    }
    scratch[0] = any;
  }
  __syncthreads();
  if (scratch[0] == 0.0) return;
  __shared__ int s_dc;  // DG: slot of the zero frequency (k1 = k2 = 0) in this tile, or -1
  const double* Dg = nullptr;
  if constexpr (DG) {
    mid_slots<N, G, W>(cg0, pl, s_k1, s_k2, s_wgt, s_tw);
    if (threadIdx.x == 0) s_dc = -1;
    __syncthreads();
    if (MODE != MID_APPLY && threadIdx.x < GW && s_k1[threadIdx.x] == 0 && s_k2[threadIdx.x] == 0)
      s_dc = threadIdx.x;
    __syncthreads();
    Dg = pl.D + (size_t)(cg0 / W) * N * GW;
  } else {
    mid_prologue<N, G, W, MODE>(buf, Dsm, cg0, pl, s_k1, s_k2, s_wgt, s_tw);
  }
  const double scale = 2.0 / ((double)N * N * N);
  if (CHK_FUSED_PF && DG && threadIdx.x >= 32 && threadIdx.x < 36) {  // diagonal tile -> L2 (first use: fused last stage)
    constexpr uint32_t q = N * GW * sizeof(double) / 4;
    bulk_prefetch_l2(reinterpret_cast<const char*>(Dg) + (threadIdx.x - 32) * q, q);
  }
  for (int j = 0; j < NB; ++j) {
    if (!s_act[j]) continue;
    const int b = b0 + j;
    if (CHK_FUSED_PF && MODE == MID_ITER && threadIdx.x < 4) {  // residual tile -> L2 (read in the fused last stage)
      constexpr uint32_t q = N * GW * sizeof(double2) / 4;
      bulk_prefetch_l2(reinterpret_cast<const char*>(ctl.Rh + ((size_t)b * TILES + tile) * N * GW) + threadIdx.x * q, q);
    }
    // ---- load + group combine (registers) -> smem ----
    for (int item = threadIdx.x; item < N * W; item += blockDim.x) {
      const int w = item % W, x0 = item / W;
      const size_t rbase = slab_row(sg, B, G, x0 >> nsh, b, x0 & (sg.nloc - 1), 0) + (IL ? c0 * G : c0) + w;
      double2 v[G];
#pragma unroll
      for (int g = 0; g < G; ++g) v[g] = S[rbase + (size_t)g * GSTR];
#pragma unroll
      for (int g = 1; g < G; ++g) v[g] = cmul(v[g], s_tw[g * W + w]);
      reg_fft<G, false>(v, reg_tw<N>(pl), N);
#pragma unroll
      for (int g = 0; g < G; ++g) buf[x0 * RS + g * W + w] = v[g];
    }
    __syncthreads();
    FftRecButLast<N, N, false, GW>::run(buf, X0Addr{RS}, mid_tw<N>(pl), 1);
    // ---- last stage + residual / scaling + first inverse stage (registers) ----
    double rr = 0.0, rz = 0.0;
    double2* Rt = ctl.Rh + ((size_t)b * TILES + tile) * N * GW;
    for (int item = threadIdx.x; item < GW * (N / RL); item += blockDim.x) {
      const int s = item % GW, blk = item / GW;
      double2 v[RL];
#pragma unroll
      for (int e = 0; e < RL; ++e) v[e] = buf[(blk * RL + e) * RS + s];
      dftR<RL, false>(v);
#pragma unroll
      for (int e = 0; e < RL; ++e) {
        const int pos0 = blk * RL + e;
        double D;
        if constexpr (DG) {
          // mean projection of z (solver.py:153,179): the zero-frequency coefficient is 0
          D = (pos0 == 0 && s == s_dc) ? 0.0 : __ldg(Dg + pos0 * GW + s);
        } else {
          D = Dsm[pos0 * GW + s];
        }
        v[e] = mid_point<MODE>(v[e], D, s_wgt[s], scale, s_alpha[j], Rt + (size_t)pos0 * GW + s, rr, rz);
      }
      dftR<RL, true>(v);
#pragma unroll
      for (int e = 0; e < RL; ++e) buf[(blk * RL + e) * RS + s] = v[e];
    }
    __syncthreads();
    FftRecButLast<N, N, true, GW>::run(buf, X0Addr{RS}, mid_tw<N>(pl), 1);
    // ---- inverse group combine + store (registers) ----
    for (int item = threadIdx.x; item < N * W; item += blockDim.x) {
      const int w = item % W, x0 = item / W;
      const size_t rbase = slab_row(sg, B, G, x0 >> nsh, b, x0 & (sg.nloc - 1), 0) + (IL ? c0 * G : c0) + w;
      double2 v[G];
#pragma unroll
      for (int g = 0; g < G; ++g) v[g] = buf[x0 * RS + g * W + w];
      reg_fft<G, true>(v, reg_tw<N>(pl), N);
#pragma unroll
      for (int g = 1; g < G; ++g) v[g] = cmulc(v[g], s_tw[g * W + w]);
#pragma unroll
      for (int g = 0; g < G; ++g) S[rbase + (size_t)g * GSTR] = v[g];
    }
    if (MODE != MID_APPLY) warp_partials(rr, rz, s_wsum, j);
    __syncthreads();
  }
  if (MODE != MID_APPLY) {
    const double inv = 1.0 / ((double)N * N * N);  // Parseval: (1/N^3) sum conj(X) Y
    mid_tickets<NB>(s_wsum, s_act, b0, tile, TILES, ctl, scratch, [&](int b, double t0, double t1) {
      mid_decide(ctl.st + b, ctl, b, it, t0 * inv, t1 * inv);
    });
  }
}

// ----------------------------------------------------------------------------
// kernel 2c: register-phase spectral column pass for n = 256 (x0 radix 2, 8, 8, 2)
// ----------------------------------------------------------------------------
// CTA = NB realizations x one tile (W = 2 columns x G = 8 groups = 16 slots, 256
// x0 positions; interleaved spectrum layout).  Per realization:
//   A  (thread = column w, x0 pair j, j + 128): group combine of both x0 rows in
//      registers + the radix-2 x0 stage (M = 256)                     -> smem
//   B1 (thread = slot, block, offset): radix-8 stage M = 128            smem -> smem
//   B2 (thread = slot, 16-block): radix-8 (M = 16) + radix-2 (M = 2), residual
//      update / diagonal (read from the plan's table) / Parseval, inverse   smem -> smem
//   B1' inverse M = 128 stage;  A' inverse radix-2 + group combine      -> HBM
// 8 shared-memory passes per element (the stage kernel mid_column_fused: 12).
template <int NB, int MODE>
#ifndef CHK_R256_RPF
#define CHK_R256_RPF 1
#endif
#ifndef CHK_R256_RS
#define CHK_R256_RS 18
#endif
#ifndef CHK_R256_MINB
#define CHK_R256_MINB 2
#endif
__global__ void __launch_bounds__(256, CHK_R256_MINB) mid_column_r256_kernel(double2* __restrict__ S, PlanDev pl, SolveCtl ctl,
                                                                 SlabGeo sg, int it, int B) {
  // row pitch 18: phase A / A' lanes hold (x0 pair, column) = (lane >> 1, lane & 1), so a
  // quarter warp touches {0, 1} + pitch * {0..3}: distinct 16-byte banks need pitch = 2 mod 8
  // (pitch 17 was a 2-way conflict on those four accesses: 34 M of 179 M wavefronts per launch)
  constexpr int N = 256, G = 8, W = 2, GW = G * W, RS = CHK_R256_RS;
  static_assert(IlW<N>::value == W, "interleaved spectrum layout expected at n = 256");
  static_assert(x0_radix(N, 256) == 2 && x0_radix(N, 128) == 8 && x0_radix(N, 16) == 8 && x0_radix(N, 2) == 2,
                "x0 radix order 2, 8, 8, 2");
  const int TILES = sg.tiles;
  const int nsh = __ffs(sg.nloc) - 1;
  extern __shared__ __align__(128) double2 buf[];  // [N][RS]
  __shared__ double scratch[64];
  __shared__ int s_k1[GW], s_k2[GW];
  __shared__ double s_wgt[GW];
  __shared__ double2 s_tw[GW];
  __shared__ int s_act[NB];
  __shared__ double s_alpha[NB];
  __shared__ double s_wsum[NB * 8 * 2];
  __shared__ int s_dc;
  const int bg = blockIdx.x / TILES;
  const int tile = blockIdx.x - bg * TILES;
  const int c0 = tile * W;
  const int cg0 = (sg.tile_off + tile) * W;
  const int b0 = bg * NB;
  if (threadIdx.x == 0) {
    int any = 0;
    for (int j = 0; j < NB; ++j) {
      const int b = b0 + j;
      int a = (b < B);
      if (a && MODE != MID_APPLY) a = (ctl.st[b].status == ST_ACTIVE);
      s_act[j] = a;
      s_alpha[j] = (a && MODE == MID_ITER) ? ctl.st[b].alpha : 0.0;
      any |= a;
    }
    scratch[0] = any;
    s_dc = -1;
  }
  __syncthreads();
  if (scratch[0] == 0.0) return;
  mid_slots<N, G, W>(cg0, pl, s_k1, s_k2, s_wgt, s_tw);
  __syncthreads();
  if (MODE != MID_APPLY && threadIdx.x < GW && s_k1[threadIdx.x] == 0 && s_k2[threadIdx.x] == 0)
    s_dc = threadIdx.x;
  __syncthreads();
  const double* Dg = pl.D + (size_t)(cg0 / W) * N * GW;
  const double scale = 2.0 / ((double)N * N * N);
  const int wA = threadIdx.x & 1, jA = threadIdx.x >> 1;  // phase A item (column, x0 pair)
  for (int j = 0; j < NB; ++j) {
    if (!s_act[j]) continue;
    const int b = b0 + j;
    if (CHK_R256_RPF && MODE == MID_ITER && threadIdx.x == 0)  // residual tile -> L2 before B2 reads it
      bulk_prefetch_l2(ctl.Rh + ((size_t)b * TILES + tile) * N * GW, (uint32_t)(N * GW * sizeof(double2)));
    // ---- A: loads, group combine, radix-2 stage (M = 256) ----
    {
      double2 v[2][G];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int x0 = jA + 128 * h;
        const size_t rbase = slab_row(sg, B, G, x0 >> nsh, b, x0 & (sg.nloc - 1), 0) + c0 * G + wA;
#pragma unroll
        for (int g = 0; g < G; ++g) v[h][g] = S[rbase + (size_t)g * W];
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int g = 1; g < G; ++g) v[h][g] = cmul(v[h][g], s_tw[g * W + wA]);
        reg_fft<G, false>(v[h], reg_tw<N>(pl), N);
      }
      const double2 t1 = tw_at(mid_tw<N>(pl), jA);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double2 a = cadd(v[0][g], v[1][g]);
        const double2 d = cmul(csub(v[0][g], v[1][g]), t1);
        buf[jA * RS + g * W + wA] = a;
        buf[(jA + 128) * RS + g * W + wA] = d;
      }
    }
    __syncthreads();
    // ---- B1: radix-8 stage M = 128 (stride 16) ----
    for (int item = threadIdx.x; item < 2 * 16 * GW; item += blockDim.x) {
      const int s = item % GW, jj = (item / GW) % 16, blk = item / (16 * GW);
      double2* base = buf + (blk * 128 + jj) * RS + s;
      double2 v[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) v[t] = base[16 * t * RS];
      dftR<8, false>(v);
      if (jj > 0) {
#pragma unroll
        for (int m = 1; m < 8; ++m) v[m] = cmul(v[m], tw_at(mid_tw<N>(pl), jj * m * 2));
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) base[16 * t * RS] = v[t];
    }
    __syncthreads();
    // ---- B2: last two stages, residual / diagonal / Parseval, first two inverse stages ----
    double rr = 0.0, rz = 0.0;
    {
      const int s = threadIdx.x % GW, blk = threadIdx.x / GW;  // 16 blocks of 16 positions
      double2* row = buf + (blk * 16) * RS + s;
      double2 v[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = row[e * RS];
      reg_fft<16, false>(v, reg_tw<N>(pl), N);
      double2* Rt = ctl.Rh + ((size_t)b * TILES + tile) * N * GW + (blk * 16) * GW + s;
      const double wgt = s_wgt[s];
      const double al = s_alpha[j];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int pos0 = blk * 16 + e;
        // mean projection of z (solver.py:153,179): the zero-frequency coefficient is 0
        const double D = (pos0 == 0 && s == s_dc) ? 0.0 : __ldg(Dg + pos0 * GW + s);
        v[e] = mid_point<MODE>(v[e], D, wgt, scale, al, Rt + e * GW, rr, rz);
      }
      reg_fft<16, true>(v, reg_tw<N>(pl), N);
#pragma unroll
      for (int e = 0; e < 16; ++e) row[e * RS] = v[e];
    }
    __syncthreads();
    // ---- B1': inverse M = 128 stage ----
    for (int item = threadIdx.x; item < 2 * 16 * GW; item += blockDim.x) {
      const int s = item % GW, jj = (item / GW) % 16, blk = item / (16 * GW);
      double2* base = buf + (blk * 128 + jj) * RS + s;
      double2 v[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) v[t] = base[16 * t * RS];
      if (jj > 0) {
#pragma unroll
        for (int m = 1; m < 8; ++m) v[m] = cmulc(v[m], tw_at(mid_tw<N>(pl), jj * m * 2));
      }
      dftR<8, true>(v);
#pragma unroll
      for (int t = 0; t < 8; ++t) base[16 * t * RS] = v[t];
    }
    __syncthreads();
    // ---- A': inverse radix-2 stage, inverse group combine, store ----
    {
      double2 v[2][G];
      const double2 t1 = tw_at(mid_tw<N>(pl), jA);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const double2 a = buf[jA * RS + g * W + wA];
        const double2 d = cmulc(buf[(jA + 128) * RS + g * W + wA], t1);
        v[0][g] = cadd(a, d);
        v[1][g] = csub(a, d);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        reg_fft<G, true>(v[h], reg_tw<N>(pl), N);
#pragma unroll
        for (int g = 1; g < G; ++g) v[h][g] = cmulc(v[h][g], s_tw[g * W + wA]);
        const int x0 = jA + 128 * h;
        const size_t rbase = slab_row(sg, B, G, x0 >> nsh, b, x0 & (sg.nloc - 1), 0) + c0 * G + wA;
#pragma unroll
        for (int g = 0; g < G; ++g) S[rbase + (size_t)g * W] = v[h][g];
      }
    }
    if (MODE != MID_APPLY) warp_partials(rr, rz, s_wsum, j);
    __syncthreads();
  }
  if (MODE != MID_APPLY) {
    const double inv = 1.0 / ((double)N * N * N);  // Parseval: (1/N^3) sum conj(X) Y
    mid_tickets<NB>(s_wsum, s_act, b0, tile, TILES, ctl, scratch, [&](int b, double t0, double t1) {
      mid_decide(ctl.st + b, ctl, b, it, t0 * inv, t1 * inv);
    });
  }
}


// ----------------------------------------------------------------------------
// kernel 2b: register-resident spectral column pass (n <= 128)
// ----------------------------------------------------------------------------

// Phase A (thread = column w, x0 offset j): the G-group combine and the first
// radix-RA x0 stage straight from/to global memory in registers; phase B
// (thread = slot s, block of RB = N/RA positions): the remaining x0 stages,
// residual update / diagonal scaling and the inverse stages in registers.
// Shared memory is touched twice per element per direction (one exchange each
// way).  P realizations are in flight per CTA; NB share one diagonal tile.

// RSG (with STG, a precomputed plan diagonal and one phase-B item per thread):
// the residual tile of the next realization arrives in shared memory by one
// bulk copy (TMA) issued after the current realization's phase B, and the
// thread's 16 diagonal values stay in registers for all NB realizations (no
// shared diagonal tile) -- phase B then has no global-load latency.
template <int N, int G, int W, int RA, int NB, int P, int MODE, int NT, bool STG = false, bool RSG = false>
__global__ void __launch_bounds__(NT, (STG ? 1 : 512 / NT)) mid_column_reg_kernel(double2* __restrict__ S, PlanDev pl,
                                                                      SolveCtl ctl, SlabGeo sg, int it, int B) {
  constexpr int NR = N / G;
  constexpr int N2 = N / 2;
  constexpr int H = N2 + 1;
  const int TILES = sg.tiles;  // tiles of this rank (all NR*H/W when not slab-decomposed)
  const int nsh = __ffs(sg.nloc) - 1;  // nloc is a power of two
  constexpr int GW = G * W;
  constexpr int RS = GW + 1;
  constexpr int RB = N / RA;      // positions per phase-B block
  constexpr int JA = N / RA;      // x0 stride of a phase-A butterfly
  constexpr int ITEMS_A = W * JA;
  constexpr int ITEMS_B = GW * RA;
  static_assert(NB % P == 0, "NB must be a multiple of P");
  static_assert(RA == Radix<N>::value, "phase A must be the first stage of fft_smem<N> (dig_freq order)");
  extern __shared__ __align__(128) double2 buf[];  // [P][N][RS] (aliased by the [r1][GW] coefficients)
  const int doff = mid_dsm_offset(P * N * RS, GW, pl.kind == KIND_LKR ? pl.r1 : 0);
  double* Dsm = reinterpret_cast<double*>(reinterpret_cast<char*>(buf) + doff);  // [N][GW]
  __shared__ double scratch[64];
  __shared__ int s_k1[GW], s_k2[GW];
  __shared__ double s_wgt[GW];
  __shared__ double2 s_tw[GW];
  __shared__ int s_act[NB];
  __shared__ double s_alpha[NB];
  __shared__ double s_wsum[NB * (NT / 32) * 2];  // per-warp Parseval partials (warp_partials)
  const int bg = blockIdx.x / TILES;
  const int tile = blockIdx.x - bg * TILES;
  const int c0 = tile * W;                       // first column inside this rank's chunk
  const int cg0 = (sg.tile_off + tile) * W;      // global spectral column
  const int b0 = bg * NB;

  if (threadIdx.x == 0) {
    int any = 0;
    for (int j = 0; j < NB; ++j) {
      const int b = b0 + j;
      int a = (b < B);
      if (a && MODE != MID_APPLY) a = (ctl.st[b].status == ST_ACTIVE);
      s_act[j] = a;
      s_alpha[j] = (a && MODE == MID_ITER) ? ctl.st[b].alpha : 0.0;
      any |= a;
    }
    scratch[0] = any;
  }
  __syncthreads();
  if (scratch[0] == 0.0) return;
  // STG: the phase-A tile of the next realization streams into a per-thread
  // staging area (cp.async) while the current one is transformed
  static_assert(!STG || (P == 1 && ITEMS_A == NT), "staging needs one phase-A item per thread");
  static_assert(!RSG || (STG && ITEMS_B == NT), "staged residual needs the staged variant, one phase-B item per thread");
  // RSG layout: [buf N x RS][residual tile N x GW][phase-A staging]; otherwise [buf][Dsm][staging]
  double2* rstg = reinterpret_cast<double2*>(reinterpret_cast<char*>(buf) + ((P * N * RS * 16 + 127) & ~127));
  double2* stg = RSG ? rstg + N * GW
                     : reinterpret_cast<double2*>(reinterpret_cast<char*>(Dsm) + ((N * GW * 8 + 15) & ~15));
  __shared__ alignas(8) uint64_t rbar;
  uint32_t rphase = 0;
  auto issue_r = [&](int cc) {  // RSG: bulk copy of realization cc's residual tile
    if (RSG && MODE == MID_ITER && cc < NB && s_act[cc] && threadIdx.x == 0) {
      const uint32_t bytes = (uint32_t)(N * GW * sizeof(double2));
      mbar_arrive_expect_tx(&rbar, bytes);
      bulk_g2s(rstg, ctl.Rh + ((size_t)(b0 + cc) * TILES + tile) * N * GW, bytes, &rbar);
    }
  };
  auto stage = [&](int cc) {
    if constexpr (STG) {
      if (sg.P == 1 && s_act[cc]) {
        const int w = threadIdx.x % W, j = threadIdx.x / W;
        const double2* base = S + ((size_t)(b0 + cc) * N + j) * G * (size_t)sg.ncols + c0 + w;
#pragma unroll
        for (int t = 0; t < RA; ++t)
#pragma unroll
          for (int g = 0; g < G; ++g)
            cp_async16(stg + (g * RA + t) * NT + threadIdx.x, base + (size_t)(JA * t * G + g) * sg.ncols);
      }
      cp_async_commit();
    }
  };
  // the residual tile of a realization (N x GW, contiguous) is read in phase B:
  // pull it into L2 one realization ahead (the first one under the prologue)
  auto prefetch_r = [&](int cc) {
    if (!RSG && MODE == MID_ITER && CHK_MID_RPF && threadIdx.x == 0 && cc < NB / P) {
      for (int pr = 0; pr < P; ++pr)
        if (s_act[cc * P + pr])
          bulk_prefetch_l2(ctl.Rh + ((size_t)(b0 + cc * P + pr) * TILES + tile) * N * GW,
                           (uint32_t)(N * GW * sizeof(double2)));
    }
  };
  double Dreg[RSG ? RB : 1];
  if constexpr (RSG) {
    if (threadIdx.x == 0) {
      mbar_init(&rbar, 1);
    }
    __syncthreads();
    issue_r(0);
  }
  stage(0);
  prefetch_r(0);
  if constexpr (RSG) {
    // slots, and this thread's diagonal values D[blk*RB + e][s] from the plan's table
    __shared__ int s_dc;
    mid_slots<N, G, W>(cg0, pl, s_k1, s_k2, s_wgt, s_tw);
    if (threadIdx.x == 0) s_dc = -1;
    __syncthreads();
    if (MODE != MID_APPLY && threadIdx.x < GW && s_k1[threadIdx.x] == 0 && s_k2[threadIdx.x] == 0)
      s_dc = threadIdx.x;
    __syncthreads();
    const int s = threadIdx.x % GW, blk = threadIdx.x / GW;
    const double* Dg = pl.D + (size_t)(cg0 / W) * N * GW + (blk * RB) * GW + s;
#pragma unroll
    for (int e = 0; e < RB; ++e) Dreg[e] = (blk * RB + e == 0 && s == s_dc) ? 0.0 : __ldg(Dg + e * GW);
  } else {
    mid_prologue<N, G, W, MODE>(buf, Dsm, cg0, pl, s_k1, s_k2, s_wgt, s_tw);
  }

  const double scale = 2.0 / ((double)N * N * N);
  const int ntab = N;
  for (int c = 0; c < NB / P; ++c) {
    // warm L2 with the next chunk's tile rows (W * 16 B per (x0, group) row)
    if (!STG && c + 1 < NB / P) {
      for (int i = threadIdx.x; i < P * N * G; i += blockDim.x) {
        const int pr = i / (N * G), rr = i - pr * (N * G);
        if (s_act[(c + 1) * P + pr])
          bulk_prefetch_l2(S + slab_row(sg, B, G, (rr / G) >> nsh, b0 + (c + 1) * P + pr, (rr / G) & (sg.nloc - 1),
                                        rr % G) + c0,
                           W * sizeof(double2));
      }
    }
    // ---- phase A forward: global -> registers -> smem ----
    for (int item = threadIdx.x; item < P * ITEMS_A; item += blockDim.x) {
      const int pr = item / ITEMS_A, ia = item - pr * ITEMS_A;
      if (!s_act[c * P + pr]) continue;
      const int w = ia % W, j = ia / W;
      const int bb = b0 + c * P + pr;
      double2 v[G][RA];
      if (STG && sg.P == 1) {
        cp_async_wait_all();
#pragma unroll
        for (int t = 0; t < RA; ++t)
#pragma unroll
          for (int g = 0; g < G; ++g) v[g][t] = stg[(g * RA + t) * NT + threadIdx.x];
      } else if (sg.P == 1) {  // single chunk: rows are linear in x0
        const double2* base = S + ((size_t)bb * N + j) * G * (size_t)sg.ncols + c0 + w;
#pragma unroll
        for (int t = 0; t < RA; ++t)
#pragma unroll
          for (int g = 0; g < G; ++g) v[g][t] = base[(size_t)(JA * t * G + g) * sg.ncols];
      } else {
#pragma unroll
        for (int t = 0; t < RA; ++t) {
          const int x0 = j + JA * t;
#pragma unroll
          for (int g = 0; g < G; ++g) v[g][t] = S[slab_row(sg, B, G, x0 >> nsh, bb, x0 & (sg.nloc - 1), g) + c0 + w];
        }
      }
      if constexpr (G > 1) {
#pragma unroll
        for (int g = 1; g < G; ++g) {
          const double2 tg = s_tw[g * W + w];
#pragma unroll
          for (int t = 0; t < RA; ++t) v[g][t] = cmul(v[g][t], tg);
        }
#pragma unroll
        for (int t = 0; t < RA; ++t) {
          double2 a[G];
#pragma unroll
          for (int g = 0; g < G; ++g) a[g] = v[g][t];
          reg_fft<G, false>(a, reg_tw<N>(pl), ntab);
#pragma unroll
          for (int g = 0; g < G; ++g) v[g][t] = a[g];
        }
      }
      double2* dst = buf + pr * N * RS;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        dftR<RA, false>(v[g]);
#pragma unroll
        for (int m = 0; m < RA; ++m) {
          double2 y = v[g][m];
          if (m > 0 && j > 0) y = cmul(y, tw_at(mid_tw<N>(pl), (j * m) * (ntab / N)));
          dst[(j + JA * m) * RS + g * W + w] = y;
        }
      }
    }
    __syncthreads();
    if (c + 1 < NB / P) stage(c + 1);  // overlaps phases B and A-inverse
    prefetch_r(c + 1);
    // ---- phase B: remaining stages, residual update / diagonal, inverse ----
    double accr[P], accz[P];
#pragma unroll
    for (int pr = 0; pr < P; ++pr) accr[pr] = accz[pr] = 0.0;
    for (int item = threadIdx.x; item < P * ITEMS_B; item += blockDim.x) {
      const int pr = item / ITEMS_B, ib = item - pr * ITEMS_B;
      if (!s_act[c * P + pr]) continue;
      const int s = ib % GW, blk = ib / GW;
      double2* row = buf + pr * N * RS + (blk * RB) * RS + s;
      double2 v[RB];
#pragma unroll
      for (int e = 0; e < RB; ++e) v[e] = row[e * RS];
      reg_fft<RB, false>(v, reg_tw<N>(pl), ntab);
      double rr = 0.0, rz = 0.0;
      const double wgt = s_wgt[s];
      const double al = s_alpha[c * P + pr];
      double2* Rt = ctl.Rh + ((size_t)(b0 + c * P + pr) * TILES + tile) * N * GW + (blk * RB) * GW + s;
      if constexpr (RSG) {
        if (MODE == MID_ITER) {
          mbar_wait(&rbar, rphase & 1);
          const double2* Rs = rstg + (blk * RB) * GW + s;
#pragma unroll
          for (int e = 0; e < RB; ++e) {  // mid_point<MID_ITER> with the residual from smem
            const double2 Ro = Rs[e * GW];
            const double2 R = make_double2(fma(-al, v[e].x, Ro.x), fma(-al, v[e].y, Ro.y));
            Rt[e * GW] = R;
            const double m2 = R.x * R.x + R.y * R.y;
            rr = fma(wgt, m2, rr);
            rz = fma(wgt * Dreg[e], m2, rz);
            v[e] = cscale(R, Dreg[e] * scale);
          }
        } else {
#pragma unroll
          for (int e = 0; e < RB; ++e) v[e] = mid_point<MODE>(v[e], Dreg[e], wgt, scale, al, Rt + e * GW, rr, rz);
        }
      } else {
#pragma unroll
        for (int e = 0; e < RB; ++e)
          v[e] = mid_point<MODE>(v[e], Dsm[(blk * RB + e) * GW + s], wgt, scale, al, Rt + e * GW, rr, rz);
      }
#pragma unroll
      for (int pr2 = 0; pr2 < P; ++pr2)
        if (pr2 == pr) {
          accr[pr2] += rr;
          accz[pr2] += rz;
        }
      reg_fft<RB, true>(v, reg_tw<N>(pl), ntab);
#pragma unroll
      for (int e = 0; e < RB; ++e) row[e * RS] = v[e];
    }
    __syncthreads();
    if constexpr (RSG) {  // the residual buffer is free again: fetch the next realization's tile
      if (MODE == MID_ITER && s_act[c]) ++rphase;
      issue_r(c + 1);
    }
    // ---- phase A inverse: smem -> registers -> global ----
    for (int item = threadIdx.x; item < P * ITEMS_A; item += blockDim.x) {
      const int pr = item / ITEMS_A, ia = item - pr * ITEMS_A;
      if (!s_act[c * P + pr]) continue;
      const int w = ia % W, j = ia / W;
      const double2* src = buf + pr * N * RS;
      double2 v[G][RA];
#pragma unroll
      for (int g = 0; g < G; ++g) {
#pragma unroll
        for (int m = 0; m < RA; ++m) {
          double2 y = src[(j + JA * m) * RS + g * W + w];
          if (m > 0 && j > 0) y = cmulc(y, tw_at(mid_tw<N>(pl), (j * m) * (ntab / N)));
          v[g][m] = y;
        }
        dftR<RA, true>(v[g]);
      }
      if constexpr (G > 1) {
#pragma unroll
        for (int t = 0; t < RA; ++t) {
          double2 a[G];
#pragma unroll
          for (int g = 0; g < G; ++g) a[g] = v[g][t];
          reg_fft<G, true>(a, reg_tw<N>(pl), ntab);
#pragma unroll
          for (int g = 0; g < G; ++g) v[g][t] = a[g];
        }
#pragma unroll
        for (int g = 1; g < G; ++g) {
          const double2 tg = s_tw[g * W + w];
#pragma unroll
          for (int t = 0; t < RA; ++t) v[g][t] = cmulc(v[g][t], tg);
        }
      }
      const int bb = b0 + c * P + pr;
      if (sg.P == 1) {
        double2* base = S + ((size_t)bb * N + j) * G * (size_t)sg.ncols + c0 + w;
#pragma unroll
        for (int t = 0; t < RA; ++t)
#pragma unroll
          for (int g = 0; g < G; ++g) base[(size_t)(JA * t * G + g) * sg.ncols] = v[g][t];
      } else {
#pragma unroll
        for (int t = 0; t < RA; ++t) {
          const int x0 = j + JA * t;
#pragma unroll
          for (int g = 0; g < G; ++g) S[slab_row(sg, B, G, x0 >> nsh, bb, x0 & (sg.nloc - 1), g) + c0 + w] = v[g][t];
        }
      }
    }
    // ---- per-realization Parseval partials (warp level; tickets after the loop) ----
    if (MODE != MID_APPLY) {
#pragma unroll
      for (int pr = 0; pr < P; ++pr)
        if (s_act[c * P + pr]) warp_partials(accr[pr], accz[pr], s_wsum, c * P + pr);
    }
    __syncthreads();
  }
  if (MODE != MID_APPLY) {
    const double inv = 1.0 / ((double)N * N * N);  // Parseval: (1/N^3) sum conj(X) Y
    mid_tickets<NB>(s_wsum, s_act, b0, tile, TILES, ctl, scratch, [&](int b, double t0, double t1) {
      mid_decide(ctl.st + b, ctl, b, it, t0 * inv, t1 * inv);
    });
  }
}

// ----------------------------------------------------------------------------
// kernel 3: inverse plane transform + solution / direction update
// ----------------------------------------------------------------------------
// INV_APPLY: out = z.  INV_INIT: p = z (solver.py:154).
// INV_ITER:  u += alpha_k p_k (solver.py:167; deferred here, where p_k is read
//            anyway) and, while the solve continues, p = z + beta p_k
//            (solver.py:184).  At the stopping iteration only u is updated.
enum : int { INV_APPLY = 0, INV_INIT = 1, INV_ITER = 2 };


template <int N, int G, int MODE>
__device__ __forceinline__ void inv_plane_body(const double2* __restrict__ S, double* __restrict__ out,
                                               double* __restrict__ u, const PlanDev& pl, const SolveCtl& ctl,
                                               const SlabGeo& sg, int B, int it, int bid,
                                               const CUtensorMap* tmap = nullptr) {
  constexpr int NR = N / G;
  constexpr int N2 = N / 2;
  constexpr int H = N2 + 1;
  constexpr int HP = H;
  extern __shared__ __align__(128) double2 buf[];
  __shared__ alignas(8) uint64_t bar;
  const int b = bid / (sg.nrun * G);
  const int rrun = bid - b * (sg.nrun * G);
  const int x0 = sg.run0 + rrun / G, gg = rrun - (rrun / G) * G;  // local plane, x1 group
  const size_t nb = (size_t)sg.nloc * N * N;
  double alpha = 0.0, beta = 0.0;
  bool do_p = true, do_u = false;
  if (MODE != INV_APPLY) {
    const RState* st = ctl.st + b;
    const int status = st->status;
    do_p = (status == ST_ACTIVE);
    if (MODE == INV_ITER) {
      do_u = do_p || ((status == ST_CONVERGED || status == ST_NOT_CONVERGED) && st->iters == it);
      alpha = st->alpha;
      beta = st->beta;
    }
    if (!do_p && !do_u) return;
  }
  constexpr int IW = IlW<N>::value;
  if constexpr (IW > 0) {
    if (do_p && tmap) {
      // tensor-map TMA load of the 32-byte pieces into the dense smem row
      if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_arrive_expect_tx(&bar, (uint32_t)(NR * H * sizeof(double2)));
        const int npc = sg.ncols / IW;
        for (int c = 0; c < sg.P; ++c) {
          const int row = (c * B + b) * sg.nloc + x0;
          for (int i0 = 0; i0 < npc; i0 += TmapBox<N>::value)
            tma_load_4d(buf + (size_t)c * sg.ncols + (size_t)i0 * IW, tmap, 0, gg, i0, row, &bar);
        }
      }
    } else if (do_p) {
      // interleaved layout: 16-byte cp.async copies of the 32-byte pieces
      for (int c = 0; c < sg.P; ++c) {
        const double2* src = S + slab_row(sg, B, G, c, b, x0, 0) + gg * IW;
        double2* dst = buf + (size_t)c * sg.ncols;
        for (int i = threadIdx.x; i < sg.ncols; i += blockDim.x)
          cp_async16(dst + i, src + (size_t)(i / IW) * G * IW + (i % IW));
      }
      cp_async_commit();
    }
  } else if (do_p) {
    // the slab row arrives as P column chunks (one bulk load each)
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_arrive_expect_tx(&bar, (uint32_t)(NR * H * sizeof(double2)));
      for (int c = 0; c < sg.P; ++c)
        bulk_g2s(buf + (size_t)c * sg.ncols, S + slab_row(sg, B, G, c, b, x0, gg),
                 (uint32_t)(sg.ncols * sizeof(double2)), &bar);
    }
  }
  if (MODE == INV_ITER && CHK_INV_PF && N <= 128 && threadIdx.x < NR) {
    // p and u rows of this slab are read after the transforms: warm L2 now
    const size_t ro = b * nb + ((size_t)x0 * N + gg + G * threadIdx.x) * N;
    bulk_prefetch_l2(out + ro, N * sizeof(double));
    bulk_prefetch_l2(u + ro, N * sizeof(double));
  }
  if (do_p) {
    if constexpr (IW > 0) {
      if (tmap) {
        __syncthreads();  // barrier initialised before anyone waits
        mbar_wait(&bar, 0);
      } else {
        cp_async_wait_all();
        __syncthreads();
      }
    } else {
      __syncthreads();  // barrier initialised before anyone waits
      mbar_wait(&bar, 0);
    }
    const PlaneTw<N> ptw = plane_tw<N>(pl);
    fft_smem<NR, true, H>(buf, ColAddr{HP}, ptw, N);
    c2r_pre<N>(buf, NR, HP, ptw);
    if (MODE == INV_ITER && CHK_INV_PF_LATE && N >= CHK_INV_PF_LATE_MIN && threadIdx.x < NR) {
      // n >= 256: warm L2 with this slab's p / u rows one stage (not the whole pass)
      // before they are read -- prefetched at the start they were evicted first
      const size_t ro = b * nb + ((size_t)x0 * N + gg + G * threadIdx.x) * N;
      bulk_prefetch_l2(out + ro, N * sizeof(double));
      if (do_u) bulk_prefetch_l2(u + ro, N * sizeof(double));
    }
    __syncthreads();
    fft_smem_r<N2, true, NR, X2Rule<N>::value>(buf, RowAddr{HP}, ptw, N);
  }
  double* sm = reinterpret_cast<double*>(buf);
  constexpr int Q4 = N / 4;
  // u += alpha p by the TMA engine (n = 128, where this pass is LSU-bound; measured: pair
  // pass -3.0 %, config 3 +2.1 %; the HBM- or latency-bound passes of the other sizes lose:
  // n = 64 +1.3 %, n = 256 +9 %, n = 512 +4 %): alpha p replaces the z quad this thread has
  // just read in the shared-memory row, and one bulk reduce-add per row (cp.reduce.async.bulk
  // .add.f64, performed at the L2) accumulates it into u -- the LSU pipe, which bounds this
  // pass, moves 8 instead of 16 wavefronts per row for u.  (alpha p is rounded before the
  // add, as in the reference's own `u += alpha * p`, solver.py:167.)
  constexpr bool UTMA = CHK_U_TMA && MODE == INV_ITER && N == 128;
  for (int i = threadIdx.x; i < NR * Q4; i += blockDim.x) {
    const int t = i / Q4, x2 = 4 * (i - (i / Q4) * Q4);
    const size_t idx = b * nb + ((size_t)x0 * N + gg + G * t) * N + x2;
    double z[4] = {0.0, 0.0, 0.0, 0.0};
    if (do_p) {
      ld_quad_smem(sm + t * 2 * HP, x2, z);
    }
    if (MODE == INV_APPLY || MODE == INV_INIT) {
      stv4(out + idx, z);
    } else {
      double po[4], uo[4];
      ldv4(out + idx, po);
      if (do_u) {
        if constexpr (UTMA) {
#pragma unroll
          for (int e = 0; e < 4; ++e) uo[e] = alpha * po[e];
          st_quad_smem(sm + t * 2 * HP, x2, uo);
        } else {
          ldv4(u + idx, uo);
#pragma unroll
          for (int e = 0; e < 4; ++e) uo[e] = fma(alpha, po[e], uo[e]);  // u += step p
          stv4(u + idx, uo);
        }
      }
      if (do_p) {
        double pn[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) pn[e] = fma(beta, po[e], z[e]);  // p = z + beta p
        stv4(out + idx, pn);
      }
    }
  }
  if constexpr (UTMA) {
    if (do_u) {  // CTA-uniform
      fence_proxy_async_smem();
      __syncthreads();
      if (threadIdx.x < NR) {
        const int t = threadIdx.x;
        bulk_reduce_add_f64(u + b * nb + ((size_t)x0 * N + gg + G * t) * N, sm + t * 2 * HP,
                            (uint32_t)(N * sizeof(double)));
        bulk_commit();
        bulk_wait_read0();
      }
    }
  }
}

// ----------------------------------------------------------------------------
// init / finalize reductions and the slab-mode decision kernels
// ----------------------------------------------------------------------------
// RHS statistics -> zero-RHS / mean-projection decisions (solver.py:131-148).
__device__ __forceinline__ void stats_decide(RState* st, double sum, double sumsq, double ntot) {
  const double normf = sqrt(sumsq);
  st->iters = 0;
  st->final_rel = 0.0;
  st->rz[0] = st->rz[1] = 0.0;
  st->beta = 0.0;
  st->mean_u = 0.0;
  if (!(normf > 0.0)) {  // zero right-hand side (solver.py:131-136)
    st->status = ST_CONVERGED;
    st->rhs_projected = 0;
    st->mean_f = 0.0;
  } else {
    st->status = ST_ACTIVE;
    st->rhs_projected = fabs(sum) > 1e-10 * normf ? 1 : 0;  // solver.py:139
    st->mean_f = sum / ntot;
  }
}

template <int N, int G>
__global__ void __launch_bounds__(256) rhs_stats_kernel(const double* __restrict__ f, SolveCtl ctl, SlabGeo sg) {
  constexpr int NR = N / G;
  __shared__ double scratch[64];
  const int nlg = sg.nloc * G;
  const int b = blockIdx.x / nlg;
  const int rem = blockIdx.x - b * nlg;
  const int x0 = rem / G, gg = rem - (rem / G) * G;
  const size_t nb = (size_t)sg.nloc * N * N;
  RState* st = ctl.st + b;
  double s = 0.0, s2 = 0.0;
  for (int i = threadIdx.x; i < NR * N; i += blockDim.x) {
    const int t = i / N, x2 = i - (i / N) * N;
    const double v = __ldg(f + b * nb + ((size_t)x0 * N + gg + G * t) * N + x2);
    s += v;
    s2 += v * v;
  }
  double t0, t1;
  if (reduce2_last(s, s2, ctl.part + (size_t)b * 2 * ctl.maxblk, &st->cnt, rem, nlg, scratch,
                   t0, t1)) {
    if (threadIdx.x == 0) {
      if (ctl.red_only) {
        ctl.red[4 * b] = t0;
        ctl.red[4 * b + 1] = t1;
      } else {
        stats_decide(st, t0, t1, (double)N * N * N);
      }
    }
  }
}

template <int N, int G>
__global__ void __launch_bounds__(256) mean_u_kernel(const double* __restrict__ u, SolveCtl ctl, SlabGeo sg) {
  constexpr int NR = N / G;
  __shared__ double scratch[64];
  const int nlg = sg.nloc * G;
  const int b = blockIdx.x / nlg;
  const int rem = blockIdx.x - b * nlg;
  const int x0 = rem / G, gg = rem - (rem / G) * G;
  const size_t nb = (size_t)sg.nloc * N * N;
  RState* st = ctl.st + b;
  double s = 0.0;
  for (int i = threadIdx.x; i < NR * N; i += blockDim.x) {
    const int t = i / N, x2 = i - (i / N) * N;
    s += u[b * nb + ((size_t)x0 * N + gg + G * t) * N + x2];
  }
  double t0, t1;
  if (reduce2_last(s, 0.0, ctl.part + (size_t)b * 2 * ctl.maxblk, &st->cnt, rem, nlg, scratch,
                   t0, t1)) {
    if (threadIdx.x == 0) {
      if (ctl.red_only) ctl.red[4 * b + 3] = t0;
      else st->mean_u = t0 / ((double)N * N * N);
    }
  }
}

__global__ void __launch_bounds__(256) sub_mean_kernel(double* __restrict__ u, const RState* st,
                                                       size_t nb, int B) {
  const size_t total = nb * (size_t)B;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / nb);
    u[i] -= st[b].mean_u;  // solver.py:169 (applied once: proj is linear and idempotent)
  }
}

// Slab mode: decisions from the allreduced sums red[B][4] (identical on every
// rank, so every rank takes the same decisions).
enum : int { DECIDE_STATS = 0, DECIDE_ALPHA = 1, DECIDE_MID = 2, DECIDE_MEANU = 3 };

__global__ void decide_kernel(SolveCtl ctl, const double* __restrict__ red, int B, int what, int it,
                              double ntot) {
  SolveCtl c = ctl;
  c.red_only = 0;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    RState* st = ctl.st + b;
    if (what == DECIDE_STATS) {
      stats_decide(st, red[4 * b], red[4 * b + 1], ntot);
    } else if (what == DECIDE_MEANU) {
      st->mean_u = red[4 * b + 3] / ntot;
    } else if (st->status == ST_ACTIVE) {
      if (what == DECIDE_ALPHA) {
        const double pq = red[4 * b];
        if ((!(pq > 0.0) || !isfinite(pq))) {  // solver.py:164-165
          st->status = ST_BREAKDOWN;
          st->iters = it;
        }
        st->pq = pq;
        st->alpha = st->rz[(it - 1) & 1] / pq;  // solver.py:166
      } else {
        mid_decide(st, c, b, it, red[4 * b + 1], red[4 * b + 2]);  // already / N^3
      }
    }
  }
}

}  // namespace chk

#include "chk_plane.cuh"
