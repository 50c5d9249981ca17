// chk_generic.cuh -- the PCG path for grid sizes without a fused fast path.
//
// The reference accepts any n = n0 * L with n0 a power of two >= 4 and any L >= 1
// (lattice.py:117-123,156-159; its own tests run n = 12 and 24).  The fused
// kernels of chk_kernels.cuh cover the power-of-two sizes 8..512 of the BASELINE
// configurations; every other size runs here: the same algorithm
// (solver.py:118-194) as plain device kernels -- node-wise 7-point stencil,
// the preconditioner as a direct O(n) discrete Fourier sum per axis with the
// exact table w[(j k) mod n] (no radix restriction), the diagonal evaluated from
// its factors per element, and deterministic two-stage reductions whose sums
// feed the same decision kernel as the slab mode (decide_kernel).  r stays in
// real space here (the reference's own recurrence, solver.py:168).
#pragma once

namespace chk {

__device__ __forceinline__ int gen_wrap(int j, int n) { return j < 0 ? j + n : (j >= n ? j - n : j); }

// (A p) at one node: same formulas and summation order as stencil4
// (tests/oracles.py:52-75); indices wrap by comparison, n0 is a power of two.
__device__ __forceinline__ double gen_stencil_node(const Geo& g, const double* __restrict__ beta,
                                                   const double* __restrict__ p, int x0, int x1, int x2) {
  const int n = g.n;
  const int j0[2] = {gen_wrap(x0 - 1, n), x0}, j1[2] = {gen_wrap(x1 - 1, n), x1}, j2[2] = {gen_wrap(x2 - 1, n), x2};
  double f[2][2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) f[a][b][c] = fcell(beta, g, j0[a], j1[b], j2[c]);
  const double lam = g.lam;
  const double g0p = lam + (((f[1][1][1] + f[1][1][0]) + f[1][0][1]) + f[1][0][0]) * 0.25;
  const double g0m = lam + (((f[0][1][1] + f[0][1][0]) + f[0][0][1]) + f[0][0][0]) * 0.25;
  const double g1p = lam + (((f[1][1][1] + f[1][1][0]) + f[0][1][1]) + f[0][1][0]) * 0.25;
  const double g1m = lam + (((f[1][0][1] + f[1][0][0]) + f[0][0][1]) + f[0][0][0]) * 0.25;
  const double g2p = lam + (((f[1][1][1] + f[1][0][1]) + f[0][1][1]) + f[0][0][1]) * 0.25;
  const double g2m = lam + (((f[1][1][0] + f[1][0][0]) + f[0][1][0]) + f[0][0][0]) * 0.25;
  const size_t nn = (size_t)n * n;
  const double c = p[x0 * nn + (size_t)x1 * n + x2];
  const double xm = p[j0[0] * nn + (size_t)x1 * n + x2], xp = p[gen_wrap(x0 + 1, n) * nn + (size_t)x1 * n + x2];
  const double ym = p[x0 * nn + (size_t)j1[0] * n + x2], yp = p[x0 * nn + (size_t)gen_wrap(x1 + 1, n) * n + x2];
  const double left = p[x0 * nn + (size_t)x1 * n + j2[0]], right = p[x0 * nn + (size_t)x1 * n + gen_wrap(x2 + 1, n)];
  const double q0 = g0p * (c - xp) + g0m * (c - xm);
  const double q1 = g1p * (c - yp) + g1m * (c - ym);
  const double q2 = g2p * (c - right) + g2m * (c - left);
  return (q0 + q1) + q2;
}

// Every element-wise kernel below runs a grid of (n, B) CTAs: CTA (x0, b) owns
// plane x0 of realization b; reductions leave one partial pair per CTA in
// part[b][x0][2], summed in a fixed order by gen_finalize_kernel.
__device__ __forceinline__ void gen_store_partial(double v0, double v1, double* part, double* scratch) {
  block_sum2(v0, v1, scratch);
  if (threadIdx.x == 0) {
    double* d = part + 2 * ((size_t)blockIdx.y * gridDim.x + blockIdx.x);
    d[0] = v0;
    d[1] = v1;
  }
}

// y = A x (+ partial <x, y>); st != null: only active realizations
__global__ void __launch_bounds__(256) gen_stencil_kernel(Geo g, const double* __restrict__ beta,
                                                          const double* __restrict__ x, double* __restrict__ y,
                                                          double* part, const RState* st) {
  __shared__ double scratch[64];
  const int n = g.n, b = blockIdx.y, x0 = blockIdx.x;
  if (st && st[b].status != ST_ACTIVE) return;
  const size_t nb = (size_t)n * n * n;
  const double* xb = x + b * nb;
  const double* bb = beta + (size_t)b * g.L * g.L * g.L;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    const int x1 = i / n, x2 = i - x1 * n;
    const double q = gen_stencil_node(g, bb, xb, x0, x1, x2);
    y[b * nb + (size_t)x0 * n * n + i] = q;
    acc = fma(xb[(size_t)x0 * n * n + i], q, acc);
  }
  if (part) gen_store_partial(acc, 0.0, part, scratch);
}

// out0[b * stride] (and out1) = sums of the nblk partial pairs of realization b
__global__ void __launch_bounds__(256) gen_finalize_kernel(const double* __restrict__ part, int nblk, double* out0,
                                                           double* out1, int stride) {
  __shared__ double scratch[64];
  const int b = blockIdx.x;
  double a = 0.0, c = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    a += part[2 * ((size_t)b * nblk + i)];
    c += part[2 * ((size_t)b * nblk + i) + 1];
  }
  block_sum2(a, c, scratch);
  if (threadIdx.x == 0) {
    if (out0) out0[(size_t)b * stride] = a;
    if (out1) out1[(size_t)b * stride] = c;
  }
}

// corrector load (homogenize.py:75-89 with lattice.py:335-345), any n
__device__ __forceinline__ double gen_nodal_coef(const double* __restrict__ beta, const Geo& g, int x0, int x1,
                                                 int x2) {
  const int n = g.n;
  const int a0 = gen_wrap(x0 - 1, n), a1 = gen_wrap(x1 - 1, n), a2 = gen_wrap(x2 - 1, n);
  auto c0 = [&](int j1, int j2) { return 0.5 * (fcell(beta, g, x0, j1, j2) + fcell(beta, g, a0, j1, j2)); };
  auto c1 = [&](int j2) { return 0.5 * (c0(x1, j2) + c0(a1, j2)); };
  return 0.5 * (c1(x2) + c1(a2));
}

__global__ void __launch_bounds__(256) gen_corrector_rhs_kernel(Geo g, const double* __restrict__ beta,
                                                                double* __restrict__ f, int axis, double scale) {
  const int n = g.n, b = blockIdx.y, x0 = blockIdx.x;
  const size_t nb = (size_t)n * n * n;
  const double* bb = beta + (size_t)b * g.L * g.L * g.L;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    const int x1 = i / n, x2 = i - x1 * n;
    int xp[3] = {x0, x1, x2}, xm[3] = {x0, x1, x2};
    xp[axis] = gen_wrap(xp[axis] + 1, n);
    xm[axis] = gen_wrap(xm[axis] - 1, n);
    const double cp = gen_nodal_coef(bb, g, xp[0], xp[1], xp[2]);
    const double cm = gen_nodal_coef(bb, g, xm[0], xm[1], xm[2]);
    f[b * nb + (size_t)x0 * n * n + i] = scale * (0.5 * (cp - cm));
  }
}

// sum f, sum f^2 (solver.py:131-139)
__global__ void __launch_bounds__(256) gen_stats_kernel(const double* __restrict__ f, int n, double* part) {
  __shared__ double scratch[64];
  const size_t nn = (size_t)n * n;
  const double* fp = f + ((size_t)blockIdx.y * n + blockIdx.x) * nn;
  double s = 0.0, s2 = 0.0;
  for (int i = threadIdx.x; i < (int)nn; i += blockDim.x) {
    const double v = fp[i];
    s += v;
    s2 = fma(v, v, s2);
  }
  gen_store_partial(s, s2, part, scratch);
}

// r = f - mean (when projected, solver.py:139-143), u = 0
__global__ void __launch_bounds__(256) gen_init_kernel(const double* __restrict__ f, double* __restrict__ r,
                                                       double* __restrict__ u, int n, const RState* st) {
  const size_t nn = (size_t)n * n;
  const size_t o = ((size_t)blockIdx.y * n + blockIdx.x) * nn;
  const RState* s = st + blockIdx.y;
  const double shift = s->rhs_projected ? s->mean_f : 0.0;
  for (int i = threadIdx.x; i < (int)nn; i += blockDim.x) {
    r[o + i] = f[o + i] - shift;
    u[o + i] = 0.0;
  }
}

// r -= alpha q (it >= 1, solver.py:168), spectrum buffer S = r (+ 0 i)
__global__ void __launch_bounds__(256) gen_residual_kernel(double* __restrict__ r, const double* __restrict__ q,
                                                           double2* __restrict__ S, int n, const RState* st, int it) {
  const size_t nn = (size_t)n * n;
  const size_t o = ((size_t)blockIdx.y * n + blockIdx.x) * nn;
  const RState* s = st + blockIdx.y;
  if (s->status != ST_ACTIVE) return;
  const double alpha = s->alpha;
  for (int i = threadIdx.x; i < (int)nn; i += blockDim.x) {
    double v = r[o + i];
    if (it > 0) {
      v = fma(-alpha, q[o + i], v);
      r[o + i] = v;
    }
    S[o + i] = make_double2(v, 0.0);
  }
}

// stand-alone preconditioner: S = x (+ 0 i)
__global__ void __launch_bounds__(256) gen_load_kernel(const double* __restrict__ x, double2* __restrict__ S, int n) {
  const size_t nn = (size_t)n * n;
  const size_t o = ((size_t)blockIdx.y * n + blockIdx.x) * nn;
  for (int i = threadIdx.x; i < (int)nn; i += blockDim.x) S[o + i] = make_double2(x[o + i], 0.0);
}

// One axis of the 3-D DFT of B complex n^3 arrays, in place.  CTA = TL lines
// (consecutive in the fastest index that is not the transform axis) staged in
// shared memory; each output is the direct sum over the line with the exact
// twiddle w[(j k) mod n].  zout != null (last inverse pass): the real part goes
// to zout instead.
template <bool INV>
__global__ void __launch_bounds__(256) gen_dft_axis_kernel(double2* __restrict__ S, const double2* __restrict__ tw,
                                                           int n, int axis, int TL, const RState* st,
                                                           double* __restrict__ zout) {
  extern __shared__ __align__(16) double2 gsm[];
  double2* tile = gsm;           // [n][TL]
  double2* stw = gsm + n * TL;   // [n]
  const int b = blockIdx.y;
  if (st && st[b].status != ST_ACTIVE) return;
  const size_t nn = (size_t)n * n, nb = nn * n;
  double2* Sb = S + b * nb;
  const int nlines = n * n;
  const int l0 = blockIdx.x * TL;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 w = tw[i];
    stw[i] = INV ? make_double2(w.x, -w.y) : w;
  }
  auto line_base = [&](int id) -> size_t {
    if (axis == 2) return (size_t)id * n;
    if (axis == 1) return (size_t)(id / n) * nn + (id % n);
    return (size_t)id;
  };
  const size_t estride = (axis == 2) ? 1 : (axis == 1 ? (size_t)n : nn);
  if (axis == 2) {
    for (int i = threadIdx.x; i < TL * n; i += blockDim.x) {
      const int l = i / n, j = i - l * n;
      if (l0 + l < nlines) tile[j * TL + l] = Sb[line_base(l0 + l) + j];
    }
  } else {
    for (int i = threadIdx.x; i < TL * n; i += blockDim.x) {
      const int j = i / TL, l = i - j * TL;
      if (l0 + l < nlines) tile[j * TL + l] = Sb[line_base(l0 + l) + (size_t)j * estride];
    }
  }
  __syncthreads();
  for (int o = threadIdx.x; o < TL * n; o += blockDim.x) {
    int l, k;
    if (axis == 2) {
      l = o / n;
      k = o - l * n;
    } else {
      k = o / TL;
      l = o - k * TL;
    }
    if (l0 + l >= nlines) continue;
    double ax = 0.0, ay = 0.0;
    int idx = 0;
    for (int j = 0; j < n; ++j) {
      const double2 v = tile[j * TL + l];
      const double2 w = stw[idx];
      ax = fma(v.x, w.x, fma(-v.y, w.y, ax));
      ay = fma(v.x, w.y, fma(v.y, w.x, ay));
      idx += k;
      if (idx >= n) idx -= n;
    }
    const size_t dst = line_base(l0 + l) + (size_t)k * estride;
    if (zout)
      zout[b * nb + dst] = ax;
    else
      Sb[dst] = make_double2(ax, ay);
  }
}

// S *= D / n^3, D[i,j,l] from the plan (LKR: sum_k U0[k,i] U1[k,j] U2[k,l],
// lowrank.py:141-144; Fourier kinds: spectral.py:47-52,77-95); project: the
// zero-frequency coefficient is 0 (mean projection of z, solver.py:153,179)
__global__ void __launch_bounds__(256) gen_scale_kernel(double2* __restrict__ S, PlanDev pl, int n, int project,
                                                        const RState* st) {
  const int b = blockIdx.y, i0 = blockIdx.x;
  if (st && st[b].status != ST_ACTIVE) return;
  const size_t nn = (size_t)n * n;
  double2* Sp = S + ((size_t)b * n + i0) * nn;
  const double inv = 1.0 / ((double)n * n * n);
  for (int i = threadIdx.x; i < (int)nn; i += blockDim.x) {
    const int i1 = i / n, i2 = i - i1 * n;
    double D;
    if (pl.kind == KIND_LKR) {
      const double* U0 = pl.U;
      const double* U1 = pl.U + (size_t)pl.r1 * n;
      const double* U2 = pl.U + (size_t)2 * pl.r1 * n;
      D = 0.0;
      for (int k = 0; k < pl.r1; ++k)
        D = fma(__ldg(U0 + (size_t)k * n + i0) * __ldg(U1 + (size_t)k * n + i1), __ldg(U2 + (size_t)k * n + i2), D);
    } else {
      const double gsum = (__ldg(pl.lam + i0) + __ldg(pl.lam + i1)) + __ldg(pl.lam + i2);
      if (pl.kind == KIND_REGULARIZED && pl.delta > 0.0)
        D = 1.0 / (gsum + pl.delta);
      else
        D = (gsum > 0.0) ? 1.0 / gsum : 0.0;
    }
    if (project && i0 == 0 && i == 0) D = 0.0;
    const double2 v = Sp[i];
    Sp[i] = make_double2(v.x * (D * inv), v.y * (D * inv));
  }
}

// sum r^2, sum r z (solver.py:171,180)
__global__ void __launch_bounds__(256) gen_dots_kernel(const double* __restrict__ r, const double* __restrict__ z,
                                                       int n, double* part, const RState* st) {
  __shared__ double scratch[64];
  const size_t nn = (size_t)n * n;
  const size_t o = ((size_t)blockIdx.y * n + blockIdx.x) * nn;
  double rr = 0.0, rz = 0.0;
  if (st[blockIdx.y].status == ST_ACTIVE) {
    for (int i = threadIdx.x; i < (int)nn; i += blockDim.x) {
      const double v = r[o + i];
      rr = fma(v, v, rr);
      rz = fma(v, z[o + i], rz);
    }
  }
  gen_store_partial(rr, rz, part, scratch);
}

// it == 0: p = z (solver.py:154).  it >= 1: u += alpha p (solver.py:167) for
// realizations that were active in this iteration, p = z + beta p while the
// solve continues (solver.py:184) -- the conditions of inv_plane_body.
__global__ void __launch_bounds__(256) gen_update_kernel(double* __restrict__ p, double* __restrict__ u,
                                                         const double* __restrict__ z, int n, const RState* st,
                                                         int it) {
  const size_t nn = (size_t)n * n;
  const size_t o = ((size_t)blockIdx.y * n + blockIdx.x) * nn;
  const RState* s = st + blockIdx.y;
  const int status = s->status;
  const bool do_p = (status == ST_ACTIVE);
  const bool do_u = it > 0 && (do_p || ((status == ST_CONVERGED || status == ST_NOT_CONVERGED) && s->iters == it));
  if (!do_p && !do_u) return;
  const double alpha = s->alpha, beta = s->beta;
  for (int i = threadIdx.x; i < (int)nn; i += blockDim.x) {
    if (it == 0) {
      p[o + i] = z[o + i];
    } else {
      const double po = p[o + i];
      if (do_u) u[o + i] = fma(alpha, po, u[o + i]);
      if (do_p) p[o + i] = fma(beta, po, z[o + i]);
    }
  }
}

// sum u (final projection, solver.py:169)
__global__ void __launch_bounds__(256) gen_sum_kernel(const double* __restrict__ u, int n, double* part) {
  __shared__ double scratch[64];
  const size_t nn = (size_t)n * n;
  const double* up = u + ((size_t)blockIdx.y * n + blockIdx.x) * nn;
  double s = 0.0;
  for (int i = threadIdx.x; i < (int)nn; i += blockDim.x) s += up[i];
  gen_store_partial(s, 0.0, part, scratch);
}

}  // namespace chk
