// chk_plane.cuh -- the plane-pass kernels (forward / inverse / paired).
//
// Bodies: fwd_plane_body / inv_plane_body (chk_kernels.cuh).  A register-staged
// variant of both passes (stencil feeding the first radix-8 row stage in
// registers, R2C post-processing fused into the column stage, last stages to /
// from HBM directly; 7 instead of 11 shared-memory operations per element) was
// measured slower on B200 (config 3 paired pass 4.0 ms vs 3.0 ms: twice the
// load instructions of the quad stencil, 94-144 registers or spills, and no TMA
// bulk load in the inverse pass) and was dropped; see DESIGN.md section 7.
#pragma once

namespace chk {

// --------------------------------------------------------------------------
// plane-pass kernels
// --------------------------------------------------------------------------
template <int N, int G, int MODE, bool ALLIN>
__global__ void __launch_bounds__(PlaneNT<N>::value, PlaneNT<N>::minb) fwd_plane_kernel(Geo g, const double* __restrict__ beta,
                                                        const double* __restrict__ src, double* __restrict__ u,
                                                        double2* __restrict__ S, PlanDev pl,
                                                        SolveCtl ctl, SlabGeo sg, int B, int it,
                                                        const __grid_constant__ CUtensorMap tmap, int use_tmap) {
  fwd_plane_body<N, G, MODE, ALLIN>(g, beta, src, u, S, pl, ctl, sg, B, it, blockIdx.x,
                                    (IlW<N>::value > 0 && use_tmap) ? &tmap : nullptr);
}

template <int N, int G, int MODE>
__global__ void __launch_bounds__(PlaneNT<N>::value, PlaneNT<N>::minb) inv_plane_kernel(const double2* __restrict__ S,
                                                        double* __restrict__ out, double* __restrict__ u,
                                                        PlanDev pl, SolveCtl ctl, SlabGeo sg, int B, int it,
                                                        const __grid_constant__ CUtensorMap tmap, int use_tmap) {
  inv_plane_body<N, G, MODE>(S, out, u, pl, ctl, sg, B, it, blockIdx.x,
                             (IlW<N>::value > 0 && use_tmap) ? &tmap : nullptr);
}

// Paired plane pass: the forward pass of one half of the batch (q = A p, FFT;
// fp64-pipe and latency heavy) and the inverse pass of the other half (iFFT,
// u / p updates; HBM heavy) in ONE launch, their CTAs interleaved so that both
// kinds are co-resident on every SM.  The two halves are half an iteration
// apart (solver driver), so the launch has no internal dependency.
struct FwdArgs {
  Geo g;
  const double* beta;
  const double* p;
  double* u;
  double2* S;
  SolveCtl ctl;
  int B, it, blocks;
};
struct InvArgs {
  const double2* S;
  double* p;
  double* u;
  SolveCtl ctl;
  int B, it, blocks;
};

template <int N, int G, bool ALLIN>
__global__ void __launch_bounds__(PlaneNT<N>::value, PlaneNT<N>::minb) pair_plane_kernel(FwdArgs fa, InvArgs ia, PlanDev pl, SlabGeo sg) {
  const int m = fa.blocks < ia.blocks ? fa.blocks : ia.blocks;
  const int bx = blockIdx.x;
  bool fwd;
  int bid;
  if (bx < 2 * m) {
    fwd = (bx & 1) == 0;
    bid = bx >> 1;
  } else {
    fwd = fa.blocks > m;
    bid = bx - m;
  }
  if (fwd)
    fwd_plane_body<N, G, FWD_Q, ALLIN>(fa.g, fa.beta, fa.p, fa.u, fa.S, pl, fa.ctl, sg, fa.B, fa.it, bid);
  else
    inv_plane_body<N, G, INV_ITER>(ia.S, ia.p, ia.u, pl, ia.ctl, sg, ia.B, ia.it, bid);
}

}  // namespace chk
