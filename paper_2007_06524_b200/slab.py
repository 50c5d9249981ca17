"""Slab decomposition of ONE grid over several GPUs.

Rank r of P owns planes x0 in [r n/P, (r+1) n/P) of p, u and f and one chunk of
the spectral columns (the residual spectrum lives there and never moves).  Per
PCG iteration (pcg_solve, solver.py:161-185):

  halo exchange of p (first/last local plane, periodic)      -> stencil
  FWD_Q  : q = A p, x2/x1 transforms, rank-local p.Ap       -> allreduce -> alpha
  all_to_all (x0 slabs -> column chunks)
  MID    : x0 transform, R -= alpha Q, ||r||^2, z = D R, r.z -> allreduce -> stop / beta
  all_to_all (column chunks -> x0 slabs)
  INV    : inverse transforms, u += alpha p, p = z + beta p

The collectives run between kernel launches on the caller's stream
(torch.distributed over NCCL: NVLink/NVSwitch on one node); every rank takes
the same decisions from bit-identical allreduced scalars.  ``LocalComm``
executes the same schedule for P virtual ranks inside one process (explicit
device copies between phases, no kernel ever waits on another) -- this is how
the decomposition is verified on a single GPU.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .solver import BatchResult, SolveOptions, make_preconditioner

STATS, STATS_DECIDE, FWD_INIT, MID, MID_DECIDE, INV, FWD_Q, ALPHA_DECIDE, MEANU, MEANU_APPLY = range(10)


class ChkSlab(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32)]


# ----------------------------------------------------------------------------
# communicators (operate on lists of per-rank tensors held by this process)
# ----------------------------------------------------------------------------


class TorchComm:
    """One rank per process: torch.distributed collectives (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allreduce(self, reds):
        (red,) = reds
        self.dist.all_reduce(red, op=self.dist.ReduceOp.SUM, group=self.group)

    def all_to_all(self, outs, ins):
        (out,), (inp,) = outs, ins
        self.dist.all_to_all_single(out, inp, group=self.group)

    def halo(self, firsts, lasts, los, his):
        """lo[r] <- last plane of rank r-1, hi[r] <- first plane of rank r+1 (periodic)."""
        (first,), (last,), (lo,), (hi,) = firsts, lasts, los, his
        P, r = self.P, self.rank
        if P == 1:
            lo.copy_(last)
            hi.copy_(first)
            return
        dist = self.dist
        prv, nxt = (r - 1) % P, (r + 1) % P
        ops = [dist.P2POp(dist.isend, last.contiguous(), nxt, self.group),
               dist.P2POp(dist.irecv, lo, prv, self.group),
               dist.P2POp(dist.isend, first.contiguous(), prv, self.group),
               dist.P2POp(dist.irecv, hi, nxt, self.group)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()


class LocalComm:
    """P virtual ranks in one process (lists of length P), same semantics as TorchComm."""

    def __init__(self, P):
        self.P = P

    def allreduce(self, reds):
        total = reds[0].clone()
        for t in reds[1:]:
            total += t
        for t in reds:
            t.copy_(total)

    def all_to_all(self, outs, ins):
        P = self.P
        for r in range(P):
            src = ins[r].view(P, -1)
            for s in range(P):
                outs[s].view(P, -1)[r].copy_(src[s])

    def halo(self, firsts, lasts, los, his):
        P = self.P
        for r in range(P):
            los[r].copy_(lasts[(r - 1) % P])
            his[r].copy_(firsts[(r + 1) % P])


# ----------------------------------------------------------------------------
# one rank's buffers and phase launcher
# ----------------------------------------------------------------------------


class SlabRank:
    """Device buffers of rank ``rank`` of ``P`` for a batch of B realizations."""

    def __init__(self, config, beta_cells, f_local, P: int, rank: int, opts: SolveOptions, device=None):
        torch = _lib.require_cuda()
        self.torch = torch
        self.lib = _lib.load()
        self.config = config
        n = config.n
        if n % P:
            raise ValueError(f"nranks {P} must divide n = {n}")
        self.n, self.P, self.rank, self.nloc = n, P, rank, n // P
        self.opts = opts
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        beta = torch.as_tensor(np.asarray(beta_cells, dtype=np.float64)) if not isinstance(beta_cells, torch.Tensor) else beta_cells
        self.beta = beta.reshape(-1, config.L ** 3).to(dev, torch.float64).contiguous()
        self.B = self.beta.shape[0]
        nn = n * n
        self.f = f_local.reshape(self.B, self.nloc * nn).to(dev, torch.float64).contiguous()
        self.u = torch.empty_like(self.f)
        self.p = torch.empty_like(self.f)
        self.grid = _lib.grid_struct(3, n, config.L, config.n0, config.k, config.offset, config.lam)
        self.slab = ChkSlab(P, rank)
        self.plan = make_preconditioner(3, n, opts).plan
        ne = int(self.lib.chk_slab_exchange_elems(ctypes.byref(self.grid), ctypes.byref(self.slab), self.B))
        if ne == 0:
            raise ValueError("unsupported slab geometry")
        self.xa = torch.empty(2 * ne, dtype=torch.float64, device=dev)
        self.xb = torch.empty(2 * ne, dtype=torch.float64, device=dev)
        self.halo_lo = torch.empty(self.B, nn, dtype=torch.float64, device=dev)
        self.halo_hi = torch.empty(self.B, nn, dtype=torch.float64, device=dev)
        self.red = torch.zeros(self.B, 4, dtype=torch.float64, device=dev)
        wb = int(self.lib.chk_slab_workspace_bytes(ctypes.byref(self.grid), self.plan.handle,
                                                   ctypes.byref(self.slab), self.B, opts.max_iter))
        if wb == 0:
            raise ValueError("unsupported slab geometry")
        self.ws = torch.empty(wb, dtype=torch.uint8, device=dev)
        self.copts = _lib.ChkPcgOpts(float(opts.tol), int(opts.max_iter), int(bool(opts.precond_residual_stopping)))

    def planes(self):
        v = self.p.view(self.B, self.nloc, self.n * self.n)
        return v[:, 0].contiguous(), v[:, self.nloc - 1].contiguous()

    def phase(self, ph: int, it: int = 0):
        vp = ctypes.c_void_p
        rc = self.lib.chk_slab_phase(
            ctypes.byref(self.grid), self.plan.handle, ctypes.byref(self.slab), ph, it,
            vp(self.beta.data_ptr()), vp(self.f.data_ptr()), vp(self.u.data_ptr()), vp(self.p.data_ptr()),
            vp(self.xa.data_ptr()), vp(self.xb.data_ptr()), vp(self.halo_lo.data_ptr()),
            vp(self.halo_hi.data_ptr()), vp(self.red.data_ptr()), self.B, ctypes.byref(self.copts),
            vp(self.ws.data_ptr()), self.ws.numel(), _lib.stream_handle())
        _lib.check(rc)

    def read_state(self, history=False):
        B, mi = self.B, self.opts.max_iter
        its = np.zeros(B, np.int32)
        fin = np.zeros(B)
        st = np.zeros(B, np.int32)
        proj = np.zeros(B, np.int32)
        hist = np.zeros((B, mi)) if history else None
        vp = ctypes.c_void_p
        _lib.check(self.lib.chk_slab_read_state(
            ctypes.byref(self.grid), ctypes.byref(self.slab), B, mi, vp(self.ws.data_ptr()),
            its.ctypes.data_as(vp), fin.ctypes.data_as(vp), st.ctypes.data_as(vp), proj.ctypes.data_as(vp),
            hist.ctypes.data_as(vp) if hist is not None else None, _lib.stream_handle()))
        return its, fin, st, proj, hist


def slab_solve(ranks: list, comm, poll_every: int = 2) -> BatchResult:
    """Run the batched PCG over the ranks held by this process (all P for
    LocalComm, one for TorchComm).  Returns rank-local u in ``result.u``
    (list of [B, nloc*n*n] tensors) and the (rank-identical) reports."""
    opts = ranks[0].opts

    def each(ph, it=0):
        for r in ranks:
            r.phase(ph, it)

    def reds():
        comm.allreduce([r.red for r in ranks])

    each(STATS)
    reds()
    each(STATS_DECIDE)
    each(FWD_INIT)
    comm.all_to_all([r.xb for r in ranks], [r.xa for r in ranks])
    each(MID, 0)
    reds()
    each(MID_DECIDE, 0)
    comm.all_to_all([r.xa for r in ranks], [r.xb for r in ranks])
    each(INV, 0)
    for it in range(1, opts.max_iter + 1):
        pl = [r.planes() for r in ranks]
        comm.halo([f for f, _ in pl], [l for _, l in pl], [r.halo_lo for r in ranks],
                  [r.halo_hi for r in ranks])
        each(FWD_Q, it)
        reds()
        each(ALPHA_DECIDE, it)
        comm.all_to_all([r.xb for r in ranks], [r.xa for r in ranks])
        each(MID, it)
        reds()
        each(MID_DECIDE, it)
        comm.all_to_all([r.xa for r in ranks], [r.xb for r in ranks])
        each(INV, it)
        if it % poll_every == 0 or it == opts.max_iter:
            _, _, st, _, _ = ranks[0].read_state()
            if not np.any(st == 3):  # every rank holds the same status words
                break
    each(MEANU)
    reds()
    each(MEANU_APPLY)
    its, fin, st, proj, hist = ranks[0].read_state(history=True)
    st = np.where(st == 3, _lib.CHK_NOT_CONVERGED, st)
    return BatchResult(u=[r.u for r in ranks], iterations=its, final_residual=fin, status=st,
                       rhs_projected=proj, history=hist, launches=0)
