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
the same decisions from bit-identical allreduced scalars.  With ``chunks`` > 1
the plane phases run in plane chunks and each all_to_all is split the same
way: the exchange of chunk k (asynchronous NCCL work on its own stream) runs
under the FWD kernels of chunk k+1, and the return exchange of chunk k+1 under
the INV kernels of chunk k; the halo of p travels under the interior planes.
The convergence poll is a stream-ordered copy of the status words into pinned
memory checked one poll later (no host synchronisation on the iteration).  ``LocalComm``
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

    def all_to_all_planes(self, outs, ins, shape, p0, p1):
        """Exchange of the rows of local planes [p0, p1) only (buffers viewed as
        [P][B][nloc][row]; each (destination, realization) block is contiguous):
        grouped point-to-point sends / receives (ncclSend / ncclRecv under one
        group on NCCL), asynchronous -- returns the pending requests (finish()
        makes the current stream wait for them)."""
        (out,), (inp,) = outs, ins
        dist, P, r = self.dist, self.P, self.rank
        o = out.view(shape)[:, :, p0:p1]
        i = inp.view(shape)[:, :, p0:p1]
        o[r].copy_(i[r])
        ops = []
        for k in range(1, P):
            dst, src = (r + k) % P, (r - k) % P
            for b in range(shape[1]):
                ops.append(dist.P2POp(dist.isend, i[dst, b], dst, self.group))
                ops.append(dist.P2POp(dist.irecv, o[src, b], src, self.group))
        return (dist.batch_isend_irecv(ops) if ops else []), None

    def finish(self, pending):
        works, unpack = pending
        for w in works:
            w.wait()
        if unpack is not None:
            unpack[0].copy_(unpack[1])

    def halo(self, firsts, lasts, los, his, async_op=False):
        """lo[r] <- last plane of rank r-1, hi[r] <- first plane of rank r+1 (periodic)."""
        (first,), (last,), (lo,), (hi,) = firsts, lasts, los, his
        P, r = self.P, self.rank
        if P == 1:
            lo.copy_(last)
            hi.copy_(first)
            return ([], None) if async_op else None
        dist = self.dist
        prv, nxt = (r - 1) % P, (r + 1) % P
        ops = [dist.P2POp(dist.isend, last.contiguous(), nxt, self.group),
               dist.P2POp(dist.irecv, lo, prv, self.group),
               dist.P2POp(dist.isend, first.contiguous(), prv, self.group),
               dist.P2POp(dist.irecv, hi, nxt, self.group)]
        reqs = dist.batch_isend_irecv(ops)
        if async_op:
            return reqs, None
        for req in reqs:
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

    def all_to_all_planes(self, outs, ins, shape, p0, p1):
        P = self.P
        for r in range(P):
            src = ins[r].view(shape)
            for s in range(P):
                outs[s].view(shape)[r, :, p0:p1].copy_(src[s, :, p0:p1])
        return [], None

    def finish(self, pending):
        pass

    def halo(self, firsts, lasts, los, his, async_op=False):
        P = self.P
        for r in range(P):
            los[r].copy_(lasts[(r - 1) % P])
            his[r].copy_(firsts[(r + 1) % P])
        return ([], None) if async_op else None


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

    def xshape(self):
        """Exchange buffers as [P][B][nloc][row] float64 views."""
        return (self.P, self.B, self.nloc, -1)

    def status_async(self, out):
        """Stream-ordered copy of the B status words into ``out`` (pinned int32)."""
        _lib.check(self.lib.chk_slab_status_async(
            ctypes.byref(self.grid), ctypes.byref(self.slab), self.B, self.opts.max_iter,
            ctypes.c_void_p(self.ws.data_ptr()), ctypes.c_void_p(out.data_ptr()), _lib.stream_handle()))

    def phase(self, ph: int, it: int = 0, planes=None):
        vp = ctypes.c_void_p
        p0, cnt = planes if planes is not None else (0, -1)
        rc = self.lib.chk_slab_phase_planes(
            ctypes.byref(self.grid), self.plan.handle, ctypes.byref(self.slab), ph, it, int(p0), int(cnt),
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


def plane_chunks(nloc: int, chunks: int) -> list:
    """Plane ranges of a chunked plane phase: the interior planes [1, nloc-1) in
    ``chunks`` pieces first (they need no halo), then the two edge planes."""
    if chunks <= 1 or nloc < 4:
        return [(0, nloc)]
    inner = nloc - 2
    k = min(chunks, inner)
    cuts = [1 + (inner * j) // k for j in range(k + 1)]
    return [(cuts[j], cuts[j + 1]) for j in range(k)] + [(0, 1), (nloc - 1, nloc)]


def slab_solve(ranks: list, comm, poll_every: int = 2, chunks: int = 1) -> BatchResult:
    """Run the batched PCG over the ranks held by this process (all P for
    LocalComm, one for TorchComm).  Returns rank-local u in ``result.u``
    (list of [B, nloc*n*n] tensors) and the (rank-identical) reports.

    chunks > 1: plane phases and their all_to_all exchanges in plane chunks
    (overlapped with NCCL); the convergence poll is asynchronous (one poll of
    look-ahead), so the host never waits on the current iteration."""
    torch = ranks[0].torch
    opts = ranks[0].opts
    shape = ranks[0].xshape()
    pieces = plane_chunks(ranks[0].nloc, chunks)

    def each(ph, it=0, planes=None):
        for r in ranks:
            r.phase(ph, it, planes)

    def reds():
        comm.allreduce([r.red for r in ranks])

    def forward(ph, it):
        """plane phase ph (FWD_INIT / FWD_Q) then exchange x0 slabs -> column chunks"""
        if len(pieces) == 1:
            each(ph, it)
            return [("all", None)]
        pend = []
        for (p0, p1) in pieces:
            if p0 == 0 and halo_pending[0] is not None:
                comm.finish(halo_pending[0])
                halo_pending[0] = None
            each(ph, it, (p0, p1 - p0))
            pend.append(comm.all_to_all_planes([r.xb for r in ranks], [r.xa for r in ranks], shape, p0, p1))
        return pend

    def after_forward(pend):
        if pend and pend[0][0] == "all":
            comm.all_to_all([r.xb for r in ranks], [r.xa for r in ranks])
            return
        for pd in pend:
            comm.finish(pd)

    def backward(it):
        """exchange column chunks -> x0 slabs, then INV, chunk by chunk"""
        if len(pieces) == 1:
            comm.all_to_all([r.xa for r in ranks], [r.xb for r in ranks])
            each(INV, it)
            return
        pend = [comm.all_to_all_planes([r.xa for r in ranks], [r.xb for r in ranks], shape, p0, p1)
                for (p0, p1) in pieces]
        for (p0, p1), pd in zip(pieces, pend):
            comm.finish(pd)
            each(INV, it, (p0, p1 - p0))

    halo_pending = [None]
    each(STATS)
    reds()
    each(STATS_DECIDE)
    after_forward(forward(FWD_INIT, 0))
    each(MID, 0)
    reds()
    each(MID_DECIDE, 0)
    backward(0)
    # asynchronous convergence poll: status words -> pinned host every poll_every
    # iterations, read one poll later
    stat = [torch.empty(ranks[0].B, dtype=torch.int32).pin_memory() for _ in range(2)]
    evs = [torch.cuda.Event(), torch.cuda.Event()]
    npoll = 0
    for it in range(1, opts.max_iter + 1):
        pl = [r.planes() for r in ranks]
        halo = comm.halo([f for f, _ in pl], [l for _, l in pl], [r.halo_lo for r in ranks],
                         [r.halo_hi for r in ranks], async_op=True)
        if len(pieces) == 1:
            comm.finish(halo)
        else:
            halo_pending[0] = halo
        pend = forward(FWD_Q, it)
        reds()
        each(ALPHA_DECIDE, it)
        after_forward(pend)
        each(MID, it)
        reds()
        each(MID_DECIDE, it)
        backward(it)
        if it % poll_every == 0 or it == opts.max_iter:
            if npoll > 0:
                prev = (npoll - 1) & 1
                evs[prev].synchronize()
                if not np.any(stat[prev].numpy() == 3):  # every rank holds the same status words
                    break
            cur = npoll & 1
            ranks[0].status_async(stat[cur])
            evs[cur].record()
            npoll += 1
    each(MEANU)
    reds()
    each(MEANU_APPLY)
    its, fin, st, proj, hist = ranks[0].read_state(history=True)
    st = np.where(st == 3, _lib.CHK_NOT_CONVERGED, st)
    return BatchResult(u=[r.u for r in ranks], iterations=its, final_residual=fin, status=st,
                       rhs_projected=proj, history=hist, launches=0)
