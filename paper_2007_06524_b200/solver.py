"""Mean-projected PCG on the GPU: drop-in for the reference solver.py.

``pcg_solve(A, f, opts, precond)`` keeps the reference contract
(solver.py:118-194): returns ``(u, PcgReport)``, projects a RHS with a
non-negligible mean and flags it, returns zero for a zero RHS, reports (does
not raise) non-convergence, raises :class:`SolverBreakdown` on p'Ap <= 0 or a
non-finite residual.  ``pcg_solve_batched`` is the realization batcher that
runs B independent solves in one set of kernels.
"""

from __future__ import annotations

import ctypes
import functools
import re
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigurationError, SolverBreakdown
from .lowrank import DevicePlan, _device_apply, _plan_for

PRECONDITIONERS = ("fourier", "lkr", "regularized")


@dataclass(frozen=True)
class SolveOptions:
    """solver.py:32-58."""

    tol: float = 1e-8
    max_iter: int = 500
    preconditioner: str = "fourier"
    eps_rank: float = 1e-8
    delta: float = 0.0
    precond_residual_stopping: bool = False

    def __post_init__(self):
        if self.tol <= 0.0:
            raise ConfigurationError(f"tolerance must be positive, got {self.tol}")
        if self.max_iter < 1:
            raise ConfigurationError(f"max_iter must be >= 1, got {self.max_iter}")
        if self.preconditioner not in PRECONDITIONERS:
            raise ConfigurationError(
                f"preconditioner must be one of {PRECONDITIONERS}, got {self.preconditioner!r}")
        if self.delta < 0.0:
            raise ConfigurationError(f"delta must be >= 0, got {self.delta}")


@dataclass(frozen=True)
class PcgReport:
    """solver.py:61-70."""

    iterations: int
    residuals: tuple
    converged: bool
    final_residual: float
    preconditioner: str
    rhs_projected: bool = False


@dataclass(frozen=True)
class Preconditioner:
    """solver.py:73-76; ``plan`` is the device plan the batched solver consumes."""

    name: str
    apply: object
    plan: object = None


def _device_index() -> int:
    torch = _lib.require_cuda()
    return int(torch.cuda.current_device())


@functools.lru_cache(maxsize=8)
def _cached_preconditioner(d: int, n: int, kind: str, eps_rank: float, delta: float,
                           device: int = 0) -> Preconditioner:
    """solver.py:79-93 (same names; the apply is the device pipeline).  Keyed
    also by the CUDA device: a plan's buffers live on the device it was built on."""
    plan = _plan_for(d, n, kind, eps_rank, delta, device)
    if kind == "fourier":
        name = "fourier"
    elif kind == "regularized":
        name = f"regularized(delta={delta})"
    else:
        name = f"lkr(eps={eps_rank},rank={plan.r1})"
    return Preconditioner(name, lambda x: _device_apply(plan, x), plan)


def make_preconditioner(d: int, n: int, opts: SolveOptions) -> Preconditioner:
    """solver.py:96-100."""
    eps_rank = opts.eps_rank if opts.preconditioner == "lkr" else 0.0
    delta = opts.delta if opts.preconditioner == "regularized" else 0.0
    return _cached_preconditioner(d, n, opts.preconditioner, eps_rank, delta, _device_index())


_NAME_RE = {
    "lkr": re.compile(r"^lkr\(eps=([^,]+),rank=(\d+)\)$"),
    "regularized": re.compile(r"^regularized\(delta=([^)]+)\)$"),
}


def _device_preconditioner(precond, d: int, n: int) -> Preconditioner:
    """The device-plan preconditioner equivalent to ``precond``: ours as is; a
    reference-built ``Preconditioner(name, apply)`` from its make_preconditioner
    (solver.py:79-100) is recognised by its name (``fourier``,
    ``regularized(delta=...)``, ``lkr(eps=...,rank=R)``).  Any other callable has
    no device plan: ValueError (the GPU path has no host fallback)."""
    plan = getattr(precond, "plan", None)
    if isinstance(plan, DevicePlan):
        if plan.n != n:
            raise ValueError(f"preconditioner is for n = {plan.n}, operator has n = {n}")
        if plan.device != _device_index():
            return make_preconditioner(d, n, SolveOptions(
                preconditioner=plan.kind, eps_rank=plan.eps_rank or 1e-8, delta=plan.delta))
        return precond
    name = str(getattr(precond, "name", ""))
    if name == "fourier":
        return make_preconditioner(d, n, SolveOptions(preconditioner="fourier"))
    m = _NAME_RE["regularized"].match(name)
    if m:
        return make_preconditioner(d, n, SolveOptions(preconditioner="regularized", delta=float(m.group(1))))
    m = _NAME_RE["lkr"].match(name)
    if m:
        p = make_preconditioner(d, n, SolveOptions(preconditioner="lkr", eps_rank=float(m.group(1))))
        if p.plan.r1 != int(m.group(2)):
            raise ValueError(f"{name}: the rebuilt factors have rank {p.plan.r1}")
        return p
    raise ValueError(f"preconditioner {name!r} has no device plan: build it with make_preconditioner "
                     f"(kinds {PRECONDITIONERS})")


def project_mean_zero(x):
    """solver.py:103-106."""
    x = np.asarray(x, dtype=float)
    return x - x.mean()


def residual(A, u, f) -> float:
    """solver.py:109-115 (A.apply runs the device stencil)."""
    f = np.asarray(f, dtype=float)
    norm_f = float(np.linalg.norm(f))
    Au = A.apply(np.asarray(u, dtype=float))
    norm_r = float(np.linalg.norm(f - np.asarray(Au)))
    if norm_f == 0.0:
        return norm_r
    return norm_r / norm_f


@dataclass
class BatchResult:
    """Raw per-realization outputs of :func:`pcg_solve_batched`."""

    u: object              # torch (B, n^3) on the device
    iterations: np.ndarray
    final_residual: np.ndarray
    status: np.ndarray     # 0 converged, 1 not converged, 2 breakdown
    rhs_projected: np.ndarray
    history: np.ndarray | None
    launches: int

    def report(self, b: int, name: str) -> PcgReport:
        its = int(self.iterations[b])
        res = tuple(float(v) for v in self.history[b, :its]) if self.history is not None else ()
        return PcgReport(iterations=its, residuals=res, converged=bool(self.status[b] == 0),
                         final_residual=float(self.final_residual[b]), preconditioner=name,
                         rhs_projected=bool(self.rhs_projected[b]))


class Workspace:
    """Reusable device workspace for repeated batched solves."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device):
        import torch

        device = torch.device(device)
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = None
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        return self.buf


_default_ws = Workspace()


def pcg_solve_batched(A, F, opts: SolveOptions | None = None, precond: Preconditioner | None = None,
                      out=None, record_history: bool = True, workspace: Workspace | None = None):
    """B independent mean-projected PCG solves on one GPU.

    A: ``StiffnessBatch`` (or ``StiffnessOperator`` for B = 1); F: (B, n^3)
    float64 device tensor.  Returns a :class:`BatchResult` (u stays on the
    device).
    """
    torch = _lib.require_cuda()
    from .operators import StiffnessBatch, StiffnessOperator

    opts = opts or SolveOptions()
    batch = _as_batch(A)
    if precond is None:
        precond = make_preconditioner(3, batch.n, opts)
    precond = _device_preconditioner(precond, 3, batch.n)
    plan = precond.plan
    n = batch.n
    size = n ** 3
    B = batch.B
    if F.numel() != B * size:  # solver.py:128-130 -> operators.py:304-305
        raise ValueError(f"load has {F.numel()} entries, expected {B} x {size}")
    Fd = F.reshape(B, size)
    if Fd.dtype != torch.float64 or Fd.device.type != "cuda":
        Fd = Fd.to("cuda", torch.float64)
    Fd = Fd.contiguous()
    u = out if out is not None else torch.empty_like(Fd)
    lib = _lib.load()
    ws_bytes = int(lib.chk_pcg_workspace_bytes(ctypes.byref(batch.grid), plan.handle, B, opts.max_iter))
    if ws_bytes == 0:
        raise ValueError("unsupported grid for the GPU path")
    ws = (workspace or _default_ws).get(ws_bytes, Fd.device)
    its = np.zeros(B, dtype=np.int32)
    fin = np.zeros(B, dtype=np.float64)
    st = np.zeros(B, dtype=np.int32)
    proj = np.zeros(B, dtype=np.int32)
    hist = np.zeros((B, opts.max_iter), dtype=np.float64) if record_history else None
    copts = _lib.ChkPcgOpts(float(opts.tol), int(opts.max_iter), int(bool(opts.precond_residual_stopping)))
    vp = ctypes.c_void_p
    _lib.check(lib.chk_pcg_solve_batched(
        ctypes.byref(batch.grid), plan.handle, vp(batch.beta.data_ptr()), vp(Fd.data_ptr()),
        vp(u.data_ptr()), B, ctypes.byref(copts), its.ctypes.data_as(vp), fin.ctypes.data_as(vp),
        st.ctypes.data_as(vp), proj.ctypes.data_as(vp),
        hist.ctypes.data_as(vp) if hist is not None else None, vp(ws.data_ptr()), ws.numel(),
        _lib.stream_handle()))
    return BatchResult(u=u, iterations=its, final_residual=fin, status=st, rhs_projected=proj,
                       history=hist, launches=int(lib.chk_last_launch_count()))


def pcg_solve_host(config, beta_host, F_host, opts: SolveOptions | None = None,
                   precond: Preconditioner | None = None, chunk: int | None = None, out=None,
                   record_history: bool = True, workspace: Workspace | None = None):
    """Batched solve from HOST buffers (numpy / pinned torch CPU tensors): the
    reference-facing call with host<->device copies inside.  The batch runs in
    chunks with uploads/downloads overlapped with the solves (chk_pcg_solve_host).
    Returns a BatchResult whose ``u`` is the host (B, n^3) array."""
    torch = _lib.require_cuda()
    opts = opts or SolveOptions()
    n = config.n
    if precond is None:
        precond = make_preconditioner(3, n, opts)
    precond = _device_preconditioner(precond, 3, n)
    plan = precond.plan
    beta = beta_host if isinstance(beta_host, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(beta_host, dtype=np.float64)))
    Fh = F_host if isinstance(F_host, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(F_host, dtype=np.float64)))
    B = Fh.shape[0]
    beta = beta.reshape(B, -1).contiguous()
    Fh = Fh.reshape(B, -1).contiguous()
    U = out if out is not None else torch.empty_like(Fh)
    if chunk is None:
        # 3 lanes x chunks of B/8, but at least ~4M DOF per chunk (per-solve overheads):
        # measured best for configs 2, 3, 4 (16, 32, 2 realizations)
        chunk = max(1, (B + 7) // 8, -(-(4 << 20) // n ** 3))
    grid = _lib.grid_struct(3, n, config.L, config.n0, config.k, config.offset, config.lam)
    lib = _lib.load()
    wb = int(lib.chk_pcg_host_workspace_bytes(ctypes.byref(grid), plan.handle, min(chunk, B), opts.max_iter))
    if wb == 0:
        raise ValueError("unsupported grid for the GPU path")
    ws = (workspace or _default_ws).get(wb, torch.device("cuda", torch.cuda.current_device()))
    its = np.zeros(B, np.int32)
    fin = np.zeros(B)
    st = np.zeros(B, np.int32)
    proj = np.zeros(B, np.int32)
    hist = np.zeros((B, opts.max_iter)) if record_history else None
    copts = _lib.ChkPcgOpts(float(opts.tol), int(opts.max_iter), int(bool(opts.precond_residual_stopping)))
    vp = ctypes.c_void_p
    _lib.check(lib.chk_pcg_solve_host(
        ctypes.byref(grid), plan.handle, vp(beta.data_ptr()), vp(Fh.data_ptr()), vp(U.data_ptr()), B,
        int(chunk), ctypes.byref(copts), its.ctypes.data_as(vp), fin.ctypes.data_as(vp),
        st.ctypes.data_as(vp), proj.ctypes.data_as(vp), hist.ctypes.data_as(vp) if hist is not None else None,
        vp(ws.data_ptr()), ws.numel(), _lib.stream_handle()))
    return BatchResult(u=U, iterations=its, final_residual=fin, status=st, rhs_projected=proj,
                       history=hist, launches=int(lib.chk_last_launch_count()))


def pcg_solve_seeds(config, seeds, opts: SolveOptions | None = None, precond: Preconditioner | None = None,
                    rhs=1, chunk: int | None = None, out=None, record_history: bool = True,
                    workspace: Workspace | None = None):
    """Seeds to solutions: realization ``seeds[m]`` is drawn on the GPU
    (bit-identical to sample_realization), its load is the device corrector RHS
    along direction ``rhs`` (int, the PCG load of homogenize.py:110) or row m of
    a host array ``rhs`` (B, n^3), and u comes back to the host ``out`` (pinned
    (B, n^3) tensor or new).  Chunked over lanes like pcg_solve_host; the
    host-side work per realization is the SeedSequence hash of its seed."""
    from .lattice import contrast_args, philox_keys

    torch = _lib.require_cuda()
    opts = opts or SolveOptions()
    n = config.n
    if precond is None:
        precond = make_preconditioner(3, n, opts)
    precond = _device_preconditioner(precond, 3, n)
    plan = precond.plan
    kind, b0, b1 = contrast_args(config)
    keys = philox_keys(seeds)
    B = keys.shape[0]
    f_host = None
    direction = 0
    if isinstance(rhs, (int, np.integer)):
        direction = int(rhs)
        if not 1 <= direction <= 3:
            raise ValueError(f"direction must be in 1..3, got {direction}")
    else:
        f_host = rhs if isinstance(rhs, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.asarray(rhs, dtype=np.float64)))
        f_host = f_host.reshape(B, -1).contiguous()
    U = out if out is not None else torch.empty((B, n ** 3), dtype=torch.float64).pin_memory()
    if chunk is None:
        chunk = max(1, (B + 7) // 8, -(-(4 << 20) // n ** 3))
    grid = _lib.grid_struct(3, n, config.L, config.n0, config.k, config.offset, config.lam)
    lib = _lib.load()
    wb = int(lib.chk_pcg_host_workspace_bytes(ctypes.byref(grid), plan.handle, min(chunk, B), opts.max_iter))
    if wb == 0:
        raise ValueError("unsupported grid for the GPU path")
    ws = (workspace or _default_ws).get(wb, torch.device("cuda", torch.cuda.current_device()))
    its = np.zeros(B, np.int32)
    fin = np.zeros(B)
    st = np.zeros(B, np.int32)
    proj = np.zeros(B, np.int32)
    hist = np.zeros((B, opts.max_iter)) if record_history else None
    copts = _lib.ChkPcgOpts(float(opts.tol), int(opts.max_iter), int(bool(opts.precond_residual_stopping)))
    vp = ctypes.c_void_p
    _lib.check(lib.chk_pcg_solve_seeds(
        ctypes.byref(grid), plan.handle, keys.ctypes.data_as(vp), float(config.coverage_prob), kind, b0, b1,
        vp(f_host.data_ptr()) if f_host is not None else None, direction, vp(U.data_ptr()), B, int(chunk),
        ctypes.byref(copts), its.ctypes.data_as(vp), fin.ctypes.data_as(vp), st.ctypes.data_as(vp),
        proj.ctypes.data_as(vp), hist.ctypes.data_as(vp) if hist is not None else None,
        vp(ws.data_ptr()), ws.numel(), _lib.stream_handle()))
    return BatchResult(u=U, iterations=its, final_residual=fin, status=st, rhs_projected=proj,
                       history=hist, launches=int(lib.chk_last_launch_count()))


def _as_batch(A):
    """StiffnessBatch of ``A``: ours (StiffnessBatch / StiffnessOperator), or a
    realization-carrying operator.  The reference's StiffnessOperator holds only
    Kronecker terms (operators.py:96-131) -- build the device operator from the
    same realization with ``assemble_stiffness(r)`` (ValueError otherwise)."""
    from .operators import StiffnessBatch, StiffnessOperator

    if isinstance(A, StiffnessOperator):
        return A._batch
    if isinstance(A, StiffnessBatch):
        return A
    r = getattr(A, "realization", None)
    if r is not None:
        return StiffnessOperator(r)._batch
    raise ValueError(f"{type(A).__name__} is not a device stiffness operator: build it with "
                     f"paper_2007_06524_b200.assemble_stiffness(realization)")


def pcg_solve(A, f, opts: SolveOptions | None = None, precond: Preconditioner | None = None):
    """Drop-in for solver.py:118-194 on the GPU."""
    torch = _lib.require_cuda()
    opts = opts or SolveOptions()
    if getattr(A, "d", 3) != 3:
        raise ValueError("the GPU path implements d = 3 only")
    if precond is None:
        precond = make_preconditioner(A.d, A.n, opts)
    is_np = not isinstance(f, torch.Tensor)
    ft = torch.as_tensor(np.asarray(f, dtype=np.float64)) if is_np else f
    res = pcg_solve_batched(A, ft.reshape(1, -1), opts, precond)
    if res.status[0] == _lib.CHK_BREAKDOWN:
        raise SolverBreakdown(f"PCG breakdown (p'Ap <= 0 or non-finite residual) at iteration "
                              f"{int(res.iterations[0])}")
    if res.rhs_projected[0]:
        warnings.warn("right-hand side has a nonzero mean; projecting it out")
    report = res.report(0, precond.name)
    u = res.u.reshape(-1)
    return (u.cpu().numpy() if is_np else u), report
