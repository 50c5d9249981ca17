"""Low Kronecker rank (LKR) preconditioner: host setup + device apply.

Setup is a restatement of the reference lowrank.py:53-180 (exp-sum quadrature
of 1/x, canonical factors, dc fix) and produces bit-identical factors
(tests/test_host_api.py pins them against tests/golden/small.npz, which came
from the reference).  The factors are uploaded once into a device plan and
consumed as-is: the middle FFT pass evaluates D[i,j,l] = sum_k U0[k,i] U1[k,j]
U2[k,l] on the fly, so the n^3 diagonal never exists.
"""

from __future__ import annotations

import ctypes
import functools
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import QuadratureFailure
from .spectral import EigenSpectrum, fourier_eigenvalues

MAX_RANK = 256
_VALIDATION_POINTS = 4096


@dataclass(frozen=True)
class ExpSumQuadrature:
    """lowrank.py:26-50."""

    nodes: np.ndarray
    weights: np.ndarray
    a: float
    b: float
    eps: float
    achieved: float

    @property
    def rank(self) -> int:
        return len(self.nodes)


def _trapezoid_rule(rank: int, eps: float, rho: float):
    """lowrank.py:53-64."""
    s_min = math.log(eps / (8.0 * rho))
    s_max = math.log(math.log(8.0 / eps) + 4.0)
    s = np.linspace(s_min, s_max, rank)
    step = s[1] - s[0]
    nodes = np.exp(s)
    return nodes, step * nodes


def _sup_rel_error(nodes, weights, rho: float) -> float:
    """lowrank.py:67-71."""
    y = np.geomspace(1.0, rho, _VALIDATION_POINTS)
    with np.errstate(under="ignore"):
        approx = np.exp(-np.outer(y, nodes)) @ weights
    return float(np.max(np.abs(approx * y - 1.0)))


def exp_sum_quadrature(a: float, b: float, eps: float, max_rank: int = MAX_RANK) -> ExpSumQuadrature:
    """Minimal-rank exponential sum for 1/x on [a, b] (lowrank.py:74-120)."""
    if not (0.0 < a < b):
        raise ValueError(f"need 0 < a < b, got a={a}, b={b}")
    if eps <= 0.0:
        raise ValueError(f"tolerance must be positive, got {eps}")
    rho = b / a

    def error_at(rank):
        nodes, weights = _trapezoid_rule(rank, eps, rho)
        return _sup_rel_error(nodes, weights, rho)

    rank, previous = 8, 2
    best = math.inf
    while rank <= max_rank:
        err = error_at(rank)
        best = min(best, err)
        if err <= eps:
            break
        previous, rank = rank, rank * 2
    else:
        raise QuadratureFailure(
            f"no rank <= {max_rank} reaches eps={eps} on [{a}, {b}]; best sup relative error {best:.3e}",
            best_error=best, rank=max_rank)
    lo, hi = previous, rank
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if error_at(mid) <= eps:
            hi = mid
        else:
            lo = mid
    nodes, weights = _trapezoid_rule(hi, eps, rho)
    achieved = _sup_rel_error(nodes, weights, rho)
    return ExpSumQuadrature(nodes=nodes / a, weights=weights / a, a=float(a), b=float(b),
                            eps=float(eps), achieved=achieved)


@dataclass(frozen=True)
class CanonicalTensor:
    """entry(i) = sum_k prod_l factors[l][k, i_l] (lowrank.py:123-144)."""

    d: int
    n: int
    factors: tuple

    @property
    def rank(self) -> int:
        return self.factors[0].shape[0]

    def value(self, idx) -> float:
        prod = self.factors[0][:, idx[0]].copy()
        for axis in range(1, self.d):
            prod *= self.factors[axis][:, idx[axis]]
        return float(prod.sum())


def canonical_reciprocal(spectrum: EigenSpectrum, d: int, eps: float) -> CanonicalTensor:
    """lowrank.py:147-165."""
    if d not in (2, 3):
        raise ValueError(f"dimension must be 2 or 3, got {d}")
    lam = spectrum.values
    positive = lam[lam > 0.0]
    a = float(positive.min())
    b = float(d * lam.max())
    quad = exp_sum_quadrature(a, b, eps)
    with np.errstate(under="ignore"):
        base = np.exp(-np.outer(quad.nodes, lam))
    scale = quad.weights ** (1.0 / d)
    factor = scale[:, None] * base
    return CanonicalTensor(d=d, n=spectrum.n, factors=(factor,) * d)


def dc_correction(t: CanonicalTensor) -> CanonicalTensor:
    """lowrank.py:168-180: one extra rank-1 term zeroing the origin entry."""
    origin = t.value((0,) * t.d)
    new_factors = []
    for axis in range(t.d):
        e0 = np.zeros((1, t.n))
        e0[0, 0] = -origin if axis == 0 else 1.0
        new_factors.append(np.vstack([t.factors[axis], e0]))
    return CanonicalTensor(d=t.d, n=t.n, factors=tuple(new_factors))


# ----------------------------------------------------------------------------
# device plans
# ----------------------------------------------------------------------------


class DevicePlan:
    """Owns a chk_precond_plan (device twiddles + factors / eigenvalues)."""

    def __init__(self, kind: str, n: int, tensor: CanonicalTensor | None = None,
                 delta: float = 0.0, eps_rank: float = 0.0):
        torch = _lib.require_cuda()
        lib = _lib.load()
        self.kind = kind
        self.n = n
        self.delta = float(delta)
        self.eps_rank = float(eps_rank)
        self.device = int(torch.cuda.current_device())  # the plan's buffers live here
        handle = ctypes.c_void_p()
        eig = np.ascontiguousarray(fourier_eigenvalues(n).values, dtype=np.float64)
        if kind == "lkr":
            fac = np.ascontiguousarray(np.stack(tensor.factors), dtype=np.float64)
            self.r1 = fac.shape[1]
            self._fac = fac
            rc = lib.chk_precond_plan_create(_lib.PRECOND_KIND[kind], n, self.r1,
                                             fac.ctypes.data_as(ctypes.c_void_p),
                                             eig.ctypes.data_as(ctypes.c_void_p), 0.0,
                                             ctypes.byref(handle))
        else:
            self.r1 = 0
            rc = lib.chk_precond_plan_create(_lib.PRECOND_KIND[kind], n, 0, None,
                                             eig.ctypes.data_as(ctypes.c_void_p), self.delta,
                                             ctypes.byref(handle))
        _lib.check(rc)
        self.handle = handle

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib._lib is not None:
            _lib._lib.chk_precond_plan_destroy(h)
            self.handle = None

    def workspace_bytes(self, B: int) -> int:
        return int(_lib.load().chk_precond_workspace_bytes(self.handle, B))


def _plan_for(d: int, n: int, kind: str, eps_rank: float, delta: float, device: int | None = None) -> DevicePlan:
    """Cached device plan, keyed by the CUDA device it lives on (current device
    when ``device`` is None)."""
    if device is None:
        device = int(_lib.require_cuda().cuda.current_device())
    return _plan_on(d, n, kind, eps_rank, delta, int(device))


@functools.lru_cache(maxsize=8)
def _plan_on(d: int, n: int, kind: str, eps_rank: float, delta: float, device: int) -> DevicePlan:
    if d != 3:
        raise ValueError("the GPU path implements d = 3 only")
    torch = _lib.require_cuda()
    with torch.cuda.device(device):
        if kind == "lkr":
            t = dc_correction(canonical_reciprocal(fourier_eigenvalues(n), d, eps_rank))
            return DevicePlan("lkr", n, t, eps_rank=eps_rank)
        return DevicePlan(kind, n, delta=delta)


def _device_apply(plan: DevicePlan, x):
    """z = Re ifftn(D fftn x) for a vector (n^3,) or a batch (B, n^3); numpy in ->
    numpy out, torch CUDA in -> torch out."""
    torch = _lib.require_cuda()
    n = plan.n
    size = n ** 3
    is_np = not isinstance(x, torch.Tensor)
    xt = torch.as_tensor(np.asarray(x, dtype=np.float64)) if is_np else x
    if xt.dtype != torch.float64:
        raise ValueError("preconditioner input must be float64")
    shape = tuple(xt.shape)
    if shape == (size,):
        B = 1
    elif len(shape) == 2 and shape[1] == size:
        B = shape[0]
    else:
        raise ValueError(f"expected vector of length {size}, got shape {shape}")
    dev = torch.device("cuda", plan.device)
    with torch.cuda.device(dev):
        xd = xt.to(dev).contiguous()
        zd = torch.empty_like(xd)
        ws = torch.empty(plan.workspace_bytes(B), dtype=torch.uint8, device=dev)
        lib = _lib.load()
        _lib.check(lib.chk_precond_apply(plan.handle, ctypes.c_void_p(xd.data_ptr()),
                                         ctypes.c_void_p(zd.data_ptr()), B,
                                         ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                         _lib.stream_handle()))
    if is_np:
        return zd.cpu().numpy()
    return zd


def apply_lkr_preconditioner(t: CanonicalTensor, x):
    """y = F* (sum_k u1^k o u2^k o u3^k) . (F x) (lowrank.py:183-192) on the GPU."""
    size = t.n ** t.d
    shape = tuple(getattr(x, "shape", np.shape(x)))
    if shape != (size,) and not (len(shape) == 2 and shape[1] == size):
        raise ValueError(f"expected vector of length {size}, got shape {shape}")
    plan = _tensor_plan(t)
    return _device_apply(plan, x)


_TENSOR_PLANS: dict = {}


def _tensor_plan(t: CanonicalTensor) -> DevicePlan:
    torch = _lib.require_cuda()
    key = (id(t), int(torch.cuda.current_device()))
    hit = _TENSOR_PLANS.get(key)
    if hit is not None and hit[0] is t:
        return hit[1]
    plan = DevicePlan("lkr", t.n, t)
    _TENSOR_PLANS[key] = (t, plan)
    return plan
