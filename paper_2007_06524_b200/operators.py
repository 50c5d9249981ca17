"""Device stiffness operator: drop-in for ``StiffnessOperator`` / ``assemble_stiffness``.

The reference materialises a CSR matrix per realization (operators.py:96-131,
278-285) and multiplies with it in the PCG loop (solver.py:150,162).  Here the
operator keeps only the compact per-cell contrast array on the device and
``matrix() @ x`` runs the matrix-free fp64 stencil kernel (chk_stencil_apply),
which equals the reference CSR product (tests/oracles.py:35-82 form).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .lattice import LatticeConfig, Realization


class StiffnessBatch:
    """B realizations sharing one grid shape; ``beta`` is a device tensor (B, L^3)."""

    def __init__(self, config: LatticeConfig, beta_cells):
        torch = _lib.require_cuda()
        if config.d != 3:
            raise ValueError("the GPU path implements d = 3 only")
        self.config = config
        beta = torch.as_tensor(np.asarray(beta_cells, dtype=np.float64)) if not isinstance(
            beta_cells, torch.Tensor) else beta_cells
        self.beta = beta.reshape(-1, config.L ** 3).to(device="cuda", dtype=torch.float64).contiguous()
        self.B = self.beta.shape[0]
        self.grid = _lib.grid_struct(3, config.n, config.L, config.n0, config.k, config.offset,
                                     config.lam)

    @property
    def d(self) -> int:
        return 3

    @property
    def n(self) -> int:
        return self.config.n

    @property
    def shape(self) -> tuple:
        size = self.n ** 3
        return (size, size)

    def matvec(self, x, with_dot: bool = False):
        """y = A x for x of shape (B, n^3) (device).  Returns y or (y, <x, y>)."""
        torch = _lib.require_cuda()
        xd = x.to("cuda", torch.float64).contiguous()
        y = torch.empty_like(xd)
        xy = torch.empty(self.B, dtype=torch.float64, device=xd.device) if with_dot else None
        _lib.check(_lib.load().chk_stencil_apply(
            ctypes.byref(self.grid), ctypes.c_void_p(self.beta.data_ptr()),
            ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(y.data_ptr()),
            ctypes.c_void_p(xy.data_ptr()) if with_dot else None, self.B, _lib.stream_handle()))
        return (y, xy) if with_dot else y


class DeviceStencilMatrix:
    """What ``StiffnessOperator.matrix()`` returns: an object with ``@``."""

    def __init__(self, op: "StiffnessOperator"):
        self._op = op
        self.shape = op.shape

    def __matmul__(self, x):
        return self._op.apply(x)

    dot = __matmul__


class StiffnessOperator:
    """Single-realization operator with the reference's duck type (.d, .n,
    .shape, .lam, .matrix(), .apply())."""

    def __init__(self, r: Realization):
        r = Realization.coerce(r)
        self.realization = r
        self.config = r.config
        self.lam = float(r.config.lam)
        self._batch = StiffnessBatch(r.config, r.beta_cells.reshape(1, -1))

    @property
    def d(self) -> int:
        return self.config.d

    @property
    def n(self) -> int:
        return self.config.n

    @property
    def shape(self) -> tuple:
        size = self.n ** self.d
        return (size, size)

    @property
    def beta(self):
        return self._batch.beta

    def matrix(self) -> DeviceStencilMatrix:
        return DeviceStencilMatrix(self)

    def apply(self, x):
        torch = _lib.require_cuda()
        size = self.n ** self.d
        is_np = not isinstance(x, torch.Tensor)
        xt = torch.as_tensor(np.asarray(x, dtype=np.float64)) if is_np else x
        if tuple(xt.shape) != (size,):
            raise ValueError(f"expected vector of length {size}, got shape {tuple(xt.shape)}")
        y = self._batch.matvec(xt.reshape(1, size)).reshape(size)
        return y.cpu().numpy() if is_np else y


def assemble_stiffness(r: Realization, agglomerate: bool = True) -> StiffnessOperator:
    """Drop-in for operators.py:278-285 (``agglomerate`` is accepted and ignored:
    the matrix-free operator has no Kronecker terms to merge).  ``r`` may be a
    realization built by the reference package itself (same fields)."""
    return StiffnessOperator(r)
