"""ctypes binding of the C ABI in include/chk_pcg.h (libchkpcg.so, built in-tree).

This is the same binding a maintainer of the reference would add (see
INTEGRATION.md).  There is no fallback: if the shared library or a CUDA device
is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ConfigurationError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libchkpcg.so")

CHK_OK, CHK_EINVAL, CHK_EUNSUPPORTED, CHK_ECUDA = 0, 1, 2, 3
CHK_CONVERGED, CHK_NOT_CONVERGED, CHK_BREAKDOWN = 0, 1, 2
PRECOND_KIND = {"fourier": 0, "lkr": 1, "regularized": 2}
CONTRAST_KIND = {"fixed": 0, "two_value": 1}


class ChkGrid(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("n", ctypes.c_int32), ("L", ctypes.c_int32),
                ("n0", ctypes.c_int32), ("k", ctypes.c_int32), ("offset", ctypes.c_int32),
                ("lam", ctypes.c_double)]


class ChkPcgOpts(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_iter", ctypes.c_int32),
                ("precond_residual_stopping", ctypes.c_int32)]


_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_dbl = ctypes.c_double
_sz = ctypes.c_size_t
_gp = ctypes.POINTER(ChkGrid)

# name -> (restype, argtypes); the complete exported surface of chk_pcg.h
SIGNATURES = {
    "chk_abi_version": (_i32, []),
    "chk_last_error": (ctypes.c_char_p, []),
    "chk_last_launch_count": (ctypes.c_int64, []),
    "chk_profile_enable": (_i32, [_i32]),
    "chk_profile_read": (_i32, [_vp, _vp]),
    "chk_stencil_apply": (_i32, [_gp, _vp, _vp, _vp, _vp, _i32, _vp]),
    "chk_corrector_rhs": (_i32, [_gp, _vp, _vp, _i32, _i32, _dbl, _vp]),
    "chk_precond_plan_create": (_i32, [_i32, _i32, _i32, _vp, _vp, _dbl, ctypes.POINTER(_vp)]),
    "chk_precond_plan_destroy": (_i32, [_vp]),
    "chk_precond_workspace_bytes": (_sz, [_vp, _i32]),
    "chk_precond_apply": (_i32, [_vp, _vp, _vp, _i32, _vp, _sz, _vp]),
    "chk_pcg_workspace_bytes": (_sz, [_gp, _vp, _i32, _i32]),
    "chk_pcg_solve_batched": (_i32, [_gp, _vp, _vp, _vp, _vp, _i32, ctypes.POINTER(ChkPcgOpts),
                                     _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "chk_pcg_host_workspace_bytes": (_sz, [_gp, _vp, _i32, _i32]),
    "chk_pcg_solve_host": (_i32, [_gp, _vp, _vp, _vp, _vp, _i32, _i32, ctypes.POINTER(ChkPcgOpts),
                                  _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "chk_sample_cells": (_i32, [_gp, _vp, _dbl, _i32, _dbl, _dbl, _vp, _i32, _vp]),
    "chk_pcg_solve_seeds": (_i32, [_gp, _vp, _vp, _dbl, _i32, _dbl, _dbl, _vp, _i32, _vp, _i32, _i32,
                                   ctypes.POINTER(ChkPcgOpts), _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "chk_slab_exchange_elems": (_sz, [_gp, _vp, _i32]),
    "chk_slab_workspace_bytes": (_sz, [_gp, _vp, _vp, _i32, _i32]),
    "chk_slab_phase": (_i32, [_gp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                              _i32, ctypes.POINTER(ChkPcgOpts), _vp, _sz, _vp]),
    "chk_slab_phase_planes": (_i32, [_gp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                     _vp, _vp, _i32, ctypes.POINTER(ChkPcgOpts), _vp, _sz, _vp]),
    "chk_slab_status_async": (_i32, [_gp, _vp, _i32, _i32, _vp, _vp, _vp]),
    "chk_slab_read_state": (_i32, [_gp, _vp, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
}

_lib = None


def load():
    """Load libchkpcg.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("CHK_LIB_PATH", LIB_PATH)  # alternative builds (A/B experiments)
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == CHK_OK:
        return
    msg = load().chk_last_error().decode(errors="replace")
    if rc in (CHK_EINVAL, CHK_EUNSUPPORTED):
        raise ValueError(msg)
    raise RuntimeError(f"CUDA failure in libchkpcg: {msg}")


def grid_struct(d, n, L, n0, k, offset, lam) -> ChkGrid:
    if d != 3:
        raise ConfigurationError("the GPU path implements d = 3 only")
    return ChkGrid(d, n, L, n0, k, offset, float(lam))


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2007_06524_b200 needs a CUDA device (B200, sm_100a); none visible")
    load()
    return torch


def stream_handle():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
