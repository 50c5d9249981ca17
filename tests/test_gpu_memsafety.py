"""Memory-safety checks of the kernels on the GPU (compute-sanitizer is closed on
this pool: it left GPUs needing a reset).  Every device buffer the C ABI touches
is carved out of a larger allocation whose guard regions hold a sentinel
pattern; after the call the guards must be intact (no out-of-bounds write), the
inputs unchanged, and a workspace pre-filled with NaN garbage must give the
bit-identical result of a zeroed one (no read of memory the kernels did not
write first).  Covers every grid size of the path, the paired n = 128 schedule,
the fused n >= 256 middle passes, the generic kernels of the other sizes, the
stand-alone operators and the host pipeline."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2007_06524_b200 as chk  # noqa: E402
from paper_2007_06524_b200 import solver  # noqa: E402

GUARD = 1 << 16  # elements of each guard region
SENT = -7.77e77


def guarded(shape_or_src, dtype=torch.float64, fill=None):
    """(view, backing): view of the requested shape inside a sentinel-guarded buffer."""
    if isinstance(shape_or_src, torch.Tensor):
        src = shape_or_src
        n = src.numel()
    else:
        src = None
        n = int(np.prod(shape_or_src))
    back = torch.full((n + 2 * GUARD,), SENT if dtype == torch.float64 else 0x5A, dtype=dtype, device="cuda")
    v = back[GUARD:GUARD + n]
    if src is not None:
        v.copy_(src.reshape(-1))
        shape = src.shape
    else:
        shape = shape_or_src
        if fill is not None:
            v.fill_(fill)
    return v.view(shape), back


def guards_ok(back, dtype=torch.float64):
    s = SENT if dtype == torch.float64 else 0x5A
    return bool((back[:GUARD] == s).all()) and bool((back[-GUARD:] == s).all())


class GuardedWorkspace(solver.Workspace):
    def __init__(self, fill_byte):
        super().__init__()
        self.fill_byte = fill_byte
        self.back = None

    def get(self, nbytes, device):
        self.back = torch.full((nbytes + 2 * GUARD,), 0x5A, dtype=torch.uint8, device=device)
        self.buf = self.back[GUARD:GUARD + nbytes]
        self.buf.fill_(self.fill_byte)
        return self.buf


CASES = [(2, 4, 0.1, 3, 1e-8), (4, 4, 0.1, 3, 1e-8), (8, 4, 0.1, 2, 1e-8), (16, 4, 0.1, 4, 1e-8),
         (32, 4, 0.01, 40, 1e-8), (64, 4, 0.1, 2, 1e-10), (32, 16, 0.1, 1, 1e-8),
         (3, 4, 0.1, 3, 1e-8), (5, 8, 0.1, 2, 1e-8), (1, 4, 0.1, 2, 1e-8)]  # generic sizes n = 12, 40, 4


@pytest.mark.parametrize("L,n0,lam,B,tol", CASES, ids=[f"n{L * n0}xB{B}" for L, n0, lam, B, tol in CASES])
def test_solver_guards_and_poisoned_workspace(L, n0, lam, B, tol):
    cfg = chk.LatticeConfig(d=3, L=L, n0=n0, alpha="1/2", lam=lam)
    seeds = [chk.derive_seed(0, m) for m in range(B)]
    beta_src = chk.sample_cells_device(cfg, seeds)
    F_src = chk.corrector_rhs_batched(chk.StiffnessBatch(cfg, beta_src), 1)
    opts = chk.SolveOptions(tol=tol, preconditioner="lkr", max_iter=60)
    P = chk.make_preconditioner(3, cfg.n, opts)
    results = []
    for fill in (0x00, 0xFF):  # zeroed vs NaN-garbage workspace
        beta, bb = guarded(beta_src)
        F, fb = guarded(F_src)
        U, ub = guarded(tuple(F_src.shape))
        ws = GuardedWorkspace(fill)
        res = chk.pcg_solve_batched(chk.StiffnessBatch(cfg, beta), F, opts, P, out=U, workspace=ws)
        torch.cuda.synchronize()
        assert guards_ok(bb) and guards_ok(fb) and guards_ok(ub), "out-of-bounds write next to an argument"
        assert guards_ok(ws.back, torch.uint8), "out-of-bounds write next to the workspace"
        assert torch.equal(beta, beta_src) and torch.equal(F, F_src), "an input was modified"
        assert np.all(res.status == 0)
        results.append((U.clone(), res.iterations.copy(), res.history.copy()))
    assert torch.equal(results[0][0], results[1][0]), "result depends on workspace garbage"
    assert np.array_equal(results[0][1], results[1][1]) and np.array_equal(results[0][2], results[1][2])


@pytest.mark.parametrize("n", [16, 64, 128, 256, 512, 12, 36])
def test_operators_guards(n):
    import ctypes

    from paper_2007_06524_b200 import _lib

    lib = _lib.load()
    B = 1 if n == 512 else 2
    cfg = chk.LatticeConfig(d=3, L=n // 4, n0=4, alpha="1/2", lam=0.1)
    beta_src = chk.sample_cells_device(cfg, [chk.derive_seed(1, m) for m in range(B)])
    gen = torch.Generator(device="cuda").manual_seed(n)
    x_src = torch.randn((B, n ** 3), dtype=torch.float64, device="cuda", generator=gen)
    beta, bb = guarded(beta_src)
    x, xb = guarded(x_src)
    y, yb = guarded((B, n ** 3))
    xy, xyb = guarded((B,))
    A = chk.StiffnessBatch(cfg, beta)
    vp = ctypes.c_void_p
    _lib.check(lib.chk_stencil_apply(ctypes.byref(A.grid), vp(beta.data_ptr()), vp(x.data_ptr()), vp(y.data_ptr()),
                                     vp(xy.data_ptr()), B, _lib.stream_handle()))
    torch.cuda.synchronize()
    assert guards_ok(bb) and guards_ok(xb) and guards_ok(yb) and guards_ok(xyb)
    assert torch.equal(x, x_src)
    ref_y = y.clone()
    P = chk.make_preconditioner(3, n, chk.SolveOptions(preconditioner="lkr"))
    for fill in (0x00, 0xFF):
        z, zb = guarded((B, n ** 3))
        wsb = P.plan.workspace_bytes(B)
        ws, wsg = guarded((wsb,), dtype=torch.uint8)
        ws.fill_(fill)
        _lib.check(lib.chk_precond_apply(P.plan.handle, vp(x.data_ptr()), vp(z.data_ptr()), B, vp(ws.data_ptr()),
                                         wsb, _lib.stream_handle()))
        torch.cuda.synchronize()
        assert guards_ok(zb) and guards_ok(wsg, torch.uint8) and guards_ok(xb)
        assert torch.equal(x, x_src)
        if fill == 0x00:
            z0 = z.clone()
        else:
            assert torch.equal(z, z0), "preconditioner output depends on workspace garbage"
    # the matvec is deterministic too
    _lib.check(lib.chk_stencil_apply(ctypes.byref(A.grid), vp(beta.data_ptr()), vp(x.data_ptr()), vp(y.data_ptr()),
                                     vp(xy.data_ptr()), B, _lib.stream_handle()))
    assert torch.equal(y, ref_y)


def test_seeds_pipeline_guards():
    cfg = chk.LatticeConfig(d=3, L=16, n0=4, alpha="1/2", lam=0.1)
    seeds = [chk.derive_seed(0, m) for m in range(7)]
    opts = chk.SolveOptions(tol=1e-8, preconditioner="lkr")
    outs = []
    for fill in (0x00, 0xFF):
        ws = GuardedWorkspace(fill)
        U = torch.empty((7, cfg.n ** 3), dtype=torch.float64).pin_memory()
        res = chk.pcg_solve_seeds(cfg, seeds, opts, chunk=3, out=U, workspace=ws)
        assert guards_ok(ws.back, torch.uint8)
        assert np.all(res.status == 0)
        outs.append((U.clone(), res.iterations.copy()))
    assert torch.equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
