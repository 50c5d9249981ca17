"""Multi-process host logic of the realization sharding (world_size 2, gloo, CPU).

The GPU solve is replaced by the CPU oracle so the test exercises exactly the
partitioning, seed derivation by global index and the ordered gather that the
GPU ranks run.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_06524_b200.sharding import gather_records, shard_range, solve_shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_solve(config, seeds, opts):
    from oracle import checkerhom_oracle as orc

    its, fin, st, nu = [], [], [], []
    fac = orc.lkr_factors(config.n)
    dg = orc.lkr_diagonal(fac)
    k, off = config.k, config.offset
    for s in seeds:
        beta = orc.sample_beta_cells(config.L, config.lam, s)
        F = orc.cell_field(beta, config.n0, k, off)
        f = orc.pcg_rhs_corrector(F, 1)
        A = orc.StencilMatrix(F, config.lam)
        u, rep = orc.pcg_solve(A.__matmul__, f, lambda x: orc.apply_lkr(fac, x, dg), tol=opts.tol)
        its.append(rep.iterations)
        fin.append(rep.final_residual)
        st.append(0 if rep.converged else 1)
        nu.append(float(np.linalg.norm(u)))
    return its, fin, st, nu


def _worker(rank, world, port, total, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2007_06524_b200 as chk

    cfg = chk.LatticeConfig(d=3, L=2, n0=4, alpha="1/2", lam=0.1)
    opts = chk.SolveOptions(tol=1e-8, preconditioner="lkr")
    local = solve_shard(cfg, total, 0, opts, rank, world, solve_fn=_oracle_solve)
    merged = gather_records(local, world)
    if rank == 0:
        q.put([(r.index, r.iterations, r.final_residual, r.norm_u) for r in merged])
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_covers_exactly():
    for total in (1, 7, 64, 256):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_range(total, r, world)
                seen.extend(range(lo, hi))
            assert seen == list(range(total))


def test_two_rank_gloo_matches_single_process():
    total = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    import paper_2007_06524_b200 as chk

    cfg = chk.LatticeConfig(d=3, L=2, n0=4, alpha="1/2", lam=0.1)
    single = solve_shard(cfg, total, 0, chk.SolveOptions(tol=1e-8, preconditioner="lkr"), 0, 1,
                         solve_fn=_oracle_solve)
    assert [g[0] for g in got] == list(range(total))
    for g, s in zip(got, single):
        assert g[1] == s.iterations
        assert g[2] == s.final_residual and g[3] == s.norm_u
