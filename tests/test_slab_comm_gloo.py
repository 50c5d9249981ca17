"""Host-side communication schedule of the slab decomposition over real
processes (world_size 2 and 4, gloo, CPU tensors): TorchComm must give exactly
what LocalComm (the single-process emulation used by the GPU tests) gives."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_06524_b200.slab import LocalComm, TorchComm


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data(r, P):
    g = torch.Generator().manual_seed(100 + r)
    red = torch.randn(3, 4, generator=g, dtype=torch.float64)
    x = torch.randn(P * 6, generator=g, dtype=torch.float64)
    first = torch.randn(3, 5, generator=g, dtype=torch.float64)
    last = torch.randn(3, 5, generator=g, dtype=torch.float64)
    # exchange buffers [P][B][nloc][row] for the plane-chunked all_to_all (B = 1, 2)
    xs = [torch.randn(P * B * 6 * 3, generator=g, dtype=torch.float64) for B in (1, 2)]
    return red, x, first, last, xs


CHUNKS = [(1, 3), (3, 5), (0, 1), (5, 6)]  # slab.plane_chunks order for nloc = 6


def _worker(rank, P, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    comm = TorchComm()
    red, x, first, last, _ = _data(rank, P)
    comm.allreduce([red])
    out = torch.empty_like(x)
    comm.all_to_all([out], [x])
    lo, hi = torch.empty_like(first), torch.empty_like(first)
    comm.halo([first], [last], [lo], [hi])
    red2, x2, first2, last2, xs = _data(rank, P)
    lo2, hi2 = torch.empty_like(first), torch.empty_like(first)
    comm.finish(comm.halo([first2], [last2], [lo2], [hi2], async_op=True))
    assert torch.equal(lo2, lo) and torch.equal(hi2, hi)
    planes = []
    for B, xin in zip((1, 2), xs):
        xo = torch.full_like(xin, float("nan"))
        pend = [comm.all_to_all_planes([xo], [xin], (P, B, 6, -1), p0, p1) for p0, p1 in CHUNKS]
        for pd in pend:
            comm.finish(pd)
        planes.append(xo)
    # numpy copies: tensors through a multiprocessing queue travel as shared-memory handles
    # served by this process, which may exit before the parent has fetched them
    q.put((rank, red.numpy().copy(), out.numpy().copy(), lo.numpy().copy(), hi.numpy().copy(),
           [p.numpy().copy() for p in planes]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("P", [2, 4])
def test_torchcomm_matches_localcomm(P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, q)) for r in range(P)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(P):
        r, red, out, lo, hi, planes = q.get(timeout=120)
        got[r] = (torch.from_numpy(red), torch.from_numpy(out), torch.from_numpy(lo), torch.from_numpy(hi),
                  [torch.from_numpy(p) for p in planes])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    data = [_data(r, P) for r in range(P)]
    comm = LocalComm(P)
    reds = [d[0].clone() for d in data]
    comm.allreduce(reds)
    outs = [torch.empty_like(d[1]) for d in data]
    comm.all_to_all(outs, [d[1] for d in data])
    los = [torch.empty_like(d[2]) for d in data]
    his = [torch.empty_like(d[2]) for d in data]
    comm.halo([d[2] for d in data], [d[3] for d in data], los, his)
    for bi, B in enumerate((1, 2)):
        xins = [d[4][bi] for d in data]
        xouts = [torch.full_like(x, float("nan")) for x in xins]
        for p0, p1 in CHUNKS:
            comm.all_to_all_planes(xouts, xins, (P, B, 6, -1), p0, p1)
        full = [torch.empty_like(x) for x in xins]
        comm.all_to_all(full, xins)  # the chunks together = one whole exchange
        for r in range(P):
            assert torch.equal(got[r][4][bi], xouts[r]) and torch.equal(xouts[r], full[r])
    for r in range(P):
        assert torch.allclose(got[r][0], reds[r], rtol=1e-15, atol=1e-15)
        assert torch.equal(got[r][1], outs[r])
        assert torch.equal(got[r][2], los[r]) and torch.equal(got[r][3], his[r])
