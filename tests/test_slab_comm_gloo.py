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
    return red, x, first, last


def _worker(rank, P, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    comm = TorchComm()
    red, x, first, last = _data(rank, P)
    comm.allreduce([red])
    out = torch.empty_like(x)
    comm.all_to_all([out], [x])
    lo, hi = torch.empty_like(first), torch.empty_like(first)
    comm.halo([first], [last], [lo], [hi])
    q.put((rank, red, out, lo, hi))
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
        r, red, out, lo, hi = q.get(timeout=120)
        got[r] = (red, out, lo, hi)
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
    for r in range(P):
        assert torch.allclose(got[r][0], reds[r], rtol=1e-15, atol=1e-15)
        assert torch.equal(got[r][1], outs[r])
        assert torch.equal(got[r][2], los[r]) and torch.equal(got[r][3], his[r])
