"""Benchmark of the batched fp64 PCG hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one batched PCG solve (LKR preconditioner, eps_rank 1e-8) of a whole
BASELINE configuration batch to the reference stop rule: config 3 by default
(n = 128, 256 realizations, contrast {1,100}, corrector RHS, tol 1e-8).
Inputs (cell contrasts, RHS) are seeded synthetic data with the reference's
generator; 4.3 GB per vector, far above the 126 MB L2, so no L2 flush is needed.

value  = DOF-iterations/s over all ranks (sum n^3 * iterations / max-over-ranks
         device time of K steps).  Realizations/s is reported beside it.
e2e    = the same metric through the reference-facing call with HOST buffers:
         H2D of beta + f from pinned memory, the solve, D2H of u + reports.
Multi-GPU: `--gpus N` starts N ranks itself (or run it under torchrun); the
configured batch is sharded 256/N per GPU by global realization index (strong
scaling, no data-path collective); config 5 runs slab-decomposed.
--impl reference: the reference algorithm on host cores (the CPU oracle port,
oracle/checkerhom_oracle.py -- the reference is pure Python and cannot be
compiled or shipped), process pool over all host threads, bounded sample.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "PCG DOF-iterations/s (fp64) and realizations/s vs HBM roofline, 1/2/4/8 GPU"
UNIT = "DOF-iterations/s"

# (L, n0, lam, batch, tol, rhs) -- BASELINE.json configs (SURVEY §8d mapping)
CONFIG_NAMES = {
    1: "3D L=8 n0=4 (n=32) x1, lam=0.1 (a in {0.1,1}), corrector RHS, tol 1e-8",
    2: "3D L=16 n0=4 (n=64) x64, lam=0.1, corrector RHS, tol 1e-8",
    3: "3D L=32 n0=4 (n=128) x256, lam=0.01 (contrast 100), corrector RHS, tol 1e-8",
    4: "3D L=64 n0=4 (n=256) x16, lam=0.1, Gaussian RHS, tol 1e-10",
    5: "3D L=32 n0=16 (n=512) x1, lam=0.1, corrector RHS, tol 1e-8",
}
CFG = {
    1: dict(L=8, n0=4, lam=0.1, batch=1, tol=1e-8, rhs="corrector"),
    2: dict(L=16, n0=4, lam=0.1, batch=64, tol=1e-8, rhs="corrector"),
    3: dict(L=32, n0=4, lam=0.01, batch=256, tol=1e-8, rhs="corrector"),
    4: dict(L=64, n0=4, lam=0.1, batch=16, tol=1e-10, rhs="gaussian"),
    5: dict(L=32, n0=16, lam=0.1, batch=1, tol=1e-8, rhs="corrector"),
}

# algorithmic HBM bytes per DOF per launch of each kernel class
def kernel_bytes_per_dof(n):
    spec = 8.0 * (n // 2 + 1) / (n // 2)  # half spectrum, complex128, per real DOF
    return {
        "fwd_plane": 8.0 + spec,                  # read p; write Q' (stencil + R2C/x1 FFT of q)
        "mid_column": 4.0 * spec,                 # read Q', R; write R, Z'
        "inv_plane": spec + 32.0,                 # read Z', p, u; write u, p
    }


KERNEL_CLASSES = ["stencil_dot", "fwd_plane", "mid_column", "inv_plane", "plane_pair"]  # index = profiler class
B_ALG = 104.0  # SURVEY §8d algorithmic bytes per DOF-iteration (whole iteration)


def measured_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        sm = []
        smax = None
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                smax = float(s[1])
            except ValueError:
                continue
            for i, nm in enumerate(names):
                if s[2 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def config_dict(cfg_id, world, slab=False):
    """The `config` object of the JSON line -- identical for our arm and the
    reference arm at the same N."""
    c = CFG[cfg_id]
    n = c["n0"] * c["L"]
    d = {"workload": f"config{cfg_id}: {CONFIG_NAMES[cfg_id]}", "n": n, "realizations": c["batch"],
         "preconditioner": "lkr eps_rank=1e-8", "tol": c["tol"],
         "l2": "inputs 8*n^3*B bytes per vector >> 126 MB L2 (no flush needed)"}
    if slab:
        d["parallelism"] = f"slab x{world} (x0 planes; NCCL halo + all_to_all + allreduce)"
    else:
        d["parallelism"] = f"realization sharding x{world} (contiguous global-index blocks, no collective)"
    return d


def launch_ranks(args):
    """`python bench.py --gpus N` without torchrun: start N ranks (one process per
    GPU, 127.0.0.1 rendezvous) running this same command; rank 0 prints the line."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


class Dist:
    """Rank bookkeeping + the few collectives the bench needs (barrier, max/sum of
    a float vector); backend nccl on GPUs, gloo for the CPU dry run."""

    def __init__(self, backend):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = backend
        self.dev = None
        if backend == "nccl":
            torch.cuda.set_device(self.local if self.world > 1 else 0)
            self.dev = torch.device("cuda", torch.cuda.current_device())
        if self.world > 1:
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group("gloo")

    def barrier(self):
        import torch

        if self.world > 1:
            self.dist.barrier()
        if self.backend == "nccl":
            torch.cuda.synchronize()

    def reduce(self, vals, op):
        import torch

        t = torch.tensor(vals, dtype=torch.float64, device=self.dev if self.backend == "nccl" else "cpu")
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return [float(v) for v in t.cpu()]

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def run_dry(args):
    """CPU dry run of the multi-rank harness (gloo): the launcher, the sharding of
    the configured batch by global index, and the max-over-ranks reduction, with
    the GPU solve replaced by a stub that reports a fixed iteration count."""
    from paper_2007_06524_b200.lattice import derive_seed
    from paper_2007_06524_b200.sharding import shard_range

    D = Dist("gloo")
    c = CFG[args.config]
    n = c["n0"] * c["L"]
    lo, hi = shard_range(c["batch"], D.rank, D.world)
    seeds = [derive_seed(0, m) for m in range(lo, hi)]
    D.barrier()
    t0 = time.perf_counter()
    its = 40 * len(seeds) * args.steps  # stub: 40 iterations per realization
    dt = time.perf_counter() - t0 + 1e-3
    D.barrier()
    mx = D.reduce([dt], "max")
    tot = D.reduce([float(its) * n ** 3, float(len(seeds) * args.steps)], "sum")
    per_rank = D.reduce([float(len(seeds)) if r == D.rank else 0.0 for r in range(D.world)], "sum")
    if D.rank == 0:
        print(json.dumps({"metric": METRIC, "value": tot[0] / mx[0], "unit": UNIT, "n_gpus": D.world,
                          "steps": args.steps, "warmup": args.warmup, "scaling": "strong", "dry_run": True,
                          "realizations_per_rank": [int(v) for v in per_rank],
                          "first_seed_index_per_rank": [shard_range(c["batch"], r, D.world)[0]
                                                        for r in range(D.world)],
                          "config": config_dict(args.config, D.world)}), flush=True)
    D.close()


def run_ours(args):
    import torch

    import paper_2007_06524_b200 as chk
    from paper_2007_06524_b200 import _lib
    from paper_2007_06524_b200.sharding import shard_range

    D = Dist("nccl")
    world, rank, dev = D.world, D.rank, D.dev
    cfg_id = args.config
    c = CFG[cfg_id]
    # strong scaling: the configured batch (config 3: 256 realizations) is split
    # into contiguous global-index blocks, 256/N per GPU (sharding.shard_range)
    lo, hi = shard_range(c["batch"], rank, world)
    per_rank = hi - lo
    lat = chk.LatticeConfig(d=3, L=c["L"], n0=c["n0"], alpha="1/2", lam=c["lam"])
    n = lat.n
    nb = n ** 3
    seeds = [chk.derive_seed(0, m) for m in range(lo, hi)]
    beta = chk.sample_cells_device(lat, seeds)  # bit-identical to sample_realization
    A = chk.StiffnessBatch(lat, beta)
    f_gauss = None
    if c["rhs"] == "corrector":
        F = chk.corrector_rhs_batched(A, 1)
    else:
        f_gauss = np.stack([np.random.default_rng(s).standard_normal(nb) for s in seeds])
        f_gauss -= f_gauss.mean(axis=1, keepdims=True)
        F = torch.from_numpy(f_gauss).to(dev)
    opts = chk.SolveOptions(tol=c["tol"], preconditioner="lkr", eps_rank=1e-8)
    P = chk.make_preconditioner(3, n, opts)
    U = torch.empty_like(F)
    ws = chk.solver.Workspace()
    lib = _lib.load()

    def one_step():
        return chk.pcg_solve_batched(A, F, opts, P, out=U, record_history=False, workspace=ws)

    for _ in range(args.warmup):
        res = one_step()
    D.barrier()
    clocks = ClockSampler(dev.index)
    clocks.start()
    lib.chk_profile_enable(1)
    stream = torch.cuda.current_stream()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    dof_its = 0
    launches = 0
    reals = 0
    D.barrier()
    ev0.record(stream)
    for _ in range(args.steps):
        res = one_step()
        dof_its += int(np.sum(res.iterations)) * nb
        launches += res.launches
        reals += per_rank
        assert np.all(res.status == 0), "a realization did not converge"
    ev1.record(stream)
    D.barrier()
    clk = clocks.stop()
    ms = float(ev0.elapsed_time(ev1))
    prof_ms = np.zeros(5, dtype=np.float64)
    prof_n = np.zeros(5, dtype=np.int64)
    lib.chk_profile_read(prof_ms.ctypes.data_as(ctypes.c_void_p), prof_n.ctypes.data_as(ctypes.c_void_p))
    lib.chk_profile_enable(0)

    # --- the two operators stand-alone (north_star: >= 60 % of the HBM roofline
    # for the matvec and the preconditioner apply at n >= 128), same batch ------
    standalone = standalone_ops(lib, A, F, U, P, args.steps, torch)

    # --- e2e: seeds -> host solutions through the public API -----------------
    # pcg_solve_seeds: host SeedSequence hashes -> Philox keys (H2D) -> cells drawn
    # on the device -> corrector load on the device -> solve -> u D2H (pinned),
    # chunked over lanes so copies and convergence tails overlap other chunks
    U_h = torch.empty((per_rank, nb), dtype=torch.float64).pin_memory()
    f_h = torch.from_numpy(f_gauss).pin_memory() if f_gauss is not None else None
    ws_h = chk.solver.Workspace()
    del U
    ws.buf = None
    torch.cuda.empty_cache()
    e2e_ms = []
    for step in range(args.warmup + args.steps):
        D.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        step_seeds = chk.derive_seeds(0, range(lo, hi))  # the host work of the step (SeedSequence hashes)
        res_e = chk.pcg_solve_seeds(lat, step_seeds, opts, P, rhs=f_h if f_h is not None else 1, out=U_h,
                                    record_history=False, workspace=ws_h, chunk=args.e2e_chunk or None)
        t1.record(stream)
        D.barrier()
        if step >= args.warmup:
            e2e_ms.append(float(t0.elapsed_time(t1)))
    assert np.array_equal(res_e.iterations, res.iterations), "e2e iterations differ from the device-resident solve"
    e2e_dof_its = int(np.sum(res_e.iterations)) * nb  # identical inputs every step
    h2d = per_rank * 16 + (f_h.numel() * 8 if f_h is not None else 0)
    d2h = U_h.numel() * 8 + per_rank * (4 + 8 + 4 + 4)

    # --- max over ranks -------------------------------------------------------
    ms_max, e2e_max = D.reduce([ms, float(np.mean(e2e_ms))], "max")
    dof_total, reals_total, launches_total, e2e_dof_total, h2d_tot, d2h_tot = D.reduce(
        [float(dof_its), float(reals), float(launches), float(e2e_dof_its), float(h2d), float(d2h)], "sum")

    if rank == 0:
        peak, peak_kind = measured_peaks()
        value = dof_total / (ms_max / 1e3)
        per_kernel = {}
        kb = kernel_bytes_per_dof(n)
        dof_it_rank = dof_its  # rank 0's own work, for the live kernel figures
        if prof_n[4] > 0:
            # paired solve: every realization-iteration runs one forward and one inverse
            # plane pass, nearly all of them inside pair_plane launches (the first forward
            # and the last inverse pass of a half run alone): account the three classes
            # together as one kernel doing fwd + inv bytes per DOF-iteration
            kb["plane_pair"] = kb["fwd_plane"] + kb["inv_plane"]
            prof_ms[4] += prof_ms[1] + prof_ms[3]
            prof_n[4] += prof_n[1] + prof_n[3]
            prof_ms[1] = prof_ms[3] = 0.0
            prof_n[1] = prof_n[3] = 0
        for i, name in enumerate(KERNEL_CLASSES):
            if name not in kb or prof_n[i] == 0 or prof_ms[i] <= 0:
                continue
            achieved = kb[name] * dof_it_rank / (prof_ms[i] / 1e3) / 1e9
            per_kernel[name] = {"ms_total": round(prof_ms[i], 3), "launches": int(prof_n[i]),
                                "avg_us": round(1e3 * prof_ms[i] / prof_n[i], 2),
                                "alg_bytes_per_dof": round(kb[name], 3),
                                "achieved_gbs": round(achieved, 1),
                                "frac": round(achieved / peak, 3),
                                "share": round(prof_ms[i] / max(1e-9, prof_ms.sum()), 3)}
        dom = max(per_kernel, key=lambda k: per_kernel[k]["ms_total"]) if per_kernel else None
        traffic = None
        prof_json = os.path.join(REPO, "profiles", "ncu_traffic.json")
        if dom and os.path.exists(prof_json):
            # ncu --set full dram__bytes_read+write of the same kernel (profiles/), per DOF,
            # scaled to the DOF one launch processes on average in this run
            ncu_name = {"fwd_plane": "fwd_plane_kernel",
                        "mid_column": ("mid_column_reg_kernel" if n <= 128 else
                                       "mid_column_r256_kernel" if n == 256 else "mid_column_fused_kernel"),
                        "inv_plane": "inv_plane_kernel", "plane_pair": "pair_plane_kernel"}.get(dom)
            tj = json.load(open(prof_json)).get(f"config{cfg_id}", {}).get(ncu_name)
            if tj:
                per_launch_dof = dof_it_rank / max(1, per_kernel[dom]["launches"])
                traffic = {"bytes_per_launch": round(tj["dram_bytes_per_dof"] * per_launch_dof),
                           "bytes_per_dof": tj["dram_bytes_per_dof"], "source": tj["source"]}
        roofline = None
        if dom:
            d = per_kernel[dom]
            roofline = {"bound": "hbm", "kernel": dom, "achieved": d["achieved_gbs"], "peak": peak,
                        "peak_kind": peak_kind, "unit": "GB/s", "frac": d["frac"],
                        "traffic": traffic,
                        "alg_bytes_per_dof": d["alg_bytes_per_dof"],
                        "iteration_frac_104B": round(value / world * B_ALG / 1e9 / peak, 3)}
        cpu = cpu_baseline(cfg_id) if (world == 1 and not args.no_cpu_baseline) else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference seeded generator: derive_seed(0,m), Philox cells, corrector/Gaussian RHS)",
            "config": config_dict(cfg_id, world),
            "realizations_per_gpu": per_rank,
            "realizations_per_s": reals_total / (ms_max / 1e3),
            "dof_iterations": dof_total,
            "roofline": roofline,
            "kernels": per_kernel,
            "e2e": {"value": e2e_dof_total / (e2e_max / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d_tot), "d2h_bytes_per_step": int(d2h_tot),
                    "ms_per_step": e2e_max,
                    "realizations_per_s": c["batch"] / (e2e_max / 1e3),
                    "path": ("pcg_solve_seeds: seeds -> SeedSequence keys (host) -> Philox cells + corrector "
                             "load on the device -> solve -> u to pinned host memory"
                             if f_h is None else
                             "pcg_solve_seeds with the host Gaussian loads (numpy default_rng, generated "
                             "before the timed region) uploaded per chunk")},
            "standalone": standalone,
            "gpu_launches": int(launches_total),
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    D.close()


def standalone_ops(lib, A, F, Y, P, reps, torch):
    """Event-timed chk_stencil_apply (y = A x with <x, y>; reads x, writes y, plus
    the L^3 cells: 16 + 8 L^3/n^3 B/DOF) and chk_precond_apply (z = P r through
    the forward plane, middle and inverse passes: 8 + 4 x 8.1 + 8 = 48.5 B/DOF)
    over the whole batch, on the current stream, after one warm-up launch."""
    B, nb = F.shape
    n = round(nb ** (1.0 / 3.0))
    peak, _ = measured_peaks()
    stream = torch.cuda.current_stream()
    vp = ctypes.c_void_p
    xy = torch.empty(B, dtype=torch.float64, device=F.device)
    wsb = int(lib.chk_precond_workspace_bytes(P.plan.handle, B))
    ws = torch.empty(wsb, dtype=torch.uint8, device=F.device)
    spec = 8.0 * (n // 2 + 1) / (n // 2)
    cells = 8.0 * A.beta.shape[1] / nb
    ops = {
        "stencil_apply": (16.0 + cells, lambda: lib.chk_stencil_apply(
            ctypes.byref(A.grid), vp(A.beta.data_ptr()), vp(F.data_ptr()), vp(Y.data_ptr()),
            vp(xy.data_ptr()), B, vp(stream.cuda_stream))),
        "precond_apply": (16.0 + 4.0 * spec, lambda: lib.chk_precond_apply(
            P.plan.handle, vp(F.data_ptr()), vp(Y.data_ptr()), B, vp(ws.data_ptr()), wsb,
            vp(stream.cuda_stream))),
    }
    out = {}
    for name, (bpd, call) in ops.items():
        assert call() == 0, name
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(reps):
            assert call() == 0, name
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = bpd * B * nb / (ms / 1e3) / 1e9
        out[name] = {"ms_per_launch": round(ms, 3), "alg_bytes_per_dof": round(bpd, 3),
                     "achieved_gbs": round(gbs, 1), "peak_gbs": peak, "frac": round(gbs / peak, 3),
                     "dof_per_launch": int(B * nb)}
    del ws
    return out


# ---------------------------------------------------------------------------
# CPU side: the reference algorithm (oracle port) on host cores
# ---------------------------------------------------------------------------


def _cpu_solve(cfg_id, m):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from threadpoolctl import threadpool_limits

    from oracle import checkerhom_oracle as orc

    with threadpool_limits(1):
        t0 = time.perf_counter()
        beta, F, f = orc.config_problem(cfg_id, m)
        fac = _cpu_solve.fac.get(cfg_id) if hasattr(_cpu_solve, "fac") else None
        if fac is None:
            fac = orc.lkr_factors(F.shape[0])
            _cpu_solve.fac = getattr(_cpu_solve, "fac", {})
            _cpu_solve.fac[cfg_id] = fac
        dg = orc.lkr_diagonal(fac)
        A = orc.StencilMatrix(F, CFG[cfg_id]["lam"])
        t1 = time.perf_counter()
        u, rep = orc.pcg_solve(A.__matmul__, f, lambda x: orc.apply_lkr(fac, x, dg), tol=CFG[cfg_id]["tol"])
        t2 = time.perf_counter()
    return rep.iterations, F.shape[0] ** 3, t2 - t1, t1 - t0


def cpu_baseline(cfg_id):
    """Single-core oracle solve of realization 0 of the workload (bounded sample)."""
    its, nb, t_solve, t_setup = _cpu_solve(cfg_id, 0)
    return {"value": its * nb / t_solve, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"config{cfg_id} realization m=0: full PCG solve ({its} iterations) with the "
                      f"numpy oracle (oracle/checkerhom_oracle.py), 1 thread, {t_solve:.1f} s"}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from concurrent.futures import ProcessPoolExecutor

    cfg_id = args.config
    c = CFG[cfg_id]
    n = c["n0"] * c["L"]
    per_worker_gb = 0.5 * (n / 128) ** 3 + 0.2
    try:
        import psutil

        mem_gb = psutil.virtual_memory().available / 2 ** 30
    except Exception:  # noqa: BLE001
        mem_gb = 64.0
    cores = os.cpu_count() or 1
    workers = max(1, min(cores, c["batch"], int(mem_gb * 0.6 / per_worker_gb)))
    rates = []
    m_next = 0
    with ProcessPoolExecutor(max_workers=workers) as pool:
        for step in range(args.warmup + args.steps):
            ms = list(range(m_next, m_next + workers))
            m_next += workers
            t0 = time.perf_counter()
            out = list(pool.map(_cpu_solve, [cfg_id] * workers, [m % c["batch"] for m in ms]))
            dt = time.perf_counter() - t0
            if step >= args.warmup:
                rates.append(sum(o[0] * o[1] for o in out) / dt)
    value = float(np.mean(rates))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "impl": "reference", "data": "synthetic (same generator as our arm)",
            "config": config_dict(cfg_id, world, slab=cfg_id == 5 and world > 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                             "sample": f"per step {workers} realizations of config{cfg_id} solved to the "
                                       f"reference stop rule, one per process (pattern of "
                                       f"homogenize.py:149-161), 1 BLAS thread each"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_slab(args):
    """Config 5 on N > 1 GPUs: one n = 512 grid slab-decomposed over the ranks
    (strong scaling; NCCL halo exchange, all_to_all transposes, allreduces)."""
    import torch
    import torch.distributed as dist

    import paper_2007_06524_b200 as chk
    from paper_2007_06524_b200 import slab

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world == 1 and "MASTER_ADDR" not in os.environ:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29517", RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    c = CFG[args.config]
    lat = chk.LatticeConfig(d=3, L=c["L"], n0=c["n0"], alpha="1/2", lam=c["lam"])
    n, nloc = lat.n, lat.n // world
    beta = np.stack([chk.sample_realization(lat, chk.derive_seed(0, m)).beta_cells.ravel()
                     for m in range(c["batch"])])
    A = chk.StiffnessBatch(lat, beta)
    F = chk.corrector_rhs_batched(A, 1)  # full field on every rank, local planes kept
    Floc = F.reshape(c["batch"], n, n * n)[:, rank * nloc:(rank + 1) * nloc].contiguous()
    del F, A
    opts = chk.SolveOptions(tol=c["tol"], preconditioner="lkr", eps_rank=1e-8)
    R = slab.SlabRank(lat, beta, Floc, world, rank, opts, device=dev)
    comm = slab.TorchComm()

    def step():
        return slab.slab_solve([R], comm, chunks=args.slab_chunks)

    for _ in range(args.warmup):
        res = step()
    dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev.index)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dof_its = 0
    for _ in range(args.steps):
        res = step()
        dof_its += int(np.sum(res.iterations)) * n ** 3
    e1.record()
    dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    # e2e: host buffers of this rank's planes in, u out
    f_h = Floc.cpu().pin_memory()
    u_h = torch.empty_like(f_h).pin_memory()
    e2e = []
    for k in range(args.warmup + args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        R.f.copy_(f_h.reshape(R.f.shape), non_blocking=True)
        res = step()
        u_h.copy_(res.u[0].reshape(u_h.shape), non_blocking=True)
        t1.record()
        torch.cuda.synchronize()
        if k >= args.warmup:
            e2e.append(t0.elapsed_time(t1))
    e2e_ms = torch.tensor([float(np.mean(e2e))], dtype=torch.float64, device=dev)
    dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        peak, peak_kind = measured_peaks()
        value = dof_its / (float(ms) / 1e3)
        per_step = int(np.sum(res.iterations)) * n ** 3
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(ms) / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference seeded generator)",
            "config": config_dict(args.config, world, slab=True),
            "realizations_per_s": c["batch"] * args.steps / (float(ms) / 1e3),
            "roofline": {"bound": "hbm", "kernel": "whole iteration", "unit": "GB/s", "peak": peak * world,
                         "peak_kind": peak_kind, "achieved": round(value * B_ALG / 1e9, 1),
                         "frac": round(value * B_ALG / 1e9 / (peak * world), 3), "traffic": None},
            "e2e": {"value": per_step / (float(e2e_ms) / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": int(f_h.numel() * 8) * world,
                    "d2h_bytes_per_step": int(u_h.numel() * 8) * world, "ms_per_step": float(e2e_ms)},
            "gpu_launches": None, "clocks": clk, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3, choices=sorted(CFG))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-chunk", type=int, default=0,
                    help="realizations per pipelined chunk of the host-buffer solve (default B/4)")
    ap.add_argument("--slab", action="store_true",
                    help="force the slab-decomposed path (default for config 5 when N > 1)")
    ap.add_argument("--slab-chunks", type=int, default=4,
                    help="plane chunks of the slab phases (exchange overlapped with the next chunk)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU (gloo) run of the multi-rank harness with a stub solve (tests)")
    args = ap.parse_args()
    if os.environ.get("CHK_DEBUG_FLAGS"):
        sys.exit("bench.py: CHK_DEBUG_FLAGS is set; refusing to time a run")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.slab or (args.config == 5 and int(os.environ.get("WORLD_SIZE", "1")) > 1):
        run_slab(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
