"""Benchmark of the mpkrylov hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg4|cfg1|cfg2|cfg3|cfg5] [--precond ...]

Workload (default): BASELINE.json configs[3] = cfg4, the largest single-GPU
configuration: the 2048 x 2048 9-point convection-diffusion system
(n = 4,194,304, nnz = 37,724,164), b = A*1, double-double BiCGSTAB with
binary64 ILU(0) ("ilu0-mixed"), 200 fixed iterations.  One step = one
time-to-solve as the reference counts it (solvers.py:426-445): the ILU(0)
factorization plus the 200 iterations.  metric = iterations per second.

  value : matrix and b resident in HBM (mpk_solve_dev), device-timed with
          CUDA events on the library stream, max over ranks.
  e2e   : the C-ABI call a user makes (mpk_solve with pinned host b/x, new
          matrix values copied in first) -- host<->device copies inside.
  cold_time_to_solve_s : one cold solve through the C ABI on a matrix never
          seen before (upload + level analysis + sweep-plan build/autotune +
          factorization + 200 iterations + copies), host wall clock.
  roofline : the dominant kernel (the ILU(0)-mixed apply = forward + backward
          sweep) -- algorithmic bytes / event-timed duration against the
          measured HBM peak, plus its critical-path bound; roofline_spmv: the
          mixed SpMV kernel (HBM fraction, FP64-pipe share from ncu).
  cpu_baseline : the C restatement of the reference (oracle/, "port") on
          this host's cores on a bounded sample (cfg4: the factorization plus
          3 iterations, extrapolated to the 200-iteration time-to-solve).

Multi-GPU: one process per GPU.  `--gpus N` without torchrun re-launches
itself under torch.distributed.run.  cfg4 at N > 1: ONE system row-block
sharded (SpMV / vector rows split, ILU(0) sweeps replicated -- the
triangular solve does not shard without changing the preconditioner;
NCCL all-gathers), "scaling": "strong".  cfg5: the 64 independent systems
split 64/N per GPU ("strong"; --cfg5-weak: 8 per GPU).  cfg1-3: replicas.
--impl reference: the reference's algorithm on the host cores (C port in
oracle/; the Python reference cannot travel to the box), rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import pathlib
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "precond. Krylov iters/s & time-to-solve (DD/TD/QD); % of HBM/FP64 roofline"
UNIT = "iterations/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"
TRAFFIC = ROOT / "profiles" / "r02_traffic.json"
PRECOND_CODE = {"none": 0, "ilu0-mixed": 1, "ilu0": 2}
LAB = {"dd": 2, "td": 3, "qd": 4}
# Critical-path model of the shuffle-wavefront sweep (csrc/swf.cu), cycles
# per DAG level on the dependency chain through one row: forward = shuffle
# hand-off + dmul + 2 dependent dsub + select; backward = shuffle + dmul + 3
# dsub + the Markstein division (dmul + 2 fma) + select.  Primitive
# latencies measured on B200 (tools/ubench/wfprim.cu, profiles/r02_*):
# DADD/DMUL/DFMA 8 cycles dependent, SHFL ~24, FSEL ~6.
CP_FWD_CYCLES = 24 + 8 + 2 * 8 + 6
CP_BWD_CYCLES = 24 + 8 + 3 * 8 + 3 * 8 + 6


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ---------------------------------------------------------------------
# workload description
# ---------------------------------------------------------------------
def cfg5_systems(rank: int, world: int, weak: bool):
    per = 8 if weak else max(1, 64 // world)
    return list(range(rank * per, rank * per + per))


def cells_for(config: str, rank: int, world: int, weak: bool = False):
    """[(problem, method, k)] solved by this rank in one step."""
    from paper_2504_14498_b200 import problems

    if config == "cfg5":
        out = []
        for s in cfg5_systems(rank, world, weak):
            p = problems.cfg5(s)
            for m in p.methods:
                out.append((p, m, 4))
        return out
    p = problems.CONFIGS[config]()
    return [(p, m, LAB[pr]) for pr in p.precisions for m in p.methods]


def apply_bytes(n, nnz, c):
    """ILU(0) apply = nnz(8c+4) + 4(n+1) + 4n + 4F."""
    return nnz * (8 * c + 4) + 4 * (n + 1) + 4 * n + 4 * 8 * c * n


def spmv_bytes(n, nnz, c, k):
    """SpMV = nnz(8c+4) + 4(n+1) + X + V, X = F (M^-1 output)."""
    return nnz * (8 * c + 4) + 4 * (n + 1) + 8 * c * n + 8 * c * k * n


def config_dict(args, world):
    d = {"workload": args.config}
    if args.config == "cfg4":
        d.update({"system": "2D convection-diffusion, 9-point, 2048x2048 (n=4194304, "
                            "nnz=37724164), Pe=5, b=A*1",
                  "cells": "bicgstab x dd, 200 fixed iterations", "precond": args.precond,
                  "step": "one time-to-solve: ILU(0) factorization + 200 iterations",
                  "l2_policy": "per-kernel working sets 570-620 MB > 126 MB L2 "
                               "(no flush needed); iterations chained"})
        if world > 1:
            d["parallelism"] = (f"one system, rows sharded over {world} GPUs; ILU(0) sweeps "
                                "replicated; NCCL all-gathers")
    elif args.config == "cfg5":
        per = 8 if args.cfg5_weak else 64 // world
        d.update({"system": f"{per * world} random nonsymmetric n=50000 systems, {per} per GPU",
                  "cells": "cgs,bicgstab x qd", "tol": 1e-40, "precond": args.precond,
                  "l2_policy": "8 systems x 100 MB working set per GPU; cells concurrent"})
    elif args.config == "cfg2":
        d.update({"system": "random nonsymmetric n=20000, 12 off-diag/row, seed 2",
                  "cells": "bicg,cgs,bicgstab,gpbicg x td,qd", "tol": 1e-30,
                  "precond": args.precond,
                  "l2_policy": "inputs L2-resident (4 MB per kernel); iterations chained"})
    elif args.config == "cfg3":
        d.update({"system": "complex shifted 7-point Laplacian 48^3, b=U(-1,1)+iU(-1,1)",
                  "cells": "gpbicg,bicgstab x complex dd", "tol": 1e-24,
                  "precond": args.precond,
                  "l2_policy": "working set ~150 MB per iteration, partly L2-resident"})
    else:
        d.update({"system": "2D upwind convection-diffusion 5-point 64x64, Pe=10",
                  "cells": "bicgstab x dd", "tol": 1e-20, "precond": args.precond,
                  "l2_policy": "inputs L2-resident (0.4 MB); iterations chained"})
    return d


# ---------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------
class Cell:
    """One (system, method, precision) solve: the matrix uploaded twice (a
    device-resident copy for `value` and one whose values are re-sent every
    e2e step), b formed on the device in working precision (b = A x_true),
    pinned host b / x for the e2e call."""

    def __init__(self, L, _lib, p, method, k, ctx_dev):
        import torch

        self.p, self.method, self.k = p, method, k
        self.L, self._lib = L, _lib
        self.cx = p.val_im is not None
        rp = _lib.i64(p.row_ptr)
        ci = _lib.i64(p.col_idx)
        vre = _lib.f64(p.val_re)
        vim = None if p.val_im is None else _lib.f64(p.val_im)
        vre_p = torch.empty(len(vre), dtype=torch.float64, pin_memory=True).numpy()
        vre_p[:] = vre
        vim_p = None
        if vim is not None:
            vim_p = torch.empty(len(vim), dtype=torch.float64, pin_memory=True).numpy()
            vim_p[:] = vim
        self.host_csr = (rp, ci, vre_p, vim_p)
        self.m_e2e = self._upload(ctx_dev, rp, ci, vre, vim)
        self.m = self._upload(ctx_dev, rp, ci, vre, vim)
        self.ctx = ctx_dev
        n = p.n
        if p.b64 is not None:
            b_re = np.zeros((n, k))
            b_re[:, 0] = np.real(p.b64)
            b_im = None
            if self.cx:
                b_im = np.zeros((n, k))
                b_im[:, 0] = np.imag(p.b64)
        else:
            xr = np.zeros((n, k))
            xr[:, 0] = np.real(p.x_true)
            xi = None
            if self.cx:
                xi = np.zeros((n, k))
                xi[:, 0] = np.imag(p.x_true)
            b_re = np.zeros((n, k))
            b_im = np.zeros((n, k)) if self.cx else None
            _lib.check(L.mpk_spmv_mixed(self.m, ctypes.c_int(k), _lib.dptr(xr), _lib.dptr(xi),
                                        _lib.dptr(b_re), _lib.dptr(b_im), ctypes.c_int(0)),
                       "spmv")
        self.b_re = torch.empty((n, k), dtype=torch.float64, pin_memory=True).numpy()
        self.b_re[:] = b_re
        self.b_im = None
        if self.cx:
            self.b_im = torch.empty((n, k), dtype=torch.float64, pin_memory=True).numpy()
            self.b_im[:] = b_im
        self.x_re = torch.empty((n, k), dtype=torch.float64, pin_memory=True).numpy()
        self.x_im = (torch.empty((n, k), dtype=torch.float64, pin_memory=True).numpy()
                     if self.cx else None)
        ld = int(L.mpk_plane_ld(ctypes.c_int64(n)))
        planes = k * (2 if self.cx else 1)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.d_b = torch.zeros(planes * ld + 4, dtype=torch.float64, device=dev)
        self.d_x = torch.zeros(planes * ld + 4, dtype=torch.float64, device=dev)
        self.max_iter = p.max_iter if p.max_iter is not None else 3 * n
        self.hist_cap = 2 * self.max_iter + 2
        self.d_h = torch.zeros(self.hist_cap * k + 4, dtype=torch.float64, device=dev)
        torch.cuda.synchronize()
        _lib.check(L.mpk_to_planar(ctx_dev, ctypes.c_int64(n), ctypes.c_int(k),
                                   _lib.dptr(self.b_re), _lib.dptr(self.b_im),
                                   ctypes.c_void_p(self.d_b.data_ptr())), "to_planar")

    def _upload(self, ctx, rp, ci, vre, vim):
        L, _lib, p = self.L, self._lib, self.p
        h = ctypes.c_void_p()
        _lib.check(L.mpk_csr_upload(ctx, ctypes.c_int64(p.n), ctypes.c_int64(p.nnz),
                                    _lib.dptr(rp), _lib.dptr(ci), _lib.dptr(vre),
                                    _lib.dptr(vim), ctypes.byref(h)), "upload")
        return h

    def h2d_bytes(self):
        c = 2 if self.cx else 1
        return 8 * c * self.p.nnz + 8 * c * self.k * self.p.n

    def d2h_bytes(self):
        c = 2 if self.cx else 1
        return 8 * c * self.k * self.p.n + 8 * 16


def cold_solve(L, _lib, ctx, p, method, k):
    """One cold time-to-solve through the C ABI: a fresh upload (level
    analysis, sweep plans and their autotuning), factorization, the solve,
    host b in / x out.  Host wall clock, synchronised."""
    n = p.n
    rp, ci, vre = _lib.i64(p.row_ptr), _lib.i64(p.col_idx), _lib.f64(p.val_re)
    vim = None if p.val_im is None else _lib.f64(p.val_im)
    cx = vim is not None
    x = np.zeros((n, k))
    x[:, 0] = 1.0 if p.x_true is None else np.real(p.x_true)
    b = np.zeros((n, k))
    bi = np.zeros((n, k)) if cx else None
    xo, xoi = np.zeros((n, k)), (np.zeros((n, k)) if cx else None)
    t0 = time.perf_counter()
    h = ctypes.c_void_p()
    _lib.check(L.mpk_csr_upload(ctx, ctypes.c_int64(n), ctypes.c_int64(p.nnz), _lib.dptr(rp),
                                _lib.dptr(ci), _lib.dptr(vre), _lib.dptr(vim),
                                ctypes.byref(h)), "upload")
    L.mpk_ctx_synchronize(ctx)
    t1 = time.perf_counter()
    # b = A x_true in working precision on the device (untimed below)
    _lib.check(L.mpk_spmv_mixed(h, ctypes.c_int(k), _lib.dptr(x), None, _lib.dptr(b),
                                _lib.dptr(bi), ctypes.c_int(0)), "spmv")
    t2 = time.perf_counter()
    rep = _lib.MpkReport()
    max_iter = p.max_iter if p.max_iter is not None else 3 * n
    _lib.check(L.mpk_solve(h, ctypes.c_int(_lib.METHOD_CODE[method]), ctypes.c_int(k),
                           ctypes.c_double(p.eps_rel), ctypes.c_double(p.eps_abs),
                           ctypes.c_int64(max_iter), _lib.dptr(b), _lib.dptr(bi),
                           _lib.dptr(xo), _lib.dptr(xoi), None, ctypes.c_int64(0),
                           ctypes.byref(rep)), "solve")
    t3 = time.perf_counter()
    L.mpk_csr_free(h)
    return {"total_s": (t1 - t0) + (t3 - t2), "upload_analysis_plans_s": t1 - t0,
            "factor_s": rep.factor_ms / 1e3, "solve_s": (t3 - t2) - rep.factor_ms / 1e3,
            "iterations": int(rep.iterations)}


def run_ours(args, rank, world, local_rank):
    import torch

    torch.cuda.set_device(local_rank)
    from paper_2504_14498_b200 import _lib

    L = _lib.lib()
    L.mpk_ctx_stream.restype = ctypes.c_void_p
    ctx = _lib.context(local_rank)
    stream = torch.cuda.ExternalStream(L.mpk_ctx_stream(ctx), device=local_rank)
    pre = PRECOND_CODE[args.precond]

    # one context (= CUDA stream) per cell when cells run concurrently, like
    # the reference harness's thread pool over cells (bench.py:211-215)
    def new_ctx():
        h = ctypes.c_void_p()
        _lib.check(L.mpk_ctx_create(ctypes.c_int(local_rank), ctypes.byref(h)), "ctx")
        _lib.check(L.mpk_ctx_set_option(h, ctypes.c_int(_lib.MPK_OPT_PRECOND),
                                        ctypes.c_int64(pre)), "precond")
        return h

    triples = cells_for(args.config, rank, world, args.cfg5_weak)
    concurrent = args.concurrent and len(triples) > 1
    if not concurrent:
        _lib.check(L.mpk_ctx_set_option(ctx, ctypes.c_int(_lib.MPK_OPT_PRECOND),
                                        ctypes.c_int64(pre)), "precond")
    cells = [Cell(L, _lib, p, m, k, new_ctx() if concurrent else ctx) for (p, m, k) in triples]
    dist = world > 1
    if dist:
        import torch.distributed as tdist

    def barrier():
        torch.cuda.synchronize()
        if dist:
            tdist.barrier()

    def make_jobs(dev: bool):
        J = (_lib.MpkJob * len(cells))()
        for j, c in enumerate(cells):
            J[j].m = c.m if dev else c.m_e2e
            J[j].method = _lib.METHOD_CODE[c.method]
            J[j].k = c.k
            J[j].eps_rel = c.p.eps_rel
            J[j].eps_abs = c.p.eps_abs
            J[j].max_iter = c.max_iter
            if dev:
                J[j].b_re = c.d_b.data_ptr()
                J[j].x_re = c.d_x.data_ptr()
                J[j].hist = c.d_h.data_ptr()
                J[j].hist_cap = c.hist_cap
            else:
                J[j].b_re = c.b_re.ctypes.data
                J[j].b_im = c.b_im.ctypes.data if c.b_im is not None else None
                J[j].x_re = c.x_re.ctypes.data
                J[j].x_im = c.x_im.ctypes.data if c.x_im is not None else None
                J[j].val_re = c.host_csr[2].ctypes.data
                J[j].val_im = (c.host_csr[3].ctypes.data
                               if c.host_csr[3] is not None else None)
        return J

    jobs_dev, jobs_e2e = make_jobs(True), make_jobs(False)

    def run_jobs(J, dev: bool):
        if concurrent:
            _lib.check(L.mpk_run_jobs(J, ctypes.c_int(len(cells)), ctypes.c_int(1 if dev else 0)),
                       "mpk_run_jobs")
        else:
            for j in range(len(cells)):
                _lib.check(L.mpk_run_jobs(ctypes.byref(J[j]), ctypes.c_int(1),
                                          ctypes.c_int(1 if dev else 0)), "job")
        return [J[j].rep for j in range(len(cells))]

    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    iters = launches = 0
    factor_ms = []
    with Clocks(local_rank) as clk:
        for _ in range(args.warmup):
            run_jobs(jobs_dev, True)
        barrier()
        clk.samples.clear()
        e0.record(stream)
        for _ in range(args.steps):
            reps = run_jobs(jobs_dev, True)
            iters += sum(r.iterations for r in reps)
            launches += sum(r.launches for r in reps)
            factor_ms.append(max(r.factor_ms for r in reps))
        torch.cuda.synchronize()
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    # e2e through the C ABI with host buffers
    for _ in range(max(1, args.warmup // 2)):
        run_jobs(jobs_e2e, False)
    barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2e_iters = 0
    h2d = d2h = 0
    e2.record(stream)
    for _ in range(args.steps):
        reps = run_jobs(jobs_e2e, False)
        for c, r in zip(cells, reps):
            e2e_iters += r.iterations
            h2d += c.h2d_bytes()
            d2h += c.d2h_bytes()
    torch.cuda.synchronize()
    e3.record(stream)
    barrier()
    e2e_ms = e2.elapsed_time(e3)
    # kernel probes (after the timed regions): the ILU(0)-mixed apply and
    # the mixed SpMV of the first cell's matrix, CUDA events on its stream
    c0 = cells[0]
    probe = {}
    if args.precond == "ilu0-mixed":
        bad, stc = ctypes.c_int64(0), ctypes.c_int32(0)
        _lib.check(L.mpk_ilu0_factor(c0.m, ctypes.byref(bad), ctypes.byref(stc)), "factor")
        avg = ctypes.c_double(0)
        _lib.check(L.mpk_bench_apply(c0.m, ctypes.c_int(c0.k), ctypes.c_int(10),
                                     ctypes.byref(avg)), "bench_apply")
        probe["apply_ms"] = avg.value
        info = (ctypes.c_int64 * 12)()
        _lib.check(L.mpk_sweep_info(c0.m, info, ctypes.c_int(12)), "sweep_info")
        probe["sweep_info"] = list(info)
    avg = ctypes.c_double(0)
    _lib.check(L.mpk_bench_spmv(c0.m, ctypes.c_int(c0.k), ctypes.c_int(10), ctypes.byref(avg)),
               "bench_spmv")
    probe["spmv_ms"] = avg.value
    cold = None
    if rank == 0 and not args.no_cold:
        cold = cold_solve(L, _lib, ctx, c0.p, c0.method, c0.k)
    vals = torch.tensor([ms, e2e_ms, float(iters), float(e2e_iters)], dtype=torch.float64,
                        device="cuda")
    if dist:
        mx = vals.clone()
        tdist.all_reduce(mx[:2], op=tdist.ReduceOp.MAX)
        tot = vals.clone()
        tdist.all_reduce(tot[2:], op=tdist.ReduceOp.SUM)
        ms, e2e_ms = float(mx[0]), float(mx[1])
        iters, e2e_iters = float(tot[2]), float(tot[3])
    return {"ms": ms, "e2e_ms": e2e_ms, "iters": iters, "e2e_iters": e2e_iters,
            "launches": launches, "h2d": h2d // max(1, args.steps),
            "d2h": d2h // max(1, args.steps), "clocks": clk.summary(), "probe": probe,
            "p": c0.p, "k": c0.k, "cold": cold,
            "factor_ms": statistics.median(factor_ms) if factor_ms else None}


def run_sharded(args, rank, world, local_rank):
    """cfg4 over N GPUs: ONE system, row-block sharded BiCGSTAB (csrc/shard.cuh;
    SpMV / vector rows split, ILU(0) sweeps in full on every rank, NCCL
    all-gathers of partials and sweep inputs).  value = that system's
    iterations / device time (max over ranks) -> strong scaling."""
    import torch

    torch.cuda.set_device(local_rank)
    import paper_2504_14498_b200 as mpk
    from paper_2504_14498_b200 import _lib, problems
    from paper_2504_14498_b200.sharded import Communicator, ShardedSolver

    L = _lib.lib()
    dist = world > 1
    if dist:
        import torch.distributed as tdist
        comm = Communicator.nccl(local_rank)
    else:
        comm = Communicator.local(1)[0]
    p = problems.CONFIGS[args.config]()
    P = mpk.Precision.DD
    A = mpk.CsrMatrix.from_binary64(p.n, p.row_ptr, p.col_idx, p.val_re, None, P)
    sv = ShardedSolver(A, P, comm, local_rank)
    k = 2
    xt = mpk.DenseVector.from_float64(np.real(p.x_true), P)
    b = mpk.spmv_mixed(A.demoted(), xt)
    b_pin = torch.empty((p.n, k), dtype=torch.float64, pin_memory=True).numpy()
    b_pin[:] = b.re
    x_pin = torch.empty((p.n, k), dtype=torch.float64, pin_memory=True).numpy()
    sv.load_b(b)
    max_iter = p.max_iter if p.max_iter is not None else 3 * p.n
    stream = torch.cuda.ExternalStream(L.mpk_ctx_stream(sv.ctx), device=local_rank)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            tdist.barrier()

    iters = launches = 0
    with Clocks(local_rank) as clk:
        for _ in range(args.warmup):
            sv.solve_dev(p.eps_rel, p.eps_abs, max_iter)
        barrier()
        clk.samples.clear()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            rep = sv.solve_dev(p.eps_rel, p.eps_abs, max_iter)
            iters += int(rep.iterations)
            launches += int(rep.launches)
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    barrier()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    e2e_iters = 0
    for _ in range(args.steps):
        _lib.check(L.mpk_to_planar(sv.ctx, ctypes.c_int64(p.n), ctypes.c_int(k),
                                   _lib.dptr(b_pin), None,
                                   ctypes.c_void_p(sv.d_b.data_ptr())), "to_planar")
        rep = sv.solve_dev(p.eps_rel, p.eps_abs, max_iter)
        _lib.check(L.mpk_from_planar(sv.ctx, ctypes.c_int64(p.n), ctypes.c_int(k),
                                     ctypes.c_void_p(sv.d_x.data_ptr()), _lib.dptr(x_pin),
                                     None, ctypes.c_int(0)), "from_planar")
        e2e_iters += int(rep.iterations)
    e3.record(stream)
    barrier()
    e2e_ms = e2.elapsed_time(e3)
    probe = {}
    avg = ctypes.c_double(0)
    _lib.check(L.mpk_bench_apply(sv.m, ctypes.c_int(k), ctypes.c_int(5), ctypes.byref(avg)),
               "bench_apply")
    probe["apply_ms"] = avg.value
    info = (ctypes.c_int64 * 12)()
    _lib.check(L.mpk_sweep_info(sv.m, info, ctypes.c_int(12)), "sweep_info")
    probe["sweep_info"] = list(info)
    _lib.check(L.mpk_bench_spmv(sv.m, ctypes.c_int(k), ctypes.c_int(5), ctypes.byref(avg)),
               "bench_spmv")
    probe["spmv_ms"] = avg.value
    vals = torch.tensor([ms, e2e_ms], dtype=torch.float64, device="cuda")
    if dist:
        tdist.all_reduce(vals, op=tdist.ReduceOp.MAX)
    ms, e2e_ms = float(vals[0]), float(vals[1])
    comm.close()
    return {"ms": ms, "e2e_ms": e2e_ms, "iters": float(iters), "e2e_iters": float(e2e_iters),
            "launches": launches, "h2d": 8 * k * p.n * world, "d2h": 8 * k * p.n * world,
            "clocks": clk.summary(), "probe": probe, "p": p, "k": k, "cold": None,
            "sharded": True, "factor_ms": None}


# ---------------------------------------------------------------------
# CPU: the reference's algorithm (oracle/ C port) on the host cores
# ---------------------------------------------------------------------
def _rhs(oracle, p, k):
    n = p.n
    if p.b64 is not None:
        b_re = np.zeros((n, k))
        b_re[:, 0] = np.real(p.b64)
        b_im = None
        if p.val_im is not None:
            b_im = np.zeros((n, k))
            b_im[:, 0] = np.imag(p.b64)
        return b_re, b_im
    x = np.zeros((n, k))
    x[:, 0] = np.real(p.x_true)
    xi = None
    if p.val_im is not None:
        xi = np.zeros((n, k))
        xi[:, 0] = np.imag(p.x_true)
    return oracle.spmv_mixed(n, p.row_ptr, p.col_idx, p.val_re, p.val_im, x, xi)


def _oracle_solve(oracle, p, m, k, max_iter):
    b_re, b_im = _rhs(oracle, p, k)
    t0 = time.perf_counter()
    rep, _, _, _ = oracle.solve(p.n, p.row_ptr, p.col_idx, p.val_re, p.val_im, m, k, b_re,
                                b_im, eps_rel=p.eps_rel, eps_abs=p.eps_abs, max_iter=max_iter)
    return rep, time.perf_counter() - t0


def cfg4_extrapolated(oracle, p, iters):
    """The C port on cfg4: the ILU(0) factorization once plus `iters`
    BiCGSTAB iterations, timed separately by the oracle; the 200-iteration
    time-to-solve is extrapolated as factor + 200 * (loop / iters)."""
    rep, _ = _oracle_solve(oracle, p, "bicgstab", 2, iters)
    t_it = rep.loop_seconds / max(1, rep.iterations)
    t_solve = rep.factor_seconds + 200 * t_it
    return {"value": 200 / t_solve, "factor_s": rep.factor_seconds, "iter_s": t_it,
            "iters": int(rep.iterations), "loop_s": rep.loop_seconds,
            "time_to_solve_s": t_solve}


def cpu_baseline_sample(config: str):
    import oracle

    threads = os.cpu_count() or 1
    oracle.set_threads(threads)
    from paper_2504_14498_b200 import problems

    if config == "cfg4":
        r = cfg4_extrapolated(oracle, problems.cfg4(), 3)
        return {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "port",
                "sample": f"cfg4: ILU(0) factorization ({r['factor_s']:.1f} s) + {r['iters']} "
                          f"BiCGSTAB iterations ({r['iter_s']:.2f} s each), C port of the "
                          f"reference on {threads} threads (row-parallel SpMV/axpy, sequential "
                          f"sweeps and dots as the reference); extrapolated 200-iteration "
                          f"time-to-solve {r['time_to_solve_s']:.0f} s"}
    if config == "cfg5":
        sample = [(problems.cfg5(0), "bicgstab", 4)]
    else:
        p = problems.CONFIGS[config]()
        sample = [(p, "bicgstab", LAB[pr]) for pr in p.precisions]
    it, t = 0, 0.0
    for p, m, k in sample:
        rep, dt = _oracle_solve(oracle, p, m, k, p.max_iter if p.max_iter else 3 * p.n)
        it += rep.iterations
        t += dt
    return {"value": it / t, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{config}: " + ", ".join(f"{m} k={k} full solve" for _, m, k in sample)
                      + f" ({it} iterations, {t:.1f} s, C port of the reference on "
                        f"{threads} threads)"}


def run_reference(args, world):
    """--impl reference: the reference's algorithm on the host cores (the C
    port in oracle/; the Python reference cannot travel to the box).
    cfg4: one run of `steps` BiCGSTAB iterations after the factorization
    (each step = one iteration, timed by the port), value = the extrapolated
    200-iteration time-to-solve rate.  Other configs: one full cell per
    step, cycling through the cells."""
    import oracle
    from paper_2504_14498_b200 import problems

    threads = os.cpu_count() or 1
    oracle.set_threads(threads)
    base = {"metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True,
            "scaling": ("strong" if args.config == "cfg4" or (args.config == "cfg5"
                                                              and not args.cfg5_weak)
                        else "weak"),
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE.json generators)",
            "config": config_dict(args, world), "impl": "reference"}
    if args.config == "cfg4":
        c1 = problems.cfg1()  # warm-up: page in the port, untimed
        for _ in range(min(args.warmup, 1)):
            _oracle_solve(oracle, c1, "bicgstab", 2, 5)
        r = cfg4_extrapolated(oracle, problems.cfg4(), args.steps)
        v = r["value"]
        sample = (f"cfg4: factorization ({r['factor_s']:.1f} s) + {r['iters']} BiCGSTAB "
                  f"iterations ({r['iter_s']:.2f} s each) on {threads} threads; value = 200 / "
                  f"(factor + 200 * iteration), the extrapolated time-to-solve "
                  f"{r['time_to_solve_s']:.0f} s")
        out = dict(base, value=v, ms_per_step=1000 * r["iter_s"],
                   time_to_solve_s=r["time_to_solve_s"])
    else:
        cells = cells_for(args.config, 0, 1, args.cfg5_weak)
        for s in range(args.warmup):
            p, m, k = cells[s % len(cells)]
            _oracle_solve(oracle, p, m, k, p.max_iter if p.max_iter else 3 * p.n)
        it, t = 0, 0.0
        for s in range(args.steps):
            p, m, k = cells[(args.warmup + s) % len(cells)]
            rep, dt = _oracle_solve(oracle, p, m, k, p.max_iter if p.max_iter else 3 * p.n)
            it += rep.iterations
            t += dt
        v = it / t if t > 0 else 0.0
        sample = (f"one full {args.config} solve per step, cycling {len(cells)} cells; "
                  f"C restatement of the reference on {threads} threads")
        out = dict(base, value=v, ms_per_step=1000 * t / args.steps)
    out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                           "sample": sample}
    out["e2e"] = {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    return out


# ---------------------------------------------------------------------
# launcher
# ---------------------------------------------------------------------
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args):
    """`bench.py --gpus N` outside torchrun: re-exec under
    torch.distributed.run with N ranks (NCCL_DEBUG=INFO keeps the
    communicator log the driver counts ranks from)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", str(pathlib.Path(__file__).resolve()),
           *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.run(cmd, env=env).returncode


def launch_check(world, rank):
    """--launch-check: the multi-rank plumbing alone (gloo, no GPU)."""
    import torch
    import torch.distributed as tdist

    if world > 1:
        tdist.init_process_group("gloo")
    t = torch.tensor([1.0])
    if world > 1:
        tdist.all_reduce(t)
        tdist.barrier()
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "ranks_seen": int(t.item())}),
              flush=True)
    if world > 1:
        tdist.destroy_process_group()


def roofline_blocks(res, args, hbm, peak_src, sm_mhz):
    p, k = res["p"], res["k"]
    c = 2 if p.val_im is not None else 1
    probe = res["probe"]
    traffic = {}
    if TRAFFIC.exists():
        traffic = json.loads(TRAFFIC.read_text()).get(f"{args.config}:{args.precond}", {})
    blocks = {}
    if "apply_ms" in probe:
        ab = apply_bytes(p.n, p.nnz, c)
        ach = ab / (probe["apply_ms"] * 1e-3) / 1e9
        info = probe.get("sweep_info", [0] * 12)
        plan = {0: "sync-free global", 1: "single-CTA", 2: "cluster", 3: "ring",
                4: "lane-chunk wavefront (wf.cu)", 5: "shuffle wavefront (swf.cu)"}.get(info[2])
        lev_f, lev_b = int(info[0]), int(info[1])
        bound_ms = (lev_f * CP_FWD_CYCLES + lev_b * CP_BWD_CYCLES) / (sm_mhz * 1e3)
        t = traffic.get("sweep", {})
        blocks["sweep"] = {
            "bound": "hbm", "kernel": f"ILU(0)-mixed apply (forward + backward sweep), plan: "
                                      f"{plan}", "achieved": ach, "peak": hbm,
            "unit": "GB/s", "frac": ach / hbm, "traffic": t.get("dram_bytes_per_launch"),
            "algorithmic_bytes": ab, "avg_ms": probe["apply_ms"], "peak_source": peak_src,
            "critical_path": {
                "levels": [lev_f, lev_b],
                "model_cycles_per_level": [CP_FWD_CYCLES, CP_BWD_CYCLES],
                "model": "per DAG level one dependent row: shuffle hand-off 24 + dmul 8 + "
                         "2 (fwd) / 3 (bwd) dsub 8 each + bwd Markstein division 24 + "
                         "select 6 cycles",
                "sm_mhz": sm_mhz, "bound_ms": bound_ms,
                "frac": bound_ms / probe["apply_ms"]},
            "traffic_source": t.get("source")}
    sb = spmv_bytes(p.n, p.nnz, c, k)
    ach = sb / (probe["spmv_ms"] * 1e-3) / 1e9
    t = traffic.get("spmv", {})
    blocks["spmv"] = {
        "bound": "hbm", "kernel": f"mixed SpMV y = A x (binary64 A, x an F vector, y "
                                  f"{ {2: 'DD', 3: 'TD', 4: 'QD'}[k]})",
        "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
        "traffic": t.get("dram_bytes_per_launch"), "algorithmic_bytes": sb,
        "avg_ms": probe["spmv_ms"], "peak_source": peak_src,
        "fp64_pipe_pct": t.get("fp64_pipe_pct"), "traffic_source": t.get("source")}
    if probe.get("sweep_info", [0] * 3)[2] == 5 and p.n >= (1 << 18) and c == 1 and args.precond == "ilu0-mixed":
        # cfg4-class systems: inside a solve this SpMV does not run as a kernel of
        # its own -- pspmv_kernel (csrc/units.cu) forms A z chunk by chunk beside the
        # backward phase of the sweep that produces z
        blocks["spmv"]["in_solve"] = (
            "pipelined beside the backward sweep on the 84 SMs it leaves idle "
            "(pspmv_kernel); exposed per SpMV site: the dot-product row kernel only "
            "(profiles/r02_launch_summary_cfg4_final.txt)")
    return blocks


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cold", action="store_true", help="skip the cold time-to-solve")
    ap.add_argument("--precond", default="ilu0-mixed", choices=list(PRECOND_CODE),
                    help="preconditioner of every cell (the paper's ILU(0)_d = ilu0-mixed, "
                         "ILU(0) = ilu0 at working precision, or none)")
    ap.add_argument("--shard", action="store_true",
                    help="cfg4: the row-block sharded path also at N=1")
    ap.add_argument("--cfg5-weak", action="store_true",
                    help="cfg5: 8 systems per GPU (weak scaling) instead of 64/N")
    ap.add_argument("--serial", dest="concurrent", action="store_false",
                    help="run the cells of a step one after another")
    ap.add_argument("--launch-check", action="store_true",
                    help="only check the multi-rank launch (gloo; no GPU)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and (args.impl == "ours"
                                                             or args.launch_check):
        sys.exit(relaunch(args))
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.launch_check:
        launch_check(world, rank)
        return
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, max(world, args.gpus))), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.config == "cfg4" and (world > 1 or args.shard):
        res = run_sharded(args, rank, world, local_rank)
    else:
        res = run_ours(args, rank, world, local_rank)
    if rank != 0:
        if world > 1:
            import torch.distributed as tdist

            tdist.destroy_process_group()
        return
    peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = ("MEASURED_PEAKS.json hbm_gbs" if PEAKS.exists()
                else "fallback B200_PROFILING.md")
    sm_mhz = res["clocks"].get("sm_mhz") or float(peaks.get("sm_max_mhz", 1965.0))
    blocks = roofline_blocks(res, args, hbm, peak_src, sm_mhz)
    value = res["iters"] / (res["ms"] * 1e-3)
    e2e = res["e2e_iters"] / (res["e2e_ms"] * 1e-3)
    sharded = bool(res.get("sharded"))
    # cfg4: one system (rows sharded at N > 1); cfg5: 64 systems split 64/N
    scaling = ("strong" if (sharded or args.config == "cfg4"
                            or (args.config == "cfg5" and not args.cfg5_weak)) else "weak")
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms"] / args.steps,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE.json generators, DESIGN.md 6)",
        "config": config_dict(args, world),
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(res["h2d"]),
                "d2h_bytes_per_step": int(res["d2h"])},
        "gpu_launches": int(res["launches"]),
        "clocks": res["clocks"],
        # the dominant kernel: the ILU(0)-mixed apply (the SpMV when another
        # preconditioner is selected: its applies are not the binary64 sweep)
        "roofline": blocks.get("sweep", blocks["spmv"]),
        "roofline_spmv": blocks["spmv"],
        "iterations_per_step": res["iters"] / args.steps / (1 if sharded else world),
        "time_to_solve_s": res["ms"] / args.steps / 1e3,
    }
    if res.get("factor_ms") is not None:
        out["factor_ms"] = res["factor_ms"]
    if res.get("cold"):
        out["cold_time_to_solve_s"] = res["cold"]
    if world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline_sample(args.config)
        except Exception as e:  # pragma: no cover
            out["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as tdist

        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
