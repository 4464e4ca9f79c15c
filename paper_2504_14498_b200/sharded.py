"""Row-block sharded solve of ONE system over W GPUs (BASELINE cfg4).

The reference solves on one CPU thread (solvers.py:418-453); this is the
B200 extension of ``solve`` for a system spread over the GPUs of one node,
one process per GPU (``torch.distributed`` for the rendezvous, NCCL for the
collectives).  What shards and what does not (csrc/shard.cuh):

* the ILU(0) factorization and both sweeps of every apply run IN FULL on
  every rank -- the triangular solve does not shard without changing the
  preconditioner (block-Jacobi ILU != ILU(0));
* SpMV rows, vector updates and reduction block partials run on the rank's
  contiguous block of ``nb = ceil(n / W)`` rows;
* exchanges, all in-place all-gathers: reduction block partials (every rank
  folds the same W*Gl partials in one fixed order, so the scalar recurrence
  and the stop decision are identical on all ranks) and the head plane of
  each sweep input (8 B per row).  Sweep outputs are then complete on every
  rank, so the SpMV rows need no halo.

BiCGSTAB only (the cfg4 method), tree reductions, ILU(0)-mixed / mixed SpMV.
``Communicator.local(W)`` builds W virtual ranks inside one process on one
GPU (device copies ordered by events, no cross-rank kernel waits) for tests.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _lib
from .ilu import PrecondMode
from .sparse import DenseVector

KMAXGRID = 592  # common.cuh kMaxGrid: partial blocks per reduction slot

__all__ = ["Communicator", "ShardedSolver", "row_blocks", "blocks_per_rank",
           "check_shardable", "solve_sharded"]


def row_blocks(n: int, world: int):
    """(nb, [(r0, r1)] per rank): rank r owns rows [r*nb, min((r+1)*nb, n))."""
    nb = -(-n // world) if world > 0 else 0
    return nb, [(min(r * nb, n), min((r + 1) * nb, n)) for r in range(world)]


def blocks_per_rank(world: int) -> int:
    """Reduction partial blocks per rank (the finalize folds world * this)."""
    return KMAXGRID // world


def check_shardable(n: int, world: int) -> None:
    nb, _ = row_blocks(n, world)
    if world * nb > _lib.plane_ld(n):
        raise ValueError(f"n={n} does not split into {world} row blocks inside the "
                         f"plane stride (need W*ceil(n/W) <= {_lib.plane_ld(n)})")


def _lib_sharded():
    L = _lib.lib()
    if not getattr(L, "_sharded_types", False):
        L.mpk_comm_rank.argtypes = [ctypes.c_void_p]
        L.mpk_comm_world.argtypes = [ctypes.c_void_p]
        L.mpk_comm_destroy.argtypes = [ctypes.c_void_p]
        L._sharded_types = True
    return L


class Communicator:
    """One rank's handle of a sharded-solve group."""

    def __init__(self, handle: ctypes.c_void_p):
        self.h = handle

    @property
    def rank(self) -> int:
        return int(_lib_sharded().mpk_comm_rank(self.h))

    @property
    def world(self) -> int:
        return int(_lib_sharded().mpk_comm_world(self.h))

    @classmethod
    def nccl(cls, device: int, group=None) -> "Communicator":
        """NCCL communicator over the torch.distributed group (one GPU per
        process); rank 0 creates the unique id and broadcasts it."""
        import torch.distributed as dist

        L = _lib_sharded()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        buf = (ctypes.c_char * 128)()
        if rank == 0:
            _lib.check(L.mpk_comm_unique_id(buf), "mpk_comm_unique_id")
        obj = [bytes(buf) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        idb = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        _lib.check(L.mpk_comm_create(ctypes.c_int(device), ctypes.c_int(rank),
                                     ctypes.c_int(world), idb, ctypes.byref(h)),
                   "mpk_comm_create")
        return cls(h)

    @classmethod
    def local(cls, world: int) -> list:
        """W virtual ranks in this process (each rank's solve on its own thread)."""
        L = _lib_sharded()
        hs = (ctypes.c_void_p * world)()
        _lib.check(L.mpk_comm_create_local(ctypes.c_int(world), hs), "mpk_comm_create_local")
        return [cls(ctypes.c_void_p(hs[r])) for r in range(world)]

    def close(self) -> None:
        if self.h:
            _lib_sharded().mpk_comm_destroy(self.h)
            self.h = None


class ShardedSolver:
    """The whole matrix on this rank's GPU (own context / stream) plus the
    device buffers of a sharded solve; ``solve(b)`` may be called repeatedly."""

    def __init__(self, A, precision, comm: Communicator, device: int = 0):
        import torch

        L = _lib.lib()
        self.comm, self.k, self.n, self.device = comm, precision.k, A.n, device
        self.precision = precision
        self.cx = A.field == "complex"
        if self.cx:
            raise NotImplementedError("sharded solve: real systems (cfg4)")
        check_shardable(A.n, comm.world)
        self.ctx = ctypes.c_void_p()
        _lib.check(L.mpk_ctx_create(ctypes.c_int(device), ctypes.byref(self.ctx)), "ctx")
        vre = _lib.f64(np.asarray(A.val_re)[:, 0])  # demoted() head (sparse.py:245-249)
        self.m = ctypes.c_void_p()
        _lib.check(L.mpk_csr_upload(self.ctx, ctypes.c_int64(A.n), ctypes.c_int64(len(vre)),
                                    _lib.dptr(_lib.i64(A.row_ptr)), _lib.dptr(_lib.i64(A.col_idx)),
                                    _lib.dptr(vre), None, ctypes.byref(self.m)), "upload")
        ld = _lib.plane_ld(A.n)
        dev = torch.device("cuda", device)
        self.d_b = torch.zeros(self.k * ld + 4, dtype=torch.float64, device=dev)
        self.d_x = torch.zeros(self.k * ld + 4, dtype=torch.float64, device=dev)
        self.d_h = None
        torch.cuda.synchronize(dev)  # the library works on its own stream

    def load_b(self, b: DenseVector) -> None:
        _lib.check(_lib.lib().mpk_to_planar(self.ctx, ctypes.c_int64(self.n), ctypes.c_int(self.k),
                                            _lib.dptr(_lib.f64(b.re)), None,
                                            ctypes.c_void_p(self.d_b.data_ptr())), "to_planar")

    def solve_dev(self, eps_rel: float, eps_abs: float, max_iter: int, hist_cap: int = 0):
        """Device-resident solve (b already loaded); returns the MpkReport."""
        import torch

        L = _lib_sharded()
        if hist_cap and (self.d_h is None or self.d_h.numel() < hist_cap * self.k):
            self.d_h = torch.zeros(hist_cap * self.k + 4, dtype=torch.float64,
                                   device=self.d_b.device)
            torch.cuda.synchronize(self.d_b.device)
        rep = _lib.MpkReport()
        _lib.check(L.mpk_solve_dev_sharded(
            self.m, self.comm.h, ctypes.c_int(_lib.METHOD_CODE["bicgstab"]),
            ctypes.c_int(self.k), ctypes.c_double(eps_rel), ctypes.c_double(eps_abs),
            ctypes.c_int64(max_iter), ctypes.c_void_p(self.d_b.data_ptr()),
            ctypes.c_void_p(self.d_x.data_ptr()),
            ctypes.c_void_p(self.d_h.data_ptr() if hist_cap else 0),
            ctypes.c_int64(hist_cap), ctypes.byref(rep)), "mpk_solve_dev_sharded")
        return rep

    def x_host(self) -> DenseVector:
        x = DenseVector.zeros(self.n, self.precision, "real")
        _lib.check(_lib.lib().mpk_from_planar(self.ctx, ctypes.c_int64(self.n), ctypes.c_int(self.k),
                                              ctypes.c_void_p(self.d_x.data_ptr()),
                                              _lib.dptr(x.re), None, ctypes.c_int(0)),
                   "from_planar")
        return x

    def history(self, rep) -> list:
        hn = min(int(rep.hist_len), (self.d_h.numel() - 4) // self.k if self.d_h is not None else 0)
        if hn <= 0:
            return []
        h = self.d_h[: hn * self.k].view(hn, self.k).cpu().numpy()
        return [tuple(r) for r in h]

    def close(self) -> None:
        L = _lib.lib()
        if self.m:
            L.mpk_csr_free(self.m)
            self.m = None
        if self.ctx:
            L.mpk_ctx_destroy(self.ctx)
            self.ctx = None


def solve_sharded(A, b: DenseVector, cfg, comm: Communicator, device: int = 0):
    """``solve(A, b, cfg)`` (solvers.py:418-453) for BiCGSTAB with ILU(0)-mixed,
    row-block sharded over ``comm``'s ranks.  Returns a SolveReport; x is
    complete on every rank."""
    from .solvers import SolveReport, _breakdown_string

    if cfg.method != "bicgstab":
        raise NotImplementedError("sharded solve: method 'bicgstab' only")
    if cfg.spmv_mode != "mixed" or cfg.precond != PrecondMode.ILU0_MIXED:
        raise NotImplementedError("sharded solve: ILU0_MIXED with spmv_mode='mixed'")
    if A.n != b.n:
        raise ValueError("matrix/vector dimension mismatch")
    t0 = time.perf_counter()
    s = ShardedSolver(A, cfg.precision, comm, device)
    try:
        s.load_b(b)
        max_iter = cfg.resolved_max_iter(A.n)
        rep = s.solve_dev(cfg.eps_rel, cfg.eps_abs, max_iter, hist_cap=2 * max_iter + 2)
        x = s.x_host() if rep.has_x else None
        hist = s.history(rep)
    finally:
        s.close()
    out = SolveReport(method="bicgstab", precision=cfg.precision.label,
                      precond=cfg.precond.value, spmv_mode=cfg.spmv_mode,
                      iterations=int(rep.iterations), converged=bool(rep.converged),
                      total_seconds=time.perf_counter() - t0,
                      breakdown=_breakdown_string(rep), x=x, history=hist,
                      factor_seconds=rep.factor_ms * 1e-3,
                      solve_seconds=rep.solve_ms * 1e-3)
    if rep.breakdown not in (7, 8, 9):
        out.final_recursive_relres = float(rep.final_recursive_relres)
        out.true_relres = float(rep.true_relres)
    return out
