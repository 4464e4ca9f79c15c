"""Multi-rank logic on CPU (gloo, world_size 2): cfg5-style independent
systems sharded across ranks and gathered, checked against a serial run.
The per-system solve here is the CPU oracle (the device path is exercised
by the GPU tests); what is under test is the sharding / gather plumbing
that bench.py uses for --config cfg5."""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2504_14498_b200.sharding import shard


def test_shard_covers_every_unit_once():
    for n in (0, 1, 7, 64):
        for w in (1, 2, 3, 8):
            seen = []
            for r in range(w):
                seen += list(shard(n, r, w))
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _systems():
    from paper_2504_14498_b200 import problems

    out = []
    for s in range(4):
        rp, ci, v, xt = problems.random_nonsym(300, 6, 900 + s)
        out.append((rp, ci, v, xt))
    return out


def _solve(sys_):
    import oracle

    rp, ci, v, xt = sys_
    n = len(rp) - 1
    x = np.zeros((n, 2))
    x[:, 0] = xt
    b, _ = oracle.spmv_mixed(n, rp, ci, v, None, x)
    rep, xr, _, hist = oracle.solve(n, rp, ci, v, None, "bicgstab", 2, b, eps_rel=1e-25)
    return {"it": int(rep.iterations), "conv": bool(rep.converged),
            "hist": [list(h) for h in hist]}


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2504_14498_b200.sharding import gather_reports

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    systems = _systems()
    local = {i: _solve(systems[i]) for i in shard(len(systems), rank, world)}
    merged = gather_reports(local, world)
    if rank == 0:
        q.put(merged)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_gather(orc):
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    serial = [_solve(s) for s in _systems()]
    assert merged == serial


# ---------------------------------------------------------------------------
# row-block sharded solve (csrc/shard.cuh, paper_2504_14498_b200/sharded.py):
# the partition and the two in-place all-gather layouts it relies on, run
# with gloo over 2 ranks.  Each rank fills ITS row block / partial blocks
# exactly like the device kernels (rows [r*nb, (r+1)*nb), partial blocks
# [r*Gl, (r+1)*Gl) of every slot) and all-gathers in place; afterwards every
# rank must hold the single-process arrays.
# ---------------------------------------------------------------------------
def test_row_blocks_and_partial_blocks():
    from paper_2504_14498_b200.sharded import KMAXGRID, blocks_per_rank, row_blocks

    for n in (1, 7, 4096, 4194304):
        for w in (1, 2, 4, 8):
            nb, blk = row_blocks(n, w)
            rows = [i for r0, r1 in blk for i in range(r0, r1)]
            assert rows == list(range(n)) and w * nb >= n
            assert w * blocks_per_rank(w) <= KMAXGRID


def _sharded_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2504_14498_b200.sharded import KMAXGRID, blocks_per_rank, row_blocks

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 1000
    nb, blk = row_blocks(n, world)
    r0, r1 = blk[rank]
    rng = np.random.default_rng(0)
    full = rng.standard_normal(world * nb)  # the head plane every rank needs
    plane = np.full(world * nb, np.nan)
    plane[r0:r1] = full[r0:r1]
    # in-place all-gather of rank ranges (NCCL: recvbuf = plane, send = own range)
    chunks = [torch.empty(nb, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(chunks, torch.from_numpy(plane[rank * nb:(rank + 1) * nb].copy()))
    gathered = torch.cat(chunks).numpy()
    # reduction partials: slot-major [slot][KMAXGRID][8]; rank owns blocks
    gl = blocks_per_rank(world)
    part = np.zeros((2, KMAXGRID, 8))
    for s in range(2):
        for g in range(gl):
            part[s, rank * gl + g, :] = 100 * s + rank * gl + g
    for s in range(2):
        flat = part[s].reshape(-1)
        cnk = [torch.empty(gl * 8, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(cnk, torch.from_numpy(flat[rank * gl * 8:(rank + 1) * gl * 8].copy()))
        flat[: world * gl * 8] = torch.cat(cnk).numpy()
    if rank == 0:
        q.put((gathered[:n].tolist(), part.tolist()))
    else:
        q.put(None)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_sharded_exchange_layout():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got = [r for r in res if r is not None][0]
    from paper_2504_14498_b200.sharded import KMAXGRID, blocks_per_rank, row_blocks

    nb, _ = row_blocks(1000, 2)
    full = np.random.default_rng(0).standard_normal(2 * nb)
    assert np.array_equal(np.asarray(got[0]), full[:1000])
    part = np.asarray(got[1])
    gl = blocks_per_rank(2)
    for s in range(2):
        assert np.array_equal(part[s, : 2 * gl, 0], 100 * s + np.arange(2 * gl))


def test_bench_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks
    (torch.distributed.run, 127.0.0.1); the launch check runs the rank
    plumbing over gloo and rank 0 reports n_gpus = 2."""
    import json
    import pathlib
    import subprocess
    import sys

    root = pathlib.Path(__file__).resolve().parents[1]
    env = {k: v for k, v in __import__("os").environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--launch-check"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["ranks_seen"] == 2
