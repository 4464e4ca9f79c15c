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
