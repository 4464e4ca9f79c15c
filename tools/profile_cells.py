"""Profiling driver: solve the cells of one config once each (after one
warm-up pass), device-resident, so `ncu` launch lists map onto one step.

    python tools/profile_cells.py [cfg2] [--cells bicgstab:4,cgs:3] [--passes 1]
"""

from __future__ import annotations

import argparse
import ctypes
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="cfg2")
    ap.add_argument("--cells", default="")
    ap.add_argument("--passes", type=int, default=1)
    ap.add_argument("--warm", type=int, default=100, help="cells in the warm-up pass")
    args = ap.parse_args()
    import torch

    from paper_2504_14498_b200 import _lib

    torch.cuda.set_device(0)
    L = _lib.lib()
    ctx = _lib.context(0)
    want = None
    if args.cells:
        want = {(c.split(":")[0], int(c.split(":")[1])) for c in args.cells.split(",")}
    cells = [bench.Cell(L, _lib, p, m, k, ctx)
             for (p, m, k) in bench.cells_for(args.config, 0, 1)
             if want is None or (m, k) in want]
    for c in cells[: args.warm]:  # warm-up pass
        c.run_dev()
    torch.cuda.synchronize()
    for _ in range(args.passes):
        for c in cells:
            r = c.run_dev()
            print(f"{c.method} k={c.k}: it={r.iterations} factor={r.factor_ms:.3f} ms "
                  f"loop={r.solve_ms:.3f} ms launches={r.launches}", flush=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
