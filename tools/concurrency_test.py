"""Do independent solves on separate contexts/streams overlap?"""
import ctypes, sys, time, pathlib, os
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from concurrent.futures import ThreadPoolExecutor
import torch
import bench
from paper_2504_14498_b200 import _lib
torch.cuda.set_device(0)
L = _lib.lib()
def ctx():
    h = ctypes.c_void_p(); _lib.check(L.mpk_ctx_create(ctypes.c_int(0), ctypes.byref(h))); return h
cells_spec = [c for c in bench.cells_for("cfg2", 0, 1) if c[1] == sys.argv[1]] if len(sys.argv) > 1 else bench.cells_for("cfg2", 0, 1)
N = 8
spec = (cells_spec * 8)[:N]
cells = [bench.Cell(L, _lib, p, m, k, ctx()) for (p, m, k) in spec]
for c in cells: c.run_dev()
torch.cuda.synchronize()
t0 = time.perf_counter()
for c in cells: c.run_dev()
torch.cuda.synchronize(); t1 = time.perf_counter()
with ThreadPoolExecutor(N) as ex: list(ex.map(lambda c: c.run_dev(), cells))
torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"serial {1e3*(t1-t0):.1f} ms, threaded {1e3*(t2-t1):.1f} ms, per-cell loop ms", [round(c.rep.solve_ms,1) for c in cells])
