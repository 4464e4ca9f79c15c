"""Wall time of N identical concurrent solves (mpk_run_jobs) for N=1,2,4,8,16."""
import ctypes, sys, time, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
import bench
from paper_2504_14498_b200 import _lib
torch.cuda.set_device(0)
L = _lib.lib()
method = sys.argv[1] if len(sys.argv) > 1 else "bicgstab"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
spec = [c for c in bench.cells_for("cfg2", 0, 1) if c[1] == method and c[2] == k][0]
def ctx():
    h = ctypes.c_void_p(); _lib.check(L.mpk_ctx_create(ctypes.c_int(0), ctypes.byref(h))); return h
cells = [bench.Cell(L, _lib, spec[0], spec[1], spec[2], ctx()) for _ in range(16)]
def jobs(cs):
    J = (_lib.MpkJob * len(cs))()
    for j, c in enumerate(cs):
        J[j].m = c.m; J[j].method = _lib.METHOD_CODE[c.method]; J[j].k = c.k
        J[j].eps_rel = c.p.eps_rel; J[j].eps_abs = c.p.eps_abs; J[j].max_iter = c.max_iter
        J[j].b_re = c.d_b.data_ptr(); J[j].x_re = c.d_x.data_ptr(); J[j].hist = c.d_h.data_ptr(); J[j].hist_cap = c.hist_cap
    return J
for N in (1, 2, 4, 8, 16):
    J = jobs(cells[:N])
    L.mpk_run_jobs(J, N, 1); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        _lib.check(L.mpk_run_jobs(J, N, 1))
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"N={N:2d}: {dt*1e3:7.2f} ms per batch, {dt*1e3/N:6.2f} ms per solve, loop ms {[round(J[j].rep.solve_ms,1) for j in range(min(N,4))]}")
