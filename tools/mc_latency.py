"""Launch single-element MC ops (n=1) so ncu shows each op's latency."""
import ctypes, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2504_14498_b200 import _lib as L
for k in (2, 3, 4):
    a = np.zeros((1, 8)); b = np.zeros((1, 8))
    a[0, 0] = 1.2345678901234567; a[0, 1] = 1e-17; b[0, 0] = 0.987654321; b[0, 1] = -3e-18
    a = np.ascontiguousarray(a[:, :k] if True else a); b = np.ascontiguousarray(b[:, :k])
    for op in (0, 2, 3, 4, 6):
        o = np.zeros((1, k)); oi = np.zeros((1, k))
        cx = op in (5, 6)
        L.check(L.lib().mpk_mc_elementwise(L.context(), ctypes.c_int(op), ctypes.c_int(k), ctypes.c_int64(1), L.dptr(a), L.dptr(a if cx else None), L.dptr(b), L.dptr(b if cx else None), L.dptr(o), L.dptr(oi if cx else None)))
print("ok")
