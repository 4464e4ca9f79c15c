import sys, numpy as np, ctypes, subprocess
sys.path.insert(0, '.')
op, k = int(sys.argv[1]), int(sys.argv[2])
from paper_2504_14498_b200 import _lib as L
g = np.load('tests/golden/mc_ops.npz')
a, b = g[f"k{k}_a"], g[f"k{k}_b"]
if op == 7: a = g[f"k{k}_renorm_in"]
if op == 4: a = g[f"k{k}_sqrt_in"]
if op in (5, 6): a, b = g[f"k{k}_car"], g[f"k{k}_cbr"]
cx = op in (5, 6)
n = a.shape[0]; o = np.zeros((n, k)); oi = np.zeros((n, k)) if cx else None
ai = L.f64(g[f"k{k}_cai"]) if cx else None; bi = L.f64(g[f"k{k}_cbi"]) if cx else None
rc = L.lib().mpk_mc_elementwise(L.context(), ctypes.c_int(op), ctypes.c_int(k), ctypes.c_int64(n), L.dptr(L.f64(a)), L.dptr(ai), L.dptr(L.f64(b)), L.dptr(bi), L.dptr(o), L.dptr(oi))
print(op, k, rc, L.last_error() if rc else "")
