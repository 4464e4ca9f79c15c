"""Wavefront sweep diagnostics: per-group start/end (globaltimer) of the
last apply.  MPK_SWEEP_PICK=wf MPK_WF_DEBUG=1 python tools/wf_probe.py cfg4"""
import ctypes, os, sys, pathlib
os.environ.setdefault("MPK_SWEEP_PICK", "wf")
os.environ.setdefault("MPK_WF_DEBUG", "2")
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2504_14498_b200 import _lib, problems
name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
L = _lib.lib(); ctx = _lib.context(0)
if name.startswith("st9_"):  # 9-point stencil on an nx x ny grid (nx fastest)
    nx, ny = map(int, name[4:].split("_"))
    rng = np.random.default_rng(1)
    rows, cols = [], []
    for y in range(ny):
        for x in range(nx):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    if 0 <= x + dx < nx and 0 <= y + dy < ny:
                        rows.append(y * nx + x); cols.append((y + dy) * nx + x + dx)
    rows = np.array(rows); cols = np.array(cols)
    n = nx * ny
    v = rng.uniform(-1, 0, len(rows)); v[rows == cols] = 9.0
    rp = np.zeros(n + 1, np.int64); np.add.at(rp, rows + 1, 1); rp = np.cumsum(rp)
    ci = cols; nnz = len(ci); vim = None
elif name.startswith("cd9_"):
    rp, ci, v = problems.convdiff9(int(name[4:]), 5.0)[:3]
    n, nnz, vim = len(rp) - 1, len(ci), None
else:
    p = problems.CONFIGS[name]()
    rp, ci, v, n, nnz = p.row_ptr, p.col_idx, p.val_re, p.n, p.nnz
    vim = None if p.val_im is None else _lib.f64(p.val_im)
h = ctypes.c_void_p()
_lib.check(L.mpk_csr_upload(ctx, ctypes.c_int64(n), ctypes.c_int64(nnz), _lib.dptr(_lib.i64(rp)),
                            _lib.dptr(_lib.i64(ci)), _lib.dptr(_lib.f64(v)), _lib.dptr(vim), ctypes.byref(h)))
bad = ctypes.c_int64(); st = ctypes.c_int32()
_lib.check(L.mpk_ilu0_factor(h, ctypes.byref(bad), ctypes.byref(st)))
ms = ctypes.c_double()
_lib.check(L.mpk_bench_apply(h, ctypes.c_int(2), ctypes.c_int(3), ctypes.byref(ms)))
print(name, "apply ms", ms.value)
buf = np.zeros(2 * 8192, np.int64)
L.mpk_wf_debug(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(len(buf)))
st_ = buf[0::2]; en = buf[1::2]
ng = int(np.count_nonzero(en))
if ng < 2:
    sys.exit(0)
t0 = st_[:ng].min()
s = (st_[:ng] - t0) / 1e3; e = (en[:ng] - t0) / 1e3
half = ng // 2
for lo, hi, tag in ((0, half, "fwd"), (half, ng, "bwd")):
    d = e[lo:hi] - s[lo:hi]
    print(f"{tag}: groups {hi-lo}, dur us min/med/max {d.min():.1f}/{np.median(d):.1f}/{d.max():.1f}; "
          f"end of first {e[lo]:.1f}, end of last {e[hi-1]:.1f}; end gaps med "
          f"{np.median(np.diff(e[lo:hi])):.2f} us")
    print("   first ends:", np.round(e[lo:lo+6], 1), "last ends:", np.round(e[hi-4:hi], 1))

b2 = np.zeros(4096, np.int64)
L.mpk_wf_debug2(b2.ctypes.data_as(ctypes.c_void_p))
q = b2[:4096].reshape(1024, 4)
q = q[:int(np.count_nonzero(q[:, 0]))]
seg = np.diff(q, axis=1)
nxt = q[1:, 0] - q[:-1, 3]
print("per-step segments (median cycles): wait", np.median(seg[:, 0]), "loads+rhs", np.median(seg[:, 1]),
      "chain+pub", np.median(seg[:, 2]), "prefetch+sync+loop", np.median(nxt))
