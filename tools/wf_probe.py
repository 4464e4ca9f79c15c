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
L.mpk_wf_debug3(None, ctypes.c_int(1))
_lib.check(L.mpk_bench_apply(h, ctypes.c_int(2), ctypes.c_int(1), ctypes.byref(ms)))
sl = np.zeros(8192, np.int32)
L.mpk_wf_debug3(sl.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(0))
sb, sd = sl & 0xffff, sl >> 16
print("slow-path steps per group: staged-not-ready (fwd, bwd totals)", sb[:64].sum(), sb[64:128].sum(), "; division test failed", sd[:128].sum())
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
m = int(np.count_nonzero(b2[:3072]))
cb = b2[3072:].reshape(256, 4).astype(np.int64)
st = b2[:m]
# chunk c boundary: last step stamp of chunk c-1 (t=7) -> cb[c,0..3] -> step stamp c*8
rows = []
for c in range(2, min(200, m // 8 - 1)):
    rows.append([cb[c, 0] - st[c * 8 - 1], cb[c, 1] - cb[c, 0], cb[c, 2] - cb[c, 1], cb[c, 3] - cb[c, 2], st[c * 8] - cb[c, 3]])
print("chunk boundary median cycles [t7 body+refill, rec_wait, deps_issue, rhs_issue, wait_group]:", np.median(np.array(rows), axis=0))
d = np.diff(b2[:m])
print("group0 step cycles: n", m, "median", np.median(d), "mean", round(d.mean(), 1))
print("  by t%8:", [int(np.median(d[t::8])) for t in range(8)])

b4 = np.zeros(4096, np.int64)
L.mpk_wf_debug4(b4.ctypes.data_as(ctypes.c_void_p))
g0 = b2[:2112].astype(np.float64); g1 = b4[:2112].astype(np.float64)
if g1[100] > 0 and g0[200] > 0:
    # consumer step x needs producer step x+63; measure time(consumer x) - time(producer x+63)
    xs = np.arange(0, 2112 - 64, 100)
    print("group1 step x minus group0 step x+63 (us):", [round((g1[x] - g0[x + 63]) / 1e3, 2) for x in xs])
    tau0 = np.median(np.diff(g0[:2000])); tau1 = np.median(np.diff(g1[:2000]))
    print("median step ns g0/g1:", tau0, tau1, " lag in steps at x=1000:", round((g1[1000] - g0[1000]) / tau0, 1))

d4 = np.diff(g1[:2000]) if g1[10] > 0 else None
if d4 is not None:
    print("bwd group 0 step ns: median", np.median(d4), "mean", round(d4.mean(), 1),
          "by t%8:", [int(np.median(d4[t::8])) for t in range(8)])
