"""Device time of the binary64 ILU(0) factorization per config (event-timed
inside mpk_ilu0_factor; second call, warm)."""
import ctypes, sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2504_14498_b200 import _lib, problems
L = _lib.lib(); ctx = _lib.context(0)
L.mpk_ilu0_factor.restype = ctypes.c_int
for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg4"]:
    p = (problems.CONFIGS[name](0) if name == "cfg5" else problems.CONFIGS[name]())
    h = ctypes.c_void_p()
    vim = None if p.val_im is None else _lib.f64(p.val_im)
    _lib.check(L.mpk_csr_upload(ctx, ctypes.c_int64(p.n), ctypes.c_int64(p.nnz), _lib.dptr(_lib.i64(p.row_ptr)),
                                _lib.dptr(_lib.i64(p.col_idx)), _lib.dptr(_lib.f64(p.val_re)), _lib.dptr(vim), ctypes.byref(h)))
    bad = ctypes.c_int64(); st = ctypes.c_int32()
    rep = _lib.MpkReport()
    for _ in range(2):
        _lib.check(L.mpk_ilu0_factor(h, ctypes.byref(bad), ctypes.byref(st)))
    # factor_ms is reported through a solve report; use a 1-iteration solve
    import numpy as np
    k = 2
    b = np.zeros((p.n, k)); b[:, 0] = 1.0
    bi = np.zeros((p.n, k)) if p.val_im is not None else None
    x = np.zeros((p.n, k)); xi = np.zeros((p.n, k)) if bi is not None else None
    _lib.check(L.mpk_solve(h, ctypes.c_int(2), ctypes.c_int(k), ctypes.c_double(1e-30), ctypes.c_double(1e-300),
                           ctypes.c_int64(1), _lib.dptr(b), _lib.dptr(bi), _lib.dptr(x), _lib.dptr(xi), None,
                           ctypes.c_int64(0), ctypes.byref(rep)))
    print(f"{name}: n={p.n} nnz={p.nnz} factor {rep.factor_ms:.3f} ms")
