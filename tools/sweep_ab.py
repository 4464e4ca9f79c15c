"""A/B the sweep variants (MPK_SWEEP_VAR) on cfg2 / cfg1 / cfg3 applies."""
import ctypes, os, subprocess, sys, pathlib, json
ROOT = pathlib.Path(__file__).resolve().parents[1]
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, str(ROOT))
    import numpy as np
    from paper_2504_14498_b200 import _lib, problems
    L = _lib.lib(); ctx = _lib.context(0)
    out = {}
    for name in sys.argv[2:]:
        p = problems.CONFIGS[name]()
        h = ctypes.c_void_p()
        vim = None if p.val_im is None else _lib.f64(p.val_im)
        _lib.check(L.mpk_csr_upload(ctx, ctypes.c_int64(p.n), ctypes.c_int64(p.nnz), _lib.dptr(_lib.i64(p.row_ptr)), _lib.dptr(_lib.i64(p.col_idx)), _lib.dptr(_lib.f64(p.val_re)), _lib.dptr(vim), ctypes.byref(h)))
        bad = ctypes.c_int64(); st = ctypes.c_int32()
        import time
        t0 = time.perf_counter(); _lib.check(L.mpk_ilu0_factor(h, ctypes.byref(bad), ctypes.byref(st))); tf = time.perf_counter() - t0
        ms = ctypes.c_double()
        _lib.check(L.mpk_bench_apply(h, ctypes.c_int(2), ctypes.c_int(30), ctypes.byref(ms)))
        out[name] = {"apply_ms": ms.value, "factor_s": tf}
        L.mpk_csr_free(h)
    print(json.dumps(out))
else:
    for v in ("0", "1", "2", "3"):
        env = dict(os.environ, MPK_SWEEP_VAR=v)
        r = subprocess.run([sys.executable, __file__, "child", *sys.argv[1:]], env=env, capture_output=True, text=True)
        print("VAR", v, r.stdout.strip(), r.stderr.strip()[-300:])
