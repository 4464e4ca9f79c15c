"""A/B the sweep implementations on ILU(0) applies of the named configs.

    python tools/sweep_ab.py [--env 'A=1 B=2' ...] cfg1 cfg2 ...
Each --env set runs in its own process (settings are read at upload)."""
import ctypes, os, subprocess, sys, pathlib, json
ROOT = pathlib.Path(__file__).resolve().parents[1]
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, str(ROOT))
    import numpy as np
    from paper_2504_14498_b200 import _lib, problems
    L = _lib.lib(); ctx = _lib.context(0)
    out = {}
    for name in sys.argv[2:]:
        p = problems.cfg5(0) if name == "cfg5" else problems.CONFIGS[name]()
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
    args = sys.argv[1:]
    envs, names = [], []
    while args:
        a = args.pop(0)
        if a == "--env":
            envs.append(args.pop(0))
        else:
            names.append(a)
    for e in envs or ["MPK_SWEEP_VAR=3"]:
        env = dict(os.environ, **dict(kv.split("=") for kv in e.split()))
        r = subprocess.run([sys.executable, __file__, "child", *names], env=env, capture_output=True, text=True)
        print(f"[{e}]", r.stdout.strip(), r.stderr.strip()[-300:], flush=True)
