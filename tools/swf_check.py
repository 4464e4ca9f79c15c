"""Shuffle-wavefront sweep plan (csrc/swf.cu): bitwise check against the C
oracle and apply timing per sweep plan, one process per plan setting.

    python tools/swf_check.py [--env 'MPK_SWEEP_PICK=swf' ...] cd9_97 cfg1 cfg4
"""
import ctypes, hashlib, json, os, pathlib, subprocess, sys, time
ROOT = pathlib.Path(__file__).resolve().parents[1]
MATS = {
    "cd5_64": lambda pr: pr.convdiff5(64, 10.0)[:3],
    "cd9_97": lambda pr: pr.convdiff9(97, 5.0)[:3],
    "cd9_200": lambda pr: pr.convdiff9(200, 5.0)[:3],
    "cd9_1000": lambda pr: pr.convdiff9(1000, 5.0)[:3],
    "cfg1": lambda pr: (lambda p: (p.row_ptr, p.col_idx, p.val_re))(pr.cfg1()),
    "cfg4": lambda pr: (lambda p: (p.row_ptr, p.col_idx, p.val_re))(pr.cfg4()),
}
if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import oracle.oracle as orc
    import paper_2504_14498_b200 as mpk
    from paper_2504_14498_b200 import _lib, problems
    from paper_2504_14498_b200.sparse import device_matrix
    out = {}
    for name in sys.argv[2:]:
        rp, ci, v = MATS[name](problems)
        n = len(rp) - 1
        A = mpk.CsrMatrix.from_binary64(n, rp, ci, v, None, mpk.Precision.DD)
        t0 = time.perf_counter()
        F = mpk.ilu0_factorize_demoted(A)
        tf = time.perf_counter() - t0
        rng = np.random.default_rng(5)
        r_re = rng.standard_normal((n, 2))
        r = mpk.DenseVector(r_re.copy(), None, mpk.Precision.DD)
        if os.environ.get("SWF_FORCE_RERUN") == "1":
            _lib.lib().mpk_swf_debug(None, ctypes.c_int(3))
        z = mpk.ilu0_apply_mixed(F, r)
        z2 = mpk.ilu0_apply_mixed(F, r)
        rec = {"factor_s": tf, "z_sha": hashlib.sha256(z.re.tobytes()).hexdigest()[:16],
               "repeat_equal": bool(np.array_equal(z.re.view(np.uint64), z2.re.view(np.uint64)))}
        if n <= 5_000_000 and os.environ.get("SWF_ORACLE", "1") == "1":
            rc, lre, lim = orc.ilu0_factor(n, rp, ci, v, None)[:3]
            _, zr, _ = orc.ilu0_apply_mixed(n, rp, ci, lre, lim, r_re, None)
            rec["oracle_bitwise"] = bool(np.array_equal(z.re.view(np.uint64), zr.view(np.uint64)))
            if not rec["oracle_bitwise"]:
                bad = np.nonzero(z.re[:, 0].view(np.uint64) != zr[:, 0].view(np.uint64))[0]
                rec["first_bad"] = int(bad[0]) if len(bad) else -1
                rec["nbad"] = int(len(bad))
        ms = ctypes.c_double()
        d = F._dev
        _lib.check(_lib.lib().mpk_bench_apply(d.h, ctypes.c_int(2), ctypes.c_int(20),
                                              ctypes.byref(ms)))
        rec["apply_ms"] = ms.value
        out[name] = rec
    print(json.dumps(out))
elif __name__ == "__main__":
    args = sys.argv[1:]
    envs, names = [], []
    while args:
        a = args.pop(0)
        if a == "--env":
            envs.append(args.pop(0))
        else:
            names.append(a)
    for e in envs or ["MPK_VERBOSE=1"]:
        env = dict(os.environ, **dict(kv.split("=") for kv in e.split()))
        r = subprocess.run([sys.executable, __file__, "child", *names], env=env,
                           capture_output=True, text=True)
        print(f"[{e}]", r.stdout.strip(), r.stderr.strip()[-1500:], flush=True)
