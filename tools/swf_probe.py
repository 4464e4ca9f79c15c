"""Per-group timing of the shuffle-wavefront sweep (MPK_SWF_DEBUG stamps).

    MPK_SWEEP_PICK=swf python tools/swf_probe.py cfg4 [W...]
Prints per phase: total span, per-group duration (min/median/max), and the
start delay between consecutive groups (intra-CTA and cross-CTA hops)."""
import ctypes, json, os, pathlib, subprocess, sys
ROOT = pathlib.Path(__file__).resolve().parents[1]
if len(sys.argv) > 2 and sys.argv[1] == "child":
    sys.path.insert(0, str(ROOT))
    import numpy as np
    import paper_2504_14498_b200 as mpk
    from paper_2504_14498_b200 import _lib, problems
    sys.path.insert(0, str(ROOT / "tools"))
    from swf_check import MATS
    rp, ci, v = MATS[sys.argv[2]](problems)
    n = len(rp) - 1
    A = mpk.CsrMatrix.from_binary64(n, rp, ci, v, None, mpk.Precision.DD)
    F = mpk.ilu0_factorize_demoted(A)
    L = _lib.lib()
    ms = ctypes.c_double()
    _lib.check(L.mpk_bench_apply(F._dev.h, ctypes.c_int(2), ctypes.c_int(3), ctypes.byref(ms)))
    L.mpk_swf_debug(None, ctypes.c_int(int(os.environ.get("SWF_DBG", "1"))))
    _lib.check(L.mpk_bench_apply(F._dev.h, ctypes.c_int(2), ctypes.c_int(1), ctypes.byref(ms)))
    buf = (ctypes.c_longlong * (4 * 4096))()
    L.mpk_swf_debug(buf, ctypes.c_int(0))
    a = np.array(buf[:], dtype=np.int64).reshape(2, 4096, 2)
    W = int(os.environ.get("MPK_SSWEEP_W", "4"))
    out = {"apply_ms": ms.value}
    for ph, nm in ((0, "fwd"), (1, "bwd")):
        st, en = a[ph, :, 0], a[ph, :, 1]
        ng = int(np.count_nonzero(st))
        st, en = st[:ng], en[:ng]
        t0 = st.min()
        dur = (en - st) / 1e3
        d = np.diff(st) / 1e3
        intra = [d[i] for i in range(len(d)) if (i + 1) % W != 0]
        cross = [d[i] for i in range(len(d)) if (i + 1) % W == 0]
        out[nm] = {"groups": ng, "span_us": float((en.max() - t0) / 1e3),
                   "dur_us_min_med_max": [float(dur.min()), float(np.median(dur)), float(dur.max())],
                   "hop_intra_us_med": float(np.median(intra)) if intra else None,
                   "hop_cross_us_med": float(np.median(cross)) if cross else None,
                   "first_starts_us": [float(x) for x in (st[:10] - t0) / 1e3]}
    wb = (ctypes.c_int * 128)()
    L.mpk_swf_debugw(wb)
    out["warp_slots_fwd"] = list(wb[:8])
    if os.environ.get("SWF_DBG") == "2":
        cb = (ctypes.c_longlong * (2 * 2 * 512 * 6))()
        L.mpk_swf_debugc(cb)
        c = np.array(cb[:], dtype=np.int64).reshape(2, 2, 512, 6)
        names = ["ready_wait", "rec_wait", "steps", "x", "arrive"]
        for ph in range(2):
            for g in range(2):
                x = c[ph, g]
                x = x[x[:, 0] > 0]
                if len(x) < 3:
                    continue
                rec = {"n": int(len(x)), "chunk": float(np.median(x[1:, 0] - x[:-1, 0]))}
                for i, nm in enumerate(names):
                    rec[nm] = float(np.median(x[:, i + 1] - x[:, i]))
                out[f"chunks_ph{ph}_g{g}"] = rec
    print(json.dumps(out))
else:
    name = sys.argv[1]
    for w in sys.argv[2:] or ["4"]:
        env = dict(os.environ, MPK_SWEEP_PICK="swf", MPK_SSWEEP_W=w)
        r = subprocess.run([sys.executable, __file__, "child", name], env=env,
                           capture_output=True, text=True)
        print(f"[W={w}]", r.stdout.strip(), r.stderr.strip()[-800:], flush=True)
