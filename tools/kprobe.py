"""Factor + a few ILU(0)-mixed applies + a few mixed SpMVs of one config (ncu target).

usage: python tools/kprobe.py cfg4 [k] [reps]     (cfg5 = system 0)
"""
import ctypes
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2504_14498_b200 import _lib, problems  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
L = _lib.lib()
ctx = _lib.context(0)
p = problems.CONFIGS[name](0) if name == "cfg5" else problems.CONFIGS[name]()
h = ctypes.c_void_p()
vim = None if p.val_im is None else _lib.f64(p.val_im)
_lib.check(L.mpk_csr_upload(ctx, ctypes.c_int64(p.n), ctypes.c_int64(p.nnz),
                            _lib.dptr(_lib.i64(p.row_ptr)), _lib.dptr(_lib.i64(p.col_idx)),
                            _lib.dptr(_lib.f64(p.val_re)), _lib.dptr(vim), ctypes.byref(h)))
bad = ctypes.c_int64()
st = ctypes.c_int32()
_lib.check(L.mpk_ilu0_factor(h, ctypes.byref(bad), ctypes.byref(st)))
ms = ctypes.c_double()
_lib.check(L.mpk_bench_apply(h, ctypes.c_int(k), ctypes.c_int(reps), ctypes.byref(ms)))
print(name, "apply ms", ms.value)
_lib.check(L.mpk_bench_spmv(h, ctypes.c_int(k), ctypes.c_int(reps), ctypes.byref(ms)))
print(name, "spmv ms", ms.value)
