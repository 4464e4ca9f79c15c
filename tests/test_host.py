"""CPU-side checks of the product: the C-ABI library loads and exports the
header's symbols, host MC scalar arithmetic is bitwise the reference's,
the problem generators reproduce the inputs the golden runs used, and
the drop-in API validates like the reference (ValueError paths)."""

from __future__ import annotations

import ctypes
import pathlib
import re

import numpy as np
import pytest

from conftest import ROOT, bits_equal, golden


def test_library_exports_every_header_symbol():
    from paper_2504_14498_b200 import _lib

    L = _lib.lib()
    hdr = (ROOT / "include" / "mpk_b200.h").read_text()
    declared = set(re.findall(r"\b(mpk_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name


def test_error_free_transformations_match_reference():
    """two_sum / two_prod exports over the whole exponent range, incl. the
    overflowing and underflowing cases (mc_scalar.npz, reference _mccore.py:19-51)."""
    import paper_2504_14498_b200 as mpk

    g = golden("mc_scalar.npz")
    ts = np.array([mpk.two_sum(a, b) for a, b in g["eft_in"]])
    tp = np.array([mpk.two_prod(a, b) for a, b in g["eft_in"]])
    assert np.array_equal(ts, g["two_sum"], equal_nan=True)
    assert np.array_equal(tp, g["two_prod"], equal_nan=True)
    finite = np.isfinite(g["two_prod"]).all(axis=1)
    assert bits_equal(tp[finite], g["two_prod"][finite])


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_mc_scalar_strings_and_complex_match_reference(k):
    """MCFloat.to_string (exact and 7 digits), from_string, and complex
    mul / div / sqrt, against the reference's outputs (mc_scalar.npz)."""
    import paper_2504_14498_b200 as mpk

    g = golden("mc_scalar.npz")
    P = mpk.Precision.from_k(k)
    vals = [mpk.MCFloat(tuple(v)) for v in g[f"k{k}_vals"]]
    assert [v.to_string() for v in vals] == list(g[f"k{k}_str"])
    assert [v.to_string(7) for v in vals] == list(g[f"k{k}_str7"])
    for v, s in zip(vals, g[f"k{k}_str"]):  # exact strings round-trip bitwise
        assert bits_equal(mpk.MCFloat.from_string(str(s), P).components, v.components)
    parsed = [mpk.MCFloat.from_string(str(t), P).components for t in g[f"k{k}_parse_in"]]
    assert bits_equal(np.array(parsed), g[f"k{k}_parse"])
    zs = [mpk.MCComplex(vals[i], vals[i + 1]) for i in range(0, 58, 2)]
    for name, res in (("cmul", [zs[i] * zs[i + 1] for i in range(len(zs) - 1)]),
                      ("cdiv", [zs[i] / zs[i + 1] for i in range(len(zs) - 1)]),
                      ("csqrt", [z.sqrt() for z in zs])):
        got = np.array([(z.re.components, z.im.components) for z in res])
        assert bits_equal(got, g[f"k{k}_{name}"]), name
    with pytest.raises(ValueError):
        mpk.MCFloat.from_string("not a number", P)
    with pytest.raises(ValueError):
        (-abs(vals[0]) - 1.0).sqrt()


def test_library_is_sm100a():
    so = ROOT / "paper_2504_14498_b200" / "_lib" / "libmpkb200.so"
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("k", [2, 3, 4])
def test_host_mc_scalars_bitwise(k):
    import paper_2504_14498_b200 as mpk

    g = golden("mc_ops.npz")
    P = mpk.Precision.from_k(k)
    a, b = g[f"k{k}_a"][:120], g[f"k{k}_b"][:120]
    for i in range(len(a)):
        x, y = mpk.MCFloat(tuple(a[i])), mpk.MCFloat(tuple(b[i]))
        assert bits_equal((x + y).components, g[f"k{k}_add"][i])
        assert bits_equal((x - y).components, g[f"k{k}_sub"][i])
        assert bits_equal((x * y).components, g[f"k{k}_mul"][i])
    idx = g[f"k{k}_div_idx"][:60]
    for j, i in enumerate(idx):
        q = mpk.MCFloat(tuple(g[f"k{k}_a"][i])) / mpk.MCFloat(tuple(g[f"k{k}_b"][i]))
        assert bits_equal(q.components, g[f"k{k}_div"][j])
    for i in range(40):
        s = mpk.MCFloat(tuple(g[f"k{k}_sqrt_in"][i])).sqrt()
        assert bits_equal(s.components, g[f"k{k}_sqrt"][i])
    for i in range(40):
        za = mpk.MCComplex(mpk.MCFloat(tuple(g[f"k{k}_car"][i])),
                           mpk.MCFloat(tuple(g[f"k{k}_cai"][i])))
        zb = mpk.MCComplex(mpk.MCFloat(tuple(g[f"k{k}_cbr"][i])),
                           mpk.MCFloat(tuple(g[f"k{k}_cbi"][i])))
        m = za * zb
        d = za / zb
        assert bits_equal(m.re.components, g[f"k{k}_cmul_re"][i])
        assert bits_equal(m.im.components, g[f"k{k}_cmul_im"][i])
        assert bits_equal(d.re.components, g[f"k{k}_cdiv_re"][i])
        assert bits_equal(d.im.components, g[f"k{k}_cdiv_im"][i])
    assert P.k == k


def test_problem_generators_match_golden_inputs():
    from paper_2504_14498_b200 import problems

    assert problems.cfg1().checksum() == str(golden("solver_cfg1.npz")["cfg1_checksum"])
    assert problems.cfg2().checksum() == str(golden("solver_cfg2.npz")["cfg2_checksum"])
    assert problems.cfg3().checksum() == str(golden("solver_cfg3.npz")["cfg3_checksum"])
    assert problems.cfg5(0).checksum() == str(golden("solver_cfg5.npz")["cfg5_0_checksum"])


def test_cfg_shapes():
    from paper_2504_14498_b200 import problems

    p1 = problems.cfg1()
    assert (p1.n, p1.nnz) == (4096, 20224)
    p3 = problems.cfg3(m=48)
    assert (p3.n, p3.nnz) == (110592, 760320)
    p4 = problems.cfg4(m=64)  # full size is exercised by bench.py
    assert p4.nnz == (3 * 64 - 2) ** 2
    p2 = problems.cfg2()
    assert p2.n == 20000 and 250_000 < p2.nnz < 270_000
    # strictly increasing columns, diagonal present in every row
    for p in (p1, p2, p3):
        rp, ci = p.row_ptr, p.col_idx
        row = np.repeat(np.arange(p.n), np.diff(rp))
        assert np.all((np.diff(ci) > 0) | (np.diff(row) > 0))
        assert np.count_nonzero(ci == row) == p.n


def test_api_validation_errors():
    import paper_2504_14498_b200 as mpk

    P = mpk.Precision.DD
    with pytest.raises(ValueError, match="unknown method"):
        mpk.SolverConfig(method="gmres")
    with pytest.raises(ValueError, match="mixed SpMV needs"):
        mpk.SolverConfig(precision=mpk.Precision.F64, spmv_mode="mixed")
    with pytest.raises(ValueError, match="eps_rel"):
        mpk.SolverConfig(eps_rel=0.0)
    with pytest.raises(ValueError, match="strictly increasing"):
        mpk.CsrMatrix(2, np.array([0, 2, 3]), np.array([1, 0, 1]),
                      np.ones((3, 2)), None, P)
    with pytest.raises(ValueError, match="row_ptr"):
        mpk.CsrMatrix(2, np.array([0, 2, 2]), np.array([0, 1, 1]),
                      np.ones((3, 2)), None, P)
    assert mpk.PrecondMode.from_label("ilu0-mixed") is mpk.PrecondMode.ILU0_MIXED
    assert mpk.Precision.from_label("qd").k == 4


def test_product_does_not_import_oracle():
    pkg = ROOT / "paper_2504_14498_b200"
    for f in pkg.rglob("*.py"):
        txt = f.read_text()
        assert "import oracle" not in txt and "from oracle" not in txt, f
    for f in list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        assert "mpk_oracle" not in f.read_text(), f


def test_integration_binding_signatures():
    """The reference-side ctypes stub in INTEGRATION.md declares argtypes that
    match include/mpk_b200.h parameter for parameter (an untyped Python int
    would travel as a 32-bit c_int into an int64_t parameter)."""
    doc = (ROOT / "INTEGRATION.md").read_text()
    hdr = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "mpk_b200.h").read_text(), flags=re.S)
    stubs = dict(re.findall(r"_L\.(mpk_\w+)\.argtypes = \[(.*?)\]", doc, flags=re.S))
    assert {"mpk_csr_upload", "mpk_solve", "mpk_ctx_create", "mpk_thread_set_option",
            "mpk_csr_set_mc_values", "mpk_csr_free"} <= set(stubs)
    scalar = {"int": "c_int", "int32_t": "c_int32", "int64_t": "c_int64", "double": "c_double"}
    for fn, arglist in stubs.items():
        args = [a.strip() for a in re.sub(r"#.*", "", arglist).replace("\n", " ").split(",")
                if a.strip()]
        # POINTER(x) contains no comma, so the split is positional
        m = re.search(rf"\b{fn}\s*\((.*?)\)\s*;", hdr, flags=re.S)
        assert m, fn
        params = [p.strip() for p in m.group(1).replace("\n", " ").split(",")]
        assert len(params) == len(args), (fn, params, args)
        for prm, arg in zip(params, args):
            if "*" in prm:
                assert arg == "c_void_p" or arg.startswith("POINTER("), (fn, prm, arg)
            else:
                ctype = prm.replace("const ", "").split()[0]
                assert scalar[ctype] == arg, (fn, prm, arg)


def test_first_use_paths_do_not_self_deadlock():
    """context() creates the device context under the module lock and loads
    the library inside it; the lock must be re-entrant (a solve() as the very
    first call of a process used to hang on itself).  Checked in a fresh
    interpreter without a GPU: the call must come back (with the CUDA error
    of a GPU-less box), not block."""
    import subprocess
    import sys

    code = ("import paper_2504_14498_b200._lib as L\n"
            "try:\n    L.context()\nexcept RuntimeError as e:\n    print('returned', type(e).__name__)\n"
            "else:\n    print('returned ok')\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=str(ROOT), capture_output=True,
                         text=True, timeout=120)
    assert "returned" in out.stdout, (out.stdout, out.stderr)
