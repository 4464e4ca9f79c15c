"""Generate tests/golden/mc_scalar.npz from the UNMODIFIED reference (run here,
where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_mc_scalar.py

Host scalar API of the drop-in (reference multicomponent.py / _mccore.py):
two_sum / two_prod over the whole exponent range, MCFloat.to_string (exact and
rounded), from_string, and complex mul / div / sqrt at k = 1..4.
"""
import pathlib
import random

import numpy as np

import mpkrylov as R
from mpkrylov import _mccore

rng = random.Random(20261021)
out = {}
n = 4000
ab = np.array([[rng.uniform(-1, 1) * 2.0 ** rng.randint(-1070, 1020) for _ in range(2)]
               for _ in range(n)])
out["eft_in"] = ab
out["two_sum"] = np.array([R.two_sum(a, b) for a, b in ab])
out["two_prod"] = np.array([R.two_prod(a, b) for a, b in ab])
for k in (1, 2, 3, 4):
    P = R.Precision.from_k(k)
    vals = []
    for _ in range(60):
        t = [rng.uniform(-1, 1) * 10.0 ** rng.randint(-30, 30) * 2.0 ** (-53 * i - rng.randint(0, 4))
             for i in range(k)]
        vals.append(_mccore.renormalize(t, k))
    vals = np.array(vals)
    out[f"k{k}_vals"] = vals
    out[f"k{k}_str"] = np.array([R.MCFloat(tuple(v)).to_string() for v in vals])
    out[f"k{k}_str7"] = np.array([R.MCFloat(tuple(v)).to_string(7) for v in vals])
    texts = ["0.1", "-2.5e-300", "3.14159265358979323846264338327950288419716939937510",
             "1e308", "-0", "7"]
    out[f"k{k}_parse_in"] = np.array(texts)
    out[f"k{k}_parse"] = np.array([R.MCFloat.from_string(s, P).components for s in texts])
    zs = [R.MCComplex(R.MCFloat(tuple(vals[i])), R.MCFloat(tuple(vals[i + 1])))
          for i in range(0, 58, 2)]
    prod = [zs[i] * zs[i + 1] for i in range(len(zs) - 1)]
    quot = [zs[i] / zs[i + 1] for i in range(len(zs) - 1)]
    roots = [z.sqrt() for z in zs]
    out[f"k{k}_cmul"] = np.array([(z.re.components, z.im.components) for z in prod])
    out[f"k{k}_cdiv"] = np.array([(z.re.components, z.im.components) for z in quot])
    out[f"k{k}_csqrt"] = np.array([(z.re.components, z.im.components) for z in roots])
np.savez_compressed(pathlib.Path(__file__).with_name("mc_scalar.npz"), **out)
print("wrote mc_scalar.npz")
