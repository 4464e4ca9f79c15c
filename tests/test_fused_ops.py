"""Fused sweep primitives of the working-precision ILU(0) (
reference _mcfast.py:80-183 rmulsubK / rmulK): the library's MC code
(csrc/mc.cuh fmulsub / fmul, host build through mpk_mc_host) against the
reference's own outputs (tests/golden/mc_fused.npz), bit for bit.  The GPU
twin of the same templates is checked in tests/test_gpu_parity.py."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

from conftest import bits_equal, golden


def _host(op, k, a, b, c=None):
    from paper_2504_14498_b200 import _lib

    arr = lambda v: (ctypes.c_double * 4)(*list(v) + [0.0] * (4 - len(v)))  # noqa: E731
    o = (ctypes.c_double * 4)()
    rc = _lib.lib().mpk_mc_host(ctypes.c_int(op), ctypes.c_int(k), arr(a),
                                None if c is None else arr(c), arr(b), None, o, None)
    _lib.check(rc)
    return np.array(o[:k])


@pytest.mark.parametrize("k", [2, 3, 4])
def test_fused_mulsub_and_mul_bitwise(k):
    g = golden("mc_fused.npz")
    A, B, C = g[f"k{k}_a"], g[f"k{k}_b"], g[f"k{k}_c"]
    ms = np.array([_host(11, k, a, b, c) for a, b, c in zip(A, B, C)])
    mu = np.array([_host(12, k, a, b) for a, b in zip(A, B)])
    assert bits_equal(ms, g[f"k{k}_mulsub"])
    assert bits_equal(mu, g[f"k{k}_mul"])
