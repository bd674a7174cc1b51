"""The shared exp/log (include/eq_math.h) against libm: <= 2 ulp.

These functions are the one piece of arithmetic the GPU and the CPU oracle
share; their accuracy bounds how far device mode can drift from the
reference's glibc exp/log (SURVEY.md §8(c) precision contract)."""

import ctypes

import numpy as np
import pytest

from oracle import oracle as orc


def _call(which, x):
    L = orc.lib()
    L.eqo_math.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    L.eqo_math(which, x.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p), x.size)
    return out


def _ulps64(a, b):
    ia = a.view(np.int64); ib = b.view(np.int64)
    ia = np.where(ia < 0, np.int64(-2**63) - ia, ia)
    ib = np.where(ib < 0, np.int64(-2**63) - ib, ib)
    return np.abs(ia - ib)


def _ulps32(a, b):
    a = a.astype(np.float32); b = b.astype(np.float32)
    ia = a.view(np.int32).astype(np.int64); ib = b.view(np.int32).astype(np.int64)
    ia = np.where(ia < 0, -2**31 - ia, ia)
    ib = np.where(ib < 0, -2**31 - ib, ib)
    return np.abs(ia - ib)


rng = np.random.default_rng(0)
HOT_EXP = np.concatenate([-rng.uniform(0, 0.2, 20000),         # -phi/tau, -u/tau
                          rng.uniform(-700, 700, 20000),
                          rng.uniform(-1, 1, 20000)])
HOT_LOG = np.concatenate([rng.uniform(0.998, 1.0, 20000),        # r in (k_m, 1]
                          np.exp(rng.uniform(-700, 700, 20000)),
                          rng.uniform(1e-6, 10, 20000)])


def test_exp_f64_within_2ulp():
    assert _ulps64(_call(0, HOT_EXP), np.exp(HOT_EXP)).max() <= 2


def test_log_f64_within_2ulp():
    assert _ulps64(_call(1, HOT_LOG), np.log(HOT_LOG)).max() <= 2


def test_exp_f32_within_2ulp():
    x = np.clip(HOT_EXP, -80, 80).astype(np.float32).astype(np.float64)
    ref = np.exp(x).astype(np.float32)
    assert _ulps32(_call(2, x), ref).max() <= 2


def test_log_f32_within_2ulp():
    x = HOT_LOG.astype(np.float32).astype(np.float64)
    x = x[(x > 1e-30) & (x < 1e30)]
    ref = np.log(x).astype(np.float32)
    assert _ulps32(_call(3, x), ref).max() <= 2


@pytest.mark.parametrize("which,x,want", [(0, 0.0, 1.0), (1, 1.0, 0.0), (2, 0.0, 1.0), (3, 1.0, 0.0)])
def test_exact_points(which, x, want):
    assert _call(which, np.array([x]))[0] == want


def test_special_values():
    assert np.isinf(_call(0, np.array([800.0]))[0])
    assert _call(0, np.array([-800.0]))[0] == 0.0
    assert np.isnan(_call(1, np.array([-1.0]))[0])
    assert _call(1, np.array([0.0]))[0] == -np.inf
