"""The C-ABI library loads (no GPU needed) and exports every function that
include/*.h declares; the Python binding covers all of them."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = []
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if not fn.startswith("eventq"):
            continue
        src = open(os.path.join(ROOT, "include", fn)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^[A-Za-z_][\w \t\*]*?\b(eq_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2512_05906_b200 import build as b
    path = b.build()
    return ctypes.CDLL(path)


def test_header_declares_the_api():
    names = declared_functions()
    for must in ("eq_create", "eq_set_network", "eq_set_drive", "eq_forward", "eq_backward", "eq_run"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_2512_05906_b200 import _native
    assert set(declared_functions()) <= set(_native.EXPORTED)


def test_version_string(lib):
    lib.eq_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.eq_version()


def test_create_without_gpu_reports_an_error_not_a_crash(lib):
    """eq_create on a box with no device must return a status, never fall back."""
    from paper_2512_05906_b200 import _native
    L = _native.lib()
    cfg = _native.Config()
    cfg.kind, cfg.precision, cfg.n_neurons, cfg.n_trials, cfg.t_steps = 0, 32, 10, 1, 10
    cfg.exact_delivery = 1
    cfg.dt, cfg.tau_m, cfg.tau_syn, cfg.v_th, cfg.v_reset = 1e-3, 1.0, 0.5, 1.0, 0.0
    h = ctypes.c_void_p()
    code = L.eq_create(ctypes.byref(cfg), 0, ctypes.byref(h))
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert code == 5  # EQ_ERR_CUDA
    if h.value:
        L.eq_destroy(h)


def test_configuration_is_validated_before_the_device(lib):
    from paper_2512_05906_b200 import _native
    L = _native.lib()
    cfg = _native.Config()
    cfg.kind, cfg.precision, cfg.n_neurons, cfg.n_trials, cfg.t_steps = 0, 32, 1, 1, 10
    cfg.dt, cfg.tau_m, cfg.tau_syn, cfg.v_th, cfg.v_reset = 1e-3, 1.0, 0.5, 1.0, 0.0
    h = ctypes.c_void_p()
    assert L.eq_create(ctypes.byref(cfg), 0, ctypes.byref(h)) == 1
    assert b"n >= 2" in L.eq_last_error(h)
    L.eq_destroy(h)
