"""ctypes wrapper of the CPU oracle (oracle/eq_oracle.cpp).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libeqoracle.so")
_lib = None

KINDS = {"ring": 0, "fiforing": 1, "binaryheap": 2, "sortedarray": 3, "lossyring": 4, "donothing": 5}
STATUS = {0: "ok", 1: "ConfigurationError", 2: "CapabilityError", 3: "CausalityError",
          4: "GrazingCrossingError", 5: "InternalError"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS.get(code, str(code))


class _Cfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "kind", "n", "n_trials", "t_steps", "refractory_steps", "exact_delivery",
        "capacity", "frac_bits", "mode", "precision", "record_v", "pad")] + \
        [(n, ctypes.c_double) for n in ("dt", "tau_m", "tau_syn", "v_th", "v_reset")]


def build() -> str:
    """Compile the oracle with its Makefile (g++ only, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        vp = ctypes.c_void_p
        L.eqo_create.restype = vp
        L.eqo_create.argtypes = [ctypes.POINTER(_Cfg)]
        L.eqo_destroy.argtypes = [vp]
        L.eqo_error.restype = ctypes.c_char_p
        L.eqo_error.argtypes = [vp]
        for name in ("eqo_set_network", "eqo_set_drive", "eqo_forward", "eqo_backward",
                     "eqo_horizon"):
            getattr(L, name).restype = ctypes.c_int
        L.eqo_set_network.argtypes = [vp] * 5
        L.eqo_set_drive.argtypes = [vp] * 3
        L.eqo_forward.argtypes = [vp]
        L.eqo_backward.argtypes = [vp] * 6
        L.eqo_horizon.argtypes = [vp]
        L.eqo_spike_count.restype = ctypes.c_int64
        L.eqo_spike_count.argtypes = [vp]
        L.eqo_get_spikes.argtypes = [vp] * 7
        L.eqo_get_state.argtypes = [vp] * 3
        L.eqo_get_vtrace.argtypes = [vp] * 2
        L.eqo_get_counters.argtypes = [vp] * 2
        L.eqo_get_pending.argtypes = [vp] * 3
        L.eqo_threads.restype = ctypes.c_int
        L.eqo_philox4x32_10.argtypes = [vp] * 3
        L.eqo_poisson_drive.argtypes = [ctypes.c_int32] * 3 + [ctypes.c_double] * 3 + [ctypes.c_uint64, vp]
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def frac_bits(max_in_weight: float, bits: int) -> int:
    """Fixed-point fraction bits: largest F with 4*max_in*2^F <= 2^(bits-2).

    Restated from the engine's rule: a slot (target, step) gets
    at most two events per incoming edge, each |payload| <= |w|.
    """
    bound = 4.0 * max_in_weight
    if bound <= 0.0:
        return bits - 2
    m, e = math.frexp(bound)           # bound = m * 2^e, m in [0.5, 1)
    ceil_log2 = e - 1 if m == 0.5 else e
    return (bits - 2) - ceil_log2


class OracleSession:
    """One simulation configuration (all trials) on the CPU oracle.

    mode="reference": double + libm + reference summation order
    mode="device":    precision 32/64, eq_math exp/log, fixed-point slots
    """

    def __init__(self, *, n: int, n_trials: int, t_steps: int, kind: str = "ring",
                 dt: float = 1e-3, tau_m: float = 1.0, tau_syn: float = 0.5,
                 v_th: float = 1.0, v_reset: float = 0.0, refractory_steps: int = 0,
                 exact_delivery: bool = True, capacity: int = 0, frac_bits: int = 0,
                 mode: str = "device", precision: int = 32, record_v: bool = False):
        self.L = lib()
        cfg = _Cfg()
        cfg.kind = KINDS[kind]
        cfg.n, cfg.n_trials, cfg.t_steps = n, n_trials, t_steps
        cfg.refractory_steps = refractory_steps
        cfg.exact_delivery = int(bool(exact_delivery))
        cfg.capacity = capacity
        cfg.frac_bits = frac_bits
        cfg.mode = 0 if mode == "reference" else 1
        cfg.precision = precision
        cfg.record_v = int(bool(record_v))
        cfg.dt, cfg.tau_m, cfg.tau_syn, cfg.v_th, cfg.v_reset = dt, tau_m, tau_syn, v_th, v_reset
        self.cfg = cfg
        self.n, self.B, self.T = n, n_trials, t_steps
        self.h = self.L.eqo_create(ctypes.byref(cfg))
        self._keep = []

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.L.eqo_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def _check(self, code: int):
        if code != 0:
            raise OracleError(code, self.L.eqo_error(self.h).decode())

    def _cast(self, a: np.ndarray) -> np.ndarray:
        """Values as the working precision sees them, carried in float64."""
        a = np.asarray(a, dtype=np.float64)
        if self.cfg.mode == 1 and self.cfg.precision == 32:
            a = a.astype(np.float32).astype(np.float64)
        return np.ascontiguousarray(a)

    def set_network(self, rowptr, col, weight, delay):
        rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
        col = np.ascontiguousarray(col, dtype=np.int32)
        w = self._cast(weight)
        d = self._cast(delay)
        self._keep += [rowptr, col, w, d]
        self._check(self.L.eqo_set_network(self.h, _p(rowptr), _p(col), _p(w), _p(d)))
        self.horizon = self.L.eqo_horizon(self.h)

    def set_drive(self, mask: np.ndarray, amp):
        mask = np.ascontiguousarray(mask, dtype=np.uint32)
        amp = self._cast(amp)
        assert mask.shape == (self.B, self.T, (self.n + 31) // 32)
        self._keep += [mask, amp]
        self._check(self.L.eqo_set_drive(self.h, _p(mask), _p(amp)))

    def forward(self) -> Dict[str, np.ndarray]:
        self._check(self.L.eqo_forward(self.h))
        S = self.L.eqo_spike_count(self.h)
        step = np.empty(S, np.int32); trial = np.empty(S, np.int32); neuron = np.empty(S, np.int32)
        t = np.empty(S); a = np.empty(S); vh = np.empty(S)
        self.L.eqo_get_spikes(self.h, _p(step), _p(trial), _p(neuron), _p(t), _p(a), _p(vh))
        v = np.empty((self.B, self.n)); i = np.empty((self.B, self.n))
        self.L.eqo_get_state(self.h, _p(v), _p(i))
        cnt = np.empty((self.B, 3), np.int64)
        self.L.eqo_get_counters(self.h, _p(cnt))
        out = dict(step=step, trial=trial, neuron=neuron, t=t, a=a, vh=vh, v=v, i=i,
                   counters=cnt)
        H = self.horizon
        if self.cfg.mode == 1:
            pend = np.empty((self.B, self.n, H, 2), np.int64)
            self.L.eqo_get_pending(self.h, _p(pend), None)
        else:
            pend = np.empty((self.B, self.n, H, 2), np.float64)
            self.L.eqo_get_pending(self.h, None, _p(pend))
        out["pending"] = pend
        if self.cfg.record_v:
            tr = np.empty((self.B, self.T, self.n))
            self.L.eqo_get_vtrace(self.h, _p(tr))
            out["v_trace"] = tr
        return out

    def backward(self, vbar: np.ndarray, ibar: Optional[np.ndarray] = None):
        E = int(self._keep[1].shape[0]) if self._keep else 0
        vbar = np.ascontiguousarray(vbar, dtype=np.float64)
        ibar_ = None if ibar is None else np.ascontiguousarray(ibar, dtype=np.float64)
        gw = np.empty(E); gd = np.empty(E); ga = np.empty(self.n)
        self._check(self.L.eqo_backward(self.h, _p(vbar), _p(ibar_), _p(gw), _p(gd), _p(ga)))
        return gw, gd, ga


def threads() -> int:
    return lib().eqo_threads()


def philox4x32_10(ctr, key) -> np.ndarray:
    """Philox4x32-10 block (restated in eq_oracle.cpp; Random123 KATs pin it)."""
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().eqo_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def poisson_drive(n: int, n_trials: int, t_steps: int, dt: float, mean_interval: float,
                  pulse_duration: float, seed: int) -> np.ndarray:
    """CPU restatement of eq_poisson_drive: packed mask uint32 [B][T][ceil(n/32)]."""
    out = np.zeros((n_trials, t_steps, (n + 31) // 32), dtype=np.uint32)
    lib().eqo_poisson_drive(n, n_trials, t_steps, dt, mean_interval, pulse_duration, seed, _p(out))
    return out
