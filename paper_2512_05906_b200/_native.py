"""ctypes binding of the in-tree sm_100a library (lib/libeventq_b200.so).

There is no fallback: if the library is missing or cannot load, importing the
engine fails loudly (build it with ``python -m paper_2512_05906_b200.build`` or
``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os

from .errors import STATUS_TO_ERROR, EventQError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EQ_LIB_PATH") or os.path.join(HERE, "lib", "libeventq_b200.so")   # override: A/B runs

KIND_IDS = {"ring": 0, "fiforing": 1, "binaryheap": 2, "sortedarray": 3, "lossyring": 4, "donothing": 5}


class Config(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("precision", ctypes.c_int32), ("n_neurons", ctypes.c_int32),
        ("n_trials", ctypes.c_int32), ("t_steps", ctypes.c_int32), ("refractory_steps", ctypes.c_int32),
        ("exact_delivery", ctypes.c_int32), ("capacity", ctypes.c_int32), ("max_spikes", ctypes.c_int64),
        ("dt", ctypes.c_double), ("tau_m", ctypes.c_double), ("tau_syn", ctypes.c_double),
        ("v_th", ctypes.c_double), ("v_reset", ctypes.c_double),
        ("max_ctas", ctypes.c_int32), ("staged_queues", ctypes.c_int32),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the B200 extension is not built "
            "(run `python -m paper_2512_05906_b200.build`); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    H = ctypes.c_void_p
    sig = {
        "eq_create": (ctypes.c_int, [ctypes.POINTER(Config), ctypes.c_int, ctypes.POINTER(H)]),
        "eq_destroy": (ctypes.c_int, [H]),
        "eq_last_error": (ctypes.c_char_p, [H]),
        "eq_version": (ctypes.c_char_p, []),
        "eq_set_network": (ctypes.c_int, [H, vp, vp, vp, vp, i64, vp]),
        "eq_set_drive": (ctypes.c_int, [H, vp, vp, vp]),
        "eq_poisson_drive": (ctypes.c_int, [i32, i32, i32, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                            ctypes.c_uint64, vp, vp]),
        "eq_reset": (ctypes.c_int, [H, vp]),
        "eq_run": (ctypes.c_int, [H, i32, vp, vp]),
        "eq_forward": (ctypes.c_int, [H, vp, vp, vp, vp]),
        "eq_backward": (ctypes.c_int, [H, vp, vp, vp, vp, vp, vp]),
        "eq_get_state": (ctypes.c_int, [H, vp, vp, vp]),
        "eq_forward_jvp": (ctypes.c_int, [H, i32, vp, vp, vp, vp, vp]),
        "eq_backward_begin": (ctypes.c_int, [H, vp, vp, vp, vp, vp, vp]),
        "eq_backward_window": (ctypes.c_int, [H, i32, vp]),
        "eq_set_partition": (ctypes.c_int, [H, i32, i32]),
        "eq_set_frac_bits": (ctypes.c_int, [H, i32]),
        "eq_export_spikes": (ctypes.c_int, [H, i32, i32, vp, ctypes.POINTER(i64), vp]),
        "eq_import_spikes": (ctypes.c_int, [H, vp, i64, vp]),
        "eq_get_import_adjoints": (ctypes.c_int, [H, i32, vp, vp]),
        "eq_add_spike_adjoints": (ctypes.c_int, [H, i32, vp, i64, vp]),
        "eq_set_peers": (ctypes.c_int, [H, i32, vp, i32]),
        "eq_run_window": (ctypes.c_int, [H, i32, i32, i32, vp]),
        "eq_backward_window_peer": (ctypes.c_int, [H, i32, i32, i32, vp]),
        "eq_sync": (ctypes.c_int, [H, vp]),
        "eq_counters": (ctypes.c_int, [H, vp, vp]),
        "eq_spike_count": (i64, [H, vp]),
        "eq_get_spikes": (ctypes.c_int, [H, vp, vp, vp, vp, vp]),
        "eq_get_pending": (ctypes.c_int, [H, vp, vp]),
        "eq_horizon": (ctypes.c_int, [H]),
        "eq_frac_bits": (ctypes.c_int, [H]),
        "eq_geometry": (ctypes.c_int, [H, vp, vp]),
        "eq_launch_count": (i64, [H]),
        "eq_debug_timeline": (ctypes.c_int, [H, ctypes.c_int, vp]),
        "eq_log_capacity": (i64, [H, ctypes.POINTER(i32)]),
        "eq_debug_set_bucket_capacity": (ctypes.c_int, [H, i64]),
        "eq_debug_set_admission_slots": (ctypes.c_int, [H, i32]),
        "eq_queues_create": (ctypes.c_int, [ctypes.c_int] * 6 + [ctypes.POINTER(H)]),
        "eq_queues_destroy": (ctypes.c_int, [H]),
        "eq_queues_last_error": (ctypes.c_char_p, [H]),
        "eq_queues_capacity": (ctypes.c_int, [H]),
        "eq_queues_now": (ctypes.c_int, [H]),
        "eq_queues_enqueue": (ctypes.c_int, [H, vp, vp, vp, vp, vp, i64, vp, vp]),
        "eq_queues_pop": (ctypes.c_int, [H, vp, vp, vp, vp, vp]),
        "eq_queues_occupancy": (ctypes.c_int, [H, vp, vp]),
        "eq_queues_run_poisson": (ctypes.c_int, [H, vp, i32, i32, vp, vp, vp]),
        "eq_queues_lossy_counts": (ctypes.c_int, [H, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTED = ("eq_create", "eq_destroy", "eq_last_error", "eq_version", "eq_set_network", "eq_set_drive", "eq_poisson_drive",
            "eq_reset", "eq_run", "eq_forward", "eq_backward", "eq_get_state", "eq_forward_jvp", "eq_backward_begin", "eq_backward_window",
            "eq_set_partition", "eq_set_frac_bits", "eq_export_spikes", "eq_import_spikes",
            "eq_get_import_adjoints", "eq_add_spike_adjoints", "eq_set_peers", "eq_run_window",
            "eq_backward_window_peer", "eq_sync", "eq_counters", "eq_spike_count",
            "eq_get_spikes", "eq_get_pending", "eq_horizon", "eq_frac_bits", "eq_geometry",
            "eq_launch_count", "eq_debug_timeline", "eq_log_capacity", "eq_debug_set_bucket_capacity",
            "eq_debug_set_admission_slots",
            "eq_queues_create", "eq_queues_destroy",
            "eq_queues_last_error", "eq_queues_capacity", "eq_queues_now", "eq_queues_enqueue", "eq_queues_pop",
            "eq_queues_occupancy", "eq_queues_lossy_counts", "eq_queues_run_poisson")


def check(handle, code: int, queues: bool = False) -> None:
    if code == 0:
        return
    msg = (lib().eq_queues_last_error if queues else lib().eq_last_error)(handle)
    msg = msg.decode() if msg else ""
    raise STATUS_TO_ERROR.get(code, EventQError)(msg)
