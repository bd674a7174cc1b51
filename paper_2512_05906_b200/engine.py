"""Device engine: one C-ABI handle (include/eventq_b200.h) on one GPU.

PyTorch is only the tensor shell here: it owns the caller-side device buffers
and provides the CUDA stream; every simulation step and its reverse run inside
the sm_100a kernels of ``lib/libeventq_b200.so``.
"""

from __future__ import annotations

import ctypes
from typing import Dict, Optional, Tuple

import numpy as np
import torch

from . import _native
from .errors import ConfigurationError
from .workload import LIFConfig


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class Engine:
    """Batched R-SNN simulation of ``n_trials`` trials sharing one network.

    Mirrors ``build_rsnn`` + ``simulate`` (network.py:201-497) for every
    network kind (ring, lossyring, fiforing, binaryheap, sortedarray,
    donothing), plus the reverse pass (``backward``) the reference lacks.

    staged_queues selects the bounded-kind implementation (same results):
    0 = by admission on the calendar (default; heap, sorted, and FIFO with its
    delay on the step grid), 1 = shared-memory staged queues, 2 = HBM-resident
    queue structures.  max_ctas caps the persistent grid (partitions sharing a
    GPU); stream = a private stream (ordered after the caller's current one).
    """

    def __init__(self, n: int, n_trials: int, t_steps: int, *, kind: str = "ring",
                 precision: int = 32, lif: Optional[LIFConfig] = None, capacity: int = 0,
                 max_spikes: int = 0, device: Optional[int] = None,
                 partition: Optional[Tuple[int, int]] = None, max_ctas: int = 0,
                 stream: Optional[torch.cuda.Stream] = None, staged_queues: int = 0):
        self.L = _native.lib()
        if kind not in _native.KIND_IDS:
            raise ConfigurationError(f"unknown queue kind {kind!r}")
        lif = lif or LIFConfig()
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device)
        self.n, self.B, self.T = n, n_trials, t_steps
        self.kind, self.precision, self.lif = kind, precision, lif
        self.dtype = torch.float32 if precision == 32 else torch.float64
        cfg = _native.Config()
        cfg.kind = _native.KIND_IDS[kind]
        cfg.precision = precision
        cfg.n_neurons, cfg.n_trials, cfg.t_steps = n, n_trials, t_steps
        cfg.refractory_steps = lif.refractory_steps
        cfg.exact_delivery = int(bool(lif.exact_delivery))
        cfg.capacity = capacity
        cfg.max_spikes = max_spikes
        cfg.dt, cfg.tau_m, cfg.tau_syn = lif.dt, lif.tau_m, lif.tau_syn
        cfg.v_th, cfg.v_reset = lif.v_th, lif.v_reset
        cfg.max_ctas = max_ctas
        cfg.staged_queues = int(staged_queues)   # 0 admission, 1 smem-staged, 2 HBM structures
        self.cfg = cfg
        self._stream = stream      # None: the device's current torch stream at each call
        h = ctypes.c_void_p()
        code = self.L.eq_create(ctypes.byref(cfg), device, ctypes.byref(h))
        self.h = h
        _native.check(self.h, code)
        self._net = None
        self._drive = None
        # bumped by every call that changes the recorded forward run (spike log,
        # queues): a reverse pass saved against an older run id is stale
        self.run_id = 0
        # partitioned network (paper_2512_05906_b200.partition): this engine owns
        # neurons [offset, offset + n) of an n_global-neuron network
        self.n_global, self.offset = (n, 0) if partition is None else (int(partition[0]), int(partition[1]))
        if partition is not None:
            _native.check(self.h, self.L.eq_set_partition(self.h, self.n_global, self.offset))

    # ------------------------------------------------------------ lifetime
    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.L.eq_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def torch_stream(self) -> torch.cuda.Stream:
        return self._stream if self._stream is not None else torch.cuda.current_stream(self.device)

    @property
    def stream(self):
        """cudaStream_t for an ABI call.  With a private stream (partitions
        running concurrently) the call is ordered after the caller's current
        stream (its inputs) and the caller's stream after it (its outputs)."""
        if self._stream is not None:
            cur = torch.cuda.current_stream(self.device)
            if cur.cuda_stream != self._stream.cuda_stream:
                self._stream.wait_stream(cur)
                self._join_pending = True
        return ctypes.c_void_p(self.torch_stream.cuda_stream)

    def _join(self) -> None:
        if self._stream is not None and getattr(self, "_join_pending", False):
            torch.cuda.current_stream(self.device).wait_stream(self._stream)
            self._join_pending = False

    def _dev(self, a, dtype) -> torch.Tensor:
        if isinstance(a, torch.Tensor):
            return a.to(device=self.device, dtype=dtype).contiguous()
        return torch.as_tensor(np.ascontiguousarray(a)).to(device=self.device, dtype=dtype).contiguous()

    # ------------------------------------------------------------ inputs
    def set_network(self, rowptr, col, weight, delay) -> None:
        rp = self._dev(rowptr, torch.int64)
        cl = self._dev(col, torch.int32)
        w = self._dev(weight, self.dtype)
        d = self._dev(delay, self.dtype)
        if rp.numel() != self.n_global + 1:
            raise ConfigurationError(f"rowptr must have n+1 = {self.n_global + 1} entries")
        E = cl.numel()
        if w.numel() != E or d.numel() != E:
            raise ConfigurationError("weight/delay must have one entry per edge")
        self._net = (rp, cl, w, d)
        self.run_id += 1                     # eq_set_network resets the run
        _native.check(self.h, self.L.eq_set_network(self.h, _ptr(rp), _ptr(cl), _ptr(w), _ptr(d), E,
                                                      self.stream))
        self.n_edges = E

    def set_drive(self, mask, amp) -> None:
        m = self._dev(np.asarray(mask, dtype=np.uint32).view(np.int32) if not isinstance(mask, torch.Tensor)
                      else mask, torch.int32)
        words = (self.n + 31) // 32
        if tuple(m.shape) != (self.B, self.T, words):
            raise ConfigurationError(f"drive mask must be [{self.B}, {self.T}, {words}] uint32")
        a = self._dev(amp, self.dtype)
        if a.numel() != self.n:
            raise ConfigurationError("amplitude must have n entries")
        self._drive = (m, a)
        _native.check(self.h, self.L.eq_set_drive(self.h, _ptr(m), _ptr(a), self.stream))

    def set_poisson_drive(self, amp, mean_interval: float, pulse_duration: float, seed: int) -> None:
        """Drive generated on the device (eq_poisson_drive): the reference's
        PoissonDrive (network.py:98-155) pulse trains with a Philox stream per
        (trial, neuron) — same statistics as the reference's draws."""
        m = poisson_drive_device(self.n, self.B, self.T, self.lif.dt, mean_interval, pulse_duration, seed,
                                 device=self.device, stream=self.stream)
        self.set_drive(m, amp)

    # ------------------------------------------------------------ running
    def forward(self, record_v: bool = False) -> Dict[str, torch.Tensor]:
        v = torch.empty(self.B, self.n, dtype=self.dtype, device=self.device)
        i = torch.empty_like(v)
        tr = torch.empty(self.T, self.B, self.n, dtype=self.dtype, device=self.device) if record_v else None
        self.run_id += 1
        _native.check(self.h, self.L.eq_forward(self.h, _ptr(v), _ptr(i), _ptr(tr), self.stream))
        self._join()
        out = {"v": v, "i": i}
        if record_v:
            out["v_trace"] = tr
        return out

    def forward_jvp(self, kinds, indices):
        """Forward mode for D seeded directions at once (network.py:668-683):
        kinds[d] in {"weight", "delay", "drive"}, indices[d] = CSR edge
        (weight/delay) or neuron (drive).  Runs the whole drive from rest;
        returns (v [B, n], v_tangent [D, B, n]) in float64."""
        code = {"weight": 0, "delay": 1, "drive": 2}
        k = np.asarray([code[x] if isinstance(x, str) else int(x) for x in kinds], dtype=np.int32)
        ix = np.asarray(indices, dtype=np.int64)
        if k.shape != ix.shape or k.ndim != 1:
            raise ConfigurationError("kinds and indices must be 1-d of equal length")
        v = torch.empty(self.B, self.n, dtype=torch.float64, device=self.device)
        vt = torch.empty(len(k), self.B, self.n, dtype=torch.float64, device=self.device)
        self.run_id += 1
        _native.check(self.h, self.L.eq_forward_jvp(self.h, len(k), k.ctypes.data_as(ctypes.c_void_p),
                                                     ix.ctypes.data_as(ctypes.c_void_p), _ptr(v), _ptr(vt),
                                                     self.stream))
        return v, vt

    def state(self) -> Dict[str, torch.Tensor]:
        """Current membrane and synaptic current, [n_trials, n]."""
        v = torch.empty(self.B, self.n, dtype=self.dtype, device=self.device)
        i = torch.empty_like(v)
        _native.check(self.h, self.L.eq_get_state(self.h, _ptr(v), _ptr(i), self.stream))
        self._join()
        return {"v": v, "i": i}

    def reset(self) -> None:
        self.run_id += 1
        _native.check(self.h, self.L.eq_reset(self.h, self.stream))

    def run(self, n_steps: int, v_trace: Optional[torch.Tensor] = None) -> None:
        self.run_id += 1
        _native.check(self.h, self.L.eq_run(self.h, n_steps, _ptr(v_trace), self.stream))

    def backward(self, v_bar: torch.Tensor, i_bar: Optional[torch.Tensor] = None, want_amp: bool = True):
        vb = self._dev(v_bar, self.dtype)
        ib = None if i_bar is None else self._dev(i_bar, self.dtype)
        gw = torch.empty(self.n_edges, dtype=torch.float64, device=self.device)
        gd = torch.empty_like(gw)
        ga = torch.empty(self.n, dtype=torch.float64, device=self.device) if want_amp else None
        _native.check(self.h, self.L.eq_backward(self.h, _ptr(vb), _ptr(ib), _ptr(gw), _ptr(gd), _ptr(ga),
                                                  self.stream))
        self._join()
        return gw, gd, ga

    def backward_begin(self, v_bar: torch.Tensor, i_bar: Optional[torch.Tensor] = None, want_amp: bool = True):
        """Start a windowed reverse pass; returns the (grad_w, grad_d, grad_amp)
        buffers the windows accumulate into (final after the window at step 0)."""
        vb = self._dev(v_bar, self.dtype)
        ib = None if i_bar is None else self._dev(i_bar, self.dtype)
        gw = torch.empty(self.n_edges, dtype=torch.float64, device=self.device)
        gd = torch.empty_like(gw)
        ga = torch.empty(self.n, dtype=torch.float64, device=self.device) if want_amp else None
        self._bw = (vb, ib)
        _native.check(self.h, self.L.eq_backward_begin(self.h, _ptr(vb), _ptr(ib), _ptr(gw), _ptr(gd), _ptr(ga),
                                                        self.stream))
        return gw, gd, ga

    def backward_window(self, m_lo: int) -> None:
        _native.check(self.h, self.L.eq_backward_window(self.h, int(m_lo), self.stream))

    # ------------------------------------------------------------ partitions
    @property
    def spike_words(self) -> int:
        """int32 words per wire spike record (eq_spike_f32 / eq_spike_f64)."""
        return 4 if self.precision == 32 else 6

    def set_frac_bits(self, frac_bits: int) -> None:
        _native.check(self.h, self.L.eq_set_frac_bits(self.h, int(frac_bits)))

    def export_spikes(self, step_lo: int, step_hi: int) -> torch.Tensor:
        """Own spikes of steps [step_lo, step_hi) as wire records, int32 [n, spike_words]."""
        n = ctypes.c_int64()
        _native.check(self.h, self.L.eq_export_spikes(self.h, step_lo, step_hi, None, ctypes.byref(n), self.stream))
        out = torch.empty(n.value, self.spike_words, dtype=torch.int32, device=self.device)
        if n.value:
            _native.check(self.h, self.L.eq_export_spikes(self.h, step_lo, step_hi, _ptr(out), ctypes.byref(n),
                                                           self.stream))
        return out

    def import_spikes(self, recs: torch.Tensor) -> None:
        recs = recs.to(device=self.device, dtype=torch.int32).contiguous()
        if recs.numel() and (recs.dim() != 2 or recs.shape[1] != self.spike_words):
            raise ConfigurationError(f"spike records must be int32 [n, {self.spike_words}]")
        self._imp_keep = recs
        _native.check(self.h, self.L.eq_import_spikes(self.h, _ptr(recs), recs.shape[0] if recs.numel() else 0,
                                                       self.stream))

    def import_adjoints(self, start_step: int, n: int) -> torch.Tensor:
        out = torch.zeros(n, dtype=self.dtype, device=self.device)
        if n:
            _native.check(self.h, self.L.eq_get_import_adjoints(self.h, int(start_step), _ptr(out), self.stream))
        return out

    def add_spike_adjoints(self, step_lo: int, vals: torch.Tensor) -> None:
        v = self._dev(vals, self.dtype)
        self._adj_keep = v
        _native.check(self.h, self.L.eq_add_spike_adjoints(self.h, int(step_lo), _ptr(v), v.numel(), self.stream))

    # ------------------------------------------------------------ device-resident peer exchange
    def set_peers(self, engines, me: int) -> None:
        """Partitions of one network that read each other's spike logs directly
        (eq_set_peers): engines[k] is partition k, this engine is engines[me]."""
        arr = (ctypes.c_void_p * len(engines))(*[e.h.value for e in engines])
        self._peers = list(engines)
        _native.check(self.h, self.L.eq_set_peers(self.h, len(engines), arr, int(me)))

    def run_window(self, w: int, a_prev: int, n_steps: int) -> None:
        self.run_id += 1
        _native.check(self.h, self.L.eq_run_window(self.h, int(w), int(a_prev), int(n_steps), self.stream))

    def backward_window_peer(self, w: int, m_lo: int, a_next: int) -> None:
        _native.check(self.h, self.L.eq_backward_window_peer(self.h, int(w), int(m_lo), int(a_next), self.stream))

    def sync(self) -> None:
        """Wait for this engine's stream; raise the device error of any
        asynchronous window."""
        _native.check(self.h, self.L.eq_sync(self.h, ctypes.c_void_p(self.torch_stream.cuda_stream)))

    # ------------------------------------------------------------ queries
    def counters(self) -> np.ndarray:
        out = np.empty((self.B, 3), dtype=np.int64)
        _native.check(self.h, self.L.eq_counters(self.h, out.ctypes.data_as(ctypes.c_void_p), self.stream))
        return out

    def spike_count(self) -> int:
        n = self.L.eq_spike_count(self.h, self.stream)
        if n < 0:
            _native.check(self.h, 5)
        return int(n)

    def spikes(self) -> Dict[str, np.ndarray]:
        """Spike records sorted by (trial, step, neuron)."""
        S = self.spike_count()
        step = torch.empty(S, dtype=torch.int32, device=self.device)
        trial = torch.empty_like(step)
        neuron = torch.empty_like(step)
        t = torch.empty(S, dtype=self.dtype, device=self.device)
        if S:
            _native.check(self.h, self.L.eq_get_spikes(self.h, _ptr(step), _ptr(trial), _ptr(neuron), _ptr(t),
                                                        self.stream))
            self._join()
        st, tr, ne, tt = (x.cpu().numpy() for x in (step, trial, neuron, t))
        order = np.lexsort((ne, st, tr))
        return {"step": st[order], "trial": tr[order], "neuron": ne[order], "t": tt[order]}

    def pending(self) -> np.ndarray:
        H = self.horizon
        out = np.empty((self.B, self.n, H, 2), dtype=np.int64)
        _native.check(self.h, self.L.eq_get_pending(self.h, out.ctypes.data_as(ctypes.c_void_p), self.stream))
        return out

    @property
    def horizon(self) -> int:
        return int(self.L.eq_horizon(self.h))

    @property
    def frac_bits(self) -> int:
        return int(self.L.eq_frac_bits(self.h))

    @property
    def geometry(self):
        c = ctypes.c_int32()
        t = ctypes.c_int32()
        self.L.eq_geometry(self.h, ctypes.byref(c), ctypes.byref(t))
        return c.value, t.value

    @property
    def launch_count(self) -> int:
        return int(self.L.eq_launch_count(self.h))

    def log_capacity(self):
        """(spike-log capacity in records, times eq_run grew it)."""
        g = ctypes.c_int32()
        cap = int(self.L.eq_log_capacity(self.h, ctypes.byref(g)))
        return cap, g.value

    def debug_set_bucket_capacity(self, cap: int) -> None:
        """Test hook: shrink the ring kind's calendar buckets so events spill
        into the DRAM overflow ring (the rarely-taken path); next reset on."""
        _native.check(self.h, self.L.eq_debug_set_bucket_capacity(self.h, int(cap)))

    def debug_set_admission_slots(self, k: int) -> None:
        """Test hook (heap / sorted by admission): record arrival keys for the
        reference-order fix-ups only while a queue's room is below k; 0 sends
        every fix-up through the in-edge walk."""
        _native.check(self.h, self.L.eq_debug_set_admission_slots(self.h, int(k)))


def poisson_drive_device(n: int, n_trials: int, t_steps: int, dt: float, mean_interval: float,
                         pulse_duration: float, seed: int, device=0, stream=None) -> torch.Tensor:
    """Packed active-step masks int32 [B][T][ceil(n/32)] generated on the GPU
    (eq_poisson_drive); bitwise equal to oracle.poisson_drive."""
    L = _native.lib()
    words = (n + 31) // 32
    m = torch.empty((n_trials, t_steps, words), dtype=torch.int32, device=device)
    s = stream if stream is not None else torch.cuda.current_stream(m.device).cuda_stream
    rc = L.eq_poisson_drive(n, n_trials, t_steps, dt, mean_interval, pulse_duration, seed, _ptr(m), s)
    if rc != 0:
        raise ConfigurationError(
            f"eq_poisson_drive: invalid arguments (n={n}, trials={n_trials}, steps={t_steps}, dt={dt}, "
            f"mean_interval={mean_interval}, pulse_duration={pulse_duration})")
    return m
