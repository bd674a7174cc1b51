"""GPU-backed queues with the reference's operator API.

``make_queue(kind, capacity, max_delay_steps)`` (queues.py:636-692) returns a
``DeviceQueue`` with the EventQueue protocol (events.py:99-141):
``enqueue(SpikeEvent) -> bool``, ``pop_due() -> AggregatedPulse``,
``_pop_raw()``, ``occupancy()``, ``now``, ``kind``, ``capabilities``.
``QueueBatch`` is the batched form the hot paths use: Q queues of one kind,
enqueue of an event array in call order, one pop for all queues per step.

Both call the sm_100a library (``eq_queues_*`` in include/eventq_b200.h); there
is no host implementation to fall back to.  Kinds the network path does not
use (SingleSpike*, BitArray32, DenseOracle) are out of scope and
raise ConfigurationError naming the kind; BGPQ is rejected as the reference
rejects it (queues.py:651-655).
"""

from __future__ import annotations

import ctypes
from typing import Optional, Tuple, Union

import numpy as np
import torch

from . import _native
from .errors import ConfigurationError
from .events import AggregatedPulse, DualScalar, QueueCapabilities, QueueKind, SpikeEvent, ZERO_PULSE

_GPU_KINDS = {QueueKind.RING, QueueKind.LOSSYRING, QueueKind.FIFORING, QueueKind.SORTEDARRAY,
              QueueKind.BINARYHEAP, QueueKind.DONOTHING}

# capability flags per kind (queues.py: each class's __init__)
_CAPS = {
    QueueKind.DONOTHING: (True, True, True, True),
    QueueKind.RING: (True, True, True, False),
    QueueKind.LOSSYRING: (True, True, True, True),
    QueueKind.FIFORING: (True, False, True, True),
    QueueKind.SORTEDARRAY: (True, True, True, True),
    QueueKind.BINARYHEAP: (True, True, True, True),
    QueueKind.SINGLESPIKEHOLD: (True, True, False, True),
    QueueKind.SINGLESPIKEDROP: (True, True, False, True),
    QueueKind.BITARRAY32: (False, False, False, True),
    QueueKind.DENSEORACLE: (True, True, True, False),
}


def coerce_kind(kind: Union[QueueKind, str]) -> QueueKind:
    try:
        return QueueKind(kind)
    except ValueError:
        raise ConfigurationError(f"unknown queue kind {kind!r}") from None


def _reject(kind: QueueKind) -> None:
    if kind is QueueKind.BGPQ:
        raise ConfigurationError("bgpq is registered but unsupported: its value is GPU group "
                                 "parallelism, which a serial build cannot express")
    if kind not in _GPU_KINDS:
        raise ConfigurationError(f"{kind.value} is out of scope of the B200 build "
                                 "(ring, lossyring, fiforing, sortedarray, binaryheap, donothing)")


class QueueBatch:
    """Q independent device queues of one kind stepping together."""

    def __init__(self, kind: Union[QueueKind, str], n_queues: int, capacity: Optional[int] = None,
                 max_delay_steps: Optional[int] = None, precision: int = 64, device=None):
        self.kind = coerce_kind(kind)
        _reject(self.kind)
        self.L = _native.lib()
        self.n = n_queues
        self.precision = precision
        self.dtype = torch.float64 if precision == 64 else torch.float32
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        h = ctypes.c_void_p()
        code = self.L.eq_queues_create(_native.KIND_IDS[self.kind.value], precision, n_queues,
                                       0 if capacity is None else int(capacity),
                                       0 if max_delay_steps is None else int(max_delay_steps),
                                       self.device.index, ctypes.byref(h))
        self.h = h
        _native.check(self.h, code, queues=True)
        self.capacity = int(self.L.eq_queues_capacity(self.h))
        Q = n_queues
        self._w = torch.empty(Q, dtype=self.dtype, device=self.device)
        self._dw = torch.empty_like(self._w)
        self._wtt = torch.empty_like(self._w)
        self._has = torch.empty(Q, dtype=torch.uint8, device=self.device)

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.L.eq_queues_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def _stream(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    @property
    def now(self) -> int:
        return int(self.L.eq_queues_now(self.h))

    def enqueue(self, queue, deliver_step, weight, weight_tangent=None, time_tangent=None) -> torch.Tensor:
        """Events in call order; returns the accepted flags (bool tensor)."""
        dev, dt = self.device, self.dtype
        q = torch.as_tensor(queue, dtype=torch.int32).to(dev).contiguous()
        n = q.numel()
        s = torch.as_tensor(deliver_step, dtype=torch.int32).to(dev).contiguous()
        w = torch.as_tensor(weight, dtype=dt).to(dev).contiguous()
        dw = (torch.zeros(n, dtype=dt, device=dev) if weight_tangent is None
              else torch.as_tensor(weight_tangent, dtype=dt).to(dev).contiguous())
        tt = (torch.zeros(n, dtype=dt, device=dev) if time_tangent is None
              else torch.as_tensor(time_tangent, dtype=dt).to(dev).contiguous())
        if not (s.numel() == w.numel() == dw.numel() == tt.numel() == n):
            raise ConfigurationError("enqueue arrays must have one entry per event")
        if n and (int(q.min()) < 0 or int(q.max()) >= self.n):
            raise ConfigurationError("queue index out of range")
        acc = torch.zeros(n, dtype=torch.uint8, device=dev)
        p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _native.check(self.h, self.L.eq_queues_enqueue(self.h, p(q), p(s), p(w), p(dw), p(tt), n, p(acc),
                                                        self._stream), queues=True)
        return acc.bool()

    def pop(self) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
        """pop_due for all queues: (w, dw, wtt, has) device tensors (views reused)."""
        p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _native.check(self.h, self.L.eq_queues_pop(self.h, p(self._w), p(self._dw), p(self._wtt), p(self._has),
                                                    self._stream), queues=True)
        return self._w, self._dw, self._wtt, self._has

    def run_poisson(self, spike_bits: torch.Tensor, t_steps: int, delay: int):
        """The reference's Poisson queue benchmark stream (bench.py:183-205) for
        every queue in one launch.  spike_bits: uint32/int32 [n_queues,
        ceil(t_steps/32)] (bit s of queue q = a spike at step s).  Returns
        (delivered weight float64 [Q], accepted int64 [Q]) on the device."""
        bits = torch.as_tensor(spike_bits).to(self.device)
        if bits.dtype != torch.int32:
            bits = bits.to(torch.int32)
        bits = bits.contiguous()
        if tuple(bits.shape) != (self.n, (t_steps + 31) // 32):
            raise ConfigurationError(f"spike bits must be [{self.n}, {(t_steps + 31) // 32}]")
        delivered = torch.empty(self.n, dtype=torch.float64, device=self.device)
        accepted = torch.empty(self.n, dtype=torch.int64, device=self.device)
        _native.check(self.h, self.L.eq_queues_run_poisson(
            self.h, ctypes.c_void_p(bits.data_ptr()), int(t_steps), int(delay),
            ctypes.c_void_p(delivered.data_ptr()), ctypes.c_void_p(accepted.data_ptr()), self._stream), queues=True)
        return delivered, accepted

    def occupancy(self) -> torch.Tensor:
        out = torch.empty(self.n, dtype=torch.int32, device=self.device)
        _native.check(self.h, self.L.eq_queues_occupancy(self.h, ctypes.c_void_p(out.data_ptr()), self._stream),
                      queues=True)
        return out

    def lossy_counts(self):
        a = torch.empty(self.n, dtype=torch.int64, device=self.device)
        m = torch.empty_like(a)
        _native.check(self.h, self.L.eq_queues_lossy_counts(self.h, ctypes.c_void_p(a.data_ptr()),
                                                             ctypes.c_void_p(m.data_ptr()), self._stream),
                      queues=True)
        return a, m


class DeviceQueue:
    """One device queue with the reference EventQueue protocol."""

    def __init__(self, kind: QueueKind, capacity: Optional[int], max_delay_steps: Optional[int],
                 precision: int = 64):
        self._b = QueueBatch(kind, 1, capacity, max_delay_steps, precision)
        self.kind = self._b.kind
        caps = _CAPS[self.kind]
        cap = 0 if self.kind is QueueKind.DONOTHING else self._b.capacity
        self.capabilities = QueueCapabilities(*caps, capacity=cap)

    @property
    def now(self) -> int:
        return self._b.now

    @property
    def aliased(self) -> int:
        return int(self._b.lossy_counts()[0][0])

    @property
    def merged(self) -> int:
        return int(self._b.lossy_counts()[1][0])

    def enqueue(self, ev: SpikeEvent) -> bool:
        w = ev.weight
        acc = self._b.enqueue([0], [int(ev.deliver_step)], [float(w.primal)], [float(w.tangent)],
                              [float(ev.time_tangent)])
        return bool(acc[0])

    def _pop_raw(self):
        w, dw, wtt, has = self._b.pop()
        if not bool(has[0]):
            return None
        return (float(w[0]), float(dw[0]), float(wtt[0]))

    def pop_due(self) -> AggregatedPulse:
        raw = self._pop_raw()
        if raw is None:
            return ZERO_PULSE
        return AggregatedPulse(DualScalar(raw[0], raw[1]), raw[2])

    def occupancy(self) -> int:
        return int(self._b.occupancy()[0])


def make_queue(kind: Union[QueueKind, str], capacity: Optional[int] = None,
               max_delay_steps: Optional[int] = None, precision: int = 64) -> DeviceQueue:
    """queues.py:636-692 on the GPU (argument rules enforced by the library)."""
    kind = coerce_kind(kind)
    _reject(kind)
    return DeviceQueue(kind, capacity, max_delay_steps, precision)


def kind_capabilities(kind: Union[QueueKind, str]) -> QueueCapabilities:
    """queues.py:695-705 (a pure function of the kind; no device needed)."""
    kind = coerce_kind(kind)
    if kind is QueueKind.BGPQ:
        _reject(kind)
    caps = _CAPS[kind]
    cap = {QueueKind.DONOTHING: 0, QueueKind.DENSEORACLE: None}.get(kind, 1)
    return QueueCapabilities(*caps, capacity=cap)
