"""Event/pulse data model of the reference (pkg/src/eventq/events.py:20-96,
dual.py:19-46), restated so reference call sites keep their types.

These are plain host-side value types; the queues themselves live on the GPU
(``queues.py``)."""

from __future__ import annotations

from enum import Enum
from typing import NamedTuple, Optional


class DualScalar(NamedTuple):
    """(primal, tangent) pair, dual.py:19-46."""

    primal: float
    tangent: float = 0.0

    def __add__(self, other):  # type: ignore[override]
        return DualScalar(self.primal + other.primal, self.tangent + other.tangent)

    def __sub__(self, other):
        return DualScalar(self.primal - other.primal, self.tangent - other.tangent)

    def scale(self, c: float) -> "DualScalar":
        return DualScalar(c * self.primal, c * self.tangent)


class SpikeEvent(NamedTuple):
    """events.py:20-31: delivery step, dual weight, delivery-time tangent."""

    deliver_step: int
    weight: DualScalar
    time_tangent: float = 0.0


def unit_event(deliver_step: int) -> SpikeEvent:
    return SpikeEvent(deliver_step, DualScalar(1.0, 0.0), 0.0)


class AggregatedPulse(NamedTuple):
    """events.py:38-60: same-step deliveries merged."""

    weight: DualScalar
    weighted_time_tangent: float

    def is_zero(self) -> bool:
        return self.weight.primal == 0.0 and self.weight.tangent == 0.0 and self.weighted_time_tangent == 0.0


ZERO_PULSE = AggregatedPulse(DualScalar(0.0, 0.0), 0.0)


class QueueKind(str, Enum):
    """events.py:71-86 (same string values)."""

    DONOTHING = "donothing"
    RING = "ring"
    LOSSYRING = "lossyring"
    FIFORING = "fiforing"
    SINGLESPIKEHOLD = "singlespikehold"
    SINGLESPIKEDROP = "singlespikedrop"
    SORTEDARRAY = "sortedarray"
    BITARRAY32 = "bitarray32"
    BINARYHEAP = "binaryheap"
    DENSEORACLE = "denseoracle"
    BGPQ = "bgpq"


class QueueCapabilities(NamedTuple):
    """events.py:89-96."""

    supports_gradients: bool
    supports_heterogeneous_delay: bool
    supports_multi_spike_per_step: bool
    lossy: bool
    capacity: Optional[int]
