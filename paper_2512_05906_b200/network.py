"""Reference-shaped network API over the B200 engine.

Same names and call shapes as pkg/src/eventq/network.py so the reference's
call sites (bench.py:345-404, gradcheck.py:71-102, the tests) can switch:

* ``NetworkParams`` / ``SeedDirection``        network.py:39-95
* ``PoissonDrive``                              network.py:98-155 (same numpy draws)
* ``build_rsnn(params, seed, rng_seed)``        network.py:201-333 -> ``NetworkState``
* ``simulate(state, t_steps, drive, record)``   network.py:458-497 -> ``SimResult``
* ``PrimalRSNN(params).run(t_steps, drive)``    network.py:500-619
* ``forward_gradient(params, direction, ...)``  network.py:668-683 — here one
  forward + one reverse pass (the full gradient), dotted with the direction
* ``grad_fd_oracle``                            network.py:622-665
* ``RSNNFunction`` — the torch autograd shell: final membrane as a function of
  (weights, delays, drive amplitudes), backward = the reverse kernel.

Dense (n, n) parameter matrices map to CSR with all n-1 off-diagonal entries
per row (zero weights included), so every queue kind — bounded ones too — sees
exactly the reference's event stream.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Callable, List, Optional, Sequence, Tuple, Union

import numpy as np
import torch

from .errors import ConfigurationError, EventQError, GrazingCrossingError, NonSmoothDirectionError
from .events import DualScalar, QueueKind
from .queues import coerce_kind
from .workload import LIFConfig, Network, pack_mask


@dataclass(frozen=True)
class SeedDirection:
    """Which single scalar carries tangent 1 (network.py:39-53)."""

    param: str  # "weight" | "delay" | "drive"
    i: int
    j: int = -1

    def __post_init__(self):
        if self.param not in ("weight", "delay", "drive"):
            raise ConfigurationError(f"seed direction must be weight/delay/drive, got {self.param!r}")
        if self.param in ("weight", "delay") and self.j < 0:
            raise ConfigurationError(f"{self.param} seed needs an (i, j) edge")


@dataclass
class NetworkParams:
    """network.py:56-95: dense (n, n) matrices, diagonal unused."""

    n: int
    weights: np.ndarray
    delays: np.ndarray
    tau_m: float
    tau_syn: float
    v_th: float
    v_reset: float
    dt: float
    queue_kind: Union[QueueKind, str] = QueueKind.RING
    queue_capacity: Optional[int] = None
    refractory_steps: int = 0
    v_target: Optional[np.ndarray] = None
    exact_delivery: bool = True

    def perturbed(self, direction: SeedDirection, delta: float) -> "NetworkParams":
        if direction.param == "weight":
            w = np.array(self.weights, dtype=float, copy=True)
            w[direction.i, direction.j] += delta
            return replace(self, weights=w)
        if direction.param == "delay":
            d = np.array(self.delays, dtype=float, copy=True)
            d[direction.i, direction.j] += delta
            return replace(self, delays=d)
        raise ConfigurationError("drive directions perturb the drive, not params")

    def lif(self) -> LIFConfig:
        return LIFConfig(dt=self.dt, tau_m=self.tau_m, tau_syn=self.tau_syn, v_th=self.v_th,
                         v_reset=self.v_reset, refractory_steps=self.refractory_steps,
                         exact_delivery=self.exact_delivery)

    def csr(self) -> Network:
        n = self.n
        w = np.asarray(self.weights, dtype=float)
        d = np.asarray(self.delays, dtype=float)
        if w.shape != (n, n) or d.shape != (n, n):
            raise ConfigurationError("weights and delays must both be (n, n)")
        off = ~np.eye(n, dtype=bool)
        src, dst = np.nonzero(off)
        rowptr = np.arange(0, n * (n - 1) + 1, n - 1, dtype=np.int64)
        return Network(n=n, rowptr=rowptr, col=dst.astype(np.int32), weight=w[src, dst], delay=d[src, dst])


class PoissonDrive:
    """network.py:98-155: seeded Poisson current pulses in physical time (the
    same numpy Generator draws as the reference, so the same seed gives the
    same pulses on the same numpy)."""

    def __init__(self, n: int, mean_interval: float, amplitude: float, pulse_duration: float, t_total: float,
                 rng_seed: int):
        self.n = n
        self.amplitude = amplitude
        rng = np.random.default_rng(rng_seed)
        self.pulses: List[List[Tuple[float, float]]] = []
        for _ in range(n):
            starts = []
            t = rng.exponential(mean_interval)
            while t < t_total:
                starts.append(t)
                t += pulse_duration + rng.exponential(mean_interval)
            self.pulses.append([(s, s + pulse_duration) for s in starts])

    def active(self, t_steps: int, dt: float) -> np.ndarray:
        act = np.zeros((t_steps, self.n), dtype=bool)
        for i, intervals in enumerate(self.pulses):
            for s, e in intervals:
                lo = min(t_steps, max(0, math.ceil(s / dt)))
                hi = min(t_steps, max(0, math.ceil(e / dt)))
                act[lo:hi, i] = True
        return act

    def amplitudes(self, amp_delta: Optional[Tuple[int, float]] = None) -> np.ndarray:
        amps = np.full(self.n, float(self.amplitude))
        if amp_delta is not None:
            amps[amp_delta[0]] += amp_delta[1]
        return amps


def _drive_arrays(drive, n: int, t_steps: int, dt: float, amp_delta=None):
    """Drive as (active[T, n], amplitude[n]) from a PoissonDrive, an
    (active, amplitude) pair, a reference-style callable step -> row of
    DualScalar (constant per-neuron amplitude), or None."""
    if drive is None:
        return np.zeros((t_steps, n), bool), np.zeros(n)
    if isinstance(drive, PoissonDrive):
        return drive.active(t_steps, dt), drive.amplitudes(amp_delta)
    if isinstance(drive, tuple):
        act, amp = drive
        return np.asarray(act, bool)[:t_steps], np.asarray(amp, float)
    act = np.zeros((t_steps, n), bool)
    amp = np.zeros(n)
    for m in range(t_steps):
        row = drive(m)
        if len(row) != n:
            raise ConfigurationError(f"drive vector has {len(row)} entries for n={n}")
        for j, x in enumerate(row):
            v = float(x.primal if isinstance(x, DualScalar) or hasattr(x, "primal") else x)
            if v != 0.0:
                if act[:m, j].any() and amp[j] != v:
                    raise ConfigurationError("the B200 drive needs a constant amplitude per neuron")
                act[m, j] = True
                amp[j] = v
    return act, amp


@dataclass
class SimResult:
    loss: DualScalar
    spike_count: int
    drop_count: int
    enqueued_count: int
    raster: Optional[List[Tuple[int, int]]] = None
    voltages: Optional[np.ndarray] = None
    v_final: Optional[np.ndarray] = None
    i_final: Optional[np.ndarray] = None


class NetworkState:
    """A built network on the GPU (engine + parameters), network.py:158-185."""

    def __init__(self, params: NetworkParams, seed: Optional[SeedDirection], precision: int, device=None,
                 t_steps: int = 1):
        from .engine import Engine
        self.params = params
        self.seed = seed
        self.precision = precision
        self.kind = coerce_kind(params.queue_kind)
        self.net = params.csr()
        self.device = device
        self.engine = None
        self.t_steps = 0
        self._Engine = Engine

    def _ensure(self, t_steps: int):
        if self.engine is not None and self.t_steps == t_steps:
            return self.engine
        p = self.params
        eng = self._Engine(p.n, 1, t_steps, kind=self.kind.value, precision=self.precision, lif=p.lif(),
                           capacity=int(p.queue_capacity or 0), device=self.device)
        eng.set_network(self.net.rowptr, self.net.col, self.net.weight, self.net.delay)
        self.engine, self.t_steps = eng, t_steps
        return eng


def build_rsnn(params: NetworkParams, seed: Optional[SeedDirection] = None, rng_seed: int = 0,
               precision: int = 64, device=None) -> NetworkState:
    """Validate and assemble (network.py:201-333).  Validation that needs the
    full matrices happens here on the host with the reference's messages; the
    device repeats the CSR checks in eq_set_network."""
    n = params.n
    if n < 2:
        raise ConfigurationError(f"a recurrent network needs n >= 2, got {n}")
    w = np.asarray(params.weights, dtype=float)
    d = np.asarray(params.delays, dtype=float)
    if w.shape != (n, n) or d.shape != (n, n):
        raise ConfigurationError("weights and delays must both be (n, n)")
    kind = coerce_kind(params.queue_kind)
    if kind is QueueKind.BGPQ:
        raise ConfigurationError("bgpq is registered but unsupported: its value is GPU group parallelism, "
                                 "which a serial build cannot express")
    if kind not in (QueueKind.RING, QueueKind.LOSSYRING, QueueKind.FIFORING, QueueKind.BINARYHEAP,
                    QueueKind.SORTEDARRAY, QueueKind.DONOTHING):
        raise ConfigurationError(f"{kind.value} networks are out of scope of the B200 build "
                                 "(ring, lossyring, fiforing, binaryheap, sortedarray, donothing)")
    off = ~np.eye(n, dtype=bool)
    bad = np.argwhere(off & (d < params.dt))
    if len(bad):
        i, j = bad[0]
        raise ConfigurationError(f"delay on edge ({i},{j}) is {d[i, j]}, below one step ({params.dt})")
    if kind is QueueKind.FIFORING:
        vals = d[off]
        if (vals != vals[0]).any():
            k = int(np.argmax(vals != vals[0]))
            i, j = np.argwhere(off)[k]
            raise ConfigurationError(f"fiforing supports homogeneous delays only, but edge ({i},{j}) has "
                                     f"{d[i, j]} while another edge has {vals[0]}")
    if params.exact_delivery and abs(params.tau_m - params.tau_syn) < 1e-3 * params.tau_m:
        raise ConfigurationError("exact delivery splits the membrane/synapse eigenmodes and needs tau_m != "
                                 f"tau_syn; got {params.tau_m} and {params.tau_syn} (set exact_delivery=False)")
    if seed is not None:
        if seed.param == "drive":
            if not 0 <= seed.i < n:
                raise ConfigurationError(f"drive seed neuron {seed.i} out of range")
        elif not (0 <= seed.i < n and 0 <= seed.j < n) or seed.i == seed.j:
            raise ConfigurationError(f"seed edge ({seed.i},{seed.j}) is not a valid off-diagonal edge")
    return NetworkState(params, seed, precision, device)


def _edge_index(n: int, i: int, j: int) -> int:
    return i * (n - 1) + (j if j < i else j - 1)


def _run(state: NetworkState, t_steps: int, drive, record: bool, amp_delta=None):
    p = state.params
    act, amp = _drive_arrays(drive, p.n, t_steps, p.dt, amp_delta)
    eng = state._ensure(t_steps)
    mask = pack_mask(act)[None]
    eng.set_drive(mask, amp)
    try:
        out = eng.forward(record_v=record)
    except GrazingCrossingError:
        raise
    return eng, out, act, amp


def simulate(state: NetworkState, t_steps: int, drive=None, record: bool = False) -> SimResult:
    """network.py:458-497.  The loss tangent is filled when the state was built
    with a seed direction (via one reverse pass)."""
    if t_steps < 1:
        raise ConfigurationError(f"t_steps must be >= 1, got {t_steps}")
    p = state.params
    eng, out, act, amp = _run(state, t_steps, drive, record)
    v = out["v"][0].double().cpu().numpy()
    target = np.zeros(p.n) if p.v_target is None else np.asarray(p.v_target, dtype=float)
    loss = 0.0
    for j in range(p.n):                      # sequential, as the dual sum in network.py:486-489
        diff = float(v[j]) - float(target[j])
        loss = loss + diff * diff
    tangent = 0.0
    if state.seed is not None:
        tangent = _directional(state, eng, v, target, state.seed)
    counters = eng.counters()[0]
    res = SimResult(loss=DualScalar(loss, tangent), spike_count=int(counters[0]), drop_count=int(counters[2]),
                    enqueued_count=int(counters[0]) * (p.n - 1), v_final=v,
                    i_final=out["i"][0].double().cpu().numpy())
    if record:
        sp = eng.spikes()
        res.raster = [(int(m), int(j)) for m, j in zip(sp["step"], sp["neuron"])]
        res.voltages = out["v_trace"][:, 0].double().cpu().numpy()
    return res


def _directional(state, eng, v, target, seed: SeedDirection) -> float:
    vbar = torch.as_tensor(2.0 * (v - target)[None], dtype=eng.dtype, device=eng.device)
    gw, gd, ga = eng.backward(vbar, want_amp=seed.param == "drive")
    if seed.param == "drive":
        return float(ga[seed.i])
    x = _edge_index(state.params.n, seed.i, seed.j)
    return float((gw if seed.param == "weight" else gd)[x])


def forward_gradient(params: NetworkParams, direction: SeedDirection, t_steps: int, drive=None,
                     precision: int = 64) -> Tuple[float, SimResult]:
    """network.py:668-683: d loss / d theta along `direction` — one forward and
    one reverse pass (the reverse pass yields every direction at once)."""
    state = build_rsnn(params, seed=direction, precision=precision)
    res = simulate(state, t_steps, drive)
    return res.loss.tangent, res


def forward_gradients(params: NetworkParams, directions, t_steps: int, drive=None) -> np.ndarray:
    """The reference's forward mode (network.py:668-683) for many directions in
    ONE batched JVP run on the GPU (eq_forward_jvp; fp64, ring kind): returns
    d loss / d theta for each SeedDirection — an independent cross-check of
    the reverse pass (tests/test_gpu_jvp.py)."""
    directions = list(directions)
    state = build_rsnn(params, precision=64)
    for dr in directions:
        build_rsnn(params, seed=dr)            # the reference's seed validation
    p = state.params
    act, amp = _drive_arrays(drive, p.n, t_steps, p.dt)
    eng = state._ensure(t_steps)
    eng.set_drive(pack_mask(act)[None], amp)
    kinds, idx = [], []
    for dr in directions:
        kinds.append(dr.param)
        idx.append(dr.i if dr.param == "drive" else _edge_index(p.n, dr.i, dr.j))
    v, vt = eng.forward_jvp(kinds, idx)
    v = v[0].cpu().numpy()
    target = np.zeros(p.n) if p.v_target is None else np.asarray(p.v_target, dtype=float)
    g = 2.0 * (v - target)
    out = np.empty(len(directions))
    for d in range(len(directions)):         # sequential dual sum, network.py:486-489
        t = vt[d, 0].cpu().numpy()
        acc = 0.0
        for j in range(p.n):
            acc = acc + g[j] * t[j]
        out[d] = acc
    return out


def full_gradient(params: NetworkParams, t_steps: int, drive=None, precision: int = 64):
    """All directions at once: dL/dW and dL/dD as dense (n, n) (diagonal 0) and
    dL/d amplitude (n,)."""
    state = build_rsnn(params, precision=precision)
    p = state.params
    eng, out, act, amp = _run(state, t_steps, drive, False)
    v = out["v"][0].double()
    target = torch.zeros_like(v) if p.v_target is None else torch.as_tensor(p.v_target, dtype=torch.float64,
                                                                              device=v.device)
    gw, gd, ga = eng.backward((2.0 * (v - target))[None].to(eng.dtype))
    n = p.n
    off = ~np.eye(n, dtype=bool)
    GW = np.zeros((n, n)); GD = np.zeros((n, n))
    GW[off] = gw.cpu().numpy(); GD[off] = gd.cpu().numpy()
    return GW, GD, ga.cpu().numpy()


def grad_fd_oracle(params: NetworkParams, direction: SeedDirection, epsilon: float, t_steps: int,
                   drive=None, precision: int = 64) -> float:
    """network.py:622-665: central difference with the spike-count guard."""
    results = []
    for sign in (+1.0, -1.0):
        delta = sign * epsilon
        if direction.param == "drive":
            p, amp_delta = params, (direction.i, delta)
        else:
            p, amp_delta = params.perturbed(direction, delta), None
        st = build_rsnn(p, precision=precision)
        try:
            eng, out, _, _ = _run(st, t_steps, drive, False, amp_delta)
        except GrazingCrossingError as exc:
            raise NonSmoothDirectionError(f"{direction}: grazing crossing under perturbation {delta}: {exc}") from exc
        v = out["v"][0].double().cpu().numpy()
        target = np.zeros(p.n) if p.v_target is None else np.asarray(p.v_target, dtype=float)
        loss = 0.0
        for j in range(p.n):
            diff = float(v[j]) - float(target[j])
            loss = loss + diff * diff
        results.append((loss, int(eng.counters()[0][0])))
    (lp, sp), (lm, sm) = results
    if sp != sm:
        raise NonSmoothDirectionError(f"{direction}: spike count changed under +/-{epsilon} ({sp} vs {sm})")
    return (lp - lm) / (2.0 * epsilon)


class PrimalRSNN:
    """network.py:500-619: tangent-free forward (here: the same kernel)."""

    def __init__(self, params: NetworkParams, precision: int = 64):
        self.state = build_rsnn(params, precision=precision)
        self.params = params
        self.v = None
        self.i_syn = None
        self.spike_count = self.enqueued_count = self.drop_count = 0

    def run(self, t_steps: int, drive=None) -> None:
        eng, out, _, _ = _run(self.state, t_steps, drive, False)
        self.v = out["v"][0].double().cpu().numpy().tolist()
        self.i_syn = out["i"][0].double().cpu().numpy().tolist()
        c = eng.counters()[0]
        self.spike_count = int(c[0])
        self.enqueued_count = int(c[0]) * (self.params.n - 1)
        self.drop_count = int(c[2])


class RSNNFunction(torch.autograd.Function):
    """Final membrane V[B, n] as a differentiable function of (weight[E],
    delay[E], amplitude[n]) for a fixed drive mask; backward runs the reverse
    kernel through the same queues (gradients summed over trials)."""

    @staticmethod
    def forward(ctx, weight, delay, amplitude, engine, rowptr, col, mask):
        engine.set_network(rowptr, col, weight.detach(), delay.detach())
        engine.set_drive(mask, amplitude.detach())
        out = engine.forward()
        ctx.engine = engine
        ctx.run_id = engine.run_id
        ctx.dtypes = (weight.dtype, delay.dtype, amplitude.dtype)
        ctx.needs_amp = ctx.needs_input_grad[2]
        return out["v"]

    @staticmethod
    def backward(ctx, v_bar):
        eng = ctx.engine
        if eng.run_id != ctx.run_id:
            # the engine holds ONE recorded run (spike log + queues); a later
            # forward on it (gradient accumulation, two losses, checkpointing)
            # replaced the run this backward belongs to
            raise EventQError("RSNNFunction.backward: the engine ran another forward since this one "
                              f"(run {eng.run_id} != {ctx.run_id}); use one engine per pending backward")
        gw, gd, ga = eng.backward(v_bar.contiguous(), want_amp=ctx.needs_amp)
        dw, dd, da = ctx.dtypes
        return (gw.to(dw), gd.to(dd), None if ga is None else ga.to(da), None, None, None, None)
