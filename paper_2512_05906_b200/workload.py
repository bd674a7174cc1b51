"""Synthetic, version-stable inputs for the R-SNN hot path.

The reference draws its networks and drives from ``np.random.default_rng``
(``pkg/src/eventq/bench.py:305``, ``network.py:113``), whose streams numpy does
not promise to keep across versions.  Parity fixtures must be
regenerable on any box, so every random draw here comes from a counter-based
SplitMix64 hash: draw ``k`` of stream ``s`` under seed ``seed`` is a pure
function of ``(seed, s, k)``.

Distributions follow BASELINE.md §4 / SURVEY.md §8(d):

* topology — each source gets ``k_out`` distinct targets uniform over the other
  neurons; rows are sorted by target, matching the ascending-``j`` fan-out of
  ``network_step`` (``network.py:417``);
* weights ~ N(w_mean, w_std); delays = k·dt with k uniform on [d_lo, d_hi];
* drive — ``PoissonDrive`` semantics (``network.py:98-155``): per neuron, pulses
  start at t0 ~ Exp(mean_interval), then every ``pulse_duration + Exp(mean)``;
  a pulse [s, e) is active on steps ceil(s/dt) .. ceil(e/dt)-1.

The drive is packed as a bit mask ``[trials, steps, ceil(n/32)]`` of uint32
(bit j%32 of word j//32), the layout the CUDA kernels read.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x += np.uint64(0x9E3779B97F4A7C15)
        z = x
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def hash_u64(seed: int, stream: int, counter: np.ndarray) -> np.ndarray:
    """Counter-based 64-bit hash: the k-th draw of (seed, stream)."""
    base = _splitmix(np.array([(seed * 0x100000001B3 + stream) & 0xFFFFFFFFFFFFFFFF],
                              dtype=np.uint64))[0]
    with np.errstate(over="ignore"):
        return _splitmix(np.asarray(counter, dtype=np.uint64) ^ base)


def uniform(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    """Uniform float64 in [0, 1) from the top 53 bits."""
    k = np.arange(offset, offset + n, dtype=np.uint64)
    return (hash_u64(seed, stream, k) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def normal(seed: int, stream: int, n: int) -> np.ndarray:
    """Box-Muller normals from two uniform streams."""
    u1 = uniform(seed, stream, n)
    u2 = uniform(seed, stream + 1, n)
    u1 = 1.0 - u1  # (0, 1]
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)


@dataclass
class Network:
    """CSR out-edges of a recurrent network (rows = presynaptic sources)."""

    n: int
    rowptr: np.ndarray   # int64 [n+1]
    col: np.ndarray      # int32 [E]
    weight: np.ndarray   # float64 [E]
    delay: np.ndarray    # float64 [E] (time units)

    @property
    def n_edges(self) -> int:
        return int(self.col.shape[0])

    def dense(self, non_edge_delay: float) -> Tuple[np.ndarray, np.ndarray]:
        """Dense (n, n) weights/delays for the reference, non-edges with zero
        weight (exact for lossless queues)."""
        w = np.zeros((self.n, self.n))
        d = np.full((self.n, self.n), non_edge_delay)
        src = np.repeat(np.arange(self.n), np.diff(self.rowptr))
        w[src, self.col] = self.weight
        d[src, self.col] = self.delay
        np.fill_diagonal(w, 0.0)
        np.fill_diagonal(d, non_edge_delay)
        return w, d


def random_network(n: int, k_out: int, seed: int, dt: float = 1e-3,
                   w_mean: float = 0.003, w_std: float = 0.001,
                   delay_steps: Tuple[int, int] = (1, 64)) -> Network:
    """``k_out`` distinct random targets per source (no self loops)."""
    if n < 2:
        raise ValueError("need n >= 2")
    k_out = min(k_out, n - 1)
    # draw candidate targets in [0, n-2], shift past the source (no self loop),
    # redraw rows with duplicates until every row is distinct
    rows = np.arange(n, dtype=np.int64)
    cand = np.empty((n, k_out), dtype=np.int64)
    need = rows
    attempt = 0
    while need.size:
        cnt = need.size * k_out
        u = uniform(seed, 1000 + attempt, cnt)
        t = np.minimum((u * (n - 1)).astype(np.int64), n - 2).reshape(need.size, k_out)
        t = t + (t >= need[:, None])
        t.sort(axis=1)
        dup = (t[:, 1:] == t[:, :-1]).any(axis=1) if k_out > 1 else np.zeros(need.size, bool)
        ok = need[~dup]
        cand[ok] = t[~dup]
        need = need[dup]
        attempt += 1
        if attempt > 200 and need.size:
            # dense regime: sample by permutation per remaining row
            for i in need:
                others = np.delete(np.arange(n), i)
                key = uniform(seed, 5000 + int(i), n - 1)
                cand[i] = np.sort(others[np.argsort(key, kind="stable")[:k_out]])
            need = need[:0]
    col = cand.reshape(-1).astype(np.int32)
    E = col.shape[0]
    rowptr = np.arange(0, (n + 1) * k_out, k_out, dtype=np.int64)
    weight = w_mean + w_std * normal(seed, 2, E)
    lo, hi = delay_steps
    ks = lo + np.minimum((uniform(seed, 4, E) * (hi - lo + 1)).astype(np.int64), hi - lo)
    delay = ks.astype(np.float64) * dt
    return Network(n=n, rowptr=rowptr, col=col, weight=weight, delay=delay)


def dense_network(weights: np.ndarray, delays: np.ndarray) -> Network:
    """All-to-all CSR from dense (n, n) matrices (diagonal ignored)."""
    n = weights.shape[0]
    mask = ~np.eye(n, dtype=bool)
    src, dst = np.nonzero(mask)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum(mask.sum(axis=1))
    return Network(n=n, rowptr=rowptr, col=dst.astype(np.int32),
                   weight=weights[src, dst].astype(np.float64),
                   delay=delays[src, dst].astype(np.float64))


def poisson_drive_mask(n: int, t_steps: int, dt: float, mean_interval: float,
                       pulse_duration: float, seed: int) -> np.ndarray:
    """Active[t_steps, n] bool with ``PoissonDrive`` semantics
    (``network.py:114-121``, ``:136-141``), one independent train per neuron."""
    t_total = t_steps * dt
    # enough draws per neuron to pass t_total with overwhelming probability
    expect = t_total / (pulse_duration + mean_interval)
    m = int(expect + 8.0 * math.sqrt(expect + 1.0) + 8)
    u = uniform(seed, 7, n * m).reshape(n, m)
    gaps = -mean_interval * np.log1p(-u)          # Exp(mean)
    starts = np.cumsum(gaps, axis=1) + pulse_duration * np.arange(m)[None, :]
    # starts[:, k] = gap_0 + sum_{1..k}(gap_i + dur)
    if (starts[:, -1] < t_total).any():
        raise RuntimeError("drive draw budget exhausted; raise m")
    live = starts < t_total
    lo = np.clip(np.ceil(starts / dt), 0, t_steps).astype(np.int64)
    hi = np.clip(np.ceil((starts + pulse_duration) / dt), 0, t_steps).astype(np.int64)
    keep = live & (hi > lo)
    jj = np.broadcast_to(np.arange(n)[:, None], starts.shape)[keep]
    L = lo[keep]
    W = (hi - lo)[keep]
    flat = np.zeros(t_steps * n, dtype=bool)
    base = L * n + jj
    for off in range(int(W.max()) if W.size else 0):
        sel = W > off
        flat[base[sel] + off * n] = True
    active = flat.reshape(t_steps, n)
    return active


def pack_mask(active: np.ndarray) -> np.ndarray:
    """bool[..., n] -> uint32[..., ceil(n/32)], bit j%32 of word j//32."""
    n = active.shape[-1]
    words = (n + 31) // 32
    pad = words * 32 - n
    if pad:
        active = np.concatenate([active, np.zeros(active.shape[:-1] + (pad,), bool)], axis=-1)
    packed = np.packbits(active.astype(np.uint8), axis=-1, bitorder="little")
    return np.ascontiguousarray(packed).view(np.uint32).reshape(active.shape[:-1] + (words,))


def unpack_mask(mask: np.ndarray, n: int) -> np.ndarray:
    bits = np.unpackbits(mask.view(np.uint8), axis=-1, bitorder="little")
    return bits[..., :n].astype(bool)


@dataclass
class LIFConfig:
    """Cell constants; defaults are ``default_rsnn_params`` (bench.py:297-329)."""

    dt: float = 1e-3
    tau_m: float = 1.0
    tau_syn: float = 0.5
    v_th: float = 1.0
    v_reset: float = 0.0
    refractory_steps: int = 0
    exact_delivery: bool = True
    v_target: float = 0.25


@dataclass
class Workload:
    net: Network
    lif: LIFConfig
    n_trials: int
    t_steps: int
    mask: np.ndarray      # uint32 [B, T, W]
    amp: np.ndarray       # float64 [n]
    name: str = ""


def drive_masks(n: int, n_trials: int, t_steps: int, dt: float, seed0: int = 1000,
                mean_interval_steps: float = 16.0, duration_steps: float = 12.0) -> np.ndarray:
    """Packed masks for trials b = 0..B-1 with seeds seed0 + b."""
    out = np.empty((n_trials, t_steps, (n + 31) // 32), dtype=np.uint32)
    for b in range(n_trials):
        act = poisson_drive_mask(n, t_steps, dt, mean_interval_steps * dt,
                                 duration_steps * dt, seed0 + b)
        out[b] = pack_mask(act)
    return out


def poisson_streams(lambda_steps: float, t_steps: int, n_queues: int, seed: int) -> np.ndarray:
    """Bernoulli(1/lambda) spike streams of the reference's Poisson queue
    benchmark (restates eventq.bench.gen_poisson, bench.py:86-96: one
    SeedSequence child per queue, ``default_rng(child).random(T) < 1/lambda``).
    Returns packed bits uint32 [n_queues, ceil(T/32)].  numpy's Generator
    streams are version-dependent: the goldens pin them (tests/golden/p_*)."""
    p = 1.0 / lambda_steps
    out = np.empty((n_queues, (t_steps + 31) // 32), dtype=np.uint32)
    for q, ss in enumerate(np.random.SeedSequence(seed).spawn(n_queues)):
        out[q] = pack_mask(np.random.default_rng(ss).random(t_steps) < p)
    return out


CONFIGS = {
    # name: (n, k_out, delay steps, trials, steps)
    "C1": (1_000, 100, (1, 16), 1, 1000),
    "C2": (10_000, 100, (1, 64), 32, 1000),
    "C3": (100_000, 100, (1, 64), 32, 1000),
    "C4": (1_000_000, 100, (1, 256), 4, 1000),
}


def make_workload(name: str = "C3", n_trials: Optional[int] = None, t_steps: Optional[int] = None,
                  seed: int = 0, n: Optional[int] = None, amplitude: float = 12.0) -> Workload:
    n0, k, drange, b0, t0 = CONFIGS[name]
    n = n or n0
    B = n_trials or b0
    T = t_steps or t0
    lif = LIFConfig()
    net = random_network(n, k, seed, dt=lif.dt, delay_steps=drange)
    mask = drive_masks(n, B, T, lif.dt)
    amp = np.full(n, amplitude)
    return Workload(net=net, lif=lif, n_trials=B, t_steps=T, mask=mask, amp=amp, name=name)
