"""One network partitioned over several GPUs (BASELINE config 5).

The reference has no sharding; this is the B200 layout for a network too big
(or too slow) for one GPU.  Partition r owns the contiguous neuron range
[lo_r, hi_r): their LIF state, their queues, and the CSR restricted to edges
INTO the range (every source keeps a row, columns are local).  Steps run in
exchange windows of W <= D_min steps, D_min = min_e floor(d_e / dt): an event
emitted at step m is due no earlier than m + 1 + D_min (jumps.py:90-96), so a
window's spikes only have to reach the other partitions before the next window
starts.  Per window:

  forward   eq_run(W); export own spikes {source, trial, step, t}; all-gather;
            import the others' (rank order) — the next launch fans them out in
            its first phase.
  reverse   windows in reverse order: eq_backward_window(a) walks the phases
            down to a, then the partial dL/dt_spk over this partition's edges of
            every spike imported before forward launch a is returned to the
            spike's owner (all-gather; the owner sums the partials in rank
            order) and added before the owner's next reverse window.

dL/dw and dL/dd stay with the target's partition (no final all-reduce).
Forward results equal the unpartitioned network's bitwise (fixed-point slot
sums are order-free; every partition uses the minimum fraction bits); reverse
results differ only in the association of each spike's dL/dt_spk sum (own
edges, then other partitions in rank order).

Two transports drive the same per-partition logic: ``DistTransport``
(torch.distributed, one process per GPU — NCCL over NVLink on B200, gloo on
CPU) and ``LocalTransport`` (all partitions in one process, e.g. several
partitions on one GPU for parity tests: windows run one partition after
another, never waiting on each other inside a kernel).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from .errors import ConfigurationError


# ------------------------------------------------------------------ layout

def split_range(n: int, parts: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced neuron range [lo, hi) of partition `rank`."""
    if parts < 1 or n < parts:
        raise ConfigurationError(f"cannot split {n} neurons into {parts} partitions")
    base, extra = divmod(n, parts)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def partition_csr(rowptr, col, weight, delay, lo: int, hi: int):
    """The CSR of edges into [lo, hi): every source keeps its (possibly empty)
    row, columns become local (col - lo), row order is preserved.  Returns
    (rowptr, col, weight, delay, edge_ids) with edge_ids the global edge index
    of each local edge."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    col = np.asarray(col)
    keep = (col >= lo) & (col < hi)
    edge_ids = np.nonzero(keep)[0].astype(np.int64)
    ck = np.zeros(len(col) + 1, dtype=np.int64)
    np.cumsum(keep, out=ck[1:])
    rp = ck[rowptr]                           # kept edges before each row start
    return (rp, (col[keep] - lo).astype(np.int32), np.asarray(weight)[keep], np.asarray(delay)[keep], edge_ids)


def slice_mask(mask: np.ndarray, n: int, lo: int, hi: int) -> np.ndarray:
    """Packed drive mask [B, T, ceil(n/32)] restricted to neurons [lo, hi)."""
    from .workload import pack_mask, unpack_mask
    mask = np.asarray(mask, dtype=np.uint32)
    out = np.empty(mask.shape[:2] + ((hi - lo + 31) // 32,), dtype=np.uint32)
    for b in range(mask.shape[0]):
        out[b] = pack_mask(unpack_mask(mask[b], n)[:, lo:hi])
    return out


def min_delay_steps(delay, dt: float, dtype=np.float64) -> int:
    """D_min = min_e floor(d_e / dt) in the engine's precision (the device's
    lower delivery bound, eq_device.cuh delivery_code)."""
    d = np.asarray(delay, dtype=dtype)
    return int(np.floor(d / dtype(dt)).min()) if d.size else 1


def windows(t_steps: int, w: int) -> List[Tuple[int, int]]:
    if w < 1:
        raise ConfigurationError("exchange window must be >= 1 step")
    return [(a, min(a + w, t_steps)) for a in range(0, t_steps, w)]


# ------------------------------------------------------------------ routing (pure; CPU-tested)

def route_imports(exports: Sequence[torch.Tensor], rank: int) -> torch.Tensor:
    """Spikes partition `rank` imports: the other partitions' exports in rank order."""
    others = [e for r, e in enumerate(exports) if r != rank]
    if not others:
        return exports[rank][:0]
    return torch.cat(others, dim=0)


def route_adjoints(partials: Sequence[torch.Tensor], counts: Sequence[int], rank: int) -> torch.Tensor:
    """Sum, for partition `rank`'s exported spikes, the partial dL/dt_spk every
    other partition computed over its edges.  partials[q] is partition q's
    vector over its import block (the exports of all p != q in rank order,
    counts[p] records each); the owner adds them in ascending q."""
    P = len(counts)
    acc = None
    for q in range(P):
        if q == rank:
            continue
        off = sum(counts[p] for p in range(rank) if p != q)
        seg = partials[q][off:off + counts[rank]]
        acc = seg.clone() if acc is None else acc + seg
    if acc is None:
        return partials[rank][:0]
    return acc


# ------------------------------------------------------------------ transports

class LocalTransport:
    """All partitions in this process: collectives are list operations."""

    def __init__(self, parts: int):
        self.parts = parts


class PeerTransport:
    """All partitions in this process with the device-resident exchange
    (eq_set_peers): each partition's kernels read the other partitions' spike
    logs (forward) and import-adjoint blocks (reverse) directly — on one GPU,
    or on several with P2P access over NVLink — so the window loop makes no
    host round trip and no copy: windows are ordered by the stream (one device)
    or by CUDA events (several)."""

    def __init__(self, parts: int):
        self.parts = parts


class DistTransport:
    """One partition per process over torch.distributed (NCCL on B200)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.parts = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_gather_varlen(self, t: torch.Tensor) -> List[torch.Tensor]:
        """All-gather of a [n, ...] tensor whose n differs per rank."""
        dist = self.dist
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        ns = [torch.zeros_like(n) for _ in range(self.parts)]
        dist.all_gather(ns, n, group=self.group)
        ns = [int(x.item()) for x in ns]
        mx = max(ns)
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[:t.shape[0]] = t
        bufs = [torch.empty_like(pad) for _ in range(self.parts)]
        dist.all_gather(bufs, pad, group=self.group)
        return [b[:k] for b, k in zip(bufs, ns)]

    def min_int(self, v: int, device) -> int:
        t = torch.tensor([v], dtype=torch.int64, device=device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return int(t.item())


# ------------------------------------------------------------------ driver

@dataclass
class PartitionSpec:
    n_global: int
    lo: int
    hi: int
    edge_ids: np.ndarray      # global edge index of each local edge


class PartitionedNetwork:
    """Forward + reverse of one network over partitions.

    ``engines[k]`` is the engine of partition ``ranks[k]`` (an ``Engine``
    created with ``partition=(n_global, lo)``, network and drive set).  With a
    ``LocalTransport`` all partitions are local (ranks = 0..P-1); with a
    ``DistTransport`` exactly one is (this process's rank)."""

    def __init__(self, engines, ranks: Sequence[int], transport, window: int):
        self.engines = list(engines)
        self.ranks = list(ranks)
        self.tp = transport
        self.P = transport.parts
        self.W = int(window)
        if isinstance(transport, (LocalTransport, PeerTransport)) and self.ranks != list(range(self.P)):
            raise ConfigurationError("a local transport needs every partition")
        self.peer = isinstance(transport, PeerTransport)
        if self.peer:
            for k, e in enumerate(self.engines):
                e.set_peers(self.engines, k)
        self.counts: List[List[int]] = []     # per forward window: export count of every partition
        self.win: List[Tuple[int, int]] = []

    # -- collectives over the partitions, whatever the transport
    def _order(self) -> None:
        """Peer exchange on several streams (partitions running concurrently
        on one GPU's SM subsets, or on several GPUs): every partition's next
        window starts after every partition's current one — CUDA events, no
        host wait."""
        streams = [e.torch_stream for e in self.engines]
        if len({s.cuda_stream for s in streams}) < 2:
            return
        evs = []
        for st in streams:
            ev = torch.cuda.Event()
            ev.record(st)
            evs.append(ev)
        for st in streams:
            for ev in evs:
                st.wait_event(ev)

    def join(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Make `stream` (default: the current stream of the first engine's
        device) wait for every partition's stream."""
        stream = stream or torch.cuda.current_stream(self.engines[0].device)
        for e in self.engines:
            st = e.torch_stream
            if st.cuda_stream != stream.cuda_stream:
                ev = torch.cuda.Event()
                ev.record(st)
                stream.wait_event(ev)

    def _gather(self, mine: List[torch.Tensor]) -> List[torch.Tensor]:
        if isinstance(self.tp, LocalTransport):
            return mine
        return self.tp.all_gather_varlen(mine[0])

    def unify_frac_bits(self) -> int:
        fb = min(e.frac_bits for e in self.engines)
        if isinstance(self.tp, DistTransport):
            fb = self.tp.min_int(fb, self.engines[0].device)
        for e in self.engines:
            e.set_frac_bits(fb)
        return fb

    def forward(self, t_steps: int, sync: bool = True) -> None:
        """sync=False (peer exchange): no host wait at the end (errors surface at
        the next sync) — the whole window loop is then one stream-ordered
        sequence that a CUDA graph can capture (scripts/c5_partitioned.py --graph)."""
        self.unify_frac_bits()
        for e in self.engines:
            e.reset()
        self.counts, self.win = [], windows(t_steps, self.W)
        if self.peer:
            for w, (a, b) in enumerate(self.win):
                a_prev = self.win[w - 1][0] if w else 0
                for e in self.engines:
                    e.run_window(w, a_prev, b - a)
                self._order()
            for e in self.engines:          # deliver the last window's spikes (queue contents)
                e.run_window(len(self.win), self.win[-1][0], 0)
            self._order()
            if sync:
                for e in self.engines:
                    e.sync()
            return
        for a, b in self.win:
            for e in self.engines:
                e.run(b - a)
            exports = self._gather([e.export_spikes(a, b) for e in self.engines])
            self.counts.append([int(x.shape[0]) for x in exports])
            for e, r in zip(self.engines, self.ranks):
                e.import_spikes(route_imports(exports, r))
        # the last window's spikes are due after the run: deliver them so the
        # queues (and event counters) hold what the unpartitioned network's do
        for e in self.engines:
            e.run(0)

    def backward(self, v_bars: Sequence[torch.Tensor], want_amp: bool = True, sync: bool = True):
        grads = [e.backward_begin(vb, None, want_amp) for e, vb in zip(self.engines, v_bars)]
        if self.peer:
            self._order()
            for w in range(len(self.win) - 1, -1, -1):
                a, b = self.win[w]
                for e in self.engines:
                    e.backward_window_peer(w, a, b)
                self._order()
            if sync:
                for e in self.engines:
                    e.sync()
            return grads
        for wi in range(len(self.win) - 1, -1, -1):
            a, _ = self.win[wi]
            for e in self.engines:
                e.backward_window(a)
            if wi == 0:
                break
            # spikes of window wi-1 were imported before forward launch a
            counts = self.counts[wi - 1]
            mine = []
            for e, r in zip(self.engines, self.ranks):
                n_imp = sum(counts) - counts[r]
                mine.append(e.import_adjoints(a, n_imp))
            partials = self._gather(mine)
            lo_prev = self.win[wi - 1][0]
            for e, r in zip(self.engines, self.ranks):
                e.add_spike_adjoints(lo_prev, route_adjoints(partials, counts, r))
        return grads


class GraphedPass:
    """One partitioned forward + reverse (peer exchange) captured as a single
    CUDA graph: every window's launches on every partition's stream and the
    events that order them are recorded once; `replay()` re-runs the whole
    pass with no per-launch host work (scripts/c5_partitioned.py --graph;
    equal to the eager pass, tests/test_gpu_partition.py).

    v_bar_fn(engines) -> list of dL/dV per partition, computed on the device
    from the forward's final state (it is captured too).  The returned
    gradient buffers belong to the graph and are overwritten by each replay."""

    def __init__(self, pn: "PartitionedNetwork", t_steps: int, v_bar_fn, want_amp: bool = False):
        if not pn.peer:
            raise ValueError("graph capture needs the peer exchange (PeerTransport)")
        self.pn = pn
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            cap = torch.cuda.current_stream()
            pn.forward(t_steps, sync=False)
            pn.join(cap)
            self.grads = pn.backward(v_bar_fn(pn.engines), want_amp=want_amp, sync=False)
            pn.join(cap)

    def replay(self, sync: bool = False):
        """Run the captured pass on the current stream; sync=True waits and
        raises any device error of the windows."""
        self.graph.replay()
        if sync:
            for e in self.pn.engines:
                e.sync()
        return self.grads
