"""The golden cases: how each fixture's inputs are regenerated.

Shared by scripts/make_goldens.py (which runs the Python reference in the build
container) and the tests (which regenerate the identical inputs on any box and
check the stored SHA-256 before comparing outputs).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from paper_2512_05906_b200 import workload as wl

DT = 1e-3


@dataclass
class Case:
    name: str
    n: int
    k_out: int
    kind: str
    t_steps: int
    seed: int
    w_mean: float
    w_std: float
    delay_steps: Tuple[int, int]
    drive_seed: int
    capacity: Optional[int] = None
    refractory: int = 0
    n_dirs: Tuple[int, int, int] = (0, 0, 0)   # weight, delay, drive directions
    slow: bool = False
    exact: bool = True                         # NetworkParams.exact_delivery

    def inputs(self):
        net = wl.random_network(self.n, self.k_out, self.seed, dt=DT, w_mean=self.w_mean,
                                w_std=self.w_std, delay_steps=self.delay_steps)
        mask = wl.drive_masks(self.n, 1, self.t_steps, DT, seed0=self.drive_seed)
        amp = np.full(self.n, 12.0)
        return net, mask, amp

    @property
    def dense(self) -> bool:
        return self.k_out >= self.n - 1


def _dense(name, n, kind, cap, homog, seed, T, dirs=(0, 0, 0), refr=0, dl=None, exact=True):
    if dl is None:
        dl = (16, 16) if homog else (14, 30)
    return Case(name, n, n - 1, kind, T, seed, 0.3, 0.1, dl, 1000 + seed, cap, refr, dirs, exact=exact)


CASES: List[Case] = [
    _dense("dense_ring_n8", 8, "ring", None, False, 1, 1500, (3, 3, 1)),
    _dense("dense_heap_n8", 8, "binaryheap", None, False, 1, 1500),
    _dense("dense_sorted_n8", 8, "sortedarray", None, False, 1, 1500),
    _dense("dense_fifo_n8", 8, "fiforing", None, True, 2, 1500),
    _dense("dense_heap_cap3_n12", 12, "binaryheap", 3, False, 3, 1200),
    _dense("dense_sorted_cap3_n12", 12, "sortedarray", 3, False, 3, 1200),
    _dense("dense_fifo_cap2_n12", 12, "fiforing", 2, True, 4, 1200),
    _dense("dense_donothing_n8", 8, "donothing", None, False, 5, 600),
    _dense("dense_ring_n40", 40, "ring", None, False, 6, 1000, (3, 3, 1)),
    _dense("dense_ring_refr3_n10", 10, "ring", None, False, 7, 1000, (2, 2, 1), refr=3, dl=(2, 20)),
    Case("sparse_ring_n100", 100, 10, "ring", 1000, 8, 0.03, 0.01, (1, 16), 1000, None, 0, (4, 4, 2)),
    # LossyRingQueue networks (network.py:321-328, queues.py:126-181): capacity
    # below the horizon (31) aliases delays into earlier steps; default capacity
    # (horizon*(n-1)+1) is lossless
    _dense("dense_lossy_cap6_n10", 10, "lossyring", 6, False, 9, 1200, (3, 3, 1)),
    _dense("dense_lossy_n8", 8, "lossyring", None, False, 10, 1000, (2, 2, 1)),
    # plain step-aligned delivery (exact_delivery=False, network.py:403-408)
    _dense("dense_ring_plain_n10", 10, "ring", None, False, 11, 1200, (3, 3, 1), exact=False),
    _dense("dense_lossy_cap5_plain_n10", 10, "lossyring", 5, False, 12, 1000, (2, 2, 1), exact=False),
    _dense("dense_sorted_plain_cap3_n12", 12, "sortedarray", 3, False, 13, 1000, (2, 2, 1), exact=False),
    Case("sparse_ring_plain_n100", 100, 10, "ring", 1000, 14, 0.03, 0.01, (1, 16), 1014, None, 0, (3, 3, 1),
         exact=False),
    # BASELINE config 1: 1k neurons, K=100, delays 1..16 steps, ring, T=1000
    Case("c1_ring", 1000, 100, "ring", 1000, 0, 0.003, 0.001, (1, 16), 1000, None, 0, (2, 2, 1),
         slow=True),
]

BY_NAME = {c.name: c for c in CASES}


def pick_directions(net: wl.Network, rng_seed: int, k_w: int, k_d: int, k_a: int):
    """Directions on real (CSR) edges: ("weight"|"delay", i, j) and ("drive", i, -1)."""
    u = wl.uniform(rng_seed, 99, k_w + k_d + k_a)
    src = np.repeat(np.arange(net.n), np.diff(net.rowptr))
    E = net.n_edges
    out = []
    for q in range(k_w):
        x = int(u[q] * E)
        out.append(("weight", int(src[x]), int(net.col[x])))
    for q in range(k_d):
        x = int(u[k_w + q] * E)
        out.append(("delay", int(src[x]), int(net.col[x])))
    for q in range(k_a):
        out.append(("drive", int(u[k_w + k_d + q] * net.n), -1))
    return out


def edge_index(net: wl.Network, i: int, j: int) -> int:
    lo, hi = int(net.rowptr[i]), int(net.rowptr[i + 1])
    x = lo + int(np.searchsorted(net.col[lo:hi], j))
    assert net.col[x] == j
    return x


def ref_loss(v_final: np.ndarray, target: float = 0.25) -> float:
    """Sequential dual-sum order of simulate (network.py:484-489)."""
    loss = 0.0
    for v in v_final:
        diff = float(v) - target
        loss = loss + diff * diff
    return loss
