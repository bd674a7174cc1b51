"""Host logic of the partitioned network (paper_2512_05906_b200.partition) on
CPU: layout helpers, routing, and the window protocol over torch.distributed
(gloo, world size 2 and 3) with stand-in engines that record what they are
given.  The kernels behind the protocol are covered by test_gpu_partition.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_05906_b200 import workload as wl
from paper_2512_05906_b200.partition import (DistTransport, LocalTransport, PartitionedNetwork, min_delay_steps,
                                             partition_csr, route_adjoints, route_imports, slice_mask, split_range,
                                             windows)


def test_split_range_and_windows():
    for n in (8, 100, 1001):
        for P in (1, 2, 3, 8):
            rs = [split_range(n, P, r) for r in range(P)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
    assert windows(10, 4) == [(0, 4), (4, 8), (8, 10)]
    assert windows(8, 8) == [(0, 8)]


def test_partition_csr_keeps_every_edge_once_in_row_order():
    net = wl.random_network(300, 17, 4, delay_steps=(2, 9))
    P = 3
    seen = []
    for r in range(P):
        lo, hi = split_range(net.n, P, r)
        rp, cl, w, d, eid = partition_csr(net.rowptr, net.col, net.weight, net.delay, lo, hi)
        assert rp.shape == (net.n + 1,) and rp[-1] == len(cl)
        assert np.all((cl >= 0) & (cl < hi - lo))
        assert np.array_equal(cl + lo, net.col[eid]) and np.array_equal(w, net.weight[eid])
        src = np.repeat(np.arange(net.n), np.diff(rp))
        gsrc = np.repeat(np.arange(net.n), np.diff(net.rowptr))
        assert np.array_equal(src, gsrc[eid])            # rows preserved
        assert np.all(np.diff(eid) > 0)                  # CSR order preserved
        seen.append(eid)
    allid = np.sort(np.concatenate(seen))
    assert np.array_equal(allid, np.arange(net.n_edges))
    assert min_delay_steps(net.delay, 1e-3) == 2


def test_slice_mask_selects_the_neuron_range():
    n = 77
    mask = wl.drive_masks(n, 2, 30, 1e-3, seed0=5)
    full = np.stack([wl.unpack_mask(mask[b], n) for b in range(2)])
    part = slice_mask(mask, n, 20, 61)
    assert part.shape == (2, 30, 2)
    got = np.stack([wl.unpack_mask(part[b], 41) for b in range(2)])
    assert np.array_equal(got, full[:, :, 20:61])


def test_routing_matches_brute_force():
    rng = np.random.default_rng(0)
    for P in (2, 3, 5):
        counts = list(rng.integers(0, 6, P))
        exports = [torch.from_numpy(np.stack([np.full(c, r), np.arange(c)], 1)) for r, c in enumerate(counts)]
        for r in range(P):
            imp = route_imports(exports, r)
            exp = [(p, k) for p in range(P) if p != r for k in range(counts[p])]
            assert [tuple(x) for x in imp.tolist()] == exp
        # partial of partition q for record (p, k) = 100*q + 10*p + k
        partials = [torch.tensor([100.0 * q + 10 * p + k for p in range(P) if p != q for k in range(counts[p])],
                                 dtype=torch.float64) for q in range(P)]
        for r in range(P):
            got = route_adjoints(partials, counts, r).tolist()
            want = [sum(100.0 * q + 10 * r + k for q in range(P) if q != r) for k in range(counts[r])]
            assert got == want


class FakeEngine:
    """Records the protocol: exports (rank, window, k) records; the partial
    dL/dt_spk it returns for an imported record (p, w, k) is 1000*rank + id."""

    def __init__(self, rank, P, log):
        self.rank, self.P, self.log = rank, P, log
        self.frac_bits = 30 - rank
        self.device = torch.device("cpu")
        self.now = 0
        self.imports = {}

    def set_frac_bits(self, f):
        self.log.append(("frac", f))
        self.frac_bits = f

    def reset(self):
        self.now = 0

    def run(self, n):
        self.log.append(("run", self.now, n))
        self.now += n

    def export_spikes(self, a, b):
        cnt = (self.rank + 1) * (a // 4 + 1) % 5
        return torch.tensor([[self.rank, a, k, 0] for k in range(cnt)], dtype=torch.int32).reshape(-1, 4)

    def import_spikes(self, recs):
        self.imports[self.now] = recs.clone()
        self.log.append(("import", self.now, [tuple(x) for x in recs.tolist()]))

    def backward_begin(self, vb, ib, want_amp):
        return ("grads", self.rank)

    def backward_window(self, a):
        self.log.append(("bwd", a))

    def import_adjoints(self, a, n):
        recs = self.imports[a]
        assert recs.shape[0] == n
        rid = recs[:, 0] * 10000 + recs[:, 1] * 10 + recs[:, 2]
        return 1000.0 * self.rank + rid.double()

    def add_spike_adjoints(self, lo, vals):
        self.log.append(("adj", lo, vals.tolist()))


def _expected_adjoints(rank, P, lo):
    cnt = (rank + 1) * (lo // 4 + 1) % 5
    return [sum(1000.0 * q + rank * 10000 + lo * 10 + k for q in range(P) if q != rank) for k in range(cnt)]


def _check_log(log, rank, P, T, W):
    wins = windows(T, W)
    imports = [x for x in log if x[0] == "import"]
    assert [x[1] for x in imports] == [b for _, b in wins]
    for (a, b), imp in zip(wins, imports):
        want = [(p, a, k, 0) for p in range(P) if p != rank for k in range((p + 1) * (a // 4 + 1) % 5)]
        assert imp[2] == want
    assert [x[1] for x in log if x[0] == "bwd"] == [a for a, _ in reversed(wins)]
    adj = [x for x in log if x[0] == "adj"]
    assert [x[1] for x in adj] == [a for a, _ in reversed(wins[:-1])]
    for x in adj:
        assert x[2] == _expected_adjoints(rank, P, x[1])
    assert ("frac", 30 - (P - 1)) in log


def _worker(rank, world, port, T, W, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        log = []
        tp = DistTransport()
        # variable-length all-gather
        mine = torch.arange(rank + 2, dtype=torch.int32).reshape(-1, 1) + 10 * rank
        got = tp.all_gather_varlen(mine)
        assert [g.flatten().tolist() for g in got] == [list(range(10 * r, 10 * r + r + 2)) for r in range(world)]
        pn = PartitionedNetwork([FakeEngine(rank, world, log)], [rank], tp, window=W)
        pn.forward(T)
        pn.backward([torch.zeros(1)])
        _check_log(log, rank, world, T, W)
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_window_protocol_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    T, W = 22, 4
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, W, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}


def test_window_protocol_local_transport():
    P, T, W = 3, 22, 4
    logs = [[] for _ in range(P)]
    engines = [FakeEngine(r, P, logs[r]) for r in range(P)]
    pn = PartitionedNetwork(engines, range(P), LocalTransport(P), window=W)
    pn.forward(T)
    pn.backward([torch.zeros(1)] * P)
    for r in range(P):
        _check_log(logs[r], r, P, T, W)
