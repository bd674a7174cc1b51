"""One network partitioned into P ranges (BASELINE config 5),
all partitions on one GPU through LocalTransport — windows run partition after
partition, never waiting on each other inside a kernel.

Forward: raster, spike times, final V/I, counters and pending queue contents of
the partitions equal the unpartitioned engine's BITWISE (fixed-point slot sums
are order-free; all partitions use the common fraction bits).  The
unpartitioned engine itself equals the CPU oracle bitwise (test_gpu_parity.py);
one case here checks the partitioned raster against the oracle directly.
Reverse: each spike's dL/dt_spk is summed as (own edges) + (other partitions
in rank order) instead of one row-order sum, so gradients agree to rounding:
fp64 within 1e-10, fp32 within 1e-4 of the gradient scale.
"""

import numpy as np
import pytest

from paper_2512_05906_b200 import workload as wl
from paper_2512_05906_b200.partition import (GraphedPass, LocalTransport, PartitionedNetwork, PeerTransport, min_delay_steps,
                                             partition_csr, slice_mask, split_range)

pytestmark = pytest.mark.gpu

DT = 1e-3


def _whole(net, mask, amp, B, T, precision):
    from paper_2512_05906_b200.engine import Engine
    e = Engine(net.n, B, T, precision=precision)
    e.set_network(net.rowptr, net.col, net.weight, net.delay)
    e.set_drive(mask, amp)
    return e


def _parts(net, mask, amp, B, T, precision, P):
    from paper_2512_05906_b200.engine import Engine
    engines, ids, ranges = [], [], []
    for r in range(P):
        lo, hi = split_range(net.n, P, r)
        rp, cl, w, d, eid = partition_csr(net.rowptr, net.col, net.weight, net.delay, lo, hi)
        e = Engine(hi - lo, B, T, precision=precision, partition=(net.n, lo))
        e.set_network(rp, cl, w, d)
        e.set_drive(slice_mask(mask, net.n, lo, hi), amp[lo:hi])
        engines.append(e)
        ids.append(eid)
        ranges.append((lo, hi))
    return engines, ids, ranges


def _raster(eng, offset=0):
    s = eng.spikes()
    return np.stack([s["trial"], s["step"], s["neuron"] + offset], 1), s["t"]


def _sorted(rows, t):
    order = np.lexsort((rows[:, 2], rows[:, 1], rows[:, 0]))
    return rows[order], t[order]


def _problem(n=600, k=30, delays=(4, 20), B=2, T=300, seed=5):
    net = wl.random_network(n, k, seed, delay_steps=delays, w_mean=0.04, w_std=0.01)
    mask = wl.drive_masks(n, B, T, DT, seed0=40)
    amp = np.full(n, 12.0)
    return net, mask, amp


@pytest.mark.parametrize("precision,P,window,peer", [(32, 2, None, False), (32, 3, None, False),
                                                     (64, 3, None, False), (32, 4, 1, False), (64, 2, 2, False),
                                                     (32, 3, None, True), (64, 4, 2, True), (32, 8, None, True)])
def test_partitioned_run_equals_whole_network(precision, P, window, peer):
    """LocalTransport (host-routed exchange) and PeerTransport (each
    partition's kernels read the others' spike logs / import adjoints directly,
    no host round trip per window)."""
    B, T = 2, 300
    net, mask, amp = _problem(B=B, T=T)
    whole = _whole(net, mask, amp, B, T, precision)
    out = whole.forward()
    engines, ids, ranges = _parts(net, mask, amp, B, T, precision, P)
    dmin = min_delay_steps(net.delay, DT, np.float32 if precision == 32 else np.float64)
    assert dmin == 4
    tp = PeerTransport(P) if peer else LocalTransport(P)
    pn = PartitionedNetwork(engines, range(P), tp, window=window or dmin)
    pn.forward(T)
    assert all(e.frac_bits == whole.frac_bits for e in engines)
    # raster + spike times
    rows, ts = zip(*[_raster(e, lo) for e, (lo, _) in zip(engines, ranges)])
    got_r, got_t = _sorted(np.concatenate(rows), np.concatenate(ts))
    ref_r, ref_t = _sorted(*_raster(whole))
    assert len(ref_r) > 100
    assert np.array_equal(got_r, ref_r) and np.array_equal(got_t, ref_t)
    # state, counters, queue contents
    v = out["v"].cpu().numpy()
    i = out["i"].cpu().numpy()
    ctr = np.zeros_like(whole.counters())
    pend = whole.pending()
    for e, (lo, hi) in zip(engines, ranges):
        st = e.state()
        assert np.array_equal(st["v"].cpu().numpy(), v[:, lo:hi])
        assert np.array_equal(st["i"].cpu().numpy(), i[:, lo:hi])
        ctr += e.counters()
        assert np.array_equal(e.pending(), pend[:, lo:hi])
    assert np.array_equal(ctr, whole.counters())
    # reverse pass
    vbar = 2.0 * (out["v"].double() - 0.25)
    gw, gd, ga = (x.cpu().numpy() for x in whole.backward(vbar.to(out["v"].dtype)))
    grads = pn.backward([vbar[:, lo:hi].to(out["v"].dtype) for lo, hi in ranges])
    pw = np.zeros_like(gw)
    pd = np.zeros_like(gd)
    pa = np.zeros_like(ga)
    for (w_, d_, a_), eid, (lo, hi) in zip(grads, ids, ranges):
        pw[eid] = w_.cpu().numpy()
        pd[eid] = d_.cpu().numpy()
        pa[lo:hi] = a_.cpu().numpy()
    tol = 1e-10 if precision == 64 else 1e-4
    for got, ref in ((pw, gw), (pd, gd), (pa, ga)):
        assert np.abs(ref).max() > 0
        np.testing.assert_allclose(got, ref, rtol=tol, atol=tol * np.abs(ref).max())


@pytest.mark.parametrize("precision", [32, 64])
def test_concurrent_peer_partitions_equal_whole_network(precision):
    """Partitions on their own streams and SM shares (grid 2*SMs/P each),
    running side by side as on P GPUs, windows ordered by CUDA events: same
    raster, state and queues as the whole network; gradients to rounding."""
    import torch
    from paper_2512_05906_b200.engine import Engine
    B, T, P = 2, 300, 4
    net, mask, amp = _problem(B=B, T=T, seed=9)
    whole = _whole(net, mask, amp, B, T, precision)
    out = whole.forward()
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    engines, ids, ranges = [], [], []
    for r in range(P):
        lo, hi = split_range(net.n, P, r)
        rp, cl, w, d, eid = partition_csr(net.rowptr, net.col, net.weight, net.delay, lo, hi)
        e = Engine(hi - lo, B, T, precision=precision, partition=(net.n, lo), max_ctas=(2 * sm) // P,
                   stream=torch.cuda.Stream())
        e.set_network(rp, cl, w, d)
        e.set_drive(slice_mask(mask, net.n, lo, hi), amp[lo:hi])
        engines.append(e)
        ids.append(eid)
        ranges.append((lo, hi))
    assert engines[0].geometry[0] <= (2 * sm) // P
    pn = PartitionedNetwork(engines, range(P), PeerTransport(P), window=4)
    pn.forward(T)
    pn.join()
    rows, ts = zip(*[_raster(e, lo) for e, (lo, _) in zip(engines, ranges)])
    got_r, got_t = _sorted(np.concatenate(rows), np.concatenate(ts))
    ref_r, ref_t = _sorted(*_raster(whole))
    assert np.array_equal(got_r, ref_r) and np.array_equal(got_t, ref_t)
    v = out["v"].cpu().numpy()
    pend = whole.pending()
    for e, (lo, hi) in zip(engines, ranges):
        assert np.array_equal(e.state()["v"].cpu().numpy(), v[:, lo:hi])
        assert np.array_equal(e.pending(), pend[:, lo:hi])
    vbar = 2.0 * (out["v"].double() - 0.25)
    gw, gd, _ = (x.cpu().numpy() for x in whole.backward(vbar.to(out["v"].dtype)))
    grads = pn.backward([vbar[:, lo:hi].to(out["v"].dtype) for lo, hi in ranges])
    pn.join()
    pw = np.zeros_like(gw)
    for (w_, _, _), eid in zip(grads, ids):
        pw[eid] = w_.cpu().numpy()
    tol = 1e-10 if precision == 64 else 1e-4
    np.testing.assert_allclose(pw, gw, rtol=tol, atol=tol * np.abs(gw).max())


def test_partitioned_raster_matches_the_oracle():
    from oracle.oracle import OracleSession
    B, T, P = 1, 250, 3
    net, mask, amp = _problem(n=300, k=20, delays=(3, 12), B=B, T=T, seed=11)
    engines, _, ranges = _parts(net, mask, amp, B, T, 32, P)
    pn = PartitionedNetwork(engines, range(P), LocalTransport(P), window=3)
    pn.forward(T)
    s = OracleSession(n=net.n, n_trials=B, t_steps=T, mode="device", precision=32, frac_bits=engines[0].frac_bits)
    s.set_network(net.rowptr, net.col, net.weight, net.delay)
    s.set_drive(mask, amp)
    ref = s.forward()
    rows, ts = zip(*[_raster(e, lo) for e, (lo, _) in zip(engines, ranges)])
    got_r, got_t = _sorted(np.concatenate(rows), np.concatenate(ts))
    ref_r, ref_t = _sorted(np.stack([ref["trial"], ref["step"], ref["neuron"]], 1), ref["t"])
    assert len(ref_r) > 50
    assert np.array_equal(got_r, ref_r) and np.array_equal(got_t.astype(np.float64), ref_t)
    v = np.concatenate([e.state()["v"].double().cpu().numpy() for e in engines], axis=1)
    assert np.array_equal(v, ref["v"])


def test_window_longer_than_min_delay_is_a_causality_error():
    from paper_2512_05906_b200.errors import CausalityError
    B, T, P = 1, 200, 2
    net, mask, amp = _problem(n=300, k=20, delays=(4, 4), B=B, T=T, seed=3)
    engines, _, _ = _parts(net, mask, amp, B, T, 32, P)
    pn = PartitionedNetwork(engines, range(P), LocalTransport(P), window=7)
    with pytest.raises(CausalityError):
        pn.forward(T)


def test_partition_api_rules():
    from paper_2512_05906_b200.engine import Engine
    from paper_2512_05906_b200.errors import ConfigurationError
    with pytest.raises(ConfigurationError, match="ring kind"):
        Engine(100, 1, 10, kind="binaryheap", capacity=4, partition=(200, 0))
    with pytest.raises(ConfigurationError, match="outside"):
        Engine(100, 1, 10, partition=(150, 60))
    net, mask, amp = _problem(n=200, k=10, delays=(4, 8), B=1, T=50, seed=2)
    engines, _, _ = _parts(net, mask, amp, 1, 50, 32, 2)
    e0 = engines[0]
    e0.reset()
    e0.run(40)
    own = e0.export_spikes(0, 40)
    if own.shape[0]:
        with pytest.raises(ConfigurationError, match="not a remote spike"):
            e0.import_spikes(own)          # own spikes are not remote
    with pytest.raises(ConfigurationError, match="fraction bits"):
        e0.set_frac_bits(e0.frac_bits + 1)


@pytest.mark.parametrize("concurrent", [False, True])
def test_peer_partitions_in_one_cuda_graph_equal_eager(concurrent):
    """The peer-exchange forward + reverse has no host synchronisation inside
    (forward/backward with sync=False), so the whole sequence — every
    window's launches on every partition's stream and the CUDA events that
    order them — is captured in one CUDA graph.  Two replays give exactly the
    eager run's state and gradients (scripts/c5_partitioned.py --graph)."""
    import torch
    from paper_2512_05906_b200.engine import Engine
    B, T, P = 1, 200, 4        # one trial: each edge gets at most one gradient term per phase (bitwise)
    net, mask, amp = _problem(B=B, T=T, seed=13)
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    engines, ranges = [], []
    for r in range(P):
        lo, hi = split_range(net.n, P, r)
        rp, cl, w, d, eid = partition_csr(net.rowptr, net.col, net.weight, net.delay, lo, hi)
        e = Engine(hi - lo, B, T, precision=32, partition=(net.n, lo),
                   max_ctas=(2 * sm) // P if concurrent else 0, stream=torch.cuda.Stream() if concurrent else None)
        e.set_network(rp, cl, w, d)
        e.set_drive(slice_mask(mask, net.n, lo, hi), amp[lo:hi])
        engines.append(e)
        ranges.append((lo, hi))
    pn = PartitionedNetwork(engines, range(P), PeerTransport(P), window=4)

    def vbars():
        return [(2.0 * (e.state()["v"].double() - 0.25)).to(torch.float32) for e in engines]

    pn.forward(T)
    pn.join()
    v_ref = [e.state()["v"].clone() for e in engines]
    g_ref = [tuple(x.clone() for x in g[:2]) for g in pn.backward(vbars(), want_amp=False)]
    pn.join()
    torch.cuda.synchronize()
    gp = GraphedPass(pn, T, lambda es: vbars())
    for _ in range(2):
        grads = gp.replay(sync=True)
        for e, v in zip(engines, v_ref):
            assert torch.equal(e.state()["v"], v)
        for (gw, gd, _), (rw, rd) in zip(grads, g_ref):
            assert torch.equal(gw, rw) and torch.equal(gd, rd)
