"""Reference-shaped network API (paper_2512_05906_b200.network).

CPU tests: validation messages (network.py:213-268), dense->CSR mapping,
PoissonDrive draws equal the reference's (when /root/reference is present).
GPU tests: simulate / forward_gradient / grad_fd_oracle / PrimalRSNN /
RSNNFunction against the reference fixtures."""

import os
import sys

import numpy as np
import pytest

from golden_cases import BY_NAME, ref_loss
from paper_2512_05906_b200.errors import ConfigurationError
from paper_2512_05906_b200.network import (NetworkParams, PoissonDrive, SeedDirection, build_rsnn,
                                           _edge_index)

DT = 1e-3
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def params_for(case):
    net, mask, amp = case.inputs()
    w, d = net.dense(DT)
    p = NetworkParams(n=net.n, weights=w, delays=d, tau_m=1.0, tau_syn=0.5, v_th=1.0, v_reset=0.0, dt=DT,
                      queue_kind=case.kind, queue_capacity=case.capacity, refractory_steps=case.refractory,
                      v_target=np.full(net.n, 0.25), exact_delivery=case.exact)
    from paper_2512_05906_b200.workload import unpack_mask
    return p, (unpack_mask(mask[0], net.n), amp)


def small(n=4, kind="ring", homog=False):
    rng = np.random.default_rng(0)
    d = np.full((n, n), 16 * DT) if homog else rng.uniform(14 * DT, 30 * DT, (n, n))
    np.fill_diagonal(d, DT)
    w = rng.normal(0.3, 0.1, (n, n))
    np.fill_diagonal(w, 0.0)
    return NetworkParams(n=n, weights=w, delays=d, tau_m=1.0, tau_syn=0.5, v_th=1.0, v_reset=0.0, dt=DT,
                         queue_kind=kind)


# ------------------------------------------------------------------ CPU

def test_validation_messages_match_the_reference():
    p = small()
    p.delays[0, 2] = 0.2 * DT
    with pytest.raises(ConfigurationError, match=r"edge \(0,2\).*below one step"):
        build_rsnn(p)
    with pytest.raises(ConfigurationError, match="homogeneous"):
        build_rsnn(small(kind="fiforing"))
    q = small()
    q.n = 1
    q.weights = np.zeros((1, 1))
    q.delays = np.full((1, 1), DT)
    with pytest.raises(ConfigurationError, match="n >= 2"):
        build_rsnn(q)
    r = small()
    r.tau_syn = r.tau_m
    with pytest.raises(ConfigurationError, match="tau_m != tau_syn"):
        build_rsnn(r)
    with pytest.raises(ConfigurationError, match="not a valid off-diagonal edge"):
        build_rsnn(small(), seed=SeedDirection("weight", 1, 1))
    with pytest.raises(ConfigurationError, match="bgpq"):
        build_rsnn(small(kind="bgpq"))


def test_dense_to_csr_keeps_every_off_diagonal_pair():
    p = small(5)
    net = p.csr()
    assert net.n_edges == 20 and np.array_equal(np.diff(net.rowptr), np.full(5, 4))
    for i in range(5):
        for j in range(5):
            if i != j:
                x = _edge_index(5, i, j)
                assert net.col[x] == j and net.weight[x] == p.weights[i, j]


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not mounted")
def test_poisson_drive_draws_equal_the_reference():
    sys.path.insert(0, "/root/reference/pkg/src")
    from eventq.network import PoissonDrive as RefDrive
    a = PoissonDrive(7, 16 * DT, 12.0, 12 * DT, 0.5, 123)
    b = RefDrive(7, 16 * DT, 12.0, 12 * DT, 0.5, 123)
    assert a.pulses == b.pulses
    act = a.active(500, DT)
    rows = b.materialize(500, DT)
    ref = np.array([[x.primal != 0.0 for x in rows(m)] for m in range(500)])
    assert np.array_equal(act, ref)


# ------------------------------------------------------------------ GPU

@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dense_ring_n8", "dense_heap_cap3_n12", "dense_fifo_cap2_n12",
                                  "dense_ring_refr3_n10", "dense_ring_plain_n10", "dense_lossy_cap6_n10"])
def test_simulate_matches_reference_fixture(name):
    from paper_2512_05906_b200.network import simulate
    case = BY_NAME[name]
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    p, drive = params_for(case)
    res = simulate(build_rsnn(p), case.t_steps, drive, record=True)
    assert sorted(res.raster) == [tuple(r) for r in g["raster"].tolist()]
    assert res.spike_count == int(g["spike_count"]) and res.drop_count == int(g["drop_count"])
    assert res.enqueued_count == int(g["enqueued_count"])
    np.testing.assert_allclose(res.voltages, g["v_trace"], rtol=1e-9, atol=1e-12)
    assert res.loss.primal == pytest.approx(float(g["loss"]), rel=1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["dense_ring_n8", "dense_ring_refr3_n10", "dense_ring_plain_n10",
                                  "dense_sorted_plain_cap3_n12", "dense_lossy_cap6_n10",
                                  "dense_lossy_cap5_plain_n10"])
def test_forward_gradient_equals_reference_jvp(name):
    from paper_2512_05906_b200.network import forward_gradient
    case = BY_NAME[name]
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    p, drive = params_for(case)
    for (kind, i, j), jvp in zip(g["directions"].tolist(), g["jvp"].tolist()):
        d = SeedDirection(["weight", "delay", "drive"][kind], i, j)
        got, _ = forward_gradient(p, d, case.t_steps, drive)
        assert got == pytest.approx(jvp, rel=1e-7, abs=1e-10)


@pytest.mark.gpu
def test_full_gradient_agrees_with_directions_and_fd():
    from paper_2512_05906_b200.network import forward_gradient, full_gradient, grad_fd_oracle
    p = small(3)
    p.v_target = np.full(3, 0.2)
    drive = PoissonDrive(3, 16 * DT, 12.0, 12 * DT, 1.0, 29)
    GW, GD, GA = full_gradient(p, 1000, drive)
    d = SeedDirection("weight", 0, 1)
    jvp, res = forward_gradient(p, d, 1000, drive)
    assert res.spike_count > 0
    assert GW[0, 1] == pytest.approx(jvp, rel=1e-12)
    fd = grad_fd_oracle(p, d, 2e-3, 1000, drive)
    assert jvp == pytest.approx(fd, rel=5e-2)
    dd = SeedDirection("delay", 0, 1)
    jd, _ = forward_gradient(p, dd, 1000, drive)
    assert GD[0, 1] == pytest.approx(jd, rel=1e-12)
    assert jd == pytest.approx(grad_fd_oracle(p, dd, 4 * DT, 1000, drive), rel=5e-2, abs=1e-9)


@pytest.mark.gpu
def test_quiescent_network_has_zero_spikes_and_gradients():
    from paper_2512_05906_b200.network import forward_gradient, simulate
    p = small(3)
    res = simulate(build_rsnn(p), 300)
    assert res.spike_count == 0 and np.all(res.v_final == 0.0)
    for d in (SeedDirection("weight", 0, 1), SeedDirection("delay", 1, 0)):
        assert forward_gradient(p, d, 200)[0] == 0.0


@pytest.mark.gpu
def test_primal_twin_equals_simulate():
    from paper_2512_05906_b200.network import PrimalRSNN, simulate
    case = BY_NAME["dense_ring_n8"]
    p, drive = params_for(case)
    g = np.load(os.path.join(GOLDEN, case.name + ".npz"))
    pr = PrimalRSNN(p)
    pr.run(case.t_steps, drive)
    np.testing.assert_allclose(pr.v, g["v_final_primal"], rtol=1e-9, atol=1e-12)
    assert pr.v == simulate(build_rsnn(p), case.t_steps, drive).v_final.tolist()


@pytest.mark.gpu
def test_autograd_function_gradients():
    import torch
    from paper_2512_05906_b200.engine import Engine
    from paper_2512_05906_b200.network import RSNNFunction
    from paper_2512_05906_b200 import workload as wl
    net = wl.random_network(120, 12, 3, delay_steps=(1, 10), w_mean=0.04, w_std=0.01)
    B, T = 2, 300
    mask = torch.from_numpy(wl.drive_masks(120, B, T, DT, seed0=4).view(np.int32)).cuda()
    eng = Engine(120, B, T, precision=64)
    w = torch.tensor(net.weight, dtype=torch.float64, device="cuda", requires_grad=True)
    d = torch.tensor(net.delay, dtype=torch.float64, device="cuda", requires_grad=True)
    a = torch.full((120,), 12.0, dtype=torch.float64, device="cuda", requires_grad=True)
    rp = torch.from_numpy(net.rowptr).cuda()
    cl = torch.from_numpy(net.col).cuda()
    v = RSNNFunction.apply(w, d, a, eng, rp, cl, mask)
    loss = ((v - 0.25) ** 2).sum()
    loss.backward()
    gw, gd, ga = eng.backward((2 * (v.detach() - 0.25)))
    assert torch.equal(w.grad, gw) and torch.equal(d.grad, gd) and torch.equal(a.grad, ga)
    assert float(w.grad.abs().sum()) > 0
    # a small step along -grad lowers the loss (sanity of sign and scale)
    with torch.no_grad():
        w2 = (w - 1e-3 * w.grad / w.grad.abs().max()).detach()
    v2 = RSNNFunction.apply(w2, d.detach(), a.detach(), eng, rp, cl, mask)
    assert float(((v2 - 0.25) ** 2).sum()) < float(loss)


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not mounted")
def test_gradcheck_sampling_and_error_rule_equal_the_reference():
    """paper_2512_05906_b200.gradcheck mirrors eventq.gradcheck: the same random
    directions for the same Generator, and the same relative-error rule
    (ensemble floor) on the same (jvp, fd) pairs."""
    sys.path.insert(0, "/root/reference/pkg/src")
    import eventq.gradcheck as ref
    from paper_2512_05906_b200 import gradcheck as ours
    a = ours.sample_directions(10, 40, np.random.default_rng(11))
    b = ref.sample_directions(10, 40, np.random.default_rng(11))
    assert [(d.param, d.i, d.j) for d in a] == [(d.param, d.i, d.j) for d in b]
    pairs = [(0.5, 0.49), (1e-4, 3e-4), (-0.2, -0.21), (0.01, 0.0)]
    mk = lambda m: [m.DirectionCheck(None, j, f, None, 1e-3, "ok") for j, f in pairs] + \
        [m.DirectionCheck(None, 9.0, None, None, 1e-3, "non-smooth")]
    x, y = mk(ours), mk(ref)
    ours._fill_relative_errors(x)
    ref._fill_relative_errors(y)
    assert [c.rel_err for c in x] == [c.rel_err for c in y]
    assert ours.direction_epsilon(a[1], small(), 1e-3, 4.0) == ref.direction_epsilon(b[1], small(), 1e-3, 4.0)
