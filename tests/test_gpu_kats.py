"""The reference's known-answer tests for this path, through the GPU engine
(fp64, ring kind) — SURVEY.md §8(c):

* analytic single-spike delay gradient (pkg/tests/test_acceptance.py:80-102,
  test_jumps.py:197-218): dI(T)/dd = (w/tau_s) e^{-(T - t_post)/tau_s}, 1e-9;
* exact LIF spike time tau_m ln 2 at any dt (test_neuro.py:131-146), 1e-10;
* a crossing is delivered 16 samples later over a 16-step delay
  (test_network.py:117-137);
* gradient locality: edges out of a silent neuron get exactly 0
  (test_network.py:216-226)."""

import math

import numpy as np
import pytest
import torch

from paper_2512_05906_b200 import workload as wl
from paper_2512_05906_b200.engine import Engine

pytestmark = pytest.mark.gpu


def _csr(n, edges):
    """edges: list of (src, dst, w, d) -> rowptr, col, w, d (rows ascending)."""
    edges = sorted(edges)
    rowptr = np.zeros(n + 1, np.int64)
    for s, _, _, _ in edges:
        rowptr[s + 1] += 1
    rowptr = np.cumsum(rowptr)
    col = np.array([e[1] for e in edges], np.int32)
    w = np.array([e[2] for e in edges], np.float64)
    d = np.array([e[3] for e in edges], np.float64)
    return rowptr, col, w, d


def _pulse_mask(n, t_steps, who, start, width):
    act = np.zeros((t_steps, n), bool)
    act[start:start + width, who] = True
    return wl.pack_mask(act)[None]


def test_analytic_delay_gradient():
    dt, T = 1e-3, 200
    lif = wl.LIFConfig(dt=dt)
    w01, d01 = 0.01, 37.25 * dt                       # off-grid delay: t_post between samples
    rowptr, col, w, d = _csr(2, [(0, 1, w01, d01)])
    eng = Engine(2, 1, T, precision=64, lif=lif)
    eng.set_network(rowptr, col, w, d)
    eng.set_drive(_pulse_mask(2, T, 0, 5, 3), np.array([500.0, 0.0]))
    eng.forward()
    sp = eng.spikes()
    assert len(sp["t"]) >= 1 and set(sp["neuron"].tolist()) == {0}
    gw, gd, _ = eng.backward(torch.zeros(1, 2, dtype=torch.float64),
                             i_bar=torch.tensor([[0.0, 1.0]], dtype=torch.float64))
    want = sum(w01 / lif.tau_syn * math.exp(-(T * dt - (t + d01)) / lif.tau_syn) for t in sp["t"])
    got = float(gd[0])
    assert got > 0                                     # jump-rule sign
    assert abs(got - want) / abs(want) < 1e-9, (got, want)


@pytest.mark.parametrize("dt", [2e-3, 1e-3, 5e-4])
def test_lif_spike_time_is_exact_at_any_dt(dt):
    T = int(1.0 / dt)
    rowptr, col, w, d = _csr(2, [(0, 1, 1e-6, dt)])
    eng = Engine(2, 1, T, precision=64, lif=wl.LIFConfig(dt=dt))
    eng.set_network(rowptr, col, w, d)
    act = np.zeros((T, 2), bool)
    act[:, 0] = True                                   # constant drive 2.0 from t = 0
    eng.set_drive(wl.pack_mask(act)[None], np.array([2.0, 0.0]))
    eng.forward()
    sp = eng.spikes()
    assert abs(sp["t"][0] - math.log(2.0)) < 1e-10     # lif_firing_period(1, 1, 2) = ln 2


def test_single_forced_spike_fans_out_at_delay():
    dt, T = 1e-3, 60
    rowptr, col, w, d = _csr(3, [(s, t, 0.05, 16 * dt) for s in range(3) for t in range(3) if s != t])
    eng = Engine(3, 1, T, precision=64)
    eng.set_network(rowptr, col, w, d)
    eng.set_drive(_pulse_mask(3, T, 0, 5, 3), np.array([500.0, 0.0, 0.0]))
    eng.reset()
    seen = {1: None, 2: None}
    for step in range(T):
        eng.run(1)
        i = eng.state()["i"][0].cpu().numpy()
        for j in (1, 2):
            if seen[j] is None and i[j] != 0.0:
                seen[j] = step
    sp = eng.spikes()
    assert set(sp["neuron"].tolist()) == {0}
    crossing_step = int(sp["step"][0]) + 1             # the reference's ThresholdCrossing.step = loop step + 1
    for j in (1, 2):
        assert seen[j] is not None and seen[j] - crossing_step == 16


def test_gradient_locality_silent_edges_are_exactly_zero():
    dt, T = 1e-3, 400
    rng = np.random.default_rng(21)
    edges = [(s, t, float(rng.normal(0.02, 0.005)), float(rng.integers(1, 16)) * dt)
             for s in range(3) for t in range(3) if s != t]
    rowptr, col, w, d = _csr(3, edges)
    eng = Engine(3, 1, T, precision=64)
    eng.set_network(rowptr, col, w, d)
    eng.set_drive(_pulse_mask(3, T, 0, 5, 3), np.array([500.0, 0.0, 0.0]))
    out = eng.forward()
    sp = eng.spikes()
    assert len(sp["t"]) > 0 and set(sp["neuron"].tolist()) == {0}
    gw, gd, _ = eng.backward(2.0 * (out["v"] - 0.25))
    gw, gd = gw.cpu().numpy(), gd.cpu().numpy()
    silent = np.arange(rowptr[1], rowptr[3])            # rows of neurons 1 and 2
    assert np.all(gw[silent] == 0.0) and np.all(gd[silent] == 0.0)
    assert np.any(gw[:rowptr[1]] != 0.0)                 # the firing neuron's edges do carry gradient
