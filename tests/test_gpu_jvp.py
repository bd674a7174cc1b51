"""Batched forward mode on the GPU (eq_forward_jvp) against
(1) the unmodified reference's forward-mode JVPs stored in tests/golden and
(2) the reverse pass (grad . direction), on sparse multi-trial networks."""

import os

import numpy as np
import pytest
import torch

from golden_cases import BY_NAME
from paper_2512_05906_b200 import workload as wl

pytestmark = pytest.mark.gpu

DT = 1e-3
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name", ["dense_ring_n8", "dense_ring_refr3_n10", "dense_ring_plain_n10",
                                  "sparse_ring_plain_n100"])
def test_batched_jvp_equals_reference_forward_mode(name):
    from test_network_api import params_for
    from paper_2512_05906_b200.network import SeedDirection, forward_gradients
    case = BY_NAME[name]
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    p, drive = params_for(case)
    dirs = [SeedDirection(["weight", "delay", "drive"][k], i, j) for k, i, j in g["directions"].tolist()]
    got = forward_gradients(p, dirs, case.t_steps, drive)
    np.testing.assert_allclose(got, g["jvp"], rtol=1e-7, atol=1e-10)


@pytest.mark.parametrize("refractory,exact", [(0, True), (2, True), (0, False)])
def test_batched_jvp_equals_reverse_pass(refractory, exact):
    from paper_2512_05906_b200.engine import Engine
    net = wl.random_network(300, 25, 8, delay_steps=(1, 14), w_mean=0.04, w_std=0.01)
    B, T = 3, 400
    mask = wl.drive_masks(300, B, T, DT, seed0=55)
    amp = np.full(300, 12.0)
    eng = Engine(300, B, T, precision=64, lif=wl.LIFConfig(refractory_steps=refractory, exact_delivery=exact))
    eng.set_network(net.rowptr, net.col, net.weight, net.delay)
    eng.set_drive(mask, amp)
    out = eng.forward()
    assert eng.counters()[:, 0].sum() > 100
    vbar = 2.0 * (out["v"] - 0.25)
    gw, gd, ga = (x.cpu().numpy() for x in eng.backward(vbar))
    rng = np.random.default_rng(0)
    xs = rng.choice(net.n_edges, 6, replace=False)
    kinds = ["weight"] * 3 + ["delay"] * 3 + ["drive"] * 2
    idx = list(xs) + [5, 77]
    v, vt = eng.forward_jvp(kinds, idx)
    assert torch.equal(v, out["v"])                       # same primal trajectory
    jvp = (vt * vbar[None]).sum(dim=(1, 2)).cpu().numpy()
    ref = np.concatenate([gw[xs[:3]], gd[xs[3:]], ga[[5, 77]]])
    np.testing.assert_allclose(jvp, ref, rtol=1e-8, atol=1e-12 * np.abs(ref).max())


def test_jvp_argument_rules():
    from paper_2512_05906_b200.engine import Engine
    from paper_2512_05906_b200.errors import ConfigurationError
    net = wl.random_network(50, 5, 1, delay_steps=(1, 4))
    eng = Engine(50, 1, 20, precision=32)
    eng.set_network(net.rowptr, net.col, net.weight, net.delay)
    eng.set_drive(wl.drive_masks(50, 1, 20, DT), np.full(50, 12.0))
    with pytest.raises(ConfigurationError, match="precision 64"):
        eng.forward_jvp(["weight"], [0])
    eng64 = Engine(50, 1, 20, precision=64)
    eng64.set_network(net.rowptr, net.col, net.weight, net.delay)
    eng64.set_drive(wl.drive_masks(50, 1, 20, DT), np.full(50, 12.0))
    with pytest.raises(ConfigurationError, match="direction 0"):
        eng64.forward_jvp(["weight"], [net.n_edges])
