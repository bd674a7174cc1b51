"""Pin the CPU oracle against the Python reference's own outputs.

tests/golden/*.npz were produced by scripts/make_goldens.py running the
unmodified reference (pkg/src/eventq) on inputs that tests/golden_cases.py
regenerates here; the stored SHA-256 proves the inputs are the same.

* reference mode (double, glibc exp/log, reference summation order) must be
  BITWISE equal to the reference: raster, final I/V, per-step voltage trace,
  loss, spike/drop counters (network.py:458-497, 547-611);
* its reverse-mode gradient must equal the reference's forward-mode JVP along
  every stored direction (network.py:668-683) to 1e-9 relative;
* device mode in double (shared exp/log, fixed-point slots) must give the same
  raster and voltages within 1e-9 — the precision contract of SURVEY §8(c).
"""

import os

import numpy as np
import pytest

from golden_cases import CASES, edge_index, ref_loss
from oracle.oracle import OracleSession, frac_bits
from paper_2512_05906_b200.workload import Network

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _digest(net, mask, amp):
    import hashlib
    h = hashlib.sha256()
    for a in (net.rowptr, net.col, net.weight, net.delay, mask, amp):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _load(case):
    path = os.path.join(GOLDEN, case.name + ".npz")
    if not os.path.exists(path):
        pytest.skip(f"missing fixture {path}")
    g = np.load(path)
    net, mask, amp = case.inputs()
    assert _digest(net, mask, amp) == str(g["digest"]), "regenerated inputs differ from the fixture's"
    return g, net, mask, amp


def _session(case, net, mask, amp, mode, precision=64, record_v=False, F=0):
    s = OracleSession(n=case.n, n_trials=1, t_steps=case.t_steps, kind=case.kind, mode=mode,
                      precision=precision, capacity=case.capacity or 0,
                      refractory_steps=case.refractory, record_v=record_v, frac_bits=F,
                      exact_delivery=case.exact)
    s.set_network(net.rowptr, net.col, net.weight, net.delay)
    s.set_drive(mask, amp)
    return s


def _raster(out):
    return sorted(zip(out["step"].tolist(), out["neuron"].tolist()))


def _max_in(net: Network):
    return float(np.bincount(net.col, weights=np.abs(net.weight), minlength=net.n).max())


def _params(cases):
    return [pytest.param(c, id=c.name, marks=[pytest.mark.slow] if c.slow else []) for c in cases]


@pytest.mark.parametrize("case", _params(CASES))
def test_reference_mode_is_bitwise_reference(case):
    g, net, mask, amp = _load(case)
    rec = "v_trace" in g.files
    out = _session(case, net, mask, amp, "reference", record_v=rec).forward()
    assert _raster(out) == [tuple(r) for r in g["raster"].tolist()]
    assert np.array_equal(out["v"][0], g["v_final_primal"])
    assert np.array_equal(out["i"][0], g["i_final_primal"])
    if rec:
        assert np.array_equal(out["v_trace"][0], g["v_trace"])
    assert ref_loss(out["v"][0]) == float(g["loss"])
    spikes, enq, drops = out["counters"][0].tolist()
    assert spikes == int(g["spike_count"])
    assert drops == int(g["drop_count"])
    if case.dense:
        assert enq == int(g["enqueued_count"])


@pytest.mark.parametrize("case", _params([c for c in CASES if sum(c.n_dirs)]))
def test_reverse_mode_matches_reference_jvp(case):
    g, net, mask, amp = _load(case)
    assert len(g["jvp"]) == sum(case.n_dirs)
    s = _session(case, net, mask, amp, "reference")
    out = s.forward()
    gw, gd, ga = s.backward(2.0 * (out["v"] - 0.25))
    for (p, i, j), jvp in zip(g["directions"].tolist(), g["jvp"].tolist()):
        got = ga[i] if p == 2 else (gw if p == 0 else gd)[edge_index(net, i, j)]
        assert got == pytest.approx(jvp, rel=1e-9, abs=1e-12), (p, i, j)


@pytest.mark.parametrize("case", _params(CASES))
def test_device_mode_f64_within_contract(case):
    g, net, mask, amp = _load(case)
    s = _session(case, net, mask, amp, "device", 64, F=frac_bits(_max_in(net), 64))
    out = s.forward()
    assert _raster(out) == [tuple(r) for r in g["raster"].tolist()]
    np.testing.assert_allclose(out["v"][0], g["v_final_primal"], rtol=1e-9, atol=1e-12)
    assert out["counters"][0][2] == int(g["drop_count"])
