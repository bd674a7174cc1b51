"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

* device-mode oracle, same precision: BITWISE — raster, final V and I, pending
  ring contents (fixed-point ints), counters; reverse pass: lambda-derived
  gradients bitwise at one trial (same accumulation order), rtol 1e-12 across
  trials (double atomics reorder the trial sum), grad_amp bitwise;
* reference fixtures (Python reference outputs) in fp64: raster identical,
  voltages within 1e-9 (SURVEY §8(c) precision contract);
* fp32: the north-star tolerance rtol 1e-5 applies to floats vs an fp32
  restatement — here the restatement is bitwise, which is stronger.
"""

import os

import numpy as np
import pytest

from golden_cases import BY_NAME, CASES, edge_index
from oracle.oracle import OracleSession
from paper_2512_05906_b200 import workload as wl

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _engine(net, mask, amp, B, T, precision, kind="ring", refractory=0, capacity=0, exact=True, staged=0):
    from paper_2512_05906_b200.engine import Engine
    lif = wl.LIFConfig(refractory_steps=refractory, exact_delivery=exact)
    eng = Engine(net.n, B, T, kind=kind, precision=precision, lif=lif, capacity=capacity or 0, staged_queues=staged)
    eng.set_network(net.rowptr, net.col, net.weight, net.delay)
    eng.set_drive(mask, amp)
    return eng


def _oracle(net, mask, amp, B, T, precision, F, kind="ring", refractory=0, mode="device", capacity=0, exact=True):
    s = OracleSession(n=net.n, n_trials=B, t_steps=T, kind=kind, mode=mode, precision=precision,
                      frac_bits=F, refractory_steps=refractory, capacity=capacity or 0, exact_delivery=exact)
    s.set_network(net.rowptr, net.col, net.weight, net.delay)
    s.set_drive(mask, amp)
    return s


def _sorted_spikes(d):
    order = np.lexsort((d["neuron"], d["step"], d["trial"]))
    return np.stack([d["trial"][order], d["step"][order], d["neuron"][order]], 1), d["t"][order]


def _compare_forward(net, mask, amp, B, T, precision, refractory=0, backward=True, kind="ring", capacity=0,
                     exact=True):
    eng = _engine(net, mask, amp, B, T, precision, kind=kind, refractory=refractory, capacity=capacity, exact=exact)
    out = eng.forward()
    F = eng.frac_bits
    s = _oracle(net, mask, amp, B, T, precision, F, kind=kind, refractory=refractory, capacity=capacity, exact=exact)
    ref = s.forward()
    assert s.horizon == eng.horizon
    got = eng.spikes()
    r_g, t_g = _sorted_spikes(got)
    r_o, t_o = _sorted_spikes(ref)
    assert r_g.shape == r_o.shape and np.array_equal(r_g, r_o), "raster differs"
    assert np.array_equal(t_g.astype(np.float64), t_o)
    assert np.array_equal(out["v"].double().cpu().numpy(), ref["v"])
    assert np.array_equal(out["i"].double().cpu().numpy(), ref["i"])
    assert np.array_equal(eng.counters(), ref["counters"])
    assert np.array_equal(eng.pending(), ref["pending"])
    if backward:
        vbar = 2.0 * (out["v"].double() - 0.25)
        vbar_t = vbar.to(out["v"].dtype)
        gw, gd, ga = eng.backward(vbar_t)
        ow, od, oa = s.backward(vbar_t.double().cpu().numpy())
        gw, gd, ga = (x.cpu().numpy() for x in (gw, gd, ga))
        if B == 1:
            assert np.array_equal(gw, ow) and np.array_equal(gd, od)
        else:
            # double atomics reorder the sum over trials: 1e-12 of the gradient's scale
            np.testing.assert_allclose(gw, ow, rtol=1e-12, atol=1e-12 * np.abs(ow).max())
            np.testing.assert_allclose(gd, od, rtol=1e-12, atol=1e-12 * np.abs(od).max())
        assert np.array_equal(ga, oa)
    return eng, out


RING_LIKE = ["dense_ring_n8", "dense_ring_n40", "dense_ring_refr3_n10", "sparse_ring_n100",
             # lossy ring networks and plain (non-exact) delivery, forward and reverse
             "dense_lossy_cap6_n10", "dense_lossy_n8", "dense_ring_plain_n10", "dense_lossy_cap5_plain_n10",
             "sparse_ring_plain_n100"]


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("name", RING_LIKE)
def test_golden_inputs_bitwise_vs_oracle(name, precision):
    case = BY_NAME[name]
    net, mask, amp = case.inputs()
    _compare_forward(net, mask, amp, 1, case.t_steps, precision, refractory=case.refractory, kind=case.kind,
                     capacity=case.capacity, exact=case.exact)


@pytest.mark.parametrize("kind,cap", [("lossyring", 9), ("lossyring", 0)])
@pytest.mark.parametrize("exact", [True, False])
def test_lossy_multi_trial_bitwise_vs_oracle(kind, cap, exact):
    """Sparse net, 3 trials, delays 1..20 (horizon 21): capacity 9 aliases
    (events pop up to 12 steps early, some one step after their emission);
    capacity 0 = the reference default, lossless (== ring)."""
    net = wl.random_network(300, 30, 19, delay_steps=(1, 20), w_mean=0.02, w_std=0.01)
    B, T = 3, 400
    mask = wl.drive_masks(300, B, T, 1e-3, seed0=78)
    _compare_forward(net, mask, np.full(300, 12.0), B, T, 32, kind=kind, capacity=cap, exact=exact)


@pytest.mark.parametrize("precision", [32, 64])
def test_multi_trial_bitwise_vs_oracle(precision):
    net = wl.random_network(300, 30, 11, delay_steps=(1, 20), w_mean=0.02, w_std=0.01)
    B, T = 3, 400
    mask = wl.drive_masks(300, B, T, 1e-3, seed0=77)
    _compare_forward(net, mask, np.full(300, 12.0), B, T, precision)


@pytest.mark.parametrize("precision", [32, 64])
def test_c1_full_size_bitwise_vs_oracle(precision):
    wk = wl.make_workload("C1", n_trials=2)
    _compare_forward(wk.net, wk.mask, wk.amp, wk.n_trials, wk.t_steps, precision)


@pytest.mark.parametrize("name", RING_LIKE + ["c1_ring"])
def test_fp64_gpu_vs_reference_fixture(name):
    """Python reference outputs (fixtures) vs the GPU in fp64."""
    case = BY_NAME[name]
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        pytest.skip("fixture missing")
    g = np.load(path)
    net, mask, amp = case.inputs()
    eng = _engine(net, mask, amp, 1, case.t_steps, 64, kind=case.kind, refractory=case.refractory,
                  capacity=case.capacity, exact=case.exact)
    out = eng.forward()
    sp = eng.spikes()
    raster = np.stack([sp["step"], sp["neuron"]], 1)
    order = np.lexsort((raster[:, 1], raster[:, 0]))
    assert np.array_equal(raster[order], g["raster"])
    np.testing.assert_allclose(out["v"][0].cpu().numpy(), g["v_final_primal"], rtol=1e-9, atol=1e-12)
    # reverse mode vs the reference's forward-mode JVP along the stored directions
    if len(g["jvp"]):
        vbar = 2.0 * (out["v"] - 0.25)
        gw, gd, ga = (x.cpu().numpy() for x in eng.backward(vbar))
        for (p, i, j), jvp in zip(g["directions"].tolist(), g["jvp"].tolist()):
            got = ga[i] if p == 2 else (gw if p == 0 else gd)[edge_index(net, i, j)]
            assert got == pytest.approx(jvp, rel=1e-7, abs=1e-10), (p, i, j)


def test_trace_matches_oracle():
    case = BY_NAME["dense_ring_n8"]
    net, mask, amp = case.inputs()
    eng = _engine(net, mask, amp, 1, case.t_steps, 64)
    out = eng.forward(record_v=True)
    s = OracleSession(n=net.n, n_trials=1, t_steps=case.t_steps, mode="device", precision=64,
                      frac_bits=eng.frac_bits, record_v=True)
    s.set_network(net.rowptr, net.col, net.weight, net.delay)
    s.set_drive(mask, amp)
    ref = s.forward()
    assert np.array_equal(out["v_trace"][:, 0].cpu().numpy(), ref["v_trace"][0])


def test_stepwise_run_equals_forward():
    """eq_run in pieces (network_step granularity) == one eq_forward."""
    import torch
    case = BY_NAME["sparse_ring_n100"]
    net, mask, amp = case.inputs()
    eng = _engine(net, mask, amp, 1, case.t_steps, 32)
    full = eng.forward()["v"].clone()
    eng.reset()
    for chunk in (1, 7, 92, 400, 500):
        eng.run(chunk)
    torch.cuda.synchronize()
    v = torch.empty_like(full)
    # the handle's V is exposed through a zero-step forward copy: re-run to compare raster instead
    sp_pieces = eng.spikes()
    eng.forward()
    sp_full = eng.spikes()
    for k in ("trial", "step", "neuron", "t"):
        assert np.array_equal(sp_pieces[k], sp_full[k])
    del v


def test_donothing_counts_every_event_as_dropped():
    case = BY_NAME["dense_donothing_n8"]
    net, mask, amp = case.inputs()
    g = np.load(os.path.join(GOLDEN, case.name + ".npz"))
    eng = _engine(net, mask, amp, 1, case.t_steps, 64, kind="donothing")
    eng.forward()
    spikes, events, drops = eng.counters()[0].tolist()
    assert spikes == int(g["spike_count"]) and drops == int(g["drop_count"]) == events


def test_configuration_errors_name_the_edge():
    from paper_2512_05906_b200.errors import ConfigurationError
    net = wl.random_network(20, 5, 3, delay_steps=(1, 8))
    net.delay[7] = 0.5e-3
    src = np.repeat(np.arange(net.n), np.diff(net.rowptr))
    mask = wl.drive_masks(20, 1, 50, 1e-3)
    with pytest.raises(ConfigurationError, match=rf"edge \({src[7]},{net.col[7]}\).*below one step"):
        _engine(net, mask, np.full(20, 12.0), 1, 50, 32)


# ---------------------------------------------------------------- bounded kinds

BOUNDED = ["dense_heap_n8", "dense_sorted_n8", "dense_fifo_n8", "dense_heap_cap3_n12", "dense_sorted_cap3_n12",
           "dense_fifo_cap2_n12", "dense_sorted_plain_cap3_n12"]


def _compare_bounded(net, mask, amp, B, T, precision, kind, capacity, backward=True, exact=True, staged=0):
    eng = _engine(net, mask, amp, B, T, precision, kind=kind, capacity=capacity, exact=exact, staged=staged)
    out = eng.forward()
    s = OracleSession(n=net.n, n_trials=B, t_steps=T, kind=kind, mode="device", precision=precision,
                      frac_bits=eng.frac_bits, capacity=capacity or 0, exact_delivery=exact)
    s.set_network(net.rowptr, net.col, net.weight, net.delay)
    s.set_drive(mask, amp)
    ref = s.forward()
    r_g, t_g = _sorted_spikes(eng.spikes())
    r_o, t_o = _sorted_spikes(ref)
    assert np.array_equal(r_g, r_o), "raster differs"
    assert np.array_equal(t_g.astype(np.float64), t_o)
    assert np.array_equal(out["v"].double().cpu().numpy(), ref["v"])
    assert np.array_equal(out["i"].double().cpu().numpy(), ref["i"])
    assert np.array_equal(eng.counters(), ref["counters"])      # incl. drops
    assert np.array_equal(eng.pending(), ref["pending"])        # queue contents after the run
    return eng, out, ref


IMPLS = pytest.mark.parametrize("staged", [0, 1, 2], ids=["admission", "smem", "hbm"])


@IMPLS
@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("name", BOUNDED)
def test_bounded_kinds_bitwise_vs_oracle(name, precision, staged):
    """All three implementations of the bounded kinds: heap / sorted by
    admission on the calendar (default; the fixtures' FIFO delay is on the step grid), the
    shared-memory staged queues with the in-kernel arrival sort (capacity
    <= 64) and the HBM-resident structures."""
    case = BY_NAME[name]
    net, mask, amp = case.inputs()
    eng, out, _ = _compare_bounded(net, mask, amp, 1, case.t_steps, precision, case.kind, case.capacity,
                                   exact=case.exact, staged=staged)
    # reverse: bitwise at one trial, dropped events skipped exactly
    vbar = (2.0 * (out["v"].double() - 0.25)).to(out["v"].dtype)
    gw, gd, ga = (x.cpu().numpy() for x in eng.backward(vbar))
    s = _oracle(net, mask, amp, 1, case.t_steps, precision, eng.frac_bits, kind=case.kind, capacity=case.capacity,
                exact=case.exact)
    s.forward()
    ow, od, oa = s.backward(vbar.double().cpu().numpy())
    assert np.array_equal(gw, ow) and np.array_equal(gd, od) and np.array_equal(ga, oa)


@pytest.mark.parametrize("name", BOUNDED)
def test_bounded_fp64_vs_reference_fixture(name):
    case = BY_NAME[name]
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    net, mask, amp = case.inputs()
    eng = _engine(net, mask, amp, 1, case.t_steps, 64, kind=case.kind, capacity=case.capacity, exact=case.exact)
    out = eng.forward()
    sp = eng.spikes()
    raster = np.stack([sp["step"], sp["neuron"]], 1)
    raster = raster[np.lexsort((raster[:, 1], raster[:, 0]))]
    assert np.array_equal(raster, g["raster"])
    np.testing.assert_allclose(out["v"][0].cpu().numpy(), g["v_final_primal"], rtol=1e-9, atol=1e-12)
    spikes, events, drops = eng.counters()[0].tolist()
    assert spikes == int(g["spike_count"]) and drops == int(g["drop_count"])


@pytest.mark.parametrize("kind", ["binaryheap", "sortedarray"])
def test_bounded_multi_trial_with_drops_and_reverse(kind):
    """Sparse net, 3 trials, capacity small enough to drop: forward bitwise vs
    the oracle; the reverse pass must skip dropped events exactly (its
    gradients equal the oracle's pool-semantics reverse)."""
    net = wl.random_network(200, 20, 13, delay_steps=(1, 12), w_mean=0.05, w_std=0.02)
    B, T = 3, 400
    mask = wl.drive_masks(200, B, T, 1e-3, seed0=91)
    amp = np.full(200, 12.0)
    eng, out, ref = _compare_bounded(net, mask, amp, B, T, 32, kind, 4)
    assert eng.counters()[:, 2].sum() > 0, "capacity 4 should drop"
    vbar = (2.0 * (out["v"] - 0.25)).float()
    gw, gd, ga = (x.cpu().numpy() for x in eng.backward(vbar))
    s = OracleSession(n=200, n_trials=B, t_steps=T, kind=kind, mode="device", precision=32,
                      frac_bits=eng.frac_bits, capacity=4)
    s.set_network(net.rowptr, net.col, net.weight, net.delay)
    s.set_drive(mask, amp)
    s.forward()
    ow, od, oa = s.backward(vbar.double().cpu().numpy())
    np.testing.assert_allclose(gw, ow, rtol=1e-12, atol=1e-12 * np.abs(ow).max())
    np.testing.assert_allclose(gd, od, rtol=1e-12, atol=1e-12 * np.abs(od).max())
    assert np.array_equal(ga, oa)


@pytest.mark.parametrize("kind", ["binaryheap", "fiforing", "donothing"])
def test_bounded_single_trial_reverse_bitwise(kind):
    case = BY_NAME["dense_fifo_cap2_n12" if kind == "fiforing" else "dense_heap_cap3_n12"]
    net, mask, amp = case.inputs()
    cap = case.capacity if kind != "donothing" else 0
    from paper_2512_05906_b200.engine import Engine
    eng = Engine(net.n, 1, case.t_steps, kind=kind, precision=64, capacity=cap)
    eng.set_network(net.rowptr, net.col, net.weight, net.delay)
    eng.set_drive(mask, amp)
    out = eng.forward()
    vbar = 2.0 * (out["v"] - 0.25)
    gw, gd, ga = (x.cpu().numpy() for x in eng.backward(vbar))
    s = OracleSession(n=net.n, n_trials=1, t_steps=case.t_steps, kind=kind, mode="device", precision=64,
                      frac_bits=eng.frac_bits, capacity=cap)
    s.set_network(net.rowptr, net.col, net.weight, net.delay)
    s.set_drive(mask, amp)
    s.forward()
    ow, od, oa = s.backward(vbar.cpu().numpy())
    assert np.array_equal(gw, ow) and np.array_equal(gd, od) and np.array_equal(ga, oa)


def test_lossless_bounded_equals_ring_bitwise():
    """Without drops every kind delivers the same sums."""
    net = wl.random_network(150, 15, 17, delay_steps=(1, 10), w_mean=0.03, w_std=0.01)
    B, T = 2, 300
    mask = wl.drive_masks(150, B, T, 1e-3, seed0=5)
    amp = np.full(150, 12.0)
    outs = {}
    from paper_2512_05906_b200.engine import Engine
    for kind in ("ring", "binaryheap", "sortedarray"):
        eng = Engine(150, B, T, kind=kind, precision=32)
        eng.set_network(net.rowptr, net.col, net.weight, net.delay)
        eng.set_drive(mask, amp)
        o = eng.forward()
        outs[kind] = (o["v"].cpu().numpy(), eng.spikes()["t"], eng.pending())
    for kind in ("binaryheap", "sortedarray"):
        assert np.array_equal(outs[kind][0], outs["ring"][0])
        assert np.array_equal(outs[kind][1], outs["ring"][1])
        assert np.array_equal(outs[kind][2], outs["ring"][2])


@pytest.mark.parametrize("kind", ["binaryheap", "fiforing", "sortedarray"])
def test_bounded_stepwise_run_equals_forward(kind):
    """Bounded kinds in launch segments (each launch ends with the tail passes
    that insert its last steps' arrivals) == one launch: raster, queue contents
    and counters, with drops."""
    delays = (6, 6) if kind == "fiforing" else (1, 12)
    net = wl.random_network(160, 20, 21, delay_steps=delays, w_mean=0.05, w_std=0.02)
    B, T = 2, 300
    mask = wl.drive_masks(160, B, T, 1e-3, seed0=17)
    amp = np.full(160, 12.0)
    eng = _engine(net, mask, amp, B, T, 32, kind=kind, capacity=3)
    eng.forward()
    full = eng.spikes()
    pend = eng.pending()
    ctr = eng.counters()
    assert ctr[:, 2].sum() > 0
    eng.reset()
    for chunk in (1, 2, 37, 60, 200):
        eng.run(chunk)
    sp = eng.spikes()
    for k in ("trial", "step", "neuron", "t"):
        assert np.array_equal(sp[k], full[k])
    assert np.array_equal(eng.pending(), pend)
    assert np.array_equal(eng.counters(), ctr)


def test_c3_full_size_bitwise_vs_oracle():
    """BASELINE config 3 at full size — 100k neurons, K = 100, delays 1..64
    steps, T = 1000 — one trial in fp32: raster, spike times, final V and I,
    pending ring contents, counters and the reverse pass bitwise = oracle."""
    wk = wl.make_workload("C3", n_trials=1)
    eng, _ = _compare_forward(wk.net, wk.mask, wk.amp, 1, wk.t_steps, 32)
    assert eng.counters()[0, 1] > 10_000_000                     # a full-rate run (~4.4e7 events)


def test_c3_full_size_trials_are_independent():
    """Size-independent property at C3: two trials with the same drive give
    bitwise the same raster, state and per-trial counters as each other, while
    running concurrently with a differently driven third trial."""
    wk = wl.make_workload("C3", n_trials=2, t_steps=400)
    mask = np.stack([wk.mask[0], wk.mask[1], wk.mask[0]])
    eng = _engine(wk.net, mask, wk.amp, 3, 400, 32)
    out = eng.forward()
    v = out["v"].cpu().numpy()
    assert np.array_equal(v[0], v[2]) and not np.array_equal(v[0], v[1])
    sp = eng.spikes()
    r0 = np.stack([sp["step"][sp["trial"] == 0], sp["neuron"][sp["trial"] == 0]])
    r2 = np.stack([sp["step"][sp["trial"] == 2], sp["neuron"][sp["trial"] == 2]])
    assert r0.shape[1] > 1000 and np.array_equal(r0, r2)
    c = eng.counters()
    assert np.array_equal(c[0], c[2])


@IMPLS
@pytest.mark.parametrize("kind,cap", [("binaryheap", 8), ("sortedarray", 8), ("binaryheap", 64)])
def test_bounded_c2_size_bitwise_vs_oracle(kind, cap, staged):
    """BASELINE config 2 sizes (10k neurons, K = 100, delays 1..64, T = 1000),
    two trials, fp32: capacity 8 drops most events (the memory-pressure
    regime), capacity 64 almost none.  Raster, V, I, pending queue sums,
    counters bitwise = oracle; the reverse pass skips exactly the dropped
    events (gradients within 1e-12 of scale: fp64 atomics reorder the trial sum)."""
    wk = wl.make_workload("C2", n_trials=2)
    eng, out, ref = _compare_bounded(wk.net, wk.mask, wk.amp, 2, wk.t_steps, 32, kind, cap, staged=staged)
    c = eng.counters()
    if cap == 8:
        assert c[:, 2].sum() > 0.3 * c[:, 1].sum(), "capacity 8 should drop a large share of events"
    vbar = (2.0 * (out["v"] - 0.25)).float()
    gw, gd, ga = (x.cpu().numpy() for x in eng.backward(vbar))
    s = OracleSession(n=wk.net.n, n_trials=2, t_steps=wk.t_steps, kind=kind, mode="device", precision=32,
                      frac_bits=eng.frac_bits, capacity=cap)
    s.set_network(wk.net.rowptr, wk.net.col, wk.net.weight, wk.net.delay)
    s.set_drive(wk.mask, wk.amp)
    s.forward()
    ow, od, oa = s.backward(vbar.double().cpu().numpy())
    np.testing.assert_allclose(gw, ow, rtol=1e-12, atol=1e-12 * np.abs(ow).max())
    np.testing.assert_allclose(gd, od, rtol=1e-12, atol=1e-12 * np.abs(od).max())
    assert np.array_equal(ga, oa)
