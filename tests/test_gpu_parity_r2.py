"""GPU parity for the paths round 1 left untested ("Next round" #1).

Every test compares the sm_100a kernels (through the C ABI) with the CPU
oracle's device mode, bitwise unless stated:

* the calendar-bucket overflow -> DRAM ring spill path (forced with a tiny
  bucket capacity), forward, pending queue contents and reverse;
* the spike log growing mid-run (the persistent launch pauses at a step
  boundary, the log doubles, the run resumes) — ring and a bounded kind with
  drops (the drop bits grow with the log);
* GrazingCrossingError raised on the device (neuro.py:194-199);
* BASELINE config 2 with the FIFO kind at full size (homogeneous delay);
* the bench's own configuration: C3 x 24 trials, forward + reverse, and a
  second run of it (determinism);
* BASELINE config 4 at full size (1M neurons, delays 1..256) with the heap and
  sorted kinds at capacity 16 and 32 (most events dropped), forward + reverse.
"""

import numpy as np
import pytest

from oracle.oracle import OracleError, OracleSession
from paper_2512_05906_b200 import workload as wl

pytestmark = pytest.mark.gpu


def _engine(net, mask, amp, B, T, precision=32, kind="ring", capacity=0, max_spikes=0, exact=True, staged=0):
    from paper_2512_05906_b200.engine import Engine
    eng = Engine(net.n, B, T, kind=kind, precision=precision, capacity=capacity, max_spikes=max_spikes,
                 lif=wl.LIFConfig(exact_delivery=exact), staged_queues=staged)
    eng.set_network(net.rowptr, net.col, net.weight, net.delay)
    eng.set_drive(mask, amp)
    return eng


def _oracle(net, mask, amp, B, T, precision, F, kind="ring", capacity=0, exact=True):
    s = OracleSession(n=net.n, n_trials=B, t_steps=T, kind=kind, mode="device", precision=precision,
                      frac_bits=F, capacity=capacity, exact_delivery=exact)
    s.set_network(net.rowptr, net.col, net.weight, net.delay)
    s.set_drive(mask, amp)
    return s


def _raster(d):
    order = np.lexsort((d["neuron"], d["step"], d["trial"]))
    return np.stack([d["trial"][order], d["step"][order], d["neuron"][order]], 1), d["t"][order]


def _forward_state(eng, out):
    r, t = _raster(eng.spikes())
    return dict(raster=r, t=t.astype(np.float64), v=out["v"].double().cpu().numpy(),
                i=out["i"].double().cpu().numpy(), counters=eng.counters(), pending=eng.pending())


def _assert_forward_equal(eng, out, ref):
    got = _forward_state(eng, out)
    r_o, t_o = _raster(ref)
    assert got["raster"].shape == r_o.shape and np.array_equal(got["raster"], r_o), "raster differs"
    assert np.array_equal(got["t"], t_o)
    assert np.array_equal(got["v"], ref["v"])
    assert np.array_equal(got["i"], ref["i"])
    assert np.array_equal(got["counters"], ref["counters"])
    assert np.array_equal(got["pending"], ref["pending"])
    return got


def _assert_reverse(eng, s, out, B):
    vbar = (2.0 * (out["v"].double() - 0.25)).to(out["v"].dtype)
    gw, gd, ga = (x.cpu().numpy() for x in eng.backward(vbar))
    ow, od, oa = s.backward(vbar.double().cpu().numpy())
    if B == 1:
        assert np.array_equal(gw, ow) and np.array_equal(gd, od)
    else:
        # fp64 atomics reorder the sum over trials: 1e-12 of the gradient's scale
        np.testing.assert_allclose(gw, ow, rtol=1e-12, atol=1e-12 * np.abs(ow).max())
        np.testing.assert_allclose(gd, od, rtol=1e-12, atol=1e-12 * np.abs(od).max())
    assert np.array_equal(ga, oa)
    return gw, gd, ga


# ---------------------------------------------------------------- rare paths

@pytest.mark.parametrize("kind,cap", [("ring", 0), ("binaryheap", 6), ("sortedarray", 6)])
@pytest.mark.parametrize("precision", [32, 64])
def test_bucket_overflow_spills_to_dram_ring_bitwise(precision, kind, cap):
    """Calendar buckets of 2 events per CTA per step: nearly every event takes
    the spill path (red.add into the DRAM ring row, dirty flag, pop adds the
    row, row clear; the admission kinds also count the row's events and
    withdraw fix-up losers through it) — same raster, state, pending contents,
    drops and reverse."""
    net = wl.random_network(2000, 40, 23, delay_steps=(1, 24), w_mean=0.02, w_std=0.01)
    B, T = 2, 300
    mask = wl.drive_masks(2000, B, T, 1e-3, seed0=31)
    amp = np.full(2000, 12.0)
    eng = _engine(net, mask, amp, B, T, precision, kind=kind, capacity=cap)
    eng.debug_set_bucket_capacity(2)
    out = eng.forward()
    s = _oracle(net, mask, amp, B, T, precision, eng.frac_bits, kind=kind, capacity=cap)
    ref = s.forward()
    _assert_forward_equal(eng, out, ref)
    assert eng.counters()[:, 1].sum() > 50 * eng.geometry[0], "too few events to overflow 2-event buckets"
    _assert_reverse(eng, s, out, B)
    # and a second run on the same handle: the reset must clear the spilled rows
    out2 = eng.forward()
    _assert_forward_equal(eng, out2, ref)


@pytest.mark.parametrize("kind,cap,staged", [("ring", 0, 0), ("binaryheap", 4, 0), ("sortedarray", 4, 0),
                                              ("binaryheap", 4, 1), ("binaryheap", 4, 2)])
def test_spike_log_grows_mid_run_bitwise(kind, cap, staged):
    """max_spikes far below the run's spike count: the launch pauses at a step
    boundary whenever one more step could overflow, the log (and for bounded
    kinds the drop bits indexed by it) doubles, the run resumes — bitwise equal
    to the oracle, forward and reverse."""
    net = wl.random_network(500, 30, 29, delay_steps=(1, 12), w_mean=0.03, w_std=0.01)
    B, T = 2, 400
    mask = wl.drive_masks(500, B, T, 1e-3, seed0=41)
    amp = np.full(500, 12.0)
    eng = _engine(net, mask, amp, B, T, 32, kind=kind, capacity=cap, max_spikes=1500, staged=staged)
    out = eng.forward()
    cap0, grows = eng.log_capacity()
    assert grows >= 1 and cap0 >= eng.spike_count()
    s = _oracle(net, mask, amp, B, T, 32, eng.frac_bits, kind=kind, capacity=cap)
    ref = s.forward()
    _assert_forward_equal(eng, out, ref)
    if kind != "ring":
        assert eng.counters()[:, 2].sum() > 0
    _assert_reverse(eng, s, out, B)


def test_device_grazing_crossing_raises_like_the_reference():
    """A neuron driven to a = v_th + 5e-10 crosses threshold with slope
    (a - v_th)/tau_m below 1e-9: GrazingCrossingError (neuro.py:194-199) at the
    same step on the GPU and in the oracle."""
    from paper_2512_05906_b200.errors import GrazingCrossingError
    n, T = 2, 25_000
    net = wl.Network(n=2, rowptr=np.array([0, 1, 2], np.int64), col=np.array([1, 0], np.int32),
                     weight=np.zeros(2), delay=np.full(2, 1e-3))
    active = np.zeros((T, n), bool)
    active[:, 0] = True
    mask = wl.pack_mask(active)[None]
    amp = np.array([1.0 + 5e-10, 0.0])
    eng = _engine(net, mask, amp, 1, T, 64)
    with pytest.raises(GrazingCrossingError) as gpu_exc:
        eng.forward()
    s = _oracle(net, mask, amp, 1, T, 64, eng.frac_bits)
    with pytest.raises(OracleError) as cpu_exc:
        s.forward()
    assert cpu_exc.value.kind == "GrazingCrossingError"
    step = int(str(cpu_exc.value).rsplit("step ", 1)[1].split()[0])
    assert 20_000 < step < T
    assert f"grazing crossing at step {step} " in str(gpu_exc.value)


# ---------------------------------------------------------------- BASELINE configs at full size

def test_c2_fifo_full_size_bitwise():
    """C2 (10k neurons, K = 100, T = 1000) with the FIFO kind — homogeneous
    delay 32 steps (the reference's FIFO capability, network.py:236-240),
    capacity 16 (drops) — 2 trials, forward + reverse."""
    net = wl.random_network(10_000, 100, 0, delay_steps=(32, 32))
    B, T = 2, 1000
    mask = wl.drive_masks(10_000, B, T, 1e-3)
    amp = np.full(10_000, 12.0)
    eng = _engine(net, mask, amp, B, T, 32, kind="fiforing", capacity=16)
    out = eng.forward()
    s = _oracle(net, mask, amp, B, T, 32, eng.frac_bits, kind="fiforing", capacity=16)
    ref = s.forward()
    _assert_forward_equal(eng, out, ref)
    assert eng.counters()[:, 2].sum() > 0
    _assert_reverse(eng, s, out, B)


def test_c3_bench_configuration_24_trials_bitwise_and_deterministic():
    """The bench's workload: C3 (100k neurons, K = 100, delays 1..64, T = 1000),
    24 trials, fp32, forward + reverse vs the oracle; then the same run again on
    the same handle: raster, spike times, state, pending ring, counters and
    dL/d amplitude bitwise, per-edge gradients within 1e-12 (fp64 atomics
    reorder the 24-trial sum)."""
    import torch
    from paper_2512_05906_b200.engine import poisson_drive_device
    net = wl.random_network(100_000, 100, 0, delay_steps=(1, 64))
    B, T = 24, 1000
    mask = poisson_drive_device(100_000, B, T, 1e-3, 16e-3, 12e-3, 1234, device=0).cpu().numpy().view(np.uint32)
    amp = np.full(100_000, 12.0)
    eng = _engine(net, mask, amp, B, T, 32)
    out = eng.forward()
    s = _oracle(net, mask, amp, B, T, 32, eng.frac_bits)
    ref = s.forward()
    first = _assert_forward_equal(eng, out, ref)
    assert eng.counters()[:, 1].sum() > 5e8
    gw, gd, ga = _assert_reverse(eng, s, out, B)
    del s, ref
    out2 = eng.forward()
    second = _forward_state(eng, out2)
    for k in first:
        assert np.array_equal(first[k], second[k]), k
    vbar = (2.0 * (out2["v"].double() - 0.25)).float()
    gw2, gd2, ga2 = (x.cpu().numpy() for x in eng.backward(vbar))
    assert np.array_equal(ga, ga2)
    np.testing.assert_allclose(gw2, gw, rtol=1e-12, atol=1e-12 * np.abs(gw).max())
    np.testing.assert_allclose(gd2, gd, rtol=1e-12, atol=1e-12 * np.abs(gd).max())
    torch.cuda.synchronize()


_C4 = {}


def _c4_inputs():
    if not _C4:
        net = wl.random_network(1_000_000, 100, 0, delay_steps=(1, 256))
        _C4["net"] = net
    return _C4["net"]


@pytest.mark.parametrize("kind,cap,staged", [("binaryheap", 16, 0), ("binaryheap", 32, 0),
                                              ("sortedarray", 16, 0), ("sortedarray", 32, 0),
                                              ("binaryheap", 16, 1), ("sortedarray", 32, 2)])
def test_c4_full_size_bounded_with_drops_bitwise(kind, cap, staged):
    """C4 at full size — 1M neurons, K = 100, delays 1..256 — with the heap and
    sorted kinds at capacity 16 / 32 (the memory-pressure regime: most events
    are dropped), 2 trials, T = 300, fp32: forward bitwise incl. drops and the
    queues' pending contents, reverse skipping exactly the dropped events."""
    from paper_2512_05906_b200.engine import poisson_drive_device
    net = _c4_inputs()
    B, T = 2, 300
    mask = poisson_drive_device(net.n, B, T, 1e-3, 16e-3, 12e-3, 77, device=0).cpu().numpy().view(np.uint32)
    amp = np.full(net.n, 12.0)
    eng = _engine(net, mask, amp, B, T, 32, kind=kind, capacity=cap, staged=staged)
    out = eng.forward()
    s = _oracle(net, mask, amp, B, T, 32, eng.frac_bits, kind=kind, capacity=cap)
    ref = s.forward()
    _assert_forward_equal(eng, out, ref)
    c = eng.counters()
    assert c[:, 2].sum() > 0.2 * c[:, 1].sum(), "capacity 16/32 should drop a large share at C4"
    _assert_reverse(eng, s, out, B)


# ---------------------------------------------------------------- autograd shell

def test_rsnn_function_rejects_a_stale_backward():
    """Two forwards on one engine before the first backward: the first
    backward would read the second run's spike log — it must raise instead."""
    import torch
    from paper_2512_05906_b200.engine import Engine
    from paper_2512_05906_b200.errors import EventQError
    from paper_2512_05906_b200.network import RSNNFunction
    net = wl.random_network(200, 10, 3, delay_steps=(1, 8), w_mean=0.05, w_std=0.01)
    T = 100
    mask = torch.as_tensor(wl.drive_masks(200, 1, T, 1e-3).view(np.int32)).cuda()
    eng = Engine(200, 1, T, precision=32)
    w = torch.tensor(net.weight, dtype=torch.float32, device="cuda", requires_grad=True)
    d = torch.tensor(net.delay, dtype=torch.float32, device="cuda", requires_grad=True)
    a = torch.full((200,), 12.0, device="cuda", requires_grad=True)
    v1 = RSNNFunction.apply(w, d, a, eng, net.rowptr, net.col, mask)
    v2 = RSNNFunction.apply(w, d, a, eng, net.rowptr, net.col, mask)
    v2.sum().backward(retain_graph=True)          # the latest run: fine
    with pytest.raises(EventQError, match="ran another forward"):
        v1.sum().backward()


# ---------------------------------------------------------------- admission fix-ups

@pytest.mark.parametrize("slots", [0, 2])
@pytest.mark.parametrize("kind,cap", [("binaryheap", 3), ("sortedarray", 5)])
def test_admission_fixups_without_recorded_keys_bitwise(kind, cap, slots):
    """Heap / sorted by admission with the arrival keys recorded only while the
    queue's room is below `slots` (0: never): the reference-order fix-ups then
    take the in-edge (CSC) walk, one warp per queue, instead of ranking the
    recorded keys.  Small capacities on a K = 40 network give many contested
    steps; forward (raster, state, pending, drops) and reverse = oracle."""
    net = wl.random_network(3000, 40, 37, delay_steps=(1, 12), w_mean=0.03, w_std=0.01)
    B, T = 2, 300
    mask = wl.drive_masks(3000, B, T, 1e-3, seed0=71)
    amp = np.full(3000, 12.0)
    eng = _engine(net, mask, amp, B, T, 32, kind=kind, capacity=cap)
    eng.debug_set_admission_slots(slots)
    out = eng.forward()
    s = _oracle(net, mask, amp, B, T, 32, eng.frac_bits, kind=kind, capacity=cap)
    ref = s.forward()
    _assert_forward_equal(eng, out, ref)
    c = eng.counters()
    assert c[:, 2].sum() > 0.01 * c[:, 1].sum(), "capacity should drop a share of the events"
    _assert_reverse(eng, s, out, B)


@pytest.mark.parametrize("delay_steps,impl", [(7, 0), (7.5, 0), (7.5, 2)])
def test_fifo_homogeneous_delay_on_and_off_the_step_grid(delay_steps, impl):
    """FIFO with one homogeneous delay: on the step grid (7 dt) every event of
    a step has the same due step, so it runs by admission; off the grid
    (7.5 dt) dues of one step differ by the spike time and the reference's
    tail-key check (queues.py:220-224) can fire, so it runs the queue
    structures.  Either way the result equals the oracle: same raster, state,
    pending queues and drops, or a CapabilityError in both."""
    from paper_2512_05906_b200.errors import CapabilityError
    net = wl.random_network(400, 20, 43, delay_steps=(1, 1), w_mean=0.05, w_std=0.01)
    net.delay[:] = delay_steps * 1e-3
    B, T = 1, 300
    mask = wl.drive_masks(400, B, T, 1e-3, seed0=83)
    amp = np.full(400, 12.0)
    eng = _engine(net, mask, amp, B, T, 64, kind="fiforing", capacity=6, staged=impl)
    s = _oracle(net, mask, amp, B, T, 64, eng.frac_bits, kind="fiforing", capacity=6)
    from oracle.oracle import OracleError
    try:
        ref = s.forward()
    except OracleError as e:
        assert e.kind == "CapabilityError", str(e)
        assert delay_steps != int(delay_steps), "an on-grid delay cannot violate the FIFO order"
        with pytest.raises(CapabilityError, match="homogeneous"):
            eng.forward()
        return
    out = eng.forward()
    _assert_forward_equal(eng, out, ref)
    assert eng.counters()[:, 2].sum() > 0


def test_admission_csc_follows_the_topology_across_set_network():
    """The admission kinds keep their CSC across set_network calls while the
    topology is unchanged (training steps change weights and delays only) and
    rebuild it when the columns change — two networks with the same edge count,
    then the first network's weights rescaled: each run = oracle, drops included."""
    B, T, n = 2, 200, 800
    mask = wl.drive_masks(n, B, T, 1e-3, seed0=5)
    amp = np.full(n, 12.0)
    net_a = wl.random_network(n, 30, 51, delay_steps=(1, 10), w_mean=0.04, w_std=0.01)
    net_b = wl.random_network(n, 30, 52, delay_steps=(1, 10), w_mean=0.04, w_std=0.01)
    assert net_a.n_edges == net_b.n_edges and not np.array_equal(net_a.col, net_b.col)
    net_c = wl.Network(net_a.n, net_a.rowptr, net_a.col, net_a.weight * 1.1, net_a.delay)
    eng = _engine(net_a, mask, amp, B, T, 32, kind="binaryheap", capacity=3)
    for net in (net_a, net_b, net_c, net_a):
        eng.set_network(net.rowptr, net.col, net.weight, net.delay)
        out = eng.forward()
        s = _oracle(net, mask, amp, B, T, 32, eng.frac_bits, kind="binaryheap", capacity=3)
        _assert_forward_equal(eng, out, s.forward())
        assert eng.counters()[:, 2].sum() > 0


@pytest.mark.parametrize("kind,cap,refractory", [("binaryheap", 8, 0), ("sortedarray", 8, 3), ("fiforing", 6, 2)])
def test_admission_fp64_c2_size_with_refractory_bitwise(kind, cap, refractory):
    """The admission path in fp64 at C2 size (10k neurons, K = 100, two trials;
    FIFO with one on-grid delay), with refractory neurons: raster, state, pending
    queues and drops bitwise = the fp64 device-mode oracle, reverse pass within
    1e-12 of the gradient scale."""
    delays = (32, 32) if kind == "fiforing" else (1, 64)
    net = wl.random_network(10_000, 100, 0, delay_steps=delays)
    B, T = 2, 400
    mask = wl.drive_masks(10_000, B, T, 1e-3, seed0=1000)
    amp = np.full(10_000, 12.0)
    from paper_2512_05906_b200.engine import Engine
    eng = Engine(net.n, B, T, kind=kind, capacity=cap, precision=64,
                 lif=wl.LIFConfig(refractory_steps=refractory))
    eng.set_network(net.rowptr, net.col, net.weight, net.delay)
    eng.set_drive(mask, amp)
    out = eng.forward()
    s = OracleSession(n=net.n, n_trials=B, t_steps=T, kind=kind, mode="device", precision=64,
                      frac_bits=eng.frac_bits, capacity=cap, refractory_steps=refractory)
    s.set_network(net.rowptr, net.col, net.weight, net.delay)
    s.set_drive(mask, amp)
    _assert_forward_equal(eng, out, s.forward())
    assert eng.counters()[:, 2].sum() > 0
    _assert_reverse(eng, s, out, B)
