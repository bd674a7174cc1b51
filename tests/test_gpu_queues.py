"""The queue operator API on the GPU (paper_2512_05906_b200.queues) against the
reference queue classes (pkg/src/eventq/queues.py).

* Trace replays: tests/golden/q_*.npz were recorded from the unmodified
  reference classes (scripts/make_queue_goldens.py).  Replaying the same event
  stream through a QueueBatch must reproduce every accept flag, every pop
  (bitwise in fp64: merges happen in insertion order, as in Python) and every
  occupancy.
* Known-answer checks of the protocol (events.py:99-141): causality and
  capability errors, merge, drop, ordering, lossy aliasing, capability flags.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TRACES = ["q_ring", "q_lossyring", "q_fiforing", "q_sortedarray", "q_binaryheap", "q_donothing", "q_heap_big"]


def _batch(kind, Q, cap, maxd, precision=64):
    from paper_2512_05906_b200.queues import QueueBatch
    return QueueBatch(kind, Q, None if cap < 0 else cap, None if maxd < 0 else maxd, precision=precision)


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("name", TRACES)
def test_trace_replay_matches_reference(name, precision):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    Q, T = int(g["Q"]), int(g["T"])
    qb = _batch(str(g["kind"]), Q, int(g["capacity"]), int(g["max_delay"]), precision)
    step = g["ev_step"]
    accepted = []
    for m in range(T):
        w, dw, wtt, has = (t.cpu().numpy() for t in qb.pop())
        assert np.array_equal(has, g["pop_has"][m]), m
        if precision == 64:
            assert np.array_equal(w, g["pop_w"][m]) and np.array_equal(dw, g["pop_dw"][m])
            assert np.array_equal(wtt, g["pop_wtt"][m]), m
        else:
            np.testing.assert_allclose(w, g["pop_w"][m], rtol=1e-5, atol=1e-6)
            np.testing.assert_allclose(wtt, g["pop_wtt"][m], rtol=1e-5, atol=1e-5)
        sel = step == m
        if sel.any():
            acc = qb.enqueue(g["ev_q"][sel], g["ev_due"][sel], g["ev_w"][sel], g["ev_dw"][sel], g["ev_tt"][sel])
            accepted.append(acc.cpu().numpy())
        assert np.array_equal(qb.occupancy().cpu().numpy(), g["occ"][m]), m
    assert np.array_equal(np.concatenate(accepted).astype(np.uint8), g["ev_acc"])
    if "aliased" in g.files:
        a, mg = qb.lossy_counts()
        assert np.array_equal(a.cpu().numpy(), g["aliased"]) and np.array_equal(mg.cpu().numpy(), g["merged"])


def _ev(step, w=1.0, dw=0.0, tt=0.0):
    from paper_2512_05906_b200.events import DualScalar, SpikeEvent
    return SpikeEvent(step, DualScalar(w, dw), tt)


def _mk(kind, cap=None, maxd=None):
    from paper_2512_05906_b200.queues import make_queue
    return make_queue(kind, cap, maxd)


@pytest.mark.parametrize("kind,cap", [("ring", 6), ("lossyring", 6), ("fiforing", 6), ("sortedarray", 6),
                                      ("binaryheap", 6), ("donothing", None)])
def test_past_delivery_is_a_causality_error(kind, cap):
    from paper_2512_05906_b200.errors import CausalityError
    q = _mk(kind, cap, 6 if cap else None)
    for _ in range(3):
        q.pop_due()
    with pytest.raises(CausalityError):
        q.enqueue(_ev(1))


def test_ring_merge_and_capability_edge():
    from paper_2512_05906_b200.errors import CapabilityError
    q = _mk("ring", 5, 5)
    q.pop_due()
    assert q.enqueue(_ev(5, 2.0)) and q.enqueue(_ev(5, 0.5, 1.0, 3.0))   # offset capacity-1: fits
    assert q.occupancy() == 1
    with pytest.raises(CapabilityError, match="exceeds"):
        q.enqueue(_ev(6))
    seen = [q.pop_due() for _ in range(1, 6)]
    assert all(p.is_zero() for p in seen[:-1])
    assert seen[-1].weight.primal == 2.5 and seen[-1].weight.tangent == 1.0
    assert seen[-1].weighted_time_tangent == 1.5


def test_batch_error_applies_only_events_before_it():
    """A failing event aborts the rest of the batch in call order."""
    from paper_2512_05906_b200.errors import CapabilityError
    from paper_2512_05906_b200.queues import QueueBatch
    qb = QueueBatch("ring", 3, 4, 4)
    with pytest.raises(CapabilityError):
        qb.enqueue([0, 1, 2, 0], [1, 2, 9, 3], [1.0, 1.0, 1.0, 1.0])
    occ = qb.occupancy().cpu().tolist()
    assert occ == [1, 1, 0]   # events 0 and 1 applied; 2 failed; 3 never applied


def test_lossyring_aliases_and_counts():
    q = _mk("lossyring", 3)
    q.pop_due()
    q.enqueue(_ev(5))          # offset 4 >= capacity 3: wraps to step 2
    q.enqueue(_ev(2))
    assert q.aliased == 1 and q.merged == 1
    assert q.pop_due().is_zero()
    assert q.pop_due().weight.primal == 2.0


def test_fifo_drop_and_order_rules():
    from paper_2512_05906_b200.errors import CapabilityError
    q = _mk("fiforing", 2)
    assert q.enqueue(_ev(3, 1.0)) and q.enqueue(_ev(3, 4.0))
    assert q.enqueue(_ev(3, 9.0)) is False
    with pytest.raises(CapabilityError, match="homogeneous"):
        q.enqueue(_ev(2))
    out = [q.pop_due().weight.primal for _ in range(4)]
    assert out == [0.0, 0.0, 0.0, 5.0]


@pytest.mark.parametrize("kind", ["sortedarray", "binaryheap"])
def test_keyed_kinds_deliver_by_step_and_drop_when_full(kind):
    q = _mk(kind, 3)
    for k in (7, 2, 4):
        assert q.enqueue(_ev(k, float(k), 0.1 * k))
    assert q.enqueue(_ev(5)) is False
    assert q.occupancy() == 3
    got = {}
    for s in range(9):
        p = q.pop_due()
        if not p.is_zero():
            got[s] = p.weight.primal
    assert got == {2: 2.0, 4: 4.0, 7: 7.0}


@pytest.mark.parametrize("kind", ["sortedarray", "binaryheap", "fiforing"])
def test_equal_steps_merge_in_insertion_order(kind):
    q = _mk(kind, 4)
    vals = [0.1, 0.2, 0.3]
    for v in vals:
        q.enqueue(_ev(2, v, v))
    q.pop_due(), q.pop_due()
    p = q.pop_due()
    assert p.weight.primal == (0.1 + 0.2) + 0.3     # left-to-right float sum
    assert p.weight.tangent == (0.1 + 0.2) + 0.3


def test_make_queue_argument_rules():
    from paper_2512_05906_b200.errors import ConfigurationError
    with pytest.raises(ConfigurationError, match="lossyring"):
        _mk("ring", 3, 9)
    with pytest.raises(ConfigurationError, match="needs a capacity"):
        _mk("binaryheap")
    with pytest.raises(ConfigurationError, match="bgpq"):
        _mk("bgpq", 1, 1)
    with pytest.raises(ConfigurationError, match="unknown"):
        _mk("splaytree", 2, 2)
    with pytest.raises(ConfigurationError, match="out of scope"):
        _mk("bitarray32", None, 8)


def test_capability_flags_match_the_reference_matrix():
    from paper_2512_05906_b200.queues import kind_capabilities
    expect = {"ring": (True, True, True, False), "lossyring": (True, True, True, True),
              "fiforing": (True, False, True, True), "sortedarray": (True, True, True, True),
              "binaryheap": (True, True, True, True), "donothing": (True, True, True, True)}
    for kind, flags in expect.items():
        c = kind_capabilities(kind)
        assert (c.supports_gradients, c.supports_heterogeneous_delay, c.supports_multi_spike_per_step,
                c.lossy) == flags
        q = _mk(kind, 16 if kind != "donothing" else None, 16 if kind == "ring" else None)
        assert q.capabilities[:4] == flags


@pytest.mark.parametrize("kind", ["ring", "fiforing", "sortedarray", "binaryheap"])
def test_integer_weights_are_conserved_exactly(kind):
    from paper_2512_05906_b200.queues import QueueBatch
    from paper_2512_05906_b200 import workload as wl
    Q, T = 8, 250
    qb = QueueBatch(kind, Q, 64, 64 if kind == "ring" else None)
    tot_in = np.zeros(3)
    tot_out = np.zeros(3)
    for m in range(T + 40):
        w, dw, wtt, _ = (t.cpu().numpy() for t in qb.pop())
        tot_out += [w.sum(), dw.sum(), wtt.sum()]
        if m >= T:
            continue
        u = wl.uniform(77, m, 5 * Q).reshape(5, Q)
        qs = np.arange(Q)[u[0] < 0.5]
        if not len(qs):
            continue
        d = np.full(len(qs), 6) if kind == "fiforing" else 1 + (u[1][qs] * 30).astype(int)
        W = np.floor(u[2][qs] * 8) - 3
        DW = np.floor(u[3][qs] * 5) - 2
        TT = np.floor(u[4][qs] * 5) - 2
        assert bool(qb.enqueue(qs, m + d, W, DW, TT).all())
        tot_in += [W.sum(), DW.sum(), (W * TT).sum()]
    assert np.array_equal(tot_in, tot_out)
