"""The reference's Poisson queue benchmark (bench.py:183-291)
on the GPU queue batch: one launch runs every queue through its whole stream.

CPU: the stream generator restatement reproduces the reference's draws
(tests/golden/p_*.npz were made by scripts/make_poisson_goldens.py from the
unmodified reference).  GPU: per-queue delivered weight and accepted counts
equal the reference queues' exactly, for every kind."""

import os

import numpy as np
import pytest

from paper_2512_05906_b200 import workload as wl

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ["p_ring", "p_lossyring", "p_fiforing", "p_sortedarray", "p_binaryheap", "p_donothing"]


@pytest.mark.parametrize("name", NAMES)
def test_stream_generator_matches_reference_draws(name):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    bits = wl.poisson_streams(float(g["lam"]), int(g["T"]), int(g["Q"]), int(g["seed"]))
    assert np.array_equal(bits, g["bits"])
    assert int(np.unpackbits(bits.view(np.uint8)).sum()) == int(g["attempted"].sum())


@pytest.mark.gpu
@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("name", NAMES)
def test_poisson_run_matches_reference_queues(name, precision):
    from paper_2512_05906_b200.queues import QueueBatch
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    kind, cap, maxd = str(g["kind"]), int(g["capacity"]), int(g["max_delay"])
    delay, Q, T = int(g["delay"]), int(g["Q"]), int(g["T"])
    if kind == "ring" and maxd < 0:
        maxd = delay
    qb = QueueBatch(kind, Q, None if cap < 0 else cap, None if maxd < 0 else maxd, precision=precision)
    delivered, accepted = qb.run_poisson(g["bits"].view(np.int32), T, delay)
    assert np.array_equal(accepted.cpu().numpy(), g["accepted"])
    assert np.array_equal(delivered.cpu().numpy(), g["delivered"])
    assert qb.now == T + delay + 1
    assert int(qb.occupancy().sum()) == 0                    # drained


@pytest.mark.gpu
def test_poisson_ring_overflow_is_a_capability_error():
    from paper_2512_05906_b200.errors import CapabilityError
    from paper_2512_05906_b200.queues import QueueBatch
    bits = wl.poisson_streams(2.0, 64, 4, 1)
    qb = QueueBatch("ring", 4, 8, 8)
    with pytest.raises(CapabilityError, match="exceeds"):
        qb.run_poisson(bits.view(np.int32), 64, 10)


@pytest.mark.gpu
def test_drop_rates_equal_the_reference_records():
    import json
    from paper_2512_05906_b200.poisson import measure_drop_rate
    rows = json.load(open(os.path.join(GOLDEN, "p_droprate.json")))
    for kind, cap, lam, delay, steps, seed, rate, sin, sout in rows:
        r = measure_drop_rate(kind, lam, delay, steps, seed, capacity=cap)
        assert (r.drop_rate, r.spikes_in, r.spikes_out) == (rate, sin, sout), (kind, delay)


@pytest.mark.gpu
def test_sweeps_and_records():
    from paper_2512_05906_b200.poisson import PoissonWorkload, records_to_csv_text, sweep
    base = PoissonWorkload(20.0, 10, 64, 2000, 3)
    recs = sweep("capacity", [2, 4, 8], "binaryheap", base, reps=3, warmup=1)
    assert [r.capacity for r in recs] == [2, 4, 8]
    rates = [r.drop_rate for r in recs]
    assert rates[0] >= rates[1] >= rates[2]
    txt = records_to_csv_text(recs)
    assert txt.splitlines()[0].startswith("workload,kind,capacity,max_delay,batch,lambda")
    recs = sweep("pressure", [0.5, 1.0], "fiforing", base, capacity=2, reps=3, warmup=1)
    assert [r.delay_steps for r in recs] == [10, 20]


@pytest.mark.gpu
def test_reference_acceptance_criterion_4_drop_rates():
    """pkg/tests/test_acceptance.py:167-209 on the GPU queues, with the values the
    reference's own run printed (pkg/test_output.txt:20-24): DoNothing drops
    everything, a lossless Ring nothing, FIFORing[4] at queue pressure 0.5
    (lambda 400, delay 200 steps, 10^6 steps, seed 0) 1.99e-03 over 2511 spikes."""
    from paper_2512_05906_b200.poisson import measure_drop_rate
    assert measure_drop_rate("donothing", 400.0, 80, 200_000, 0).drop_rate == 1.0
    assert measure_drop_rate("ring", 400.0, 80, 200_000, 0, capacity=80).drop_rate == 0.0
    fifo = measure_drop_rate("fiforing", 400.0, 200, 1_000_000, 0, capacity=4)
    assert fifo.spikes_in == 2511
    assert f"{fifo.drop_rate:.2e}" == "1.99e-03"
