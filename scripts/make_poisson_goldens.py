"""Poisson queue-benchmark goldens from the UNMODIFIED reference
(pkg/src/eventq/bench.py: gen_poisson, _drive_queue).  Build container only
(imports eventq read-only).  Stores per config: the packed spike streams, and
per queue the delivered weight and accepted count of the reference queue."""

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from eventq import make_queue  # noqa: E402
from eventq.bench import PoissonWorkload, _drive_queue, gen_poisson  # noqa: E402

from paper_2512_05906_b200.workload import pack_mask  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")

# name: kind, capacity, max_delay, lambda, delay, Q, T, seed
CONFIGS = {
    "p_ring": ("ring", 8, 8, 3.0, 6, 64, 400, 11),
    "p_lossyring": ("lossyring", 4, None, 2.0, 6, 64, 400, 12),
    "p_fiforing": ("fiforing", 4, None, 1.5, 8, 64, 400, 13),
    "p_sortedarray": ("sortedarray", 4, None, 1.5, 8, 64, 400, 14),
    "p_binaryheap": ("binaryheap", 7, None, 1.2, 12, 64, 400, 15),
    "p_donothing": ("donothing", None, None, 2.0, 4, 16, 200, 16),
}


def gen(name):
    kind, cap, maxd, lam, delay, Q, T, seed = CONFIGS[name]
    wk = PoissonWorkload(lambda_steps=lam, delay_steps=delay, n_queues=Q, t_steps=T, rng_seed=seed)
    streams = gen_poisson(wk)
    act = np.zeros((Q, T), dtype=bool)
    for q, st in enumerate(streams):
        act[q, st] = True
    delivered = np.zeros(Q)
    accepted = np.zeros(Q, dtype=np.int64)
    attempted = np.zeros(Q, dtype=np.int64)
    for q in range(Q):
        qu = make_queue(kind, cap, maxd if maxd is not None else delay if kind == "ring" else None)
        d, a, n = _drive_queue(qu, streams[q].tolist(), T, delay)
        delivered[q], accepted[q], attempted[q] = d, a, n
    np.savez_compressed(os.path.join(OUT, name + ".npz"), kind=kind, capacity=-1 if cap is None else cap,
                        max_delay=-1 if maxd is None else maxd, lam=lam, delay=delay, Q=Q, T=T, seed=seed,
                        bits=pack_mask(act), delivered=delivered, accepted=accepted, attempted=attempted)
    print(name, "attempted", attempted.sum(), "accepted", accepted.sum(), "delivered", delivered.sum())


if __name__ == "__main__":
    for name in CONFIGS:
        gen(name)


# measure_drop_rate records (bench.py:408-452): kind, capacity, lambda, pressures, steps, seed
DROP = [("lossyring", 8, 20.0, (0.2, 0.5, 1.0), 20000, 5), ("fiforing", 2, 20.0, (0.2, 0.5, 1.0), 20000, 6),
        ("binaryheap", 3, 10.0, (0.5, 1.0, 2.0), 20000, 7), ("sortedarray", 3, 10.0, (0.5, 1.0, 2.0), 20000, 8)]


def gen_drop():
    from eventq.bench import measure_drop_rate
    rows = []
    for kind, cap, lam, prs, steps, seed in DROP:
        for pr in prs:
            delay = max(1, round(pr * lam))
            r = measure_drop_rate(kind, lam, delay, steps, seed, capacity=cap)
            rows.append((kind, cap, lam, delay, steps, seed, r.drop_rate, r.spikes_in, r.spikes_out))
    import json
    with open(os.path.join(OUT, "p_droprate.json"), "w") as f:
        json.dump(rows, f, indent=0)
    print("droprate rows", len(rows))


if __name__ == "__main__":
    gen_drop()
