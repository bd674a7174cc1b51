"""Queue-level golden traces from the UNMODIFIED reference queue classes.

Runs only in the build container (imports eventq read-only).  Each trace is a
seeded sequence of steps on Q independent queues of one kind: pop every queue
(_pop_raw), then enqueue a batch of events in call order.  Stored: the event
stream, every accept flag, every pop result and occupancies, so the GPU
QueueBatch can be replayed and compared bit for bit (tests/test_gpu_queues.py).
"""

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from eventq import DualScalar, SpikeEvent, make_queue  # noqa: E402

from paper_2512_05906_b200 import workload as wl  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")

# name: kind, capacity, max_delay, Q, T, mean events/step, offset range, seed
TRACES = {
    "q_ring": ("ring", 8, 8, 5, 300, 3.0, (1, 8), 1),
    "q_lossyring": ("lossyring", 4, None, 5, 300, 3.0, (1, 9), 2),
    "q_fiforing": ("fiforing", 3, None, 5, 300, 2.0, (5, 5), 3),
    "q_sortedarray": ("sortedarray", 4, None, 5, 300, 3.0, (1, 9), 4),
    "q_binaryheap": ("binaryheap", 4, None, 5, 300, 3.0, (1, 9), 5),
    "q_donothing": ("donothing", None, None, 3, 100, 2.0, (1, 5), 6),
    "q_heap_big": ("binaryheap", 64, None, 7, 400, 6.0, (1, 40), 7),
}


def gen(name):
    kind, cap, maxd, Q, T, lam, (lo, hi), seed = TRACES[name]
    queues = [make_queue(kind, cap, maxd) for _ in range(Q)]
    ev_step, ev_q, ev_due, ev_w, ev_dw, ev_tt, ev_acc = [], [], [], [], [], [], []
    pop_w = np.zeros((T, Q)); pop_dw = np.zeros((T, Q)); pop_wtt = np.zeros((T, Q))
    pop_has = np.zeros((T, Q), dtype=np.uint8)
    occ = np.zeros((T, Q), dtype=np.int32)
    cnt = 0
    for m in range(T):
        for q in range(Q):
            raw = queues[q]._pop_raw()
            if raw is not None:
                pop_has[m, q] = 1
                pop_w[m, q], pop_dw[m, q], pop_wtt[m, q] = raw
        u = wl.uniform(seed, m, 64)
        n = int(min(63, -lam * np.log1p(-u[0]) * 1.0 + 0.5))
        for k in range(n):
            x = wl.uniform(seed, 100000 + cnt, 5)
            q = int(x[0] * Q)
            off = lo + int(x[1] * (hi - lo + 1))
            w = float(np.round(x[2] * 2 - 0.5, 6))
            dw = float(x[3] - 0.5)
            tt = float(x[4] * 3 - 1.0)
            due = m + off
            ok = queues[q].enqueue(SpikeEvent(due, DualScalar(w, dw), tt))
            ev_step.append(m); ev_q.append(q); ev_due.append(due)
            ev_w.append(w); ev_dw.append(dw); ev_tt.append(tt); ev_acc.append(int(ok))
            cnt += 1
        for q in range(Q):
            occ[m, q] = queues[q].occupancy()
    extra = {}
    if kind == "lossyring":
        extra["aliased"] = np.array([q.aliased for q in queues]); extra["merged"] = np.array([q.merged for q in queues])
    np.savez_compressed(os.path.join(OUT, name + ".npz"), kind=kind, capacity=-1 if cap is None else cap,
                        max_delay=-1 if maxd is None else maxd, Q=Q, T=T,
                        ev_step=np.array(ev_step, np.int32), ev_q=np.array(ev_q, np.int32),
                        ev_due=np.array(ev_due, np.int32), ev_w=np.array(ev_w), ev_dw=np.array(ev_dw),
                        ev_tt=np.array(ev_tt), ev_acc=np.array(ev_acc, np.uint8), pop_w=pop_w, pop_dw=pop_dw,
                        pop_wtt=pop_wtt, pop_has=pop_has, occ=occ, **extra)
    print(name, "events", cnt, "accepted", sum(ev_acc), "pops", int(pop_has.sum()))


if __name__ == "__main__":
    for name in TRACES:
        gen(name)
