"""Batched forward mode (eq_forward_jvp) throughput.

    python scripts/jvp_bench.py [--config C1] [--dirs 1,8,32,128] [--reps 3]

One run = the whole T-step primal trajectory plus D seeded tangent lanes
(weights, delays and drive amplitudes, in rotation) in fp64 on the ring kind.
Prints one JSON line per D: ms per run, directional derivatives per second
and synaptic events per second of the primal (device counters).  The
reference's forward mode costs one full simulation per direction
(forward_gradient, network.py:668-683; 38.7 s per direction at C1 on one CPU
core).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2512_05906_b200 import workload as wl  # noqa: E402
from paper_2512_05906_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--n", type=int, default=0, help="override the neuron count")
    ap.add_argument("--dirs", default="1,8,32,128")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    wk = wl.make_workload(a.config, n_trials=1, n=a.n or None)
    eng = Engine(wk.net.n, 1, wk.t_steps, precision=64)
    eng.set_network(wk.net.rowptr, wk.net.col, wk.net.weight, wk.net.delay)
    eng.set_drive(wk.mask, wk.amp)
    eng.forward()
    events = int(eng.counters()[0, 1])
    rng = np.random.default_rng(0)
    for D in (int(x) for x in a.dirs.split(",")):
        kinds = [("weight", "delay", "drive")[d % 3] for d in range(D)]
        idx = [int(rng.integers(wk.net.n)) if k == "drive" else int(rng.integers(wk.net.n_edges)) for k in kinds]
        eng.forward_jvp(kinds, idx)                       # warm-up
        torch.cuda.synchronize()
        times = []
        for _ in range(a.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            eng.forward_jvp(kinds, idx)
            e.record()
            torch.cuda.synchronize()
            times.append(s.elapsed_time(e))
        ms = float(np.median(times))
        print(json.dumps({"metric": "batched JVP", "config": a.config, "neurons": wk.net.n, "steps": wk.t_steps,
                          "directions": D, "ms_per_run": ms, "directions_per_s": D / (ms * 1e-3),
                          "primal_events_per_s": events / (ms * 1e-3), "dtype": "f64",
                          "rep_ms": [round(t, 2) for t in times]}))


if __name__ == "__main__":
    main()
