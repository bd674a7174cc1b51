"""Time the UNMODIFIED Python reference on BASELINE config 1 (BASELINE.md §4,
"Reference timing"): per trial `forward_gradient` (forward + one-direction
JVP, the reference's gradient path) and `PrimalRSNN.run` (forward only),
single-threaded, trials spread over the host cores with multiprocessing as
the reference's own acceptance test does (tests/test_acceptance.py:51-54).

Runs only in the build container: it imports `eventq` read-only from
/root/reference/pkg/src, which does not exist on the GPU box (so bench.py's
reference arm times the C++ port of it instead).  Same network and drive
statistics as bench.py's C1 (K = 100 random targets, delays 1..16 steps,
PoissonDrive(16 dt, 12, 12 dt), seed 1000 + trial), non-edges embedded
densely with zero weight (exact for the ring kind).

    python scripts/python_reference_timing.py [--trials 8] [--out profiles/r2_python_reference_c1.json]
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
REF = "/root/reference/pkg/src"
DT = 1e-3
T = 1000


def _params(net):
    from eventq import NetworkParams
    w, d = net.dense(DT)
    return NetworkParams(n=net.n, weights=w, delays=d, tau_m=1.0, tau_syn=0.5, v_th=1.0, v_reset=0.0, dt=DT,
                         queue_kind="ring", v_target=np.full(net.n, 0.25))


def one_trial(b):
    sys.path.insert(0, REF)
    from eventq import SeedDirection
    from eventq.network import PoissonDrive, PrimalRSNN, forward_gradient
    from paper_2512_05906_b200 import workload as wl
    net = wl.random_network(1000, 100, 0, delay_steps=(1, 16))
    t0 = time.perf_counter()
    params = _params(net)
    i = 0
    j = int(net.col[net.rowptr[0]])
    drive = PoissonDrive(net.n, 16 * DT, 12.0, 12 * DT, T * DT, 1000 + b)
    t1 = time.perf_counter()
    jvp, res = forward_gradient(params, SeedDirection("weight", i, j), T, drive)
    t2 = time.perf_counter()
    pr = PrimalRSNN(params)
    pr.run(T, drive.materialize(T, DT))
    t3 = time.perf_counter()
    return {"trial": b, "setup_s": t1 - t0, "fwd_jvp_s": t2 - t1, "primal_s": t3 - t2,
            "spikes": int(res.spike_count), "events": int(res.enqueued_count)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=8)
    ap.add_argument("--out", default=os.path.join(REPO, "profiles", "r2_python_reference_c1.json"))
    args = ap.parse_args()
    if not os.path.isdir(REF):
        sys.exit("the reference is not mounted here (build container only)")
    import bench
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(min(cores, args.trials)) as pool:
        rows = pool.map(one_trial, range(args.trials))
    wall = time.perf_counter() - t0
    ev = sum(r["events"] for r in rows)
    ns = args.trials * 1000 * T
    fj = [r["fwd_jvp_s"] for r in rows]
    pm = [r["primal_s"] for r in rows]
    out = {
        "what": "unmodified Python reference (pkg/src/eventq), BASELINE config 1: 1k neurons, K=100, "
                "delays 1..16 steps, ring, T=1000, exact delivery",
        "host": bench.host_label(), "cores_used": min(cores, args.trials), "trials": args.trials,
        "per_trial": rows,
        "fwd_jvp": {"median_s_per_trial": float(np.median(fj)),
                    "events_per_s_single_thread": float(np.median([r["events"] / r["fwd_jvp_s"] for r in rows])),
                    "neuron_steps_per_s_single_thread": float(1000 * T / np.median(fj))},
        "primal": {"median_s_per_trial": float(np.median(pm)),
                   "events_per_s_single_thread": float(np.median([r["events"] / r["primal_s"] for r in rows]))},
        "all_cores": {"wall_s": wall, "events_per_s_fwd_jvp_plus_primal": ev / wall,
                      "note": "each trial runs forward_gradient then PrimalRSNN.run; events counted once per trial"},
        "neuron_steps": ns,
    }
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("host", "fwd_jvp", "primal")}, indent=1))


if __name__ == "__main__":
    main()
