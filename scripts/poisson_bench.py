"""The reference's Poisson queue benchmark (bench.py:217-291
run_inference_bench) on B200: every queue of the batch steps through its whole
stream inside one kernel launch (eq_queues_run_poisson).

    python scripts/poisson_bench.py [--batch 10000] [--lambda 400] [--delay 80] [--steps 100000]

One JSON line per queue kind: median time per timestep for the whole batch
(the unit of the paper's Table 3, PAPER.md:528-542 — H100/JAX numbers quoted
there for context), ns per step per queue (the reference's record field), drop
rate, spikes in/out.  Fresh queues every rep, CUDA events around the launch.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2512_05906_b200 import workload as wl  # noqa: E402
from paper_2512_05906_b200.queues import QueueBatch  # noqa: E402

# kind, capacity (None = reference default): the paper's table rows
KINDS = [("donothing", None), ("ring", None), ("lossyring", 4), ("fiforing", 4), ("sortedarray", 4),
         ("binaryheap", 7)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=10_000)
    ap.add_argument("--lambda", dest="lam", type=float, default=400.0)
    ap.add_argument("--delay", type=int, default=80)
    ap.add_argument("--steps", type=int, default=100_000)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--precision", type=int, default=32)
    args = ap.parse_args()
    bits = torch.from_numpy(wl.poisson_streams(args.lam, args.steps, args.batch, args.seed).view(np.int32)).cuda()
    attempted = int(np.unpackbits(bits.cpu().numpy().view(np.uint8)).sum())
    for kind, cap in KINDS:
        times = []
        for rep in range(args.warmup + args.reps):
            qb = QueueBatch(kind, args.batch, cap, args.delay if kind == "ring" else None, precision=args.precision)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            delivered, accepted = qb.run_poisson(bits, args.steps, args.delay)
            b.record()
            torch.cuda.synchronize()
            if rep >= args.warmup:
                times.append(a.elapsed_time(b))
            acc = int(accepted.sum())
            out = int(round(float(delivered.sum())))
            aliased = int(qb.lossy_counts()[0].sum()) if kind == "lossyring" else 0
            qb.close()
        ms = statistics.median(times)
        print(json.dumps({
            "workload": "poisson", "kind": kind, "capacity": cap, "batch": args.batch, "lambda": args.lam,
            "delay": args.delay, "steps": args.steps, "reps": args.reps, "dtype": f"f{args.precision}",
            "us_per_step_batch": ms * 1e3 / args.steps,
            "ns_per_step_per_queue": ms * 1e6 / (args.steps * args.batch),
            "drop_rate": (attempted - acc + aliased) / attempted if attempted else 0.0,
            "spikes_in": attempted, "spikes_out": out, "launch_ms": ms,
        }), flush=True)


if __name__ == "__main__":
    main()
