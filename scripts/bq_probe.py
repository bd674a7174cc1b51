"""One bounded-kind forward at C4 scale (for ncu captures of the bounded kernels).
    python scripts/bq_probe.py [--kind binaryheap] [--capacity 16] [--trials 4] [--steps 300]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="binaryheap")
    ap.add_argument("--capacity", type=int, default=16)
    ap.add_argument("--trials", type=int, default=4)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--delays", default="1,256")
    args = ap.parse_args()
    import torch
    from paper_2512_05906_b200 import workload as wl
    from paper_2512_05906_b200.engine import Engine, poisson_drive_device
    lo, hi = (int(x) for x in args.delays.split(","))
    net = wl.random_network(args.n, 100, 0, delay_steps=(lo, hi))
    mask = poisson_drive_device(args.n, args.trials, args.steps, 1e-3, 16e-3, 12e-3, 1000)
    eng = Engine(args.n, args.trials, args.steps, kind=args.kind, capacity=args.capacity)
    eng.set_network(net.rowptr, net.col, net.weight, net.delay)
    eng.set_drive(mask, np.full(args.n, 12.0))
    eng.forward()
    torch.cuda.synchronize()
    print("counters", eng.counters().sum(0))


if __name__ == "__main__":
    main()
