"""Phase timeline of the persistent kernels (needs EQ_TIMELINE=1).

    EQ_TIMELINE=1 python scripts/timeline.py [--trials 16] [--steps 200]
Prints per-phase medians/maxima over steps: neuron phase, fan-out+log phase,
barrier wait, whole step (max over CTAs)."""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("EQ_TIMELINE", "1")

from paper_2512_05906_b200.engine import Engine  # noqa: E402
import bench  # noqa: E402


ORDER = {"forward": [(5, "deliver done"), (1, "fan-out done / owner done"), (7, "adm records / log reserved"),
                     (4, "update done"),
                     (6, "clear+log done"),
                     (2, "both sides done"), (3, "barrier done")],
         "reverse": [(4, "stage done"), (5, "events done"), (1, "R-fanout done"), (6, "R-neuron done"),
                     (2, "both sides done"), (3, "barrier done")]}


def report(tl, label):
    """Per step: each mark's offset from the step start (median over steps of
    the max and the mean over CTAs)."""
    t = tl.astype(np.int64)
    ok = (t[:, :, 0] > 0) & (t[:, :, 3] > 0)
    steps = np.nonzero(ok.all(axis=1))[0]
    t = t[steps]
    step = np.abs(np.diff(t[:, :, 3].max(axis=1)))
    skew = t[:, :, 0].max(axis=1) - t[:, :, 0].min(axis=1)
    print(f"[{label}] steps={len(steps)}  step {np.median(step)/1e3:.2f} us  start-skew {np.median(skew)/1e3:.2f} us")
    t0 = t[:, :, 0]
    for k, name in ORDER[label]:
        mk = t[:, :, k]
        good = mk > 0
        if good.mean() < 0.5:
            continue
        d = np.where(good, mk - t0, 0)
        print(f"   {name:16s} max {np.median(d.max(1))/1e3:8.2f}  mean {np.median(d.sum(1) / np.maximum(good.sum(1), 1))/1e3:8.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=16)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--kind", default="ring")
    ap.add_argument("--capacity", type=int, default=0)
    ap.add_argument("--precision", type=int, default=32)
    args = ap.parse_args()
    net, mask, amp, T = bench.make_inputs(args.config, args.trials, 0)
    T = args.steps
    mask = np.ascontiguousarray(mask[:, :T])
    eng = Engine(net.n, args.trials, T, precision=args.precision, kind=args.kind, capacity=args.capacity)
    eng.set_network(net.rowptr, net.col, net.weight, net.delay)
    eng.set_drive(mask, amp)
    for _ in range(2):
        out = eng.forward()
        eng.backward(2 * (out["v"] - 0.25), want_amp=False)
    torch.cuda.synchronize()
    G, _ = eng.geometry
    for which, label in ((0, "forward"), (1, "reverse")):
        buf = np.zeros((T, G, 8), dtype=np.uint64)
        eng.L.eq_debug_timeline(eng.h, which, buf.ctypes.data_as(ctypes.c_void_p))
        report(buf, label)
    c = eng.counters()
    print("spikes", c[:, 0].sum(), "events", c[:, 1].sum())


if __name__ == "__main__":
    main()
