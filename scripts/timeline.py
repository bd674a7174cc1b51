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


def report(tl, label):
    t = tl.astype(np.int64)
    sub = t[:, :, 4:]
    ok = (t[:, :, 0] > 0)
    steps = np.nonzero(ok.all(axis=1))[0]
    t = t[steps]
    ph1 = t[:, :, 1] - t[:, :, 0]
    ph2 = t[:, :, 2] - t[:, :, 1]
    bar = t[:, :, 3] - t[:, :, 2]
    step = t[:, :, 3].max(axis=1)[1:] - t[:, :, 3].max(axis=1)[:-1]
    skew = t[:, :, 0].max(axis=1) - t[:, :, 0].min(axis=1)
    print(f"[{label}] steps={len(steps)}  (us: median over steps of max over CTAs / of mean)")
    for name, a in (("phase1", ph1), ("phase2", ph2), ("barrier", bar)):
        print(f"   {name:8s} max {np.median(a.max(1))/1e3:8.2f}  mean {np.median(a.mean(1))/1e3:8.2f}")
    print(f"   step     {np.median(step)/1e3:8.2f}   start-skew {np.median(skew)/1e3:8.2f}")
    sub = sub[steps]
    prev = t[:, :, 1]
    for k in range(4):
        mk = sub[:, :, k]
        if (mk > 0).all():
            d = mk - prev
            print(f"   sub{k}     max {np.median(d.max(1))/1e3:8.2f}  mean {np.median(d.mean(1))/1e3:8.2f}")
            prev = mk


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=16)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--config", default="C3")
    args = ap.parse_args()
    net, mask, amp, T = bench.make_inputs(args.config, args.trials, 0)
    T = args.steps
    mask = np.ascontiguousarray(mask[:, :T])
    eng = Engine(net.n, args.trials, T, precision=32)
    eng.set_network(net.rowptr, net.col, net.weight, net.delay)
    eng.set_drive(mask, amp)
    for _ in range(2):
        out = eng.forward()
        eng.backward((2 * (out["v"] - 0.25)).float(), want_amp=False)
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
