"""Generate tests/golden/*.npz by running the UNMODIFIED Python reference.

Runs only in the build container (it imports ``eventq`` read-only from
/root/reference/pkg/src); the GPU box never reads /root/reference.  Inputs are
drawn with the version-stable SplitMix generator in
``paper_2512_05906_b200.workload`` and fed to the reference as dense matrices
plus a drive callable, so the fixtures pin outputs for inputs any box can
regenerate.  A SHA-256 of the inputs is stored beside the outputs.

Usage:  python scripts/make_goldens.py [--skip-slow] [--only NAME]
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import eventq  # noqa: E402  (reference, read-only)
from eventq import DualScalar, NetworkParams, SeedDirection, build_rsnn, simulate  # noqa: E402
from eventq.network import PrimalRSNN, forward_gradient  # noqa: E402

from paper_2512_05906_b200 import workload as wl  # noqa: E402
sys.path.insert(0, os.path.join(REPO, "tests"))
import golden_cases  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")
DT = 1e-3


def input_digest(net: wl.Network, mask: np.ndarray, amp: np.ndarray) -> str:
    h = hashlib.sha256()
    for a in (net.rowptr, net.col, net.weight, net.delay, mask, amp):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def drive_fn(mask_bt: np.ndarray, amp: np.ndarray, n: int, seeded=None):
    """Reference-style drive callable from one trial's packed mask [T, W]."""
    active = wl.unpack_mask(mask_bt, n)
    zero = DualScalar(0.0, 0.0)
    rows = []
    for m in range(active.shape[0]):
        row = []
        for j in range(n):
            if active[m, j]:
                row.append(DualScalar(float(amp[j]), 1.0 if seeded == j else 0.0))
            else:
                row.append(zero)
        rows.append(row)
    return lambda step: rows[step] if step < len(rows) else rows[-1]


def ref_params(net: wl.Network, kind: str, capacity=None, v_target=0.25, dense_delay=DT,
               refractory=0, exact=True):
    w, d = net.dense(dense_delay)
    return NetworkParams(n=net.n, weights=w, delays=d, tau_m=1.0, tau_syn=0.5, v_th=1.0,
                         v_reset=0.0, dt=DT, queue_kind=kind, queue_capacity=capacity,
                         refractory_steps=refractory, v_target=np.full(net.n, v_target),
                         exact_delivery=exact)


def run_case(name: str, net: wl.Network, kind: str, t_steps: int, mask: np.ndarray,
             amp: np.ndarray, capacity=None, directions=(), record=True, refractory=0,
             dense_delay=DT, exact=True):
    t0 = time.time()
    params = ref_params(net, kind, capacity, refractory=refractory, dense_delay=dense_delay, exact=exact)
    res = simulate(build_rsnn(params), t_steps, drive_fn(mask[0], amp, net.n), record=record)
    # loss tangent-free; raster rows (step, neuron)
    raster = np.array(res.raster, dtype=np.int32).reshape(-1, 2) if record else np.zeros((0, 2), np.int32)
    out = dict(
        kind=kind, n=net.n, t_steps=t_steps, capacity=-1 if capacity is None else capacity,
        refractory=refractory, dense_delay=dense_delay, exact=exact,
        digest=input_digest(net, mask, amp),
        raster=raster, loss=res.loss.primal, spike_count=res.spike_count,
        drop_count=res.drop_count, enqueued_count=res.enqueued_count,
    )
    if record:
        if net.n * t_steps <= 100_000:   # keep fixtures small
            out["v_trace"] = res.voltages
        out["v_final"] = res.voltages[-1]
    # primal twin must be bitwise the dual's primal half (network.py:501-505)
    pr = PrimalRSNN(params)
    pr.run(t_steps, drive_fn(mask[0], amp, net.n))
    out["v_final_primal"] = np.array(pr.v)
    out["i_final_primal"] = np.array(pr.i_syn)
    dirs, jvps = [], []
    for (p, i, j) in directions:
        seed = SeedDirection(p, i, j)
        if p == "drive":
            # forward_gradient builds the drive from a PoissonDrive; seed manually
            st = build_rsnn(params, seed=None)
            r = simulate(st, t_steps, drive_fn(mask[0], amp, net.n, seeded=i))
            g = r.loss.tangent
        else:
            st = build_rsnn(params, seed=seed)
            r = simulate(st, t_steps, drive_fn(mask[0], amp, net.n))
            g = r.loss.tangent
        dirs.append((0 if p == "weight" else 1 if p == "delay" else 2, i, j))
        jvps.append(g)
    out["directions"] = np.array(dirs, dtype=np.int64).reshape(-1, 3)
    out["jvp"] = np.array(jvps, dtype=np.float64)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"{name}: kind={kind} n={net.n} T={t_steps} spikes={res.spike_count} "
          f"drops={res.drop_count} dirs={len(dirs)} {time.time() - t0:.1f}s", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-slow", action="store_true")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    for case in golden_cases.CASES:
        if args.only and case.name != args.only:
            continue
        if case.slow and args.skip_slow:
            continue
        net, mask, amp = case.inputs()
        dirs = golden_cases.pick_directions(net, case.seed, *case.n_dirs)
        run_case(case.name, net, case.kind, case.t_steps, mask, amp, capacity=case.capacity,
                 directions=dirs, refractory=case.refractory, exact=case.exact)


if __name__ == "__main__":
    main()
