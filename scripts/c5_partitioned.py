"""BASELINE config 5: one network partitioned across GPUs, spike exchange every
min-delay steps (paper_2512_05906_b200.partition).

    # P partitions of one network on ONE GPU (partition after partition per window)
    python scripts/c5_partitioned.py --parts 8 [--check]
    # one partition per GPU, NCCL over NVLink
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 scripts/c5_partitioned.py

Prints one JSON line: synaptic events/s (fwd+bwd) of the whole network, the
forward / reverse time, windows and exchange volume.  --check (single process)
also runs the unpartitioned engine and asserts the raster, final state and
pending queues are bitwise equal and the gradients agree to rounding.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", type=int, default=8, help="partitions when running in one process")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--delays", default="8,256")
    ap.add_argument("--trials", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="peer exchange: capture the whole partitioned forward + reverse (every window's "
                         "launches and stream events) in one CUDA graph and time its replays")
    ap.add_argument("--concurrent", action="store_true",
                    help="peer exchange: every partition on its own stream and SM share (grid = 2*SMs/P), "
                         "windows ordered by events — the partitions run side by side as on P GPUs")
    ap.add_argument("--exchange", default="peer", choices=["peer", "host"],
                    help="single process: device-resident peer exchange (eq_set_peers) or host-routed export/import")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_2512_05906_b200 import workload as wl
    from paper_2512_05906_b200.engine import Engine
    from paper_2512_05906_b200.partition import (DistTransport, GraphedPass, LocalTransport, PartitionedNetwork, PeerTransport,
                                                 min_delay_steps, partition_csr, slice_mask, split_range)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lo_d, hi_d = (int(x) for x in args.delays.split(","))
    t0 = time.perf_counter()
    net = wl.random_network(args.n, args.k, 0, delay_steps=(lo_d, hi_d))
    mask = wl.drive_masks(args.n, args.trials, args.steps, 1e-3, seed0=1000)
    amp = np.full(args.n, 12.0)
    t_build = time.perf_counter() - t0
    dtype = np.float32 if args.precision == 32 else np.float64
    W = min_delay_steps(net.delay, 1e-3, dtype)

    P = world if world > 1 else args.parts
    mine = [rank] if world > 1 else list(range(P))
    engines, ranges, ids = [], [], []
    for r in mine:
        lo, hi = split_range(net.n, P, r)
        rp, cl, w, d, eid = partition_csr(net.rowptr, net.col, net.weight, net.delay, lo, hi)
        conc = args.concurrent and world == 1 and args.exchange == "peer"
        sm = torch.cuda.get_device_properties(local).multi_processor_count
        e = Engine(hi - lo, args.trials, args.steps, precision=args.precision, partition=(net.n, lo), device=local,
                   max_ctas=(2 * sm) // P if conc else 0, stream=torch.cuda.Stream(local) if conc else None)
        e.set_network(rp, cl, w, d)
        e.set_drive(slice_mask(mask, net.n, lo, hi), amp[lo:hi])
        engines.append(e)
        ranges.append((lo, hi))
        ids.append(eid)
    if world > 1:
        tp = DistTransport()
    else:
        tp = PeerTransport(P) if args.exchange == "peer" else LocalTransport(P)
    pn = PartitionedNetwork(engines, mine, tp, window=W)
    stream = torch.cuda.current_stream()

    def once():
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        c = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for e in engines:                     # partitions on their own streams start after `a`
            e.torch_stream.wait_event(a)
        pn.forward(args.steps)
        pn.join(stream)
        b.record(stream)
        vbars = [(2.0 * (e.state()["v"].double() - 0.25)).to(e.dtype) for e in engines]
        for e in engines:
            e.torch_stream.wait_event(b)
        pn.backward(vbars, want_amp=False)
        pn.join(stream)
        c.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b), b.elapsed_time(c)

    once()                                   # warm-up
    if world > 1:
        dist.barrier()
    fw, bw = [], []
    graph = args.graph and world == 1 and args.exchange == "peer"
    if graph:
        v_eager = [e.state()["v"].clone() for e in engines]
        g = GraphedPass(pn, args.steps, lambda es: [(2.0 * (e.state()["v"].double() - 0.25)).to(e.dtype) for e in es])
        for _ in range(args.reps + 1):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            torch.cuda.synchronize()
            fw.append(a.elapsed_time(b))
            bw.append(0.0)
        fw, bw = fw[1:], bw[1:]
        for e in engines:
            e.sync()
        same = all(torch.equal(e.state()["v"], v) for e, v in zip(engines, v_eager))
        print(f"graph replay: V equal to the eager run: {same}", file=sys.stderr)
        if not same:
            sys.exit("graph replay differs from the eager run")
    for _ in range(0 if graph else args.reps):
        f, b = once()
        fw.append(f)
        bw.append(b)
    ctr = sum(e.counters() for e in engines)
    t = torch.tensor([np.mean(fw) + np.mean(bw), np.mean(fw), np.mean(bw)], device="cuda", dtype=torch.float64)
    ev = torch.tensor([float(ctr[:, 1].sum()), float(ctr[:, 0].sum()),
                       float(sum(sum(c) for c in pn.counts)) if pn.counts else float(ctr[:, 0].sum()) * (P - 1)],
                      device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ev)
        ev[2] /= world                        # every rank saw every count
    ms, fwd_ms, bwd_ms = (float(x) for x in t.tolist())
    events, spikes, exchanged = (float(x) for x in ev.tolist())
    res = {
        "metric": "synaptic events/sec (fwd+bwd)", "value": events / (ms / 1e3), "unit": "events/s",
        "config": {"workload": f"C5: {net.n} LIF neurons, {args.k} syn/neuron, delay {lo_d}..{hi_d} steps, ring, "
                               f"fwd+bwd T={args.steps}, {P} partitions", "trials": args.trials,
                   "processes": world, "partitions": P, "window_steps": W,
                   "exchange": "nccl-host" if world > 1 else args.exchange,
                   "concurrent_partitions": bool(args.concurrent and world == 1),
                   "ctas_per_partition": engines[0].geometry[0],
                   "windows": len(pn.win), "exchanged_spikes": exchanged,
                   "exchange_bytes": exchanged * (16 if args.precision == 32 else 24)},
        "ms_per_pass": ms, "fwd_ms": fwd_ms, "bwd_ms": bwd_ms, "spikes": spikes, "events": events,
        "build_s": t_build,
    }
    if args.check and world == 1:
        whole = Engine(net.n, args.trials, args.steps, precision=args.precision, device=local)
        whole.set_network(net.rowptr, net.col, net.weight, net.delay)
        whole.set_drive(mask, amp)
        out = whole.forward()
        ws = whole.spikes()
        ref = np.stack([ws["trial"], ws["step"], ws["neuron"]], 1)
        got = []
        for e, (lo, hi) in zip(engines, ranges):
            s = e.spikes()
            got.append(np.stack([s["trial"], s["step"], s["neuron"] + lo], 1))
        got = np.concatenate(got)
        got = got[np.lexsort((got[:, 2], got[:, 1], got[:, 0]))]
        ref = ref[np.lexsort((ref[:, 2], ref[:, 1], ref[:, 0]))]
        v = out["v"].cpu().numpy()
        ok_r = bool(np.array_equal(got, ref))
        ok_v = all(np.array_equal(e.state()["v"].cpu().numpy(), v[:, lo:hi]) for e, (lo, hi) in zip(engines, ranges))
        vbar = (2.0 * (out["v"].double() - 0.25)).to(out["v"].dtype)
        gw = whole.backward(vbar, want_amp=False)[0].cpu().numpy()
        grads = pn.backward([vbar[:, lo:hi] for lo, hi in ranges], want_amp=False)
        pw = np.zeros_like(gw)
        for (g, _, _), eid in zip(grads, ids):
            pw[eid] = g.cpu().numpy()
        res["check"] = {"raster_bitwise": ok_r, "v_bitwise": ok_v, "spikes": int(len(ref)),
                        "grad_w_max_rel_err": float(np.abs(pw - gw).max() / max(np.abs(gw).max(), 1e-300))}
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
