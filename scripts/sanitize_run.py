"""Small forward + reverse runs of every kernel family for compute-sanitizer
(scripts/sanitize.sh): ring fp32/fp64 (incl. forced bucket overflow), the
bounded kinds (staged and HBM-resident paths), lossy ring, plain delivery,
partitions with the peer exchange, the queue API and the device drive."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2512_05906_b200 import workload as wl
    from paper_2512_05906_b200.engine import Engine, poisson_drive_device
    from paper_2512_05906_b200.partition import (PartitionedNetwork, PeerTransport, partition_csr, slice_mask,
                                                 split_range)
    from paper_2512_05906_b200.queues import QueueBatch

    n, B, T = 256, 2, 60
    net = wl.random_network(n, 16, 5, delay_steps=(2, 10), w_mean=0.05, w_std=0.02)
    mask = wl.drive_masks(n, B, T, 1e-3, seed0=3)
    amp = np.full(n, 12.0)
    runs = [dict(kind="ring", precision=32), dict(kind="ring", precision=64), dict(kind="ring", bucket=2),
            dict(kind="binaryheap", capacity=4), dict(kind="sortedarray", capacity=8),
            dict(kind="fiforing", capacity=4, homog=True), dict(kind="binaryheap", capacity=100),
            dict(kind="lossyring", capacity=3), dict(kind="ring", exact=False)]
    for r in runs:
        nt = wl.random_network(n, 16, 5, delay_steps=(4, 4)) if r.get("homog") else net
        eng = Engine(n, B, T, kind=r["kind"], precision=r.get("precision", 32), capacity=r.get("capacity", 0),
                     lif=wl.LIFConfig(exact_delivery=r.get("exact", True)))
        eng.set_network(nt.rowptr, nt.col, nt.weight, nt.delay)
        eng.set_drive(mask, amp)
        if r.get("bucket"):
            eng.debug_set_bucket_capacity(r["bucket"])
        out = eng.forward()
        eng.backward((2.0 * (out["v"] - 0.25)).to(eng.dtype))
        eng.pending()
        torch.cuda.synchronize()
        print("ok", r, eng.spike_count(), flush=True)
    P = 2
    engines = []
    for k in range(P):
        lo, hi = split_range(n, P, k)
        rp, cl, w, d, _ = partition_csr(net.rowptr, net.col, net.weight, net.delay, lo, hi)
        e = Engine(hi - lo, B, T, partition=(n, lo))
        e.set_network(rp, cl, w, d)
        e.set_drive(slice_mask(mask, n, lo, hi), amp[lo:hi])
        engines.append(e)
    pn = PartitionedNetwork(engines, range(P), PeerTransport(P), window=2)
    pn.forward(T)
    pn.backward([(2.0 * (e.state()["v"] - 0.25)) for e in engines])
    torch.cuda.synchronize()
    print("ok partitions", flush=True)
    qb = QueueBatch("binaryheap", n_queues=64, capacity=4)
    q = torch.arange(64, dtype=torch.int32, device="cuda")
    qb.enqueue(q, torch.full((64,), 3, dtype=torch.int32, device="cuda"), torch.ones(64, device="cuda"),
               torch.zeros(64, device="cuda"), torch.zeros(64, device="cuda"))
    for _ in range(4):
        qb.pop()
    poisson_drive_device(n, B, T, 1e-3, 16e-3, 12e-3, 7)
    torch.cuda.synchronize()
    print("ok queues+drive", flush=True)


if __name__ == "__main__":
    main()
