"""Trial sharding + final all-reduce, world size 2 over gloo on CPU.

Each rank computes its trial block with the CPU oracle (device mode, fp32 —
the arithmetic the GPU ranks run) and the reduced gradient must equal one
process computing all trials, up to the reassociation of the final sum."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_05906_b200.parallel import shard_trials, sharded_value_and_grad


def test_shard_trials_covers_everything_once():
    for B in (2, 7, 16, 33):
        for world in (1, 2, 3, 8):
            if B < world:
                continue
            blocks = [shard_trials(B, world, r) for r in range(world)]
            seen = [t for s, c in blocks for t in range(s, s + c)]
            assert seen == list(range(B))
            assert max(c for _, c in blocks) - min(c for _, c in blocks) <= 1


def _problem():
    from paper_2512_05906_b200 import workload as wl
    net = wl.random_network(150, 15, 9, delay_steps=(1, 12), w_mean=0.04, w_std=0.01)
    return net


def _compute(net, start, count, T=250):
    from oracle.oracle import OracleSession, frac_bits
    from paper_2512_05906_b200 import workload as wl
    mask = wl.drive_masks(net.n, start + count, T, 1e-3, seed0=300)[start:start + count]
    maxin = float(np.bincount(net.col, weights=np.abs(net.weight.astype(np.float32)), minlength=net.n).max())
    s = OracleSession(n=net.n, n_trials=count, t_steps=T, mode="device", precision=32,
                      frac_bits=frac_bits(maxin, 32))
    s.set_network(net.rowptr, net.col, net.weight, net.delay)
    s.set_drive(mask, np.full(net.n, 12.0))
    out = s.forward()
    vbar = 2.0 * (out["v"] - 0.25)
    gw, gd, ga = s.backward(vbar)
    loss = float(((out["v"] - 0.25) ** 2).sum())
    return loss, torch.from_numpy(gw), torch.from_numpy(gd), torch.from_numpy(ga)


def _worker(rank, world, port, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    net = _problem()
    res = sharded_value_and_grad(lambda s, c: _compute(net, s, c), B)
    if rank == 0:
        q.put((res.loss, res.grad_w.numpy(), res.grad_d.numpy(), res.grad_amp.numpy()))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_equals_single_process():
    B = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    loss, gw, gd, ga = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    net = _problem()
    # single process over all trials: drive seeds are global, so the same inputs
    l1, w1, d1, a1 = _compute(net, 0, B)
    assert loss == pytest.approx(l1, rel=1e-12)
    np.testing.assert_allclose(gw, w1.numpy(), rtol=1e-12, atol=1e-12 * np.abs(w1.numpy()).max())
    np.testing.assert_allclose(gd, d1.numpy(), rtol=1e-12, atol=1e-12 * np.abs(d1.numpy()).max())
    np.testing.assert_allclose(ga, a1.numpy(), rtol=1e-12, atol=1e-12 * np.abs(a1.numpy()).max())
    assert np.abs(gw).max() > 0
