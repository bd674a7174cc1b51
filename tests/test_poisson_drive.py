"""On-device PoissonDrive (eq_poisson_drive).

The reference's PoissonDrive (pkg/src/eventq/network.py:98-155) draws its
exponential gaps from numpy's sequential PCG64 stream; the device generator
keeps the reference's walk and grid sampling but draws from a Philox4x32-10
stream per (trial, neuron).  Pinned here by:
  * Random123's known-answer vectors for Philox4x32-10 (oracle restatement);
  * the oracle's C walk == the reference's walk (PoissonDrive.__init__ +
    materialize, restated line by line below) fed the same Philox draws;
  * drive statistics of the oracle == those of the reference-style numpy drive;
  * GPU mask == oracle mask, bit for bit (-m gpu)."""

import math

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2512_05906_b200 import workload as wl

DT = 1e-3


def test_philox_known_answers():
    # Random123 kat_vectors, philox4x32 10 rounds: counter[4], key[2] -> out[4]
    kats = [
        ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
        ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
        ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
         [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
    ]
    for ctr, key, want in kats:
        assert orc.philox4x32_10(ctr, key).tolist() == want


def _draws(b, i, seed):
    """Exponential draws of (trial b, neuron i) as eq_drive.cu defines them."""
    call = 0
    while True:
        o = orc.philox4x32_10([call, i, b, 0x5D0F1EED], [seed & 0xFFFFFFFF, seed >> 32])
        call += 1
        for a, c in ((o[0], o[1]), (o[2], o[3])):
            u = ((int(a) >> 5) * 67108864.0 + (int(c) >> 6) + 0.5) * (1.0 / 9007199254740992.0)
            yield u


def test_oracle_walk_is_the_reference_walk():
    """PoissonDrive.__init__ (network.py:113-120) and materialize (:138-143),
    restated with the same draws (log via math.log here, the shared eq_log in
    C: the two agree to <= 2 ulp, and no grid boundary is that close here)."""
    n, B, T, mean, dur, seed = 45, 2, 300, 16 * DT, 12.5 * DT, (7 << 32) + 11
    got = orc.poisson_drive(n, B, T, DT, mean, dur, seed)
    want = np.zeros((B, T, 2), dtype=np.uint32)
    t_total = T * DT
    for b in range(B):
        for i in range(n):
            g = _draws(b, i, seed)
            starts = []
            t = -mean * math.log(next(g))
            while t < t_total:
                starts.append(t)
                t += dur + -mean * math.log(next(g))
            for s in starts:
                e = s + dur
                lo = min(T, max(0, math.ceil(s / DT)))
                hi = min(T, max(0, math.ceil(e / DT)))
                want[b, lo:hi, i >> 5] |= np.uint32(1 << (i & 31))
    assert np.array_equal(got, want)


def _stats(masks, n):
    bits = np.unpackbits(masks.view(np.uint8), bitorder="little").reshape(masks.shape[0], masks.shape[1], -1)[:, :, :n]
    duty = bits.mean()
    onsets = (bits[:, 1:] & ~bits[:, :-1]).sum() + bits[:, 0].sum()
    return duty, onsets / (masks.shape[0] * n)


def test_statistics_match_the_reference_drive():
    n, B, T = 1500, 2, 1000
    ref = wl.drive_masks(n, B, T, DT, seed0=1000)                 # numpy draws (reference PoissonDrive)
    dev = orc.poisson_drive(n, B, T, DT, 16 * DT, 12 * DT, 1000)  # Philox draws
    d_ref, p_ref = _stats(ref, n)
    d_dev, p_dev = _stats(dev, n)
    # duty ~ 12/28 minus edge effects; 3e6 samples: both within 1.5 %
    assert abs(d_dev - d_ref) < 0.015 * d_ref, (d_dev, d_ref)
    assert abs(p_dev - p_ref) < 0.03 * p_ref, (p_dev, p_ref)


def test_seed_and_trial_streams_are_distinct():
    a = orc.poisson_drive(64, 2, 200, DT, 16 * DT, 12 * DT, 5)
    b = orc.poisson_drive(64, 2, 200, DT, 16 * DT, 12 * DT, 6)
    assert not np.array_equal(a, b)
    assert not np.array_equal(a[0], a[1])


@pytest.mark.gpu
@pytest.mark.parametrize("n,B,T,mean,dur,seed", [
    (1000, 3, 500, 16, 12, 1000),
    (77, 2, 1000, 16, 12.5, (3 << 32) + 9),       # ragged word, off-grid duration, 64-bit seed
    (33, 1, 64, 0.5, 0.0, 1),                      # zero-length pulses are never active
    (100_000, 1, 1000, 16, 12, 42),
])
def test_gpu_drive_equals_oracle(n, B, T, mean, dur, seed):
    import torch
    from paper_2512_05906_b200.engine import poisson_drive_device
    m = poisson_drive_device(n, B, T, DT, mean * DT, dur * DT, seed)
    torch.cuda.synchronize()
    got = m.cpu().numpy().view(np.uint32)
    want = orc.poisson_drive(n, B, T, DT, mean * DT, dur * DT, seed)
    assert np.array_equal(got, want)
    if dur == 0:
        assert not got.any()


@pytest.mark.gpu
def test_engine_runs_on_the_device_drive():
    import torch
    from paper_2512_05906_b200.engine import Engine
    from paper_2512_05906_b200.errors import ConfigurationError
    net = wl.random_network(400, 30, 3, delay_steps=(1, 12), w_mean=0.02, w_std=0.01)
    eng = Engine(400, 2, 300, precision=32)
    eng.set_network(net.rowptr, net.col, net.weight, net.delay)
    eng.set_poisson_drive(np.full(400, 12.0), 16 * DT, 12 * DT, seed=9)
    out = eng.forward()
    torch.cuda.synchronize()
    assert eng.counters()[:, 0].sum() > 0
    # the same mask through the host path gives the same run
    mask = orc.poisson_drive(400, 2, 300, DT, 16 * DT, 12 * DT, 9)
    eng.set_drive(mask, np.full(400, 12.0))
    out2 = eng.forward()
    assert torch.equal(out["v"], out2["v"])
    with pytest.raises(ConfigurationError):
        eng.set_poisson_drive(np.full(400, 12.0), 0.0, 12 * DT, seed=1)
