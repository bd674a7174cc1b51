"""Queue-only Poisson workloads of the reference (`pkg/src/eventq/bench.py`),
run on the B200 queue batch: the single/batched inference benchmark
(`run_inference_bench`, bench.py:217-291), exact drop rates
(`measure_drop_rate`, :408-452) and the batch / capacity / pressure sweeps
(`sweep`, :458-500), with the reference's record schema (`CSV_COLUMNS`,
:39-43) so the reference's plotting reads the rows unchanged.

Every queue of a batch steps through its whole stream inside one kernel
launch (`eq_queues_run_poisson`); spike / drop counts are exactly the
reference's for the same seed (tests/test_poisson_queues.py), only the time
differs.
"""

from __future__ import annotations

import csv
import io
import json
import platform
import statistics
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch

from .errors import ConfigurationError
from .queues import QueueBatch, coerce_kind
from .workload import poisson_streams

CSV_COLUMNS = ["workload", "kind", "capacity", "max_delay", "batch", "lambda", "delay", "steps", "reps",
               "ns_per_step_per_queue", "drop_rate", "spikes_in", "spikes_out", "seed", "platform"]


def platform_label() -> str:
    try:
        name = torch.cuda.get_device_name()
    except Exception:
        name = platform.machine()
    return name.replace(",", ";")


@dataclass(frozen=True)
class PoissonWorkload:
    """Bernoulli(1/lambda) spike streams feeding one queue each (bench.py:63-84)."""

    lambda_steps: float
    delay_steps: int
    n_queues: int
    t_steps: int
    rng_seed: int

    def __post_init__(self):
        if self.lambda_steps < 1:
            raise ConfigurationError(f"lambda must be >= 1 step, got {self.lambda_steps}")
        if self.delay_steps < 1:
            raise ConfigurationError(f"delay must be >= 1 step, got {self.delay_steps}")


@dataclass
class BenchRecord:
    workload: str
    kind: str
    capacity: int
    max_delay: int
    batch: int
    lambda_steps: float
    delay_steps: int
    steps: int
    reps: int
    ns_per_step_per_queue: float
    drop_rate: float
    spikes_in: int
    spikes_out: int
    seed: int
    platform: str

    def to_row(self) -> dict:
        return {"workload": self.workload, "kind": self.kind, "capacity": self.capacity, "max_delay": self.max_delay,
                "batch": self.batch, "lambda": self.lambda_steps, "delay": self.delay_steps, "steps": self.steps,
                "reps": self.reps, "ns_per_step_per_queue": self.ns_per_step_per_queue,
                "drop_rate": self.drop_rate, "spikes_in": self.spikes_in, "spikes_out": self.spikes_out,
                "seed": self.seed, "platform": self.platform}


def write_csv(records: Sequence[BenchRecord], out) -> None:
    w = csv.DictWriter(out, fieldnames=CSV_COLUMNS, lineterminator="\n")
    w.writeheader()
    for r in records:
        w.writerow(r.to_row())


def write_json(records: Sequence[BenchRecord], out) -> None:
    json.dump([r.to_row() for r in records], out, indent=2)
    out.write("\n")


def records_to_csv_text(records: Sequence[BenchRecord]) -> str:
    buf = io.StringIO()
    write_csv(records, buf)
    return buf.getvalue()


def _run_batch(kind, capacity, max_delay, wl: PoissonWorkload, bits: torch.Tensor):
    """One fresh batch through its streams: (ms, delivered, accepted, aliased, batch)."""
    qb = QueueBatch(kind, wl.n_queues, capacity, max_delay if coerce_kind(kind).value == "ring" else None)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    delivered, accepted = qb.run_poisson(bits, wl.t_steps, wl.delay_steps)
    b.record()
    torch.cuda.synchronize()
    aliased = int(qb.lossy_counts()[0].sum()) if coerce_kind(kind).value == "lossyring" else 0
    return a.elapsed_time(b), float(delivered.sum()), int(accepted.sum()), aliased, qb


def run_inference_bench(kind, workload: PoissonWorkload, capacity: Optional[int] = None,
                        max_delay: Optional[int] = None, reps: int = 5, warmup: int = 2) -> BenchRecord:
    """Median time of the whole stream per step per queue (bench.py:217-291);
    the counts are the reference's exactly."""
    if reps < 3:
        raise ConfigurationError(f"reps must be >= 3, got {reps}")
    if warmup < 1:
        raise ConfigurationError(f"warmup must be >= 1, got {warmup}")
    k = coerce_kind(kind)
    if max_delay is None:
        max_delay = workload.delay_steps
    bits = torch.from_numpy(poisson_streams(workload.lambda_steps, workload.t_steps, workload.n_queues,
                                            workload.rng_seed).view(np.int32)).cuda()
    attempted = int(np.unpackbits(bits.cpu().numpy().view(np.uint8)).sum())
    times = []
    for rep in range(warmup + reps):
        ms, delivered, accepted, aliased, qb = _run_batch(k.value, capacity, max_delay, workload, bits)
        if rep >= warmup:
            times.append(ms)
    cap = capacity if capacity is not None else qb.capacity
    per = statistics.median(times) * 1e6 / (workload.t_steps * workload.n_queues)
    return BenchRecord("poisson", k.value, cap, max_delay, workload.n_queues, workload.lambda_steps,
                       workload.delay_steps, workload.t_steps, reps, per,
                       (attempted - accepted + aliased) / attempted if attempted else 0.0, attempted,
                       int(round(delivered)), workload.rng_seed, platform_label())


def measure_drop_rate(kind, lambda_steps: float, delay_steps: int, t_steps: int, rng_seed: int,
                      capacity: Optional[int] = None, max_delay: Optional[int] = None) -> BenchRecord:
    """Exact dropped/enqueued fraction over one seeded stream (bench.py:408-452);
    LossyRing aliasing counts as loss."""
    wl = PoissonWorkload(lambda_steps, delay_steps, 1, t_steps, rng_seed)
    if max_delay is None:
        max_delay = delay_steps
    bits = torch.from_numpy(poisson_streams(lambda_steps, t_steps, 1, rng_seed).view(np.int32)).cuda()
    attempted = int(np.unpackbits(bits.cpu().numpy().view(np.uint8)).sum())
    _, delivered, accepted, aliased, qb = _run_batch(coerce_kind(kind).value, capacity, max_delay, wl, bits)
    cap = capacity if capacity is not None else qb.capacity
    return BenchRecord("droprate", coerce_kind(kind).value, cap, max_delay, 1, lambda_steps, delay_steps, t_steps,
                       1, 0.0, (attempted - accepted + aliased) / attempted if attempted else 0.0, attempted,
                       int(round(delivered)), rng_seed, platform_label())


def sweep(axis: str, grid: Sequence[float], kind, base: PoissonWorkload, capacity: Optional[int] = None,
          reps: int = 5, warmup: int = 2) -> List[BenchRecord]:
    """One record per grid point along batch, capacity or pressure (bench.py:458-500)."""
    if not grid:
        raise ConfigurationError("sweep grid is empty")
    if list(grid) != sorted(grid):
        raise ConfigurationError("sweep grid must be ascending")
    out = []
    for point in grid:
        if axis == "batch":
            wl = PoissonWorkload(base.lambda_steps, base.delay_steps, int(point), base.t_steps, base.rng_seed)
            rec = run_inference_bench(kind, wl, capacity=capacity, reps=reps, warmup=warmup)
        elif axis == "capacity":
            rec = run_inference_bench(kind, base, capacity=int(point), max_delay=base.delay_steps, reps=reps,
                                      warmup=warmup)
        elif axis == "pressure":
            delay = max(1, round(point * base.lambda_steps))
            wl = PoissonWorkload(base.lambda_steps, delay, base.n_queues, base.t_steps, base.rng_seed)
            rec = run_inference_bench(kind, wl, capacity=capacity, reps=reps, warmup=warmup)
        else:
            raise ConfigurationError(f"sweep axis must be batch|capacity|pressure, got {axis!r}")
        rec.workload = f"sweep_{axis}"
        out.append(rec)
    return out
