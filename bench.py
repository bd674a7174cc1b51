"""Benchmark: ring-buffer forward + reverse of the R-SNN hot path (BASELINE config C3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C3] [--trials B] [--precision 32]

One bench step = one forward of T=1000 simulated steps plus its reverse pass
for the B trials this rank owns (weak scaling: B trials per GPU, trials shard
across ranks, a final NCCL all-reduce of dL/dw and dL/dd).  `value` is
synaptic events per second (one event = one (spike, out-edge) pair, counted on
the device, fwd+bwd counted once) over the whole job; `e2e` is the same metric
through the public API with the drive mask copied from pinned host memory, the
(device-resident) network handed to the engine as every training step does
(validation + edge repack), and the loss + gradients read back every step.
`variants` adds the same measurement for C3 in fp64 and for the heap and
sorted queues at C4 (memory pressure, drops), each with its roofline fraction.

--impl reference times the reference's CPU path on the host cores: the
reference is pure Python and cannot travel to the GPU box, so this runs the
C++ port of it (oracle/, pinned bitwise to the reference in
tests/test_oracle_pin.py) with OpenMP over trials, on a bounded sample of the
same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
TRAFFIC_FILE = "r2bl_traffic.json"   # DRAM bytes per launch from the committed ncu capture of the default workload


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


# ---------------------------------------------------------------- algorithmic bytes
# SURVEY.md §8(d) / BASELINE.md §4, written for element size t (4 fp32 / 8 fp64)
# and fixed-point slot word q (int32 fp32 / int64 fp64); at t = q = 4 these are
# the survey's fp32 figures (ring, exact delivery, reverse mode):
#   per neuron-step   fwd [slot 2q read + 2q clear, drive 4, I/V 4t] = 36 B
#                     bwd [adjoints 4t, reverse slot 2t]             = 24 B
#   per spike         record {t, a, v_hat} 3t + id 4, written fwd, read bwd = 16 + 16 B
#   per event         fwd [CSR 4 + 2t, slot RMW 4q]                  = 28 B
#                     bwd [CSR 4 + 2t, gather 2t, (g_w, g_d) RMW 4t] = 36 B
# bounded kinds (FIFO / heap / sorted), same rules: per event the fwd moves CSR
# 4 + 2t plus the event record {due 4, W_s q, W_m q} written at enqueue and read
# at pop; per neuron-step the queue meta 16 B replaces the slot's 4q.
def byte_model(precision=32, bounded=False):
    t = 4 if precision == 32 else 8
    q = t
    fwd_ns = (16 if bounded else 4 * q) + 4 + 4 * t
    fwd_ev = (4 + 2 * t) + (2 * (4 + 2 * q) if bounded else 4 * q)
    spike = 3 * t + 4
    return {"fwd": (fwd_ns, spike, fwd_ev), "bwd": (6 * t, spike, (4 + 2 * t) + 2 * t + 4 * t)}


def alg_bytes(neuron_steps, spikes, events, which, bounded=False, precision=32):
    a = byte_model(precision, bounded and which == "fwd")[which]
    return a[0] * neuron_steps + a[1] * spikes + a[2] * events


def host_label():
    """CPU model and logical core count of this host (the reference's
    bench.platform_label, pkg/src/eventq/bench.py:48-60, names the host too)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return f"{model} x {os.cpu_count()} logical cores"


class ClockSampler:
    """SM clocks + throttle reasons sampled in-process through NVML (no
    nvidia-smi child: its start-up stalled a timed step).  Start it before the
    warm-up; only samples inside mark_start()..mark_end() are summarised."""

    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20), ("hw_thermal_slowdown", 0x40),
               ("sw_power_cap", 0x4))

    def __init__(self, index=0, period=0.1):
        self.index, self.period = index, period
        self.rows = []
        self.t0 = self.t1 = None
        self.stop = threading.Event()
        self.ok = False

    def __enter__(self):
        if os.environ.get("EQ_NO_CLOCKS"):
            return self
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.dev = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.dev, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
            self.ok = True
        except Exception:
            self.ok = False
        return self

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.dev, nv.NVML_CLOCK_SM)
                get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                rs = get(self.dev)
                self.rows.append((time.perf_counter(), sm, rs))
            except Exception:
                pass
            self.stop.wait(self.period)

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter()

    def __exit__(self, *exc):
        self.stop.set()
        if self.ok:
            self.thread.join(timeout=2)

    def summary(self):
        rows = [r for r in self.rows if (self.t0 is None or r[0] >= self.t0) and (self.t1 is None or r[0] <= self.t1)]
        if not rows:   # timed region shorter than one period: nearest samples
            rows = self.rows[-2:]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({name for _, _, rs in rows for name, bit in self.REASONS if rs & bit})
        return {"sm_mhz": statistics.median(r[1] for r in rows), "sm_max_mhz": self.max_sm, "reasons": reasons,
                "samples": len(rows), "source": "nvml"}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_inputs(cfg, trials, rank, seed=0, delay_steps=None):
    from paper_2512_05906_b200 import workload as wl
    n, k, drange, _, T = wl.CONFIGS[cfg]
    net = wl.random_network(n, k, seed, delay_steps=delay_steps or drange)
    # trial b of rank r has drive seed 1000 + r*trials + b
    from concurrent.futures import ProcessPoolExecutor
    seeds = [1000 + rank * trials + b for b in range(trials)]
    workers = max(1, min(len(seeds), (os.cpu_count() or 2) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))))
    with ProcessPoolExecutor(workers) as ex:
        masks = list(ex.map(_one_mask, [(n, T, s) for s in seeds]))
    mask = np.stack(masks)
    return net, mask, np.full(n, 12.0), T


def _one_mask(args):
    from paper_2512_05906_b200 import workload as wl
    n, T, s = args
    return wl.pack_mask(wl.poisson_drive_mask(n, T, 1e-3, 16e-3, 12e-3, s))


# ---------------------------------------------------------------- reference arm (CPU)

def cpu_reference_sample(net, mask, amp, T, max_trials=None, steps=None, kind="ring", capacity=0):
    """The oracle (C++ port of the reference path) on host cores: forward +
    reverse over `trials` trials of the same network; returns (events/s, info)."""
    from oracle import oracle as orc
    threads = orc.threads()
    B = max_trials or min(threads, 16)
    B = min(B, mask.shape[0])
    steps = steps or T
    s = orc.OracleSession(n=net.n, n_trials=B, t_steps=steps, mode="device", precision=32, kind=kind,
                          capacity=capacity,
                          frac_bits=orc.frac_bits(float(np.bincount(net.col, weights=np.abs(net.weight),
                                                                     minlength=net.n).max()), 32))
    s.set_network(net.rowptr, net.col, net.weight, net.delay)
    s.set_drive(np.ascontiguousarray(mask[:B, :steps]), amp)
    t0 = time.perf_counter()
    out = s.forward()
    s.backward(2.0 * (out["v"] - 0.25))
    dt = time.perf_counter() - t0
    events = int(out["counters"][:, 1].sum())
    return events / dt, dict(cores=min(threads, B), trials=B, steps=steps, seconds=dt, events=events,
                             neuron_steps=B * steps * net.n)


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    # torchrun pins OMP_NUM_THREADS=1 per rank; the CPU arm alone on this host
    # uses every core (read by the OpenMP runtime when the oracle loads)
    if world > 1 or os.environ.get("OMP_NUM_THREADS") == "1":
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    from oracle import oracle as orc
    trials = args.cpu_trials or min(orc.threads(), 16)
    net, mask, amp, T = make_inputs(args.config, trials, 0, delay_steps=args.delays)
    vals = []
    info = None
    for it in range(args.warmup + args.steps):
        v, info = cpu_reference_sample(net, mask, amp, T, max_trials=args.cpu_trials, steps=args.cpu_steps,
                                       kind=args.kind, capacity=args.capacity)
        if it >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "synaptic events/sec (fwd+bwd)", "value": value,
        "unit": "events/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": f"{args.config} {args.kind} fwd+bwd (sample)", **info},
        "cpu_baseline": {"value": value, "unit": "events/s", "cores": info["cores"], "kind": "port",
                         "host": host_label(),
                         "sample": f"{info['trials']} trials x {info['steps']} steps of {args.config}"},
        "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm

def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch_under_torchrun(args) -> None:
    """`bench.py --gpus N` run as a plain process (no WORLD_SIZE): start N ranks
    on this node with torch.distributed.run and exit with their status.  NCCL
    logs its communicator setup (NCCL_DEBUG=INFO) so the transport is on record."""
    import subprocess
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    sys.exit(subprocess.call(cmd, env=env))


def launch_selftest(args):
    """Launcher check without GPUs (tests/test_bench_launch.py): every rank
    joins a gloo group and all-reduces its rank; rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world != args.gpus:
        raise SystemExit(f"launched {world} ranks for --gpus {args.gpus}")
    dist.init_process_group("gloo")
    t = torch.tensor([float(rank)])
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"n_gpus": world, "rank_sum": float(t.item())}), flush=True)
    dist.destroy_process_group()


QUEUE_IMPL = {"admission": 0, "smem": 1, "hbm": 2}   # eq_config.staged_queues


def fwd_kernel(kind, impl):
    """The forward kernel a kind runs: the ring kernel (heap / sorted by
    admission too), or a bounded-queue structure kernel."""
    if kind in ("binaryheap", "sortedarray", "fiforing") and impl == 0:
        return "k_forward (admission)"   # (a FIFO delay off the step grid runs k_forward_bounded)
    if kind in ("fiforing", "binaryheap", "sortedarray", "lossyring"):
        return "k_forward_bq" if impl == 1 and kind != "lossyring" else "k_forward_bounded"
    return "k_forward"

VARIANTS = (
    # (label, config, trials, kind, capacity, precision, delays)
    ("C3 ring fp64 (the reference's arithmetic)", "C3", 24, "ring", 0, 64, None),
    ("C2 binaryheap[64]", "C2", 32, "binaryheap", 64, 32, None),
    ("C2 fiforing[64] (homogeneous delay 32 steps)", "C2", 32, "fiforing", 64, 32, (32, 32)),
    ("C4 ring (1M neurons, delays 1..256)", "C4", 4, "ring", 0, 32, None),
    ("C4 binaryheap[16] (memory pressure, drops)", "C4", 4, "binaryheap", 16, 32, None),
    ("C4 sortedarray[16] (memory pressure, drops)", "C4", 4, "sortedarray", 16, 32, None),
    ("C4 binaryheap[32] (memory pressure, drops)", "C4", 4, "binaryheap", 32, 32, None),
    ("C4 sortedarray[32] (memory pressure, drops)", "C4", 4, "sortedarray", 32, 32, None),
    ("C2 sortedarray[64]", "C2", 32, "sortedarray", 64, 32, None),
)
_NETS = {}


def measure_variant(label, cfg, trials, kind, capacity, precision, delays, steps, warmup, local, peak):
    """One more workload timed like the headline (device-resident, CUDA events
    around each pass), reported with its own roofline fraction — the north
    star asks the heap and sort-based queues to be reported the same way."""
    import torch
    from paper_2512_05906_b200.engine import Engine, poisson_drive_device
    from paper_2512_05906_b200 import workload as wl
    n, k, drange, _, T = wl.CONFIGS[cfg]
    key = (cfg, delays or drange)
    if key not in _NETS:
        _NETS.clear()
        _NETS[key] = wl.random_network(n, k, 0, delay_steps=delays or drange)
    net = _NETS[key]
    # drive generated on the device (same PoissonDrive statistics): no host masks at 1M neurons
    mask = poisson_drive_device(n, trials, T, 1e-3, 16e-3, 12e-3, 1000, device=local)
    eng = Engine(n, trials, T, kind=kind, capacity=capacity, precision=precision, device=local)
    eng.set_network(net.rowptr, net.col, net.weight, net.delay)
    eng.set_drive(mask, np.full(n, 12.0))
    stream = torch.cuda.current_stream()
    fw, bw = [], []
    for it in range(warmup + steps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        out = eng.forward()
        e[1].record(stream)
        eng.backward((2.0 * (out["v"] - 0.25)).to(eng.dtype), want_amp=False)
        e[2].record(stream)
        torch.cuda.synchronize()
        if it >= warmup:
            fw.append(e[0].elapsed_time(e[1]))
            bw.append(e[1].elapsed_time(e[2]))
    c = eng.counters()
    spikes, events, drops = int(c[:, 0].sum()), int(c[:, 1].sum()), int(c[:, 2].sum())
    ns = trials * T * n
    bounded = kind in ("fiforing", "binaryheap", "sortedarray")
    fb = alg_bytes(ns, spikes, events, "fwd", bounded, precision)
    bb = alg_bytes(ns, spikes, events, "bwd", False, precision)
    f, b = statistics.mean(fw), statistics.mean(bw)
    dom = (fwd_kernel(kind, 0), fb, f) if f >= b else ("k_backward", bb, b)
    ach = dom[1] / (dom[2] / 1e3) / 1e9
    del eng
    torch.cuda.empty_cache()
    return {"workload": label, "value": events / ((f + b) / 1e3), "unit": "events/s", "trials": trials,
            "dtype": "f32" if precision == 32 else "f64", "fwd_ms": f, "bwd_ms": b, "events": events,
            "drops": drops, "drop_fraction": drops / max(events, 1),
            "roofline": {"kernel": dom[0], "achieved": ach, "peak": peak, "frac": ach / peak,
                         "fwd_bwd_frac": (fb + bb) / ((f + b) / 1e3) / 1e9 / peak}}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2512_05906_b200.engine import Engine
    from paper_2512_05906_b200 import workload as wl

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} is running with WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    net, mask, amp, T = make_inputs(args.config, args.trials, rank, delay_steps=args.delays)
    B = args.trials
    if args.steps_per_pass:
        T = args.steps_per_pass
        mask = np.ascontiguousarray(mask[:, :T])
    eng = Engine(net.n, B, T, kind=args.kind, capacity=args.capacity, precision=args.precision, device=local,
                 staged_queues=QUEUE_IMPL[args.queue_impl])
    eng.set_network(net.rowptr, net.col, net.weight, net.delay)
    mask_dev = torch.from_numpy(mask.view(np.int32)).to(dev)
    amp_dev = torch.from_numpy(amp).to(dev, eng.dtype)
    eng.set_drive(mask_dev, amp_dev)
    stream = torch.cuda.current_stream(dev)

    def step(ev=None):
        """One bench step: forward + reverse (+ the gradient all-reduce).  Used
        for warm-up and timing alike, and every output dies at return, so the
        timed steps never allocate (an allocation between two kernels showed
        up as a 30-90 ms gap inside a timed step)."""
        if ev:
            ev[0].record(stream)
        out = eng.forward()
        if ev:
            ev[1].record(stream)
        vbar = (2.0 * (out["v"] - 0.25)).to(eng.dtype)
        gw, gd, _ = eng.backward(vbar, want_amp=False)
        if ev:
            ev[2].record(stream)
        if world > 1:
            dist.all_reduce(gw)
            dist.all_reduce(gd)

    # ---- device-resident timing, with per-kernel events
    clocks = ClockSampler(local).__enter__()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    counters = eng.counters()
    spikes = int(counters[:, 0].sum())
    events = int(counters[:, 1].sum())
    neuron_steps = B * T * net.n

    fwd_ms, bwd_ms = [], []
    launches0 = eng.launch_count
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    t_start.record(stream)
    for k in range(args.steps):
        step(evs[k])
        fwd_ms.append((evs[k][0], evs[k][1]))
        bwd_ms.append((evs[k][1], evs[k][2]))
    t_end.record(stream)
    torch.cuda.synchronize()
    clocks.mark_end()
    clocks.__exit__(None, None, None)
    launches = eng.launch_count - launches0
    total_ms = t_start.elapsed_time(t_end)
    fwd = [a.elapsed_time(b) for a, b in fwd_ms]
    bwd = [a.elapsed_time(b) for a, b in bwd_ms]
    if os.environ.get("EQ_BENCH_VERBOSE"):
        print("fwd ms", " ".join(f"{x:.1f}" for x in fwd), "| bwd ms", " ".join(f"{x:.1f}" for x in bwd),
              file=sys.stderr, flush=True)
    t = torch.tensor([total_ms], device=dev)
    ev = torch.tensor([float(events)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ev)
    ms_per_step = float(t.item()) / args.steps
    total_events = float(ev.item())
    value = total_events / (ms_per_step / 1e3)

    # ---- end to end through the public API, pipelined like a training loop:
    # step k's drive mask is copied from pinned host memory on a copy stream
    # while step k-1 computes, and step k's loss + gradients are read back to
    # pinned host memory while step k+1 computes.  Every copy of every step is
    # inside the timed region (events on the compute stream bracket it all).
    # the network as a training loop holds it: device-resident parameters,
    # handed to the engine every step (what RSNNFunction.forward does)
    net_dev = (torch.from_numpy(net.rowptr).to(dev), torch.from_numpy(net.col).to(dev),
               torch.from_numpy(net.weight).to(dev, eng.dtype), torch.from_numpy(net.delay).to(dev, eng.dtype))
    mask_host = torch.from_numpy(mask.view(np.int32)).pin_memory()
    md = [mask_dev, torch.empty_like(mask_dev)]
    gwf = [torch.empty(net.n_edges, dtype=torch.float32, device=dev) for _ in range(2)]
    gdf = [torch.empty_like(gwf[0]) for _ in range(2)]
    lossd = [torch.empty(1, dtype=torch.float64, device=dev) for _ in range(2)]
    gw_host = [torch.empty(net.n_edges, dtype=torch.float32).pin_memory() for _ in range(2)]
    gd_host = [torch.empty_like(gw_host[0]).pin_memory() for _ in range(2)]
    loss_host = [torch.empty(1, dtype=torch.float64).pin_memory() for _ in range(2)]
    cs = torch.cuda.Stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=False)   # noqa: E731

    def e2e_run(nsteps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        h2d, comp, d2h = [ev(), ev()], [ev(), ev()], [ev(), ev()]
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        cs.wait_event(t0)
        with torch.cuda.stream(cs):
            md[0].copy_(mask_host, non_blocking=True)
            h2d[0].record(cs)
        for k in range(nsteps):
            sl = k % 2
            if k + 1 < nsteps:                       # next step's input, once step k-1 released its buffer
                if k >= 1:
                    cs.wait_event(comp[1 - sl])
                with torch.cuda.stream(cs):
                    md[1 - sl].copy_(mask_host, non_blocking=True)
                    h2d[1 - sl].record(cs)
            stream.wait_event(h2d[sl])
            if k >= 2:
                stream.wait_event(d2h[sl])           # step k-2's read-back of these buffers is done
            eng.set_network(*net_dev)                 # validation + edge repack, as every training step does
            eng.set_drive(md[sl], amp_dev)
            out = eng.forward()
            lossd[sl].copy_(((out["v"].double() - 0.25) ** 2).sum().reshape(1))
            vbar = (2.0 * (out["v"] - 0.25)).to(eng.dtype)
            gw, gd, _ = eng.backward(vbar, want_amp=False)
            if world > 1:
                dist.all_reduce(gw)
                dist.all_reduce(gd)
            gwf[sl].copy_(gw)
            gdf[sl].copy_(gd)
            comp[sl].record(stream)
            cs.wait_event(comp[sl])
            with torch.cuda.stream(cs):
                gw_host[sl].copy_(gwf[sl], non_blocking=True)
                gd_host[sl].copy_(gdf[sl], non_blocking=True)
                loss_host[sl].copy_(lossd[sl], non_blocking=True)
                d2h[sl].record(cs)
            del out, vbar, gw, gd
        for e in d2h:
            stream.wait_event(e)
        t1.record(stream)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1)

    e2e_run(args.warmup)
    e2e_ms = [e2e_run(args.steps) / args.steps]
    e2e_t = torch.tensor([statistics.mean(e2e_ms)], device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = total_events / (float(e2e_t.item()) / 1e3)

    peaks, peak_kind = read_peaks()
    peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    fwd_avg, bwd_avg = statistics.mean(fwd), statistics.mean(bwd)
    bounded = args.kind in ("fiforing", "binaryheap", "sortedarray")
    fwd_bytes = alg_bytes(neuron_steps, spikes, events, "fwd", bounded, args.precision)
    bwd_bytes = alg_bytes(neuron_steps, spikes, events, "bwd", False, args.precision)
    fwd_name = fwd_kernel(args.kind, QUEUE_IMPL[args.queue_impl])
    dom = (fwd_name, fwd_bytes, fwd_avg) if fwd_avg >= bwd_avg else ("k_backward", bwd_bytes, bwd_avg)
    achieved = dom[1] / (dom[2] / 1e3) / 1e9
    # DRAM bytes per launch of that kernel from the committed ncu --set full capture of this workload
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", TRAFFIC_FILE)) as f:
            tr = json.load(f)
        if (args.config == "C3" and B == tr.get("trials") and args.kind == "ring" and args.precision == 32
                and T == 1000 and args.delays is None):
            traffic = tr.get(dom[0])
    except Exception:
        traffic = None

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    variants = None
    if world == 1 and not args.no_variants:
        variants = []
        for v in VARIANTS:
            try:
                variants.append(measure_variant(*v, steps=min(args.steps, 3), warmup=3, local=local, peak=peak))
            except Exception as exc:  # a variant must not sink the headline line
                variants.append({"workload": v[0], "error": str(exc)})
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            v, info = cpu_reference_sample(net, mask, amp, T, max_trials=args.cpu_trials, steps=args.cpu_steps,
                                           kind=args.kind, capacity=args.capacity)
            cpu = {"value": v, "unit": "events/s", "cores": info["cores"], "kind": "port", "host": host_label(),
                   "sample": f"{info['trials']} trials x {info['steps']} steps of {args.config}, "
                             f"fwd+bwd, OpenMP over trials ({info['seconds']:.1f} s)"}
        except Exception as exc:  # the checker must not sink the bench line
            cpu = {"value": None, "unit": "events/s", "cores": None, "kind": "port", "sample": f"failed: {exc}"}
    line = {
        "metric": "synaptic events/sec (fwd+bwd)",
        "value": value,
        "unit": "events/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32" if args.precision == 32 else "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {net.n} LIF neurons, {net.n_edges // net.n} syn/neuron, "
                               f"delay {int(round(net.delay.min() / 1e-3))}..{int(round(net.delay.max() / 1e-3))} "
                               f"steps, {args.kind}" + (f"[{args.capacity}]" if args.capacity else "") +
                               f", fwd+bwd T={T}",
                   "queue_kind": args.kind, "capacity": args.capacity or None,
                   "drops_per_gpu": int(counters[:, 2].sum()),
                   "trials_per_gpu": B, "global_trials": B * world, "neurons": net.n, "steps_per_pass": T,
                   "spikes_per_gpu": spikes, "events_per_gpu": events,
                   "neuron_steps_per_sec": neuron_steps * world / (ms_per_step / 1e3),
                   "l2": "inputs larger than L2 (queue storage %.2f GB/GPU)" % (B * (eng.horizon + 1) * net.n * 8 / 1e9),
                   "parallelism": f"trial-dp{world}"},
        "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": achieved, "peak": peak,
                     "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": "profiles/" + TRAFFIC_FILE if traffic else None,
                     "alg_bytes_per_launch": dom[1], "avg_launch_ms": dom[2],
                     "fwd_ms": fwd_avg, "bwd_ms": bwd_avg,
                     # the north-star target is stated for forward + reverse together
                     "fwd_bwd": {"alg_bytes": fwd_bytes + bwd_bytes, "ms": fwd_avg + bwd_avg,
                                 "achieved": (fwd_bytes + bwd_bytes) / ((fwd_avg + bwd_avg) / 1e3) / 1e9,
                                 "frac": (fwd_bytes + bwd_bytes) / ((fwd_avg + bwd_avg) / 1e3) / 1e9 / peak}},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "events/s", "h2d_bytes_per_step": int(mask.nbytes),
                "d2h_bytes_per_step": int(2 * 4 * net.n_edges + 8)},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "variants": variants,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--trials", type=int, default=24)   # trials per GPU: 24 measured best of 8..48 (DESIGN 6.1)
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--cpu-trials", type=int, default=0)
    ap.add_argument("--cpu-steps", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the C3-fp64 / C4-heap / C4-sorted lines")
    ap.add_argument("--steps-per-pass", type=int, default=0, help="override T (debug)")
    ap.add_argument("--kind", default="ring", choices=["ring", "fiforing", "binaryheap", "sortedarray", "donothing"])
    ap.add_argument("--capacity", type=int, default=0, help="bounded kinds: events per queue")
    ap.add_argument("--queue-impl", choices=sorted(QUEUE_IMPL), default="admission",
                    help="bounded kinds: heap/sorted by admission on the calendar (default), the "
                         "shared-memory staged queues (smem) or the HBM-resident queue structures (hbm)")
    ap.add_argument("--delays", type=lambda s: tuple(int(x) for x in s.split(",")), default=None,
                    help="delay range in steps lo,hi (FIFO needs lo == hi)")
    ap.add_argument("--launch-selftest", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and (args.impl == "ours" or args.launch_selftest):
        relaunch_under_torchrun(args)
    if args.launch_selftest:
        launch_selftest(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
