"""bench.py as the driver calls it: `python bench.py --gpus N` must start N
ranks itself (torch.distributed.run) when it is not already under torchrun,
and the algorithmic byte model must reduce to SURVEY §8(d)'s fp32 figures."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_gpus_2_relaunches_two_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-selftest"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line == {"n_gpus": 2, "rank_sum": 1.0}


def test_byte_model_matches_survey_fp32_and_scales_fp64():
    import bench
    m = bench.byte_model(32)
    assert m["fwd"] == (36, 16, 28) and m["bwd"] == (24, 16, 36)
    assert bench.byte_model(32, bounded=True)["fwd"] == (36, 16, 36)
    m64 = bench.byte_model(64)
    assert m64["fwd"] == (68, 28, 52) and m64["bwd"] == (48, 28, 68)
    # 60 B per neuron-step, 32 B per spike, 64 B per event over both passes (fp32)
    assert bench.alg_bytes(1, 0, 0, "fwd") + bench.alg_bytes(1, 0, 0, "bwd") == 60
    assert bench.alg_bytes(0, 1, 0, "fwd") + bench.alg_bytes(0, 1, 0, "bwd") == 32
    assert bench.alg_bytes(0, 0, 1, "fwd") + bench.alg_bytes(0, 0, 1, "bwd") == 64
