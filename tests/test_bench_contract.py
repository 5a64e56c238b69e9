"""bench.py's reference arm (``--impl reference``): the JSON line the driver
parses, on CPU.  The arm is host-only (the oracle private MLP step), so it
runs here; one bounded step keeps the test under a minute.  Our own arm
(GPU) is checked by the gpu-marked test at the end."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(cmd, env=None):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    return [json.loads(x) for x in r.stdout.strip().splitlines() if x.startswith("{")]


def _check_line(d, world):
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["impl"] == "reference"
    assert d["n_gpus"] == world and d["higher_is_better"] is True and d["value"] > 0
    assert d["warmup"] >= 3 and d["steps"] >= 1
    assert abs(d["value"] - 64 / (d["ms_per_step"] / 1e3)) < 1e-6 * d["value"]
    assert isinstance(d["config"], dict) and "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["unit"] == d["unit"] and cb["kind"] == "port" and cb["cores"] >= 1
    assert cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_reference_arm_json_line():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    lines = _run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"], env)
    assert len(lines) == 1
    _check_line(lines[0], 1)
    assert lines[0]["config"]["parallelism"] == "single GPU"


def test_reference_arm_under_torchrun_world2():
    """Rank 0 alone runs and prints; the other rank exits 0 without work, and
    no device is touched (gloo)."""
    lines = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                  "--master-addr", "127.0.0.1", "--master-port", "29561", "bench.py", "--impl", "reference",
                  "--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert len(lines) == 1
    _check_line(lines[0], 2)
    assert lines[0]["config"]["global_batch"] == 128


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """Our arm at N=1, headline only: every key of the contract, the roofline
    and e2e objects, clocks, a positive launch count."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    lines = _run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-configs"], env)
    d = lines[-1]
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert abs(d["value"] - 64 / (d["ms_per_step"] / 1e3)) < 1e-6 * d["value"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] < 1 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
