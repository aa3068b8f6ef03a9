"""CPU: the bench.py driver contract that does not need a GPU.

- `--impl reference` prints one JSON line with the contract keys, the
  reference arm's own `cpu_baseline` and a zero-byte `e2e`;
- our arm fails loudly without a CUDA device (no CPU fallback);
- under torchrun (N=2) only rank 0 runs and prints the reference arm;
- `plan_depths` splits a solve into fused passes of at most t sweeps."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _run(*extra, timeout=600):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *extra],
                          capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)


def test_reference_arm_json_line():
    r = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-sweeps-per-step", "1")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["unit"] == "GLUP/s" and d["higher_is_better"] is True
    assert d["dtype"] == "f64" and d["steps"] == 1 and d["n_gpus"] == 1
    assert d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["value"] == d["value"] and cb["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "GLUP/s",
                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # same workload dict as our arm's N=1 line (BASELINE configs[1], C2)
    assert d["config"] == bench.workload(1, False) and d["config"]["workload"].startswith("C2")
    assert d["config"]["sweeps_per_step"] == 100
    assert {"cpu_model", "os_cpu_count", "sched_getaffinity"} <= set(cb["host"])


def test_workload_configs_name_baseline_configs():
    w1, w2, w8 = bench.workload(1, False), bench.workload(2, True), bench.workload(8, True)
    assert w1["grid"] == [512, 512, 512] and w1["sweeps_per_step"] == 100
    assert w2["grid"] == [1024, 1024, 2048] and w8["grid"] == [1024, 1024, 8192]
    assert w8["sweeps_per_step"] == 40 and w8["parallelism"] == "z-slab x8"
    assert bench.C5["n"] == (2048, 2048, 2048) and bench.C5["ts"] == (1, 4, 8)


def test_our_arm_fails_without_gpu():
    r = _run("--steps", "1", "--warmup", "3", "--quick", "--no-cpu")
    assert r.returncode != 0
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]


@pytest.mark.parametrize("total,t", [(100, 4), (100, 3), (7, 4), (1, 4), (64, 1), (10, 8)])
def test_plan_depths(total, t):
    p = bench.plan_depths(total, t)
    assert sum(p) == total
    assert all(1 <= d <= t for d in p)
    assert len(p) == -(-total // t)
    assert max(p) - min(p) <= 1


def test_reference_arm_under_torchrun_prints_once():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29533", os.path.join(ROOT, "bench.py"),
                        "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                        "--ref-sweeps-per-step", "1"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    # N>1 measures BASELINE configs[3] (C4 weak scaling), the same config dict
    # our arm prints, with the reference arm's own cpu_baseline and e2e
    assert d["config"] == bench.workload(2, True)
    assert d["config"]["workload"].startswith("C4") and d["config"]["grid"] == [1024, 1024, 2048]
    assert d["cpu_baseline"]["kind"] == "port" and d["e2e"]["value"] == d["value"]
    # torchrun exports OMP_NUM_THREADS=1; the reference arm still uses every host core
    assert d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))
