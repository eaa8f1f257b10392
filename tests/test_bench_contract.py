"""bench.py contract on the CPU: the reference arm (the oracle on a bounded C4 sample) prints one JSON
line with the keys the driver reads, and the product arm refuses to run without a GPU (no CPU
fallback)."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=300):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout)


def test_reference_arm_json_line():
    r = _run("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["unit"] == "pair-collisions/s" and d["higher_is_better"] is True
    assert d["steps"] == 1 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["dtype"] == "f64" and d["data"] == "synthetic" and d["vs_baseline"] is None
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == d["value"] and cb["cores"] >= 1 and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU refusal")
def test_product_arm_refuses_without_gpu():
    r = _run("--steps", "1", "--warmup", "3", timeout=120)
    assert r.returncode != 0
    assert "no CUDA device" in r.stderr
    assert not r.stdout.strip()


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_bench_two_ranks_one_line():
    """bench.py's N > 1 path end to end (the driver's scaling run launches it with torchrun): two ranks
    share the one GPU over gloo (NCCL refuses two ranks on one device), a small C5 grid; rank 0 alone
    prints ONE JSON line with the max-over-ranks time, the reduced diagnostics' pair count of BOTH
    shards and the migration status (nothing dropped)."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29547", os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "3", "--warmup", "3", "--nx", "16", "--ny", "16",
                        "--per-cell", "5000", "--dist-backend", "gloo", "--e2e-steps", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["steps"] == 3
    n_per_rank = 16 * 16 * 5000
    assert abs(d["config"]["pairs_per_step"] - n_per_rank) <= 0.01 * n_per_rank   # ~n/2 pairs on each of 2 ranks
    mg = d["multi_gpu"]["migration"]
    assert mg["status"][:3] == [0, 0, 0] and mg["status"][3] > 0                  # particles crossed shards
    assert d["value"] > 0 and d["gpu_launches"] > 0
