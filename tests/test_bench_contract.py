"""bench.py JSON-line contract: the reference arm (CPU oracle, runs here) and our arm (GPU) on the small C1
config print one JSON line with the keys the driver reads."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, "bench.py"] + args, cwd=ROOT, capture_output=True, text=True,
                         timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_c1():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "3", "--warmup", "1", "--cpu-threads", "2"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "modes/s" and d["higher_is_better"]
    assert d["steps"] == 3 and d["warmup"] == 1 and d["ms_per_step"] > 0
    assert d["config"]["workload"].startswith("c1: d=2 N=64 k=4")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 2 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "modes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_c1():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--config", "c1", "--steps", "3", "--warmup", "3", "--e2e-steps", "2", "--latency-steps", "2",
              "--no-cpu-baseline"])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["verified_exact_recovery"] is True
    assert d["config"]["workload"].startswith("c1: d=2 N=64 k=4")
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r) and r["peak"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["latency_single_solve"]["exact"] is True


@pytest.mark.gpu
def test_our_arm_line_shards_c3_world1():
    """--shard lines at one rank: the plan is a line shard with the NCCL record all-gather (world 1)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--config", "c3", "--shard", "lines", "--steps", "2", "--warmup", "3", "--e2e-steps", "1",
              "--latency-steps", "0", "--no-cpu-baseline", "--batch", "4"])
    assert d["scaling"] == "strong" and d["verified_exact_recovery"] is True
    assert "line shards x1" in d["config"]["parallelism"]
    d = _run(["--config", "c3", "--shard", "lines", "--exchange", "fused", "--steps", "2", "--warmup", "3",
              "--e2e-steps", "1", "--latency-steps", "0", "--no-cpu-baseline", "--batch", "4", "--fp64-steps", "0"])
    assert d["verified_exact_recovery"] is True and "CUDA IPC" in d["config"]["parallelism"]


def test_self_launch_dry_run_world2():
    """`python bench.py --gpus 2` without torchrun re-executes itself under torch.distributed.run with two ranks
    (here on gloo with a fake solve, --dry-run): one JSON line from rank 0, n_gpus = 2, the time the max over
    ranks (rank r fakes 1 + r ms per step)."""
    d = _run(["--dry-run", "--gpus", "2", "--steps", "3", "--warmup", "1"], timeout=300)
    assert d["n_gpus"] == 2 and d["dry_run"] is True and d["verified_exact_recovery"] is True
    assert abs(d["ms_per_step"] - 2.0) < 1e-9
