"""`bench.py --impl reference` keeps the driver's contract on CPU: one JSON line
from rank 0 with impl/cpu_baseline/e2e, the same workload string as our arm,
and exit 0 (a small C3 grid so it runs in seconds)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--nodes", "16",
                          "--steps", "2", "--warmup", "1", "--ref-iters", "30", "--cpu-iters", "12"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "solves/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] or abs(d["cpu_baseline"]["value"] - d["value"]) < 1e-6
    assert d["e2e"] == {"value": d["value"], "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C3 FEM Q1 16^3 nodes (n=4096), r=8")
    assert "median of 2 timed samples" in d["cpu_baseline"]["sample"]


def test_reference_arm_under_torchrun_prints_one_line():
    """N = 2 launch (gloo on CPU): rank 0 alone runs and prints; rank 1 exits 0 without work."""
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29571", os.path.join(ROOT, "bench.py"),
                          "--impl", "reference", "--gpus", "2", "--nodes", "12", "--steps", "1", "--warmup", "1",
                          "--ref-iters", "20", "--cpu-iters", "10"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
