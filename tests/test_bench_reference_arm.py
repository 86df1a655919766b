"""bench.py's host-side contract on CPU: `--impl reference` prints one JSON line
from rank 0 with impl/cpu_baseline/e2e and the same `config` dict as our arm,
its value anchored to one complete step of the same solves; `--gpus N` outside
torchrun re-launches itself with N ranks; the sharded leg's plumbing (owner
map agreement, all-gather, max-over-ranks timing) runs on 2 gloo ranks
(a small C3 grid so everything runs in seconds)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _one_line(out):
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:] + out.stderr[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--nodes", "16",
                          "--steps", "2", "--warmup", "1", "--ref-sample-iters", "4"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    d = _one_line(out)
    assert d["impl"] == "reference" and d["unit"] == "solves/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    cpu = d["cpu_baseline"]
    assert cpu["kind"] == "port" and cpu["cores"] >= 1
    assert abs(cpu["value"] - d["value"]) < 1e-6
    assert d["e2e"] == {"value": d["value"], "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # the anchor is a complete step: every solve converged to the arm's tolerance
    anc = cpu["anchor"]
    assert anc["solves"] == 16 and anc["max_rel_residual"] <= 1e-8 and min(anc["iterations"]) > 4
    assert "complete step" in cpu["sample"] and "median of 2 timed steps" in cpu["sample"]
    # the driver's consistency check: ms_per_step x steps is real time spent
    assert d["ms_per_step"] < anc["complete_step_s"] * 1e3
    import argparse
    import bench
    args = argparse.Namespace(nodes=16, r=8, tol=1e-8, max_iter=1000)
    assert d["config"] == json.loads(json.dumps(bench.workload_config(args, 1)))  # identical to our arm's dict


def test_reference_arm_maps_only_oracle_libraries():
    code = ("import sys, argparse; sys.path.insert(0, %r); import bench;"
            "a = argparse.Namespace(nodes=8, r=8, tol=1e-8, max_iter=1000, cpu_iters=2);"
            "bench._ref_setup(a, 1);"
            "maps = open('/proc/self/maps').read();"
            "print('LIBMPG' if 'libmpg' in maps else 'CLEAN')" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip().endswith("CLEAN")


def test_reference_arm_under_torchrun_prints_one_line():
    """N = 2 launch (gloo on CPU): rank 0 alone runs and prints; rank 1 exits 0 without work."""
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29571", os.path.join(ROOT, "bench.py"),
                          "--impl", "reference", "--gpus", "2", "--nodes", "12", "--steps", "1", "--warmup", "1",
                          "--ref-sample-iters", "3"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = _one_line(out)
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["solves_per_step"] == 32 and len(d["config"]["shifts"]) == 16


def test_gpus_flag_self_launches_and_plans_the_sharded_leg():
    """`bench.py --gpus 2` without WORLD_SIZE starts 2 ranks itself; --plan-only
    rehearses the sharded C4 leg's host plumbing on gloo."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plan-only"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    d = _one_line(out)
    assert d["plan_only"] and d["n_gpus"] == 2 and d["ranks_agree"]
    assert d["units_per_rank"] == [16, 16]
    assert d["allgather_rc"] == 0 and d["allgather_heads"] == [0.0, 1.0]


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plan-only"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode == 2 and "WORLD_SIZE=1" in out.stdout
