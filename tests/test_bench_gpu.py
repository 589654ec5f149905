"""bench.py keeps the driver's contract: one JSON line with the required keys, on 1 rank and
(functionally, both ranks on the one GPU with gloo for the host-side exchanges) on 2 ranks."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "clocks", "roofline"]


def last_json(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def test_bench_one_rank():
    p = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
                        "--no-sweep"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    d = last_json(p.stdout)
    for k in REQUIRED:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert set(d["roofline"]) >= {"bound", "achieved", "peak", "unit", "frac", "traffic"}
    assert d["config"]["population"] == 65536


def test_bench_two_ranks_functional():
    env = dict(os.environ, FFSGA_DIST_BACKEND="gloo", FFSGA_BENCH_DEVICE="0")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2",
                        "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-sweep"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    d = last_json(p.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["islands_per_rank"] == 4


def test_reference_arm_line_and_same_trajectory():
    """Both arms run warm-up + steps generations of the same 8 islands from the same seeds: the
    per-island best objectives they print are identical (the timed config is the pinned one), and
    the reference arm loads nothing of the product package."""
    code = ("import sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '2']; "
            "import bench; bench.main(); "
            "bad = [m for m in sys.modules if m.startswith('paper_1903_10722_b200')]; "
            "assert not bad, bad")
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    r = last_json(p.stdout)
    assert r["impl"] == "reference" and r["value"] > 0
    assert r["e2e"]["h2d_bytes_per_step"] == 0 and r["cpu_baseline"]["kind"] == "reference"
    assert r["cpu_baseline"]["cpu_model"] and r["cpu_baseline"]["nproc"] >= 1
    p = subprocess.run([sys.executable, "bench.py", "--steps", "1", "--warmup", "2", "--no-cpu-baseline",
                        "--no-sweep"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    d = last_json(p.stdout)
    assert d["generations_done"] == r["generations_done"] == 3
    assert d["island_best_objectives"] == r["island_best_objectives"]
