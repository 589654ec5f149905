"""bench.py host-side contract pieces that need no GPU."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_imports_no_product_code():
    """--impl reference runs the reference (oracle/_ref) only: the product package never loads."""
    from pyoracle import have_ref
    code = ("import sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'decoder', "
            "'--steps', '1', '--warmup', '0']; import bench; bench.main(); "
            "bad = [m for m in sys.modules if m.startswith('paper_1903_10722_b200') or m == 'torch']; "
            "assert not bad, bad")
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    line = [l for l in p.stdout.splitlines() if l.startswith("{")][-1]
    if have_ref():
        assert '"impl": "reference"' in line and '"cpu_model"' in line


def test_bench_machines_match_oracle_convention():
    import bench
    from pyoracle import synthetic_machines
    for J, S in ((500, 20), (1000, 20), (100, 10), (20, 5)):
        assert bench.synthetic_machines(J, S) == synthetic_machines(J, S)
    assert bench.synthetic_machines(500, 20) == [5, 2, 2, 8, 4, 7, 6, 5, 7, 8, 3, 8, 3, 6, 3, 5, 5, 2, 5, 2]
