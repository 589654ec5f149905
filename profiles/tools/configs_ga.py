"""GA throughput of the BASELINE configs C1-C4 on one GPU: device time in timing mode (no graph
replay) and wall clock with timing off (graph replay for launch-bound islands).

    python profiles/tools/configs_ga.py      (ONLY_SMALL=1: C1 and C2 only)
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
if os.environ.get("FFSGA_PKG_ROOT"):
    sys.path.insert(0, os.environ["FFSGA_PKG_ROOT"])
import paper_1903_10722_b200  # noqa: F401
print(paper_1903_10722_b200.__file__)
import bench
from paper_1903_10722_b200 import instance_arrays, generate_instance, estimate_emax
from paper_1903_10722_b200.islands import IslandConfig, IslandModel


def run(name, J, S, machines, couples, pop, mode, grid, steps):
    inst = generate_instance(jobs=J, stages=S, machines=machines, weight=100.0, seed=7)
    emax = estimate_emax(inst)
    cfg = IslandConfig(couples=couples, island_population=pop, generations=steps, migration_gap=500, theta=1.0,
                       seed=1, grid_shape=grid, mode=mode)
    m = IslandModel(instance_arrays(inst), emax, cfg, None, device=0)
    m.advance(3)
    m.inst.set_timing(True)
    m.inst.reset_timing()
    ev0 = m.inst.evaluations()
    m.advance(steps)
    ms = m.inst.last_step_ms()
    ev = m.inst.evaluations() - ev0
    m.inst.set_timing(False)
    import time
    m.advance(steps)  # graphs (timing off): warm the captured chunk
    t0 = time.perf_counter()
    m.advance(steps)
    wall = time.perf_counter() - t0
    print(f"{name}: {steps / (ms / 1e3):.1f} gen/s timed  ({ms / steps:.3f} ms/gen, {ev / (ms / 1e3) / 1e6:.2f} M evals/s); "
          f"untimed wall {steps / wall:.1f} gen/s")


if os.environ.get("ONLY_C4"):
    run("C4 1000x20x[2,8], 32 couples x 1024", 1000, 20, bench.synthetic_machines(1000, 20), 32, 1024, "dual", (32, 32), 10)
    sys.exit(0)
run("C1 20x5x3, 1 cellular 16x16", 20, 5, [3] * 5, 1, 256, "cellular", (16, 16), 2000)
run("C2 100x10x[2,5], dual 2048+2048", 100, 10, bench.synthetic_machines(100, 10, 2, 5), 1, 2048, "dual", (64, 32), 500)
if os.environ.get("ONLY_SMALL"):
    sys.exit(0)
run("C3 500x20x[2,8], 4 couples x 8192", 500, 20, bench.synthetic_machines(500, 20), 4, 8192, "dual", (128, 64), 20)
run("C4 1000x20x[2,8], 32 couples x 1024", 1000, 20, bench.synthetic_machines(1000, 20), 32, 1024, "dual", (32, 32), 10)
