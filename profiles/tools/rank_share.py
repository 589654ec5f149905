"""Per-rank share of the C3 GA step timed alone on one GPU: the islands rank RANK of a WORLD-rank
job owns (bench.py's island placement), advanced in timing mode, device time.

    python profiles/tools/rank_share.py WORLD RANK [steps]

A proxy for the multi-GPU bench (no collectives run; the driver's N-GPU run is authoritative).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1903_10722_b200 import instance_arrays  # noqa: E402
from paper_1903_10722_b200.islands import IslandConfig, IslandModel  # noqa: E402


class RankView:
    def __init__(self, world, rank):
        self.world, self.rank = world, rank


def main():
    world, rank = int(sys.argv[1]), int(sys.argv[2])
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    inst, emax = bench.make_instance()
    cfg = IslandConfig(couples=bench.COUPLES, island_population=bench.ISLAND_POP, generations=steps,
                       migration_gap=bench.GAP, theta=bench.THETA, seed=bench.RUN_SEED, grid_shape=bench.GRID)
    model = IslandModel(instance_arrays(inst), emax, cfg, RankView(world, rank), device=0)
    model.advance(3)
    model.inst.set_timing(True)
    model.inst.reset_timing()
    ev0 = model.inst.evaluations()
    model.advance(steps)
    ms = model.inst.last_step_ms()
    ev = model.inst.evaluations() - ev0
    e_ms, _ = model.inst.timing(0)
    b_ms, _ = model.inst.timing(1)
    print(f"world={world} rank={rank} islands={sorted(model.local)}: {steps / (ms / 1e3):.1f} gen/s  "
          f"{ms / steps:.3f} ms/gen  evals/gen={ev / steps:.0f}  decode={e_ms / steps:.3f} "
          f"breed={b_ms / steps:.3f} ms/gen (per-stream sums)")


if __name__ == "__main__":
    main()
