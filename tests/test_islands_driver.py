"""The island driver's host logic on CPU: policy, seeds, ownership, and the multi-rank protocol
(gloo, world_size 2) against single-process runs and the reference drive() semantics."""
import os
import socket

import numpy as np
import pytest

from paper_1903_10722_b200 import islands as isl


def test_policy_matches_oracle(orc):
    import ctypes as C
    rng = np.random.default_rng(1)
    for _ in range(2000):
        fa, fb = (float(x) for x in rng.uniform(0, 1e6, 2))
        if rng.random() < 0.1:
            fb = fa
        theta = float(rng.choice([0.0, 0.01, 0.5, 1.0]))
        n = int(rng.integers(1, 10000))
        b, a, d, k = C.c_double(), C.c_double(), C.c_int(), C.c_int()
        orc.lib.orc_decide(fa, fb, theta, n, C.byref(b), C.byref(a), C.byref(d), C.byref(k))
        beta, alpha, direction, migrants = isl.decide(fa, fb, theta, n)
        assert (beta, alpha, migrants) == (b.value, a.value, k.value)
        assert direction == {0: "none", 1: "a_to_b", 2: "b_to_a"}[d.value]


def test_seeds_and_shapes(orc):
    for base in (0, 1, 7, 2**63 + 5):
        for key in range(5):
            assert isl.derive_seed(base, key) == orc.derive_seed(base, key)
    assert isl.grid_shape_for(8192) == (128, 64)
    assert isl.grid_shape_for(2048) == (64, 32)
    with pytest.raises(ValueError):
        isl.grid_shape_for(7)


def test_owner_keeps_couples_together():
    for world in (1, 2, 4):
        owners = [isl.owner(i, 8, world) for i in range(8)]
        assert all(owners[2 * c] == owners[2 * c + 1] for c in range(4))
        assert sorted(set(owners)) == list(range(world))
    assert [isl.owner(i, 8, 8) for i in range(8)] == list(range(8))


def _data(orc, weight=0.0, seed=4):
    return orc.generate(8, 2, [2, 2], weight=weight, seed=seed)


def test_single_couple_equals_reference_drive(orc):
    import oracle_backend as ob
    for seed in range(1, 8):
        d = _data(orc, seed=seed)
        oi = orc.instance(d)
        emax = oi.estimate_emax()
        cfg = isl.IslandConfig(couples=1, island_population=32, generations=20, migration_gap=2, seed=seed)
        res = isl.IslandModel(d, emax, cfg, backend=ob).run()
        want = oi.run(population=64, generations=20, gap=2, seed=seed)
        assert list(res.trace_combined) == want["trace_combined"]
        assert list(res.traces[0]) == want["trace_island_a"] and list(res.traces[1]) == want["trace_island_b"]
        assert list(res.best_chromosome) == want["best_chromosome"]
        assert res.best_report["objective"] == want["best_objective"]
        assert [(e.generation, e.beta, e.alpha, e.direction, e.migrants) for e in res.migrations] == \
               [(m["generation"], m["beta"], m["alpha"], m["direction"], m["migrants"]) for m in want["migrations"]]


@pytest.mark.parametrize("mode", ["cellular", "pseudo"])
def test_single_island_modes(orc, mode):
    import oracle_backend as ob
    d = _data(orc, weight=100.0, seed=43)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    cfg = isl.IslandConfig(couples=1, island_population=16, generations=12, seed=4, mode=mode)
    res = isl.IslandModel(d, emax, cfg, backend=ob).run()
    want = oi.run(population=16, generations=12, seed=4, mode=mode)
    assert list(res.trace_combined) == want["trace_combined"]
    assert list(res.best_chromosome) == want["best_chromosome"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, couples, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle_backend as ob
        from pyoracle import Oracle
        orc = Oracle()
        d = orc.generate(8, 2, [2, 2], weight=0.0, seed=12)
        emax = orc.instance(d).estimate_emax()
        cfg = isl.IslandConfig(couples=couples, island_population=32, generations=24, migration_gap=3, seed=12)
        res = isl.IslandModel(d, emax, cfg, comm=isl.TorchComm(), backend=ob).run()
        q.put((rank, res.traces.tolist(), list(res.best_chromosome), res.best_report["objective"],
               [(e.generation, e.couple, e.direction, e.migrants) for e in res.migrations]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,couples", [(2, 1), (2, 2), (3, 1)])
def test_two_ranks_gloo_match_one_process(orc, world, couples):
    """couples=1: the couple is split over 2 ranks (migrant rows cross ranks);
    couples=2: one couple per rank (device-local migration); world 3 > 2 islands: one rank owns
    no island and still takes part in every exchange."""
    import multiprocessing as mp
    import oracle_backend as ob
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, couples, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    d = orc.generate(8, 2, [2, 2], weight=0.0, seed=12)
    emax = orc.instance(d).estimate_emax()
    cfg = isl.IslandConfig(couples=couples, island_population=32, generations=24, migration_gap=3, seed=12)
    single = isl.IslandModel(d, emax, cfg, backend=ob).run()
    assert len(single.migrations) > 0, "the test instance must exercise migration"
    for rank, traces, chrom, obj, migs in out:
        assert traces == single.traces.tolist()
        assert chrom == list(single.best_chromosome) and obj == single.best_report["objective"]
        assert migs == [(e.generation, e.couple, e.direction, e.migrants) for e in single.migrations]
