"""Reference-facing API on the GPU: the pybind module (reference Python API), whole runs through
the C++ drive() mirror, and the multi-island driver -- all bit-exact against the oracle."""
import numpy as np
import pytest

import paper_1903_10722_b200 as ffsga
from paper_1903_10722_b200 import capi, instance_arrays
from paper_1903_10722_b200 import islands as isl

pytestmark = pytest.mark.gpu


def as_data(inst):
    from pyoracle import InstanceData
    a = instance_arrays(inst)
    return InstanceData(a.num_jobs, a.num_stages, a.machines, a.proc, a.release, a.due, a.weight)


@pytest.fixture(scope="module")
def instance():
    return ffsga.generate_instance(jobs=6, stages=2, machines=[2], seed=5)


def test_evaluate_assignment(orc, instance):  # test_smoke.py:56-71
    emax = ffsga.estimate_emax(instance)
    rep = ffsga.evaluate_assignment(instance, [0] * instance.num_genes)
    want = orc.instance(as_data(instance)).score([0] * 12, emax)
    assert rep == want
    with pytest.raises(ValueError):
        ffsga.evaluate_assignment(instance, [2] * instance.num_genes)
    with pytest.raises(ValueError):
        ffsga.evaluate_assignment(instance, [0] * (instance.num_genes - 1))


def test_evaluate_batch(orc):
    inst = ffsga.generate_instance(jobs=100, stages=10, machines=[4, 2, 2, 3, 4, 4, 2, 3, 4, 5], seed=7)
    oi = orc.instance(as_data(inst))
    pop = oi.random_population(99, 0, 500)
    obj, fit = ffsga.evaluate_batch(inst, pop)
    eo, ef, _, _ = oi.score_batch(pop, oi.estimate_emax())
    assert np.array_equal(obj, eo) and np.array_equal(fit, ef)


@pytest.mark.parametrize("mode", ["dual", "cellular", "pseudo"])
def test_solve_matches_oracle(orc, instance, mode):
    got = ffsga.solve(instance, population=16, generations=12, gap=4, seed=3, mode=mode)
    want = orc.instance(as_data(instance)).run(population=16, generations=12, gap=4, seed=3, mode=mode)
    for k, v in want.items():
        assert got[k] == v, k


def test_solve_reproducible(instance):  # test_smoke.py:89-114
    first = ffsga.solve(instance, population=16, generations=12, gap=4, seed=3)
    for other in (ffsga.solve(instance, population=16, generations=12, gap=4, seed=3, workers=4),
                  ffsga.solve(instance, population=16, generations=12, gap=4, seed=3, serialized=True)):
        for k in ("best_objective", "best_chromosome", "trace_combined", "trace_island_a", "trace_island_b",
                  "migrations"):
            assert first[k] == other[k]
    assert first["timings"]["workers"] == 1
    assert ffsga.evaluate_assignment(instance, first["best_chromosome"])["objective"] == first["best_objective"]
    with pytest.raises(ValueError):
        ffsga.solve(instance, mode="unknown")


def test_solve_with_migrations(orc):
    fired = 0
    for seed in range(1, 25):
        inst = ffsga.generate_instance(jobs=8, stages=2, machines=[2, 2], weight=0.0, seed=seed)
        got = ffsga.solve(inst, population=64, generations=30, gap=1, seed=seed)
        want = orc.instance(as_data(inst)).run(population=64, generations=30, gap=1, seed=seed)
        for k, v in want.items():
            assert got[k] == v, (seed, k)
        fired += bool(want["migrations"])
    assert fired >= 3


def test_c2_config_parity(orc):
    """C2: 100x10, M in [2,5], dual, pop 4096, a short budget with one rendezvous."""
    from pyoracle import synthetic_machines
    m = synthetic_machines(100, 10, 2, 5)
    inst = ffsga.generate_instance(jobs=100, stages=10, machines=m, seed=7)
    got = ffsga.solve(inst, population=4096, generations=6, gap=3, seed=1)
    want = orc.instance(as_data(inst)).run(population=4096, generations=6, gap=3, seed=1)
    for k, v in want.items():
        assert got[k] == v, k


def test_island_model_one_couple_equals_drive(orc):
    inst = ffsga.generate_instance(jobs=8, stages=2, machines=[2, 2], weight=0.0, seed=4)
    d = as_data(inst)
    emax = ffsga.estimate_emax(inst)
    cfg = isl.IslandConfig(couples=1, island_population=32, generations=20, migration_gap=2, seed=4)
    res = isl.IslandModel(d, emax, cfg).run()
    want = orc.instance(d).run(population=64, generations=20, gap=2, seed=4)
    assert list(res.trace_combined) == want["trace_combined"]
    assert list(res.best_chromosome) == want["best_chromosome"]
    assert res.best_report["objective"] == want["best_objective"]
    assert len(res.migrations) == len(want["migrations"])


def test_island_model_multi_couple_matches_oracle_backend(orc):
    import oracle_backend as ob
    inst = ffsga.generate_instance(jobs=12, stages=3, machines=[2, 3, 2], weight=0.0, seed=9)
    d = as_data(inst)
    emax = ffsga.estimate_emax(inst)
    cfg = isl.IslandConfig(couples=3, island_population=24, generations=18, migration_gap=3, seed=9)
    dev = isl.IslandModel(d, emax, cfg).run()
    cpu = isl.IslandModel(d, emax, cfg, backend=ob).run()
    assert np.array_equal(dev.traces, cpu.traces)
    assert list(dev.best_chromosome) == list(cpu.best_chromosome)
    assert [(e.generation, e.couple, e.migrants) for e in dev.migrations] == \
           [(e.generation, e.couple, e.migrants) for e in cpu.migrations]


def test_export_import_equals_local_migration(orc):
    """The split-couple halves (export on one GPU, import on another) equal migrate_*."""
    inst = ffsga.generate_instance(jobs=10, stages=3, machines=[2, 3, 2], weight=0.0, seed=2)
    d = as_data(inst)
    emax = ffsga.estimate_emax(inst)
    ci = capi.Instance.from_data(d, emax)
    a1, b1 = capi.Cellular(ci, 8, 4, 1), capi.Pseudo(ci, 32, 2)
    a2, b2 = capi.Cellular(ci, 8, 4, 1), capi.Pseudo(ci, 32, 2)
    capi.step([a1, a2], [b1, b2], 3)
    capi.migrate_cellular_to_pseudo(a1, b1, 7)
    g, f, o = a2.export_best(7)
    b2.import_worst(g, f, o)
    assert np.array_equal(b1.members(), b2.members()) and np.array_equal(b1.read()[0], b2.read()[0])
    assert b1.archive()[1] == b2.archive()[1]
    capi.step([a1, a2], [b1, b2], 2)
    capi.migrate_pseudo_to_cellular(b1, a1, 5)
    bits, f, o = b2.export_best(5)
    a2.import_worst(bits, f, o)
    assert np.array_equal(a1.genes(), a2.genes()) and np.array_equal(a1.read()[0], a2.read()[0])


def test_cell_candidate_matches_oracle(orc):
    inst = ffsga.generate_instance(jobs=6, stages=2, machines=[2, 2], seed=4)
    d = as_data(inst)
    emax = ffsga.estimate_emax(inst)
    ci = capi.Instance.from_data(d, emax)
    dc = capi.Cellular(ci, 4, 4, 123)
    oc = orc.instance(d).cellular(emax, 4, 4, 123)
    for i in range(16):
        seed = orc.derive_seed(orc.derive_seed(123, 1), i)
        g, f, o, rep, used = dc.candidate(i, seed)
        eg, ef, eo, erep, edraws = oc.candidate(i, seed, with_draws=True)
        assert used == edraws
        if not erep:  # cell_candidate returns the current cell when the child loses (cellular.cpp:157-162)
            eg = oc.genes()[i]
        assert np.array_equal(g, eg) and (f, o, rep) == (ef, eo, erep)
        assert used >= 4 + 1 + 12  # tournaments + coin + one coin per gene


def test_evaluate_tensor_device_resident(orc):
    """a population already on the GPU (torch CUDA tensor) is scored in place,
    results stay on the device, bit-identical to the oracle; errors as the host path."""
    import torch
    inst = ffsga.generate_instance(jobs=100, stages=10, machines=[4, 2, 2, 3, 4, 4, 2, 3, 4, 5], seed=7)
    oi = orc.instance(as_data(inst))
    pop = oi.random_population(99, 0, 3000)
    g = torch.from_numpy(pop.astype(np.uint8)).cuda()
    obj, fit, mk, td = ffsga.evaluate_tensor(inst, g, full=True)
    assert obj.is_cuda and obj.dtype == torch.float64
    eo, ef, em, et = oi.score_batch(pop, oi.estimate_emax())
    for a, b in ((obj, eo), (fit, ef), (mk, em), (td, et)):
        assert np.array_equal(a.cpu().numpy().view(np.uint64), b.view(np.uint64))
    obj32, _ = ffsga.evaluate_tensor(inst, torch.from_numpy(pop).cuda())  # int32 input
    assert torch.equal(obj32, obj)
    bad = torch.from_numpy(pop[:5].copy()).cuda()
    bad[3, 7] = 9
    with pytest.raises(ValueError, match="out of range"):
        ffsga.evaluate_tensor(inst, bad)
