"""Edge cases of the decoder entry points against the reference (oracle/_ref and the C
restatement): empty batches, the host-batch pipeline across several sub-batches with an error in
the last one, single-job and single-machine stages, -0.0 and tied release dates, extreme weights."""
import os

import numpy as np
import pytest

from pyoracle import InstanceData, synthetic_machines

pytestmark = pytest.mark.gpu
WORKERS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def capi():
    from paper_1903_10722_b200 import capi
    assert capi.device_count() > 0
    return capi


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def test_empty_batches(capi, orc):
    d = orc.generate(6, 2, [2, 2], seed=1)
    inst = capi.Instance.from_data(d, orc.instance(d).estimate_emax())
    for dtype in (np.int32, np.uint8):
        obj, fit = inst.evaluate(np.zeros((0, 12), dtype=dtype))
        assert obj.shape == (0,) and fit.shape == (0,)
    b = capi.Batch(inst, 4)
    b.evaluate(0)
    assert b.results(0)[0].shape == (0,)


def test_host_pipeline_sub_batches_and_first_error(capi, ref):
    """16 389 chromosomes at 500x20 through ffsga_cuda_evaluate: three pipelined sub-batches,
    bitwise against the reference; then the same batch with out-of-range genes in the second and
    third sub-batches names the reference's first offender (batch order, then dispatch order)."""
    J, S = 500, 20
    d = ref.generate(J, S, synthetic_machines(J, S), weight=100.0, seed=7)
    ri = ref.instance(d)
    emax = ri.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    n = 2 * 8192 + 5
    pop = ri.random_population(77, 0, n)
    obj, fit, mk, td = inst.evaluate(pop, full=True)
    eo, ef, em, et = ri.score_batch(pop, emax, WORKERS)
    for a, e in ((obj, eo), (fit, ef), (mk, em), (td, et)):
        assert np.array_equal(bits(a), bits(e))
    obj8, _ = inst.evaluate(pop.astype(np.uint8))
    assert np.array_equal(bits(obj8), bits(eo))
    bad = pop.copy()
    bad[n - 3, 7 * S + 4] = 9      # third sub-batch
    bad[8192 + 11, 3 * S + 6] = 8  # second sub-batch: the first offender in batch order
    bad[8192 + 11, 2 * S + 9] = 8
    with pytest.raises(ValueError) as a:
        inst.evaluate(bad)
    with pytest.raises(ValueError) as b:
        ri.score_batch(bad[8192 + 11:8192 + 12], emax, 1)
    assert str(a.value).split(" (")[0] == str(b.value)


@pytest.mark.parametrize("J,S,M", [
    (1, 2, [1, 2]),                    # one job
    (7, 3, [1, 3, 1]),                 # single-machine stages around a parallel one
    (40, 4, [32, 2, 32, 5]),           # the widest stages the decoder groups hold
    (64, 2, [2, 1]),
])
def test_small_and_wide_shapes(capi, orc, J, S, M):
    d = orc.generate(J, S, M, seed=3)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    pop = oi.random_population(9, 0, 200)
    obj, fit, mk, td = inst.evaluate(pop, full=True)
    eo, ef, em, et = oi.score_batch(pop, emax)
    for a, e in ((obj, eo), (fit, ef), (mk, em), (td, et)):
        assert np.array_equal(bits(a), bits(e))
    m, s, c, rep = inst.decode(pop[0])
    e = oi.score(pop[0], emax, schedule=True)
    assert np.array_equal(m, e["machine"]) and np.array_equal(bits(s), bits(e["start"]))


def test_negative_zero_and_tied_releases(capi, orc):
    """Release dates of -0.0, +0.0 and exact ties (the stage-0 order breaks them by job,
    model.cpp:98-105); integer processing times make completions tie on every stage."""
    rng = np.random.default_rng(8)
    J, S, M = 48, 4, [3, 2, 4, 2]
    proc = rng.integers(1, 5, size=(J, sum(M))).astype(np.float64)
    release = rng.choice([-0.0, 0.0, 3.0, 3.0, 7.0], J)
    d = InstanceData(J, S, M, proc, release, np.abs(release) + 30.0, 2.0)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    pop = oi.random_population(4, 0, 500)
    obj, fit, mk, td = inst.evaluate(pop, full=True)
    eo, ef, em, et = oi.score_batch(pop, emax)
    for a, e in ((obj, eo), (fit, ef), (mk, em), (td, et)):
        assert np.array_equal(bits(a), bits(e))
    for g in pop[:5]:
        m, s, c, rep = inst.decode(g)
        e = oi.score(g, emax, schedule=True)
        assert np.array_equal(bits(s), bits(e["start"])) and np.array_equal(bits(c), bits(e["completion"]))


@pytest.mark.parametrize("weight", [0.0, 1e6])
def test_extreme_weights_and_clamped_fitness(capi, orc, weight):
    d = orc.generate(30, 5, [2, 3, 2, 4, 2], weight=weight, seed=12)
    oi = orc.instance(d)
    pop = oi.random_population(1, 0, 300)
    for emax in (oi.estimate_emax(), 1.0):  # 1.0: every fitness clamps to 0 (model.cpp:118)
        inst = capi.Instance.from_data(d, emax)
        obj, fit = inst.evaluate(pop)
        eo, ef, _, _ = oi.score_batch(pop, emax)
        assert np.array_equal(bits(obj), bits(eo)) and np.array_equal(bits(fit), bits(ef))


def test_joint_step_mixed_island_sizes(capi, orc):
    """One joint step over islands of different sizes and kinds (the work list interleaves their
    cells and crossed members; graph replay for the small launches) equals each island stepped
    alone by the C restatement."""
    from conftest import synthetic
    d = synthetic(orc, 30, 6, 2, 5)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    shapes = [(8, 4), (16, 16), (3, 2)]
    cs = [capi.Cellular(inst, w, h, orc.derive_seed(6, i)) for i, (w, h) in enumerate(shapes)]
    ocs = [oi.cellular(emax, w, h, orc.derive_seed(6, i)) for i, (w, h) in enumerate(shapes)]
    sizes = [32, 64, 2]
    ps = [capi.Pseudo(inst, n, orc.derive_seed(7, i)) for i, n in enumerate(sizes)]
    ops = [oi.pseudo(emax, n, orc.derive_seed(7, i)) for i, n in enumerate(sizes)]
    tc, tp = capi.step(cs, ps, 9)
    for g in range(9):
        for i, oc in enumerate(ocs):
            oc.step()
            assert tc[i, g] == oc.objective()[oc.best_index()]
        for i, op in enumerate(ops):
            op.step()
            assert tp[i, g] == op.archive()[2]
    for dc, oc in zip(cs, ocs):
        assert np.array_equal(dc.genes(), oc.genes()) and np.array_equal(bits(dc.read()[0]), bits(oc.fitness()))
    for dp, op in zip(ps, ops):
        assert np.array_equal(dp.members(), op.members()) and dp.archive()[1] == op.archive()[1]


def test_migrating_whole_islands(capi, orc):
    """k = island population (migration.cpp:40-43 allows it): every member replaced, both ways,
    locally and through device packets."""
    d = orc.generate(8, 3, [2, 3, 2], weight=0.0, seed=5)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    dc, dp = capi.Cellular(inst, 4, 4, 3), capi.Pseudo(inst, 16, 4)
    oc, op = oi.cellular(emax, 4, 4, 3), oi.pseudo(emax, 16, 4)
    capi.step([dc], [dp], 2)
    for _ in range(2):
        oc.step()
        op.step()
    capi.migrate_cellular_to_pseudo(dc, dp, 16)
    orc.lib.orc_migrate_cellular_to_pseudo(oc.ptr, op.ptr, 16)
    assert np.array_equal(dp.members(), op.members()) and dp.archive()[1] == op.archive()[1]
    capi.migrate_pseudo_to_cellular(dp, dc, 16)
    orc.lib.orc_migrate_pseudo_to_cellular(op.ptr, oc.ptr, 16)
    assert np.array_equal(dc.genes(), oc.genes()) and np.array_equal(bits(dc.read()[0]), bits(oc.fitness()))
    dc2, dp2 = capi.Cellular(inst, 4, 4, 3), capi.Pseudo(inst, 16, 4)
    capi.step([dc2], [dp2], 2)
    dp2.import_packet(dc2.export_packet(16), 16)
    dc2.import_packet(dp2.export_packet(16), 16)
    assert np.array_equal(dc2.genes(), dc.genes()) and np.array_equal(dp2.members(), dp.members())


@pytest.mark.parametrize("pk", ["1", "0"])
def test_packed_heads_near_ties(capi, orc, monkeypatch, pk):
    """Ready times a few ulps apart agree above the job bits the packed heads keep (K1's
    ready-only pass, DevInst::pk_bits): such pops are flagged and the chromosome is decoded again
    in exact (ready, job) order.  Processing times n + k * 2^-48 make completions collide or miss
    each other by ulps on every stage; with FFSGA_EVAL_PK=0 the unpacked pass runs instead."""
    monkeypatch.setenv("FFSGA_EVAL_PK", pk)
    rng = np.random.default_rng(31)
    J, S, M = 48, 4, [3, 2, 4, 2]
    proc = rng.integers(1, 5, size=(J, sum(M))) + rng.integers(0, 4, size=(J, sum(M))) * 2.0 ** -48
    release = rng.integers(0, 3, J) + rng.integers(0, 8, J) * 2.0 ** -50
    d = InstanceData(J, S, M, proc, release, release + 40.0, 1.0)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    pop = oi.random_population(6, 0, 400)
    obj, fit, mk, td = inst.evaluate(pop, full=True)
    eo, ef, em, et = oi.score_batch(pop, emax)
    for a, e in ((obj, eo), (fit, ef), (mk, em), (td, et)):
        assert np.array_equal(bits(a), bits(e))


def test_host_batch_from_page_locked_memory(capi, orc):
    """A batch already in page-locked host memory is read in place by the copy engine (no
    staging copy): three pipelined sub-batches, equal to the pageable path and to the oracle."""
    import torch
    d = orc.generate(40, 4, [2, 3, 4, 2], seed=9)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    n = 2 * 8192 + 77
    pop = oi.random_population(12, 0, n)
    for dtype, tdtype in ((np.int32, torch.int32), (np.uint8, torch.uint8)):
        pinned = torch.empty(pop.shape, dtype=tdtype, pin_memory=True).numpy()
        pinned[:] = pop.astype(dtype)
        obj, fit = inst.evaluate(pinned)
        obj2, fit2 = inst.evaluate(np.array(pinned, copy=True))
        assert np.array_equal(bits(obj), bits(obj2)) and np.array_equal(bits(fit), bits(fit2))
    eo, ef, _, _ = oi.score_batch(pop, emax)
    assert np.array_equal(bits(obj), bits(eo)) and np.array_equal(bits(fit), bits(ef))
    bad = torch.empty(pop.shape, dtype=torch.int32, pin_memory=True).numpy()
    bad[:] = pop
    bad[8192 + 5, 3] = 7
    with pytest.raises(ValueError):
        inst.evaluate(bad)
