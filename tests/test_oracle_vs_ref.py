"""Pin the C restatement to the reference itself (oracle/_ref, compiled from the reference
sources by oracle/Makefile): decoder, islands, migration, whole runs.  CPU only."""
import numpy as np
import pytest

from conftest import synthetic


@pytest.mark.parametrize("J,S,lo,hi", [(20, 5, 3, 3), (100, 10, 2, 5), (60, 7, 1, 8), (300, 20, 2, 8)])
def test_decoder(orc, ref, J, S, lo, hi):
    d = synthetic(orc, J, S, lo, hi)
    oi, ri = orc.instance(d), ref.instance(d)
    emax = ri.estimate_emax()
    assert oi.estimate_emax() == emax
    pop = ri.random_population(99, 0, 100)
    assert np.array_equal(pop, oi.random_population(99, 0, 100))
    a, b = oi.score_batch(pop, emax), ri.score_batch(pop, emax, 4)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_schedule(orc, ref):
    d = synthetic(orc, 40, 6)
    oi, ri = orc.instance(d), ref.instance(d)
    for g in ri.random_population(3, 0, 20):
        m, s, c = ri.decode(g)
        e = oi.score(g, 0.0, schedule=True)
        assert np.array_equal(m, e["machine"]) and np.array_equal(s, e["start"]) and np.array_equal(c, e["completion"])


def test_islands_step_by_step(orc, ref):
    d = synthetic(orc, 20, 5, 3, 3)
    oi, ri = orc.instance(d), ref.instance(d)
    emax = ri.estimate_emax()
    oc, rc = oi.cellular(emax, 16, 16, 5), ri.cellular(emax, 256, 5)
    op, rp = oi.pseudo(emax, 64, 6), ri.pseudo(emax, 64, 6)
    for _ in range(25):
        oc.step()
        rc.step(4)
        op.step()
        rp.step(4)
        f, o, g = rc.read(genes=True)
        assert np.array_equal(f, oc.fitness()) and np.array_equal(g, oc.genes())
        f, o, b = rp.read(bits=True)
        assert np.array_equal(f, op.fitness()) and np.array_equal(b, op.members())
        assert rp.archive()[1:] == op.archive()[1:]


@pytest.mark.parametrize("mode", ["dual", "cellular", "pseudo"])
def test_runs(orc, ref, mode):
    d = orc.generate(10, 2, [2, 2], seed=41)
    oi, ri = orc.instance(d), ref.instance(d)
    assert oi.run(population=24, generations=40, gap=10, seed=9, mode=mode) == \
        ri.run(population=24, generations=40, gap=10, seed=9, mode=mode)


def test_runs_with_migrations(orc, ref):
    fired = 0
    for seed in range(1, 30):
        d = orc.generate(8, 2, [2, 2], weight=0.0, seed=seed)
        a = orc.instance(d).run(population=64, generations=30, gap=1, seed=seed)
        b = ref.instance(d).run(population=64, generations=30, gap=1, seed=seed)
        assert a == b
        fired += bool(a["migrations"])
    assert fired >= 3
