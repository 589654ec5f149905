"""K2-K6 parity: device islands against the C restatement, every cell every generation."""
import numpy as np
import pytest

from conftest import synthetic

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    from paper_1903_10722_b200 import capi
    assert capi.device_count() > 0
    return capi


def bits_eq(a, b):
    return np.array_equal(np.asarray(a, dtype=np.float64).view(np.uint64), np.asarray(b, dtype=np.float64).view(np.uint64))


def check_cell(dc, oc):
    f, o = dc.read()
    assert bits_eq(f, oc.fitness()) and bits_eq(o, oc.objective())
    assert np.array_equal(dc.genes(), oc.genes())
    i, bf, bo = dc.best()
    assert i == oc.best_index() and bf == oc.fitness()[i] and bo == oc.objective()[i]


def test_cellular_init_and_slots(capi, orc):
    d = orc.generate(6, 2, [2, 2], seed=1)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    dc = capi.Cellular(inst, 4, 4, 2)
    oc = oi.cellular(emax, 4, 4, 2)
    check_cell(dc, oc)
    assert sorted(dc.slots(0)) == [1, 3, 4, 12]  # test_cellular.cpp:173-182
    assert np.array_equal(np.stack([dc.slots(i) for i in range(16)]), oc.slots())


@pytest.mark.parametrize("J,S,lo,hi,W,H,r,mu,xr", [
    (20, 5, 3, 3, 16, 16, 1, 0.05, 1.0),    # C1
    (6, 2, 2, 2, 4, 4, 1, 0.05, 1.0),
    (8, 3, 2, 4, 2, 2, 1, 0.3, 0.5),         # folded torus neighbourhoods
    (30, 4, 2, 8, 8, 6, 2, 0.2, 0.9),        # radius 2
    (16, 3, 2, 4, 9, 9, 4, 0.1, 0.8),        # radius 4: 40 neighbours (more than a warp's lanes)
    (50, 6, 2, 5, 5, 5, 1, 1.0, 1.0),        # every gene mutates
    (12, 3, 2, 3, 6, 2, 1, 0.0, 0.0),        # no crossover, no mutation
])
def test_cellular_steps_match_oracle(capi, orc, J, S, lo, hi, W, H, r, mu, xr):
    d = synthetic(orc, J, S, lo, hi)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    seed = orc.derive_seed(1, 0)
    dc = capi.Cellular(inst, W, H, seed, crossover=xr, mutation=mu, radius=r)
    oc = oi.cellular(emax, W, H, seed, crossover=xr, mutation=mu, radius=r)
    check_cell(dc, oc)
    gens = 100 if J * S <= 100 else 25
    for g in range(gens):
        tc, _ = capi.step([dc], [], 1)
        oc.step()
        check_cell(dc, oc)
        assert tc[0, 0] == oc.objective()[oc.best_index()]
    assert dc.generation == gens


def test_cellular_multi_generation_trace(capi, orc):
    d = synthetic(orc, 20, 5, 3, 3)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    dc = capi.Cellular(inst, 16, 16, 5)
    oc = oi.cellular(emax, 16, 16, 5)
    tc, _ = capi.step([dc], [], 40)
    want = []
    for _ in range(40):
        oc.step()
        want.append(oc.objective()[oc.best_index()])
    assert np.array_equal(tc[0], np.array(want))
    check_cell(dc, oc)


def check_pseudo(dp, op):
    f, o = dp.read()
    assert bits_eq(f, op.fitness()) and bits_eq(o, op.objective())
    assert np.array_equal(dp.members(), op.members())
    ab, af, ao = dp.archive()
    eb, ef, eo = op.archive()
    assert af == ef and ao == eo and np.array_equal(ab, eb)
    i, bf, _ = dp.best()
    assert i == op.best_index() and bf == op.fitness()[i]


@pytest.mark.parametrize("J,S,lo,hi,n,xr", [
    (6, 2, 2, 2, 16, 0.75), (20, 5, 3, 3, 64, 0.75), (13, 7, 2, 8, 40, 1.0), (100, 10, 2, 5, 128, 0.75),
    (9, 3, 1, 5, 2, 0.5), (30, 20, 2, 8, 32, 0.0),
    (40, 25, 9, 16, 32, 0.75),   # 100 bits per job: the unpack window's upper word
    (11, 30, 17, 32, 24, 0.9)])  # 150 bits per job: wider than the 128-bit unpack window
def test_pseudo_steps_match_oracle(capi, orc, J, S, lo, hi, n, xr):
    d = synthetic(orc, J, S, lo, hi)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    dp = capi.Pseudo(inst, n, 42, crossover=xr)
    op = oi.pseudo(emax, n, 42, crossover=xr)
    check_pseudo(dp, op)
    for _ in range(30):
        _, tp = capi.step([], [dp], 1)
        op.step()
        check_pseudo(dp, op)
        assert tp[0, 0] == op.archive()[2]


@pytest.mark.parametrize("split,mix", [("1", "0"), ("2", "0"), ("3", "0"), ("1", "1"), ("1", "2"), ("1", "3")])
def test_joint_step_equals_separate(capi, orc, monkeypatch, split, mix):
    # step groups (one stream per group of islands, one or both kinds per group) change no result
    monkeypatch.setenv("FFSGA_STEP_SPLIT", split)  # read when the instance is created
    monkeypatch.setenv("FFSGA_STEP_MIX", mix)
    d = synthetic(orc, 40, 6, 2, 6)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    cs = [capi.Cellular(inst, 8, 4, orc.derive_seed(3, 2 * i)) for i in range(3)]
    ps = [capi.Pseudo(inst, 32, orc.derive_seed(3, 2 * i + 1)) for i in range(2)]
    ocs = [oi.cellular(emax, 8, 4, orc.derive_seed(3, 2 * i)) for i in range(3)]
    ops = [oi.pseudo(emax, 32, orc.derive_seed(3, 2 * i + 1)) for i in range(2)]
    tc, tp = capi.step(cs, ps, 12)
    for g in range(12):
        for i, oc in enumerate(ocs):
            oc.step()
            assert tc[i, g] == oc.objective()[oc.best_index()]
        for i, op in enumerate(ops):
            op.step()
            assert tp[i, g] == op.archive()[2]
    for dc, oc in zip(cs, ocs):
        check_cell(dc, oc)
    for dp, op in zip(ps, ops):
        check_pseudo(dp, op)


def test_migration_both_directions(capi, orc):
    d = orc.generate(8, 2, [2, 2], weight=0.0, seed=4)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    dc, dp = capi.Cellular(inst, 8, 4, 11), capi.Pseudo(inst, 32, 12)
    oc, op = oi.cellular(emax, 8, 4, 11), oi.pseudo(emax, 32, 12)
    lib = orc.lib
    for rnd in range(6):
        capi.step([dc], [dp], 3)
        for _ in range(3):
            oc.step()
            op.step()
        k = 3 + rnd
        if rnd % 2 == 0:
            capi.migrate_cellular_to_pseudo(dc, dp, k)
            lib.orc_migrate_cellular_to_pseudo(oc.ptr, op.ptr, k)
        else:
            capi.migrate_pseudo_to_cellular(dp, dc, k)
            lib.orc_migrate_pseudo_to_cellular(op.ptr, oc.ptr, k)
        check_cell(dc, oc)
        check_pseudo(dp, op)
    with pytest.raises(ValueError):
        capi.migrate_cellular_to_pseudo(dc, dp, 33)


def test_install(capi, orc):
    d = orc.generate(6, 2, [2, 2], seed=19)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    dc, oc = capi.Cellular(inst, 4, 4, 55), oi.cellular(emax, 4, 4, 55)
    g = dc.genes(3)
    dc.install(7, g, 123.5, 42.25)
    oc.install(7, g, 123.5, 42.25)
    check_cell(dc, oc)
    dp, op = capi.Pseudo(inst, 8, 9), oi.pseudo(emax, 8, 9)
    b = dp.members(0)
    hi = dp.archive()[1] + 10.0
    for args in ((3, b, hi, 1.25), (4, b, hi - 5.0, 2.0)):
        dp.install(*args)
        op.install(*args)
        check_pseudo(dp, op)


def test_c3_shape_islands_match_oracle(capi, orc):
    """C3 instance shape (500 x 20, M in [2, 8]) on small islands, every member every generation."""
    d = synthetic(orc, 500, 20)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    dc = capi.Cellular(inst, 16, 8, orc.derive_seed(1, 0))
    dp = capi.Pseudo(inst, 64, orc.derive_seed(1, 1))
    oc = oi.cellular(emax, 16, 8, orc.derive_seed(1, 0))
    op = oi.pseudo(emax, 64, orc.derive_seed(1, 1))
    for _ in range(3):
        capi.step([dc], [dp], 1)
        oc.step()
        op.step()
        check_cell(dc, oc)
        check_pseudo(dp, op)
