"""K1/K7 parity: the CUDA decoder against the C restatement and the compiled reference, bitwise."""
import numpy as np
import pytest

from conftest import synthetic

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    from paper_1903_10722_b200 import capi
    assert capi.device_count() > 0, "no GPU: the device path has no CPU fallback"
    return capi


def micro(orc):
    from pyoracle import InstanceData
    # test_model.cpp:18-31: J=2, S=2, M=[2,1]
    return InstanceData(2, 2, [2, 1], [2, 3, 4, 2, 3, 1], [0, 0], [10, 10], 100.0)


def test_micro_schedule(capi, orc):
    d = micro(orc)
    inst = capi.Instance.from_data(d, 211.0)
    m, s, c, rep = inst.decode([0, 0, 0, 0])
    # test_model.cpp:57-69
    assert (s[0], c[0]) == (0.0, 2.0)
    assert (s[2], c[2]) == (2.0, 4.0)
    assert (s[1], c[1]) == (2.0, 6.0)
    assert (s[3], c[3]) == (6.0, 7.0)
    # test_model.cpp:79-88
    assert rep == dict(makespan=7.0, total_tardiness=0.0, objective=7.0, fitness=204.0, emax_used=211.0)
    obj, fit = capi.Instance.from_data(d, 5.0).evaluate([[0, 0, 0, 0]])
    assert obj[0] == 7.0 and fit[0] == 0.0  # test_model.cpp:90-95


def test_bad_gene_messages(capi, orc):
    d = micro(orc)
    inst = capi.Instance.from_data(d, 211.0)
    with pytest.raises(ValueError, match="out of range"):
        inst.evaluate([[0, 1, 0, 0]])
    with pytest.raises(ValueError, match="out of range"):
        inst.evaluate([[-1, 0, 0, 0]])
    # message matches the reference's first offending gene in dispatch order
    oi = orc.instance(d)
    for genes in ([0, 1, 0, 0], [-1, 0, 0, 0], [0, 0, 5, 0], [0, 7, 0, 7]):
        with pytest.raises(ValueError) as a:
            inst.evaluate([genes])
        with pytest.raises(ValueError) as b:
            oi.score(genes, 211.0)
        assert str(a.value).split(" (")[0] == str(b.value)


SHAPES = [(20, 5, 3, 3), (6, 2, 2, 2), (100, 10, 2, 5), (100, 20, 2, 8), (500, 20, 2, 8), (37, 7, 1, 8),
          (64, 3, 5, 16), (30, 4, 9, 32), (1, 2, 1, 2), (3, 2, 2, 2),
          (1000, 20, 2, 8), (1500, 5, 2, 6)]  # J >= 1000: three pops in flight


@pytest.mark.parametrize("J,S,lo,hi", SHAPES)
def test_random_batch_bitwise(capi, orc, J, S, lo, hi):
    d = synthetic(orc, J, S, lo, hi)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    n = 300 if J * S <= 2000 else 60
    pop = oi.random_population(99, 0, n)
    obj, fit, mk, td = inst.evaluate(pop, full=True)
    eo, ef, em, et = oi.score_batch(pop, emax)
    for a, b in ((obj, eo), (fit, ef), (mk, em), (td, et)):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_integer_times_ties(capi, orc):
    # integer processing times make equal completions (ties broken by job index) common
    for seed in range(5):
        d = orc.generate(40, 6, [2, 3, 4, 2, 3, 2], weight=1.0, seed=seed, integer_times=True)
        oi = orc.instance(d)
        emax = oi.estimate_emax()
        pop = oi.random_population(seed, 0, 400)
        obj, fit = capi.Instance.from_data(d, emax).evaluate(pop)
        eo, ef, _, _ = oi.score_batch(pop, emax)
        assert np.array_equal(obj, eo) and np.array_equal(fit, ef)


@pytest.mark.parametrize("J,S,M", [(30, 5, [3, 2, 3, 2, 3]), (1000, 4, [3, 2, 4, 2])])
def test_ready_time_ties_redecoded_exactly(capi, orc, J, S, M):
    """The decoder pops by ready time alone and decodes a chromosome again in (ready, job) order
    when two consecutive pops tie.  Small integer times make ties occur in some chromosomes and
    not in others, so CTAs mix re-decoded and kept groups; every result must still be the
    reference's, bit for bit."""
    from pyoracle import InstanceData
    rng = np.random.default_rng(17)
    proc = rng.integers(1, 400, size=(J, sum(M))).astype(np.float64)
    release = rng.integers(0, 600, J).astype(np.float64)
    due = release + rng.integers(50, 400, J)
    d = InstanceData(J, S, M, proc, release, due, 1.0)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    pop = oi.random_population(23, 0, 3000 if J < 100 else 300)
    obj, fit, mk, td = capi.Instance.from_data(d, emax).evaluate(pop, full=True)
    eo, ef, em, et = oi.score_batch(pop, emax)
    for a, b in ((obj, eo), (fit, ef), (mk, em), (td, et)):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    # both kinds occur: chromosomes whose per-machine ready times tie, and ones without ties
    def has_tie(g):
        e = oi.score(g, emax, schedule=True)
        mach = np.asarray(e["machine"]).reshape(J, S)
        comp = np.asarray(e["completion"]).reshape(J, S)
        for s in range(1, S):
            for mm in range(M[s]):
                r = comp[mach[:, s] == mm, s - 1]
                if len(np.unique(r)) < len(r):
                    return True
        return False
    if J < 100:
        ties = sum(has_tie(g) for g in pop[:300])
        assert 0 < ties < 300


def test_ties_and_out_of_range_genes_name_the_reference_job(capi, orc):
    """a chromosome whose earlier stages have equal ready times AND whose later stage
    holds several out-of-range genes must name the reference's first offender (model.cpp:81-83,
    minimum (ready, job) in that stage's dispatch order), which depends on the exact tie order."""
    from pyoracle import InstanceData
    J, S, M = 30, 5, [3, 2, 3, 2, 3]
    rng = np.random.default_rng(5)
    proc = rng.integers(1, 4, size=(J, sum(M))).astype(np.float64)
    release = rng.integers(0, 3, J).astype(np.float64)
    d = InstanceData(J, S, M, proc, release, release + 20.0, 1.0)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    pop = oi.random_population(31, 0, 150)
    checked = 0
    for i, g in enumerate(pop):
        g = g.copy()
        s_bad = 2 + i % 3
        for j in rng.choice(J, size=6, replace=False):
            g[j * S + s_bad] = M[s_bad] + int(rng.integers(0, 3))
        with pytest.raises(ValueError) as a:
            inst.evaluate([g])
        with pytest.raises(ValueError) as b:
            oi.score(g, emax)
        assert str(a.value).split(" (")[0] == str(b.value), i
        # the same chromosome inside a batch of good ones (item order, CTA-mixed redo)
        batch = np.concatenate([pop[:i], g[None, :]])
        with pytest.raises(ValueError) as c:
            inst.evaluate(batch)
        assert str(c.value).split(" (")[0] == str(b.value), i
        checked += 1
    assert checked == 150


def test_decode_schedule_matches_reference(capi, orc):
    d = synthetic(orc, 50, 6)
    oi = orc.instance(d)
    inst = capi.Instance.from_data(d, oi.estimate_emax())
    for g in oi.random_population(5, 0, 10):
        m, s, c, rep = inst.decode(g)
        e = oi.score(g, oi.estimate_emax(), schedule=True)
        assert np.array_equal(m, e["machine"]) and np.array_equal(s, e["start"])
        assert np.array_equal(c, e["completion"]) and rep["objective"] == e["objective"]


def test_device_random_population_matches(capi, orc):
    d = synthetic(orc, 100, 10, 2, 5)
    oi = orc.instance(d)
    inst = capi.Instance.from_data(d, oi.estimate_emax())
    b = capi.Batch(inst, 1000)
    b.fill_random(99, 12345, 1000)
    got = b.download(0, 1000)
    want = oi.random_population(99, 12345, 1000)
    assert np.array_equal(got, want)
    b.evaluate(1000)
    obj, fit = b.results(1000)
    eo, ef, _, _ = oi.score_batch(want, oi.estimate_emax())
    assert np.array_equal(obj, eo) and np.array_equal(fit, ef)


def test_exhaustive_small_instances(capi, orc):
    # acceptance criterion 2 (acceptance_main.cpp:161-215): J=3..5, S=2, M=2, all assignments
    import itertools
    for seed in range(6):
        J = 3 + seed % 3
        d = orc.generate(J, 2, [2, 2], seed=100 + seed)
        oi = orc.instance(d)
        emax = oi.estimate_emax()
        pop = np.array(list(itertools.product([0, 1], repeat=2 * J)), dtype=np.int32)
        obj, _ = capi.Instance.from_data(d, emax).evaluate(pop)
        sel = np.array([oi.simulate_selection(g)["objective"] for g in pop])
        assert np.array_equal(obj, sel)


def test_against_compiled_reference(capi, orc, ref):
    d = synthetic(orc, 500, 20)
    ri = ref.instance(d)
    emax = ri.estimate_emax()
    pop = ri.random_population(99, 0, 200)
    obj, fit, mk, td = capi.Instance.from_data(d, emax).evaluate(pop, full=True)
    eo, ef, em, et = ri.score_batch(pop, emax, workers=8)
    assert np.array_equal(obj, eo) and np.array_equal(fit, ef)
    assert np.array_equal(mk, em) and np.array_equal(td, et)


def test_full_size_sweep_properties(capi, orc):
    """BASELINE C5 size (1M chromosomes, 500 x 20): a spread sample is bitwise equal to the oracle
    and every result satisfies the size-independent invariants of report_from_completions."""
    d = synthetic(orc, 500, 20)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    n = 1 << 20
    b = capi.Batch(inst, n)
    b.fill_random(99, 0, n)
    b.evaluate(n)
    obj, fit, mk, td = b.results(n, full=True)
    slack = emax - obj
    assert np.array_equal(fit, np.where(slack < 0.0, 0.0, slack))
    assert np.all(mk > 0) and np.all(td >= 0) and np.all(np.isfinite(obj))
    assert np.array_equal(obj, d.weight * td + mk)
    idx = np.linspace(0, n - 1, 200).astype(np.int64)
    for i in idx[::10]:
        g = b.download(int(i), 1)[0]
        r = oi.score(g, emax)
        assert (r["objective"], r["fitness"], r["makespan"], r["total_tardiness"]) == (obj[i], fit[i], mk[i], td[i])
    want = oi.random_population(99, 12345, 1)[0]
    assert np.array_equal(b.download(12345, 1)[0], want)


# ---- the bucket-sort decoder (K1b): forced on every shape, and chosen automatically for instances
# whose processing times fall below ulp(horizon), where completions on a machine can tie

@pytest.fixture
def bucket(monkeypatch):
    monkeypatch.setenv("FFSGA_EVAL_ALGO", "bucket")  # read when an instance is created


@pytest.mark.parametrize("J,S,lo,hi", SHAPES)
def test_bucket_decoder_bitwise(capi, orc, bucket, J, S, lo, hi):
    d = synthetic(orc, J, S, lo, hi)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    pop = oi.random_population(7, 0, 200 if J * S <= 2000 else 50)
    obj, fit, mk, td = inst.evaluate(pop, full=True)
    eo, ef, em, et = oi.score_batch(pop, emax)
    for a, b in ((obj, eo), (fit, ef), (mk, em), (td, et)):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_bucket_decoder_ties_errors_schedule(capi, orc, bucket):
    for seed in range(4):
        d = orc.generate(40, 6, [2, 3, 4, 2, 3, 2], weight=1.0, seed=seed, integer_times=True)
        oi = orc.instance(d)
        emax = oi.estimate_emax()
        pop = oi.random_population(seed, 0, 300)
        obj, fit = capi.Instance.from_data(d, emax).evaluate(pop)
        eo, ef, _, _ = oi.score_batch(pop, emax)
        assert np.array_equal(obj, eo) and np.array_equal(fit, ef)
    d = micro(orc)
    inst = capi.Instance.from_data(d, 211.0)
    oi = orc.instance(d)
    for genes in ([0, 1, 0, 0], [-1, 0, 0, 0], [0, 0, 5, 0], [0, 7, 0, 7]):
        with pytest.raises(ValueError) as a:
            inst.evaluate([genes])
        with pytest.raises(ValueError) as b:
            oi.score(genes, 211.0)
        assert str(a.value).split(" (")[0] == str(b.value)
    d = synthetic(orc, 50, 6)
    oi = orc.instance(d)
    inst = capi.Instance.from_data(d, oi.estimate_emax())
    for g in oi.random_population(5, 0, 6):
        m, s, c, rep = inst.decode(g)
        e = oi.score(g, oi.estimate_emax(), schedule=True)
        assert np.array_equal(m, e["machine"]) and np.array_equal(s, e["start"])
        assert np.array_equal(c, e["completion"]) and rep["objective"] == e["objective"]


def test_sub_ulp_processing_times(capi, orc):
    """Release times near 2^53 with processing times below their ulp: start + p rounds back to
    start, so completions on one machine tie.  The merge decoder cannot order such lists; the
    instance runs on the bucket decoder automatically and still matches the reference."""
    from pyoracle import InstanceData
    rng = np.random.default_rng(3)
    J, S, M = 60, 4, [2, 3, 2, 3]
    proc = rng.choice([0.25, 0.5, 1.0, 3.0, 8.0], size=(J, sum(M)))
    release = 2.0 ** 53 + rng.integers(0, 40, J).astype(np.float64) * 2.0
    due = release + 50.0
    d = InstanceData(J, S, M, proc, release, due, 0.5)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    pop = oi.random_population(11, 0, 400)
    obj, fit, mk, td = inst.evaluate(pop, full=True)
    eo, ef, em, et = oi.score_batch(pop, emax)
    for a, b in ((obj, eo), (fit, ef), (mk, em), (td, et)):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("J,S,lo,hi", [(4000, 3, 2, 2), (9000, 2, 2, 3), (20000, 2, 2, 2)])
def test_large_jobs_wider_groups(capi, orc, J, S, lo, hi):
    """Per-chromosome state grows with J: past a warp of minimal groups the decoder switches to
    wider groups (fewer chromosomes per warp) instead of refusing the instance."""
    d = synthetic(orc, J, S, lo, hi)
    oi = orc.instance(d)
    emax = oi.estimate_emax()
    inst = capi.Instance.from_data(d, emax)
    assert inst.info()["group_lanes"] > 4
    pop = oi.random_population(5, 0, 12)
    obj, fit, mk, td = inst.evaluate(pop, full=True)
    eo, ef, em, et = oi.score_batch(pop, emax)
    for a, b in ((obj, eo), (fit, ef), (mk, em), (td, et)):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_too_many_jobs_is_a_config_error(capi, orc):
    d = synthetic(orc, 30000, 2, 2, 2)
    with pytest.raises(capi.ConfigError, match="too large"):
        capi.Instance.from_data(d, 1e12)


@pytest.mark.parametrize("algo", ["merge", "bucket"])
def test_randomized_instances_both_decoders(capi, orc, monkeypatch, algo):
    """Many random shapes (1-40 jobs... 300 jobs, 1-12 stages, 1-32 machines per stage, real and
    integer times, random weights): both decoders bit-identical to the oracle."""
    monkeypatch.setenv("FFSGA_EVAL_ALGO", algo)
    rng = np.random.default_rng(20261018)
    for case in range(24):
        J = int(rng.choice([1, 2, 5, 17, 40, 97, 300]))
        S = int(rng.integers(1, 13))
        hi = int(rng.choice([2, 4, 8, 13, 32]))
        M = [int(x) for x in rng.integers(1, hi + 1, S)]
        d = orc.generate(J, S, M, weight=float(rng.choice([0.0, 1.0, 100.0, 7.25])), seed=int(rng.integers(1, 10**6)),
                         integer_times=bool(rng.integers(0, 2)))
        oi = orc.instance(d)
        emax = oi.estimate_emax()
        inst = capi.Instance.from_data(d, emax)
        pop = oi.random_population(int(rng.integers(0, 10**6)), 0, 48)
        obj, fit, mk, td = inst.evaluate(pop, full=True)
        eo, ef, em, et = oi.score_batch(pop, emax)
        for a, b in ((obj, eo), (fit, ef), (mk, em), (td, et)):
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), (case, J, S, M)
