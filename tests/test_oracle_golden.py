"""Pin the C restatement (oracle/ffsga_oracle.c) to the reference's own golden vectors.

Every constant below comes from the reference unit tests (proj/tests/test_*.cpp, cited per
test); the doctest suite itself cannot build here (doctest.h is not vendored), so its facts are
re-encoded.  CPU only.
"""
import numpy as np
import pytest

from pyoracle import InstanceData


def test_splitmix_raw_vectors(orc):  # test_rng.cpp:15-35
    vectors = {
        0x0: [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC],
        0x1: [0x910A2DEC89025CC1, 0xBEEB8DA1658EEC67, 0xF893A2EEFB32555E, 0x71C18690EE42C90B],
        0xDEADBEEF: [0x4ADFB90F68C9EB9B, 0xDE586A3141A10922, 0x021FBC2F8E1CFC1D, 0x7466CE737BE16790],
    }
    for seed, want in vectors.items():
        r = orc.rng(seed)
        assert [r.next_u64() for _ in range(4)] == want


def test_unit_and_uniform(orc):  # test_rng.cpp:37-49
    r = orc.rng(42)
    assert [r.next_unit() for _ in range(3)] == [0.7415648787718233, 0.1599103928769201, 0.27860113025513866]
    r = orc.rng(42)
    assert [r.next_uniform(1.0, 5.0) for _ in range(3)] == [3.9662595150872932, 1.6396415715076804,
                                                             2.1144045210205547]


def test_index_and_coin(orc):  # test_rng.cpp:75-95
    r = orc.rng(77)
    seen = [0] * 5
    for _ in range(5000):
        v = r.next_index(5)
        assert 0 <= v < 5
        seen[v] += 1
    assert min(seen) > 0 and r.next_index(1) == 0
    r = orc.rng(5)
    for _ in range(100):
        assert not r.next_coin(0.0)
        assert r.next_coin(1.0)


def test_derive_seed(orc):  # test_rng.cpp:97-101
    assert orc.derive_seed(1, 0) == 0x910A2DEC89025CC1
    assert orc.derive_seed(1, 1) == 0xBEEB8DA1658EEC67
    assert orc.derive_seed(7, 3) == 0x953AEB70673E29CB


def micro():  # test_model.cpp:18-31
    return InstanceData(2, 2, [2, 1], [2, 3, 4, 2, 3, 1], [0, 0], [10, 10], 100.0)


def test_micro_schedule_and_report(orc):  # test_model.cpp:57-88
    oi = orc.instance(micro())
    r = oi.score([0, 0, 0, 0], 211.0, schedule=True)
    s, c = r["start"], r["completion"]
    assert (s[0], c[0], s[2], c[2], s[1], c[1], s[3], c[3]) == (0, 2, 2, 4, 2, 6, 6, 7)
    assert (r["makespan"], r["total_tardiness"], r["objective"], r["fitness"], r["emax_used"]) == (7, 0, 7, 204, 211)
    assert oi.score([0, 0, 0, 0], 5.0)["fitness"] == 0.0  # :90-95


def test_out_of_range_genes(orc):  # test_model.cpp:71-77
    oi = orc.instance(micro())
    for g in ([0, 1, 0, 0], [-1, 0, 0, 0]):
        with pytest.raises(ValueError, match="out of range"):
            oi.score(g, 211.0)


def test_due_boundary_and_emax(orc):  # test_model.cpp:97-123
    d = micro()
    d.due = np.array([7.0, 7.0])
    oi = orc.instance(d)
    r = oi.score([0, 0, 0, 0], 211.0)
    assert r["total_tardiness"] == 0.0 and r["objective"] == r["makespan"]
    assert orc.instance(micro()).estimate_emax() == 211.0
    d = micro()
    d.due = np.array([50.0, 60.0])
    assert orc.instance(d).estimate_emax() == 11.0
    oi = orc.instance(micro())
    assert oi.mean_job_load(0) == 6.5 and oi.mean_job_load(1) == 3.5 and oi.mean_total_load() == 10.0


def test_single_job(orc):  # test_model.cpp:125-139
    d = InstanceData(1, 2, [2, 1], [2.5, 4.0, 3.0], [1.5], [100.0], 100.0)
    r = orc.instance(d).score([1, 0], 100.0, schedule=True)
    assert r["start"][0] == 1.5 and r["completion"][0] == 5.5 and r["completion"][1] == 8.5
    assert r["makespan"] == 1.5 + 4.0 + 3.0


def test_decoder_vs_selection_oracle(orc):  # test_model.cpp:172-185 (800 chromosomes)
    for seed in (21, 22, 23, 24):
        d = orc.generate(5, 2, [2, 2], seed=seed)
        oi = orc.instance(d)
        rng = orc.rng(seed + 99)
        for _ in range(200):
            g = oi.random_chromosome(rng)
            a, b = oi.score(g, 0.0), oi.simulate_selection(g)
            assert (a["makespan"], a["total_tardiness"], a["objective"]) == \
                   (b["makespan"], b["total_tardiness"], b["objective"])


def test_bit_layout(orc):  # test_chromosome.cpp:26-60
    d = InstanceData(1, 5, [1, 2, 3, 4, 5], np.ones(15), [0.0], [1.0], 1.0)
    lay = orc.instance(d).layout
    assert list(lay.bits_per_stage[:5]) == [1, 1, 2, 2, 3] and lay.bits_per_job == 9 and lay.total_bits == 9
    assert list(lay.stage_bit_offset[:6]) == [0, 1, 2, 4, 6, 9]
    d = InstanceData(2, 2, [2, 2], np.ones(8), [0, 0], [1, 1], 1.0)
    assert list(orc.instance(d).int_to_bits([0, 1, 1, 0])) == [0, 1, 1, 0]
    d = InstanceData(1, 2, [3, 3], np.ones(6), [0.0], [1.0], 1.0)
    assert list(orc.instance(d).int_to_bits([2, 1])) == [1, 0, 0, 1]


def test_bit_wrap(orc):  # test_chromosome.cpp:77-96
    d = InstanceData(1, 2, [3, 2], np.ones(5), [0.0], [1.0], 1.0)
    oi = orc.instance(d)
    assert list(oi.bits_to_int([1, 1, 0])) == [0, 0]


def test_round_trip_small(orc):  # test_chromosome.cpp:62-75
    import itertools
    for m in range(1, 6):
        d = InstanceData(2, 2, [m, m], np.ones(4 * m), [0, 0], [1, 1], 1.0)
        oi = orc.instance(d)
        for g in itertools.product(range(m), repeat=4):
            assert list(oi.bits_to_int(oi.int_to_bits(list(g)))) == list(g)


def test_pair_step_known_streams(orc):  # test_pseudo.cpp:33-54
    import ctypes as C
    a = np.array([1, 0, 1, 0], dtype=np.uint8)
    b = np.array([0, 1, 0, 1], dtype=np.uint8)
    c1, c2 = np.empty(4, np.uint8), np.empty(4, np.uint8)
    pu8 = C.POINTER(C.c_uint8)
    st = C.c_uint64(42)
    r = orc.lib.orc_pair_step(a.ctypes.data_as(pu8), b.ctypes.data_as(pu8), 4, C.byref(st), 0.75,
                              c1.ctypes.data_as(pu8), c2.ctypes.data_as(pu8))
    assert r == 1 and list(c1) == [1, 0, 0, 1] and list(c2) == [0, 1, 1, 0]
    st = C.c_uint64(0)
    r = orc.lib.orc_pair_step(a.ctypes.data_as(pu8), b.ctypes.data_as(pu8), 4, C.byref(st), 0.75,
                              c1.ctypes.data_as(pu8), c2.ctypes.data_as(pu8))
    assert r == 0 and list(c1) == list(a) and list(c2) == list(b)


def test_grid_shapes_and_sort(orc):  # test_cellular.cpp:61-77
    import ctypes as C
    w, h = C.c_int(), C.c_int()
    for pop, want in ((256, (16, 16)), (512, (32, 16)), (32, (8, 4)), (4, (2, 2)), (12, (4, 3)), (6, (3, 2))):
        assert orc.lib.orc_grid_shape_for(pop, C.byref(w), C.byref(h)) == 0 and (w.value, h.value) == want
    for pop in (2, 7):
        assert orc.lib.orc_grid_shape_for(pop, C.byref(w), C.byref(h)) != 0

    def sort(f):
        f = np.asarray(f, dtype=np.float64)
        o = np.empty(len(f), dtype=np.int32)
        orc.lib.orc_sort_island(f.ctypes.data_as(C.POINTER(C.c_double)), len(f), o.ctypes.data_as(C.POINTER(C.c_int)))
        return list(o)
    assert sort([3.0, 1.0, 2.0]) == [0, 2, 1]
    assert sort([2.0, 2.0, 1.0]) == [0, 1, 2]
    assert sort([1.0, 2.0, 2.0]) == [1, 2, 0]


def test_neighborhoods(orc):  # test_cellular.cpp:35-59,173-182
    import ctypes as C
    slots = (C.c_int * 16)()
    n = orc.lib.orc_neighborhood_slots(0, 0, 4, 4, 1, slots)
    assert n == 4 and sorted(slots[:4]) == [1, 3, 4, 12]
    n = orc.lib.orc_neighborhood_slots(0, 0, 2, 2, 1, slots)
    assert sorted(slots[:n]) == [1, 1, 2, 2]
    n = orc.lib.orc_neighborhood_slots(8, 8, 32, 32, 2, slots)
    assert n == 12


def test_migration_formulas(orc):  # test_migration.cpp:31-64
    assert orc.lib.orc_compute_beta(80.0, 100.0) == 0.8
    assert orc.lib.orc_compute_beta(100.0, 80.0) == 0.8
    assert orc.lib.orc_compute_beta(5.0, 5.0) == 1.0
    assert orc.lib.orc_compute_alpha(0.8, 1.0) == 1.0 - 0.8
    assert orc.lib.orc_compute_alpha(0.8, 0.1) == 0.0
    import ctypes as C
    b, a, d, k = C.c_double(), C.c_double(), C.c_int(), C.c_int()
    orc.lib.orc_decide(100.0, 80.0, 1.0, 256, C.byref(b), C.byref(a), C.byref(d), C.byref(k))
    assert d.value == 1 and k.value == int(np.floor((1.0 - 0.8) * 256)) == 51


def test_whole_run_values():
    """proj/test_output.txt:10,15 record run means that the compiled reference reproduced bit for
    bit during the survey; the oracle run is checked against oracle/_ref in
    tests/test_oracle_vs_ref.py.  Here: the criterion-3 style desk run is deterministic."""
    from pyoracle import Oracle
    orc = Oracle()
    d = orc.generate(12, 2, [2, 2], seed=47)
    oi = orc.instance(d)
    r1 = oi.run(population=32, generations=60, gap=20, seed=12)
    r2 = oi.run(population=32, generations=60, gap=20, seed=12)
    assert r1 == r2
    tc, ta, tb = r1["trace_combined"], r1["trace_island_a"], r1["trace_island_b"]
    assert all(c == min(a, b) for c, a, b in zip(tc, ta, tb))
    assert all(tc[g] <= tc[g - 1] for g in range(1, 60))
    assert r1["best_objective"] == tc[-1]
