"""Reduced parity set for the checked build (device-side bounds and invariant checks standing in
for compute-sanitizer, which this GPU pool does not allow), or for compute-sanitizer itself where
it is available.

    python build.py --checked
    FFSGA_CUDA_LIB=paper_1903_10722_b200/checked/libffsga_cuda.so python profiles/tools/sanitize_set.py
    compute-sanitizer --tool racecheck python profiles/tools/sanitize_set.py [--algo bucket]

Exercises every kernel of the library at sizes the sanitizers finish in minutes, and checks
each result against the C restatement of the reference (oracle/, the checker):
  K1  k_eval DEPTH 2 (micro instance, 40x6 integer-time ties, 100x10) and DEPTH 3 (J = 1000),
      the exact re-decode on ties, out-of-range genes, K7 schedule decode;
  K1b k_eval_bkt (with --algo bucket: FFSGA_EVAL_ALGO=bucket before the instances are created);
  K2  k_random_rows; K3 k_cell_breed; K4 k_pseudo_breed; K6 k_commit / island stats
      (C1 island 16x16 for 3 generations, 100x10 pseudo island for 3 generations);
  K5  sort_island + migrate both ways, migrant packets (export/import on the device).
Exit code 0 = every comparison equal (the sanitizer's own report is the hazard count).
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algo", default="merge", choices=["merge", "bucket"])
    a = ap.parse_args()
    if a.algo == "bucket":
        os.environ["FFSGA_EVAL_ALGO"] = "bucket"
    from pyoracle import InstanceData, Oracle, synthetic_machines
    from paper_1903_10722_b200 import capi
    orc = Oracle()
    checks = 0

    def decoder(d, n, seed):
        nonlocal checks
        oi = orc.instance(d)
        emax = oi.estimate_emax()
        inst = capi.Instance.from_data(d, emax)
        pop = oi.random_population(seed, 0, n)
        obj, fit, mk, td = inst.evaluate(pop, full=True)
        eo, ef, em, et = oi.score_batch(pop, emax)
        for x, y in ((obj, eo), (fit, ef), (mk, em), (td, et)):
            assert np.array_equal(x.view(np.uint64), y.view(np.uint64))
        m, s, c, rep = inst.decode(pop[0])
        e = oi.score(pop[0], emax, schedule=True)
        assert np.array_equal(c, e["completion"]) and rep["objective"] == e["objective"]
        checks += 1
        return inst, oi, emax, pop

    # micro instance (test_model.cpp:18-31) + an out-of-range gene
    micro = InstanceData(2, 2, [2, 1], [2, 3, 4, 2, 3, 1], [0, 0], [10, 10], 100.0)
    inst = capi.Instance.from_data(micro, 211.0)
    assert inst.evaluate([[0, 0, 0, 0]])[0][0] == 7.0
    try:
        inst.evaluate([[0, 1, 0, 0]])
        raise AssertionError("bad gene accepted")
    except ValueError:
        pass
    # 40 x 6 integer times: ties -> exact re-decode (DEPTH 2)
    d = orc.generate(40, 6, [2, 3, 4, 2, 3, 2], weight=1.0, seed=3, integer_times=True)
    decoder(d, 96, 5)
    # 100 x 10 (C2 shape) and J = 1000 (DEPTH 3)
    decoder(orc.generate(100, 10, synthetic_machines(100, 10, 2, 5), seed=7), 64, 6)
    decoder(orc.generate(1000, 3, [3, 2, 4], seed=7), 16, 7)
    # K2 device init == reference stream
    inst, oi, emax, pop = decoder(orc.generate(20, 5, [3] * 5, seed=7), 8, 99)
    b = capi.Batch(inst, 64)
    b.fill_random(99, 0, 64)
    assert np.array_equal(b.download(0, 64), oi.random_population(99, 0, 64))
    b.evaluate(64)
    assert np.array_equal(b.results(64)[0], oi.score_batch(oi.random_population(99, 0, 64), emax)[0])
    # C1 island (K3 / K6) + 100 x 10 pseudo island (K4 / K6), 3 generations
    d1 = orc.generate(20, 5, [3] * 5, seed=7)
    o1 = orc.instance(d1)
    e1 = o1.estimate_emax()
    i1 = capi.Instance.from_data(d1, e1)
    dc = capi.Cellular(i1, 16, 16, orc.derive_seed(1, 0))
    oc = o1.cellular(e1, 16, 16, orc.derive_seed(1, 0))
    d2 = orc.generate(100, 10, synthetic_machines(100, 10, 2, 5), seed=7)
    o2 = orc.instance(d2)
    e2 = o2.estimate_emax()
    i2 = capi.Instance.from_data(d2, e2)
    dp = capi.Pseudo(i2, 64, orc.derive_seed(1, 1))
    op = o2.pseudo(e2, 64, orc.derive_seed(1, 1))
    for _ in range(3):
        capi.step([dc], [], 1)
        capi.step([], [dp], 1)
        oc.step()
        op.step()
        assert np.array_equal(dc.genes(), oc.genes()) and np.array_equal(dc.read()[0], oc.fitness())
        assert np.array_equal(dp.members(), op.members()) and dp.archive()[1] == op.archive()[1]
        checks += 1
    capi.step([dc], [], 2)  # graph-captured chunk
    for _ in range(2):
        oc.step()
    assert np.array_equal(dc.read()[0], oc.fitness())
    # K5: local migrations both ways and device packets, on a weight-0 pair
    d3 = orc.generate(10, 3, [2, 3, 2], weight=0.0, seed=2)
    o3 = orc.instance(d3)
    e3 = o3.estimate_emax()
    i3 = capi.Instance.from_data(d3, e3)
    a1, b1 = capi.Cellular(i3, 8, 4, 1), capi.Pseudo(i3, 32, 2)
    oa, ob = o3.cellular(e3, 8, 4, 1), o3.pseudo(e3, 32, 2)
    capi.step([a1], [b1], 2)
    for _ in range(2):
        oa.step()
        ob.step()
    capi.migrate_cellular_to_pseudo(a1, b1, 7)
    orc.lib.orc_migrate_cellular_to_pseudo(oa.ptr, ob.ptr, 7)
    capi.migrate_pseudo_to_cellular(b1, a1, 5)
    orc.lib.orc_migrate_pseudo_to_cellular(ob.ptr, oa.ptr, 5)
    assert np.array_equal(a1.genes(), oa.genes()) and np.array_equal(b1.members(), ob.members())
    a2, b2 = capi.Cellular(i3, 8, 4, 1), capi.Pseudo(i3, 32, 2)
    capi.step([a2], [b2], 2)
    b2.import_packet(a2.export_packet(7), 7)
    a2.import_packet(b2.export_packet(5), 5)
    assert np.array_equal(a1.genes(), a2.genes()) and np.array_equal(b1.members(), b2.members())
    checks += 1
    st = capi.checked_status(reset=True)
    assert st in (0, -1), f"device check {st >> 48} failed (a={(st >> 24) & 0xFFFFFF}, b={st & 0xFFFFFF})"
    if st == 0:  # the failure channel itself: an instance created with FFSGA_CHECK_SELFTEST
        os.environ["FFSGA_CHECK_SELFTEST"] = "1"
        capi.Instance.from_data(micro, 211.0).evaluate([[0, 0, 0, 0]])
        del os.environ["FFSGA_CHECK_SELFTEST"]
        assert capi.checked_status(reset=True) >> 48 == 99, "a deliberate device check failure was not reported"
    print(f"sanitize_set ({a.algo}): {checks} groups of checks equal to the oracle; "
          f"device checks: {'not a checked build' if st == -1 else 'all passed'}")


if __name__ == "__main__":
    main()
