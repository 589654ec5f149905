"""Golden vectors produced by the reference itself (tests/golden/ref_vectors.json, written by
tests/golden/make_golden.py from oracle/_ref): the C restatement must reproduce them on the CPU,
and the product (CUDA kernels behind the C ABI and the reference Python API) on the GPU -- bit for
bit, with no access to the reference at test time."""
import json
import os
import struct

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "ref_vectors.json")) as _f:
    GOLD = json.load(_f)


def hx(x):
    return struct.pack("<d", float(x)).hex()


def hexes(a):
    return [hx(v) for v in np.asarray(a, dtype=np.float64)]


def oracle_instance(orc, case):
    d = orc.generate(case["J"], case["S"], case["machines"], weight=case["weight"], seed=case["gen_seed"])
    return d, orc.instance(d)


# ------------------------------------------------------------------ CPU: the oracle is pinned
@pytest.mark.parametrize("case", GOLD["decoder"], ids=lambda c: f"{c['J']}x{c['S']}")
def test_oracle_decoder_fixture(orc, case):
    _, oi = oracle_instance(orc, case)
    emax = oi.estimate_emax()
    assert hx(emax) == case["emax"]
    pop = oi.random_population(case["pop_seed"], 0, case["n"])
    obj, fit, mk, td = oi.score_batch(pop, emax)
    assert hexes(obj) == case["objective"] and hexes(fit) == case["fitness"]
    assert hexes(mk) == case["makespan"] and hexes(td) == case["tardiness"]


@pytest.mark.parametrize("case", GOLD["cellular"], ids=lambda c: f"{c['J']}x{c['S']}")
def test_oracle_cellular_fixture(orc, case):
    _, oi = oracle_instance(orc, case)
    c = oi.cellular(oi.estimate_emax(), case["width"], case["height"], int(case["seed"]))
    trace = []
    for _ in range(case["generations"]):
        c.step()
        trace.append(hx(c.objective()[c.best_index()]))
    assert trace == case["best_objective_trace"]
    assert hexes(c.fitness()) == case["fitness"] and hexes(c.objective()) == case["objective"]


@pytest.mark.parametrize("case", GOLD["pseudo"], ids=lambda c: f"{c['J']}x{c['S']}")
def test_oracle_pseudo_fixture(orc, case):
    _, oi = oracle_instance(orc, case)
    p = oi.pseudo(oi.estimate_emax(), case["population"], int(case["seed"]))
    trace = []
    for _ in range(case["generations"]):
        p.step()
        trace.append(hx(p.archive()[2]))
    assert trace == case["archive_objective_trace"]
    assert hexes(p.fitness()) == case["fitness"] and hexes(p.objective()) == case["objective"]


def run_matches(got, case):
    assert hx(got["best_objective"]) == case["best_objective"]
    assert list(got["best_chromosome"]) == case["best_chromosome"]
    assert hexes(got["trace_combined"]) == case["trace_combined"]
    mig = [dict(generation=m["generation"], beta=hx(m["beta"]), alpha=hx(m["alpha"]), direction=m["direction"],
                migrants=m["migrants"]) for m in got["migrations"]]
    assert mig == case["migrations"]


@pytest.mark.parametrize("case", GOLD["run"], ids=lambda c: f"{c['J']}x{c['S']}-s{c['seed']}")
def test_oracle_run_fixture(orc, case):
    _, oi = oracle_instance(orc, case)
    got = oi.run(population=case["population"], generations=case["generations"], gap=case["gap"],
                 theta=case["theta"], seed=case["seed"])
    run_matches(got, case)


# ------------------------------------------------------------------ GPU: the product matches
@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["decoder"], ids=lambda c: f"{c['J']}x{c['S']}")
def test_device_decoder_fixture(orc, case):
    from paper_1903_10722_b200 import capi
    d, oi = oracle_instance(orc, case)
    inst = capi.Instance.from_data(d, struct.unpack("<d", bytes.fromhex(case["emax"]))[0])
    b = capi.Batch(inst, case["n"])
    b.fill_random(case["pop_seed"], 0, case["n"])  # device K2: random_int_chromosome(Rng(derive_seed(99, i)))
    b.evaluate(case["n"])
    obj, fit, mk, td = b.results(case["n"], full=True)
    assert hexes(obj) == case["objective"] and hexes(fit) == case["fitness"]
    assert hexes(mk) == case["makespan"] and hexes(td) == case["tardiness"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["cellular"], ids=lambda c: f"{c['J']}x{c['S']}")
def test_device_cellular_fixture(orc, case):
    from paper_1903_10722_b200 import capi
    d, oi = oracle_instance(orc, case)
    inst = capi.Instance.from_data(d, oi.estimate_emax())
    c = capi.Cellular(inst, case["width"], case["height"], int(case["seed"]))
    tc, _ = capi.step([c], [], case["generations"])
    assert hexes(tc[0]) == case["best_objective_trace"]
    fit, obj = c.read()
    assert hexes(fit) == case["fitness"] and hexes(obj) == case["objective"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["pseudo"], ids=lambda c: f"{c['J']}x{c['S']}")
def test_device_pseudo_fixture(orc, case):
    from paper_1903_10722_b200 import capi
    d, oi = oracle_instance(orc, case)
    inst = capi.Instance.from_data(d, oi.estimate_emax())
    p = capi.Pseudo(inst, case["population"], int(case["seed"]))
    _, tp = capi.step([], [p], case["generations"])
    assert hexes(tp[0]) == case["archive_objective_trace"]
    fit, obj = p.read()
    assert hexes(fit) == case["fitness"] and hexes(obj) == case["objective"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", GOLD["run"], ids=lambda c: f"{c['J']}x{c['S']}-s{c['seed']}")
def test_device_run_fixture(case):
    import paper_1903_10722_b200 as ffsga
    m = case["machines"]
    inst = ffsga.generate_instance(jobs=case["J"], stages=case["S"], machines=m, weight=case["weight"],
                                   seed=case["gen_seed"])
    got = ffsga.solve(inst, population=case["population"], generations=case["generations"], gap=case["gap"],
                      theta=case["theta"], seed=case["seed"])
    run_matches(got, case)
