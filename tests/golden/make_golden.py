"""Regenerate tests/golden/ref_vectors.json from the REFERENCE itself (oracle/_ref, the reference
sources compiled by oracle/Makefile).  Run here, where /root/reference exists:

    python build.py && python tests/golden/make_golden.py

Every floating value is stored as the hex of its IEEE-754 bits, so the fixtures pin results bit
for bit.  Chromosomes, instances and island seeds are not stored: they are regenerated from the
recorded parameters by the generator / RNG streams that tests/test_oracle_golden.py pins to the
reference's own golden vectors.
"""
import json
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import RefLib, synthetic_machines  # noqa: E402


def hx(x):
    return struct.pack("<d", float(x)).hex()


def derive_seed(base, key):  # rng.hpp:55-58 (output `key` of SplitMix64(base))
    g, m = 0x9E3779B97F4A7C15, (1 << 64) - 1
    z = (base + (key + 1) * g) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def main():
    ref = RefLib()
    out = {"source": "oracle/_ref (reference sources, -ffp-contract=off)", "decoder": [], "cellular": [],
           "pseudo": [], "run": []}
    # decoder: Evaluator::score on chromosomes of random_int_chromosome(Rng(derive_seed(99, i)))
    for (J, S, lo, hi) in [(20, 5, 3, 3), (100, 10, 2, 5), (500, 20, 2, 8), (37, 7, 1, 8)]:
        M = synthetic_machines(J, S, lo, hi)
        d = ref.generate(J, S, M, weight=100.0, seed=7)
        ri = ref.instance(d)
        emax = ri.estimate_emax()
        n = 24
        pop = ri.random_population(99, 0, n)
        obj, fit, mk, td = ri.score_batch(pop, emax)
        out["decoder"].append(dict(J=J, S=S, machines=M, gen_seed=7, weight=100.0, pop_seed=99, n=n, emax=hx(emax),
                                   objective=[hx(v) for v in obj], fitness=[hx(v) for v in fit],
                                   makespan=[hx(v) for v in mk], tardiness=[hx(v) for v in td]))
    # cellular island: CellGrid(inst, emax, W*H, params, derive_seed(1, 0)) stepped G times
    for (J, S, lo, hi, W, H, G) in [(20, 5, 3, 3, 16, 16, 12), (100, 10, 2, 5, 32, 16, 6)]:
        M = synthetic_machines(J, S, lo, hi)
        d = ref.generate(J, S, M, weight=100.0, seed=7)
        ri = ref.instance(d)
        emax = ri.estimate_emax()
        seed = derive_seed(1, 0)
        c = ri.cellular(emax, W * H, seed, width=W, height=H)
        trace = []
        for _ in range(G):
            c.step(1)
            fit, obj = c.read()
            trace.append(hx(obj[c.best_index()]))
        fit, obj = c.read()
        out["cellular"].append(dict(J=J, S=S, machines=M, gen_seed=7, weight=100.0, width=W, height=H,
                                    seed=str(seed), generations=G, best_objective_trace=trace,
                                    fitness=[hx(v) for v in fit], objective=[hx(v) for v in obj]))
    # pseudo island: PairPopulation(inst, emax, N, params, derive_seed(1, 1)) stepped G times
    for (J, S, lo, hi, N, G) in [(20, 5, 3, 3, 64, 12), (100, 10, 2, 5, 512, 6)]:
        M = synthetic_machines(J, S, lo, hi)
        d = ref.generate(J, S, M, weight=100.0, seed=7)
        ri = ref.instance(d)
        emax = ri.estimate_emax()
        seed = derive_seed(1, 1)
        p = ri.pseudo(emax, N, seed)
        trace = []
        for _ in range(G):
            p.step(1)
            trace.append(hx(p.archive()[2]))
        fit, obj = p.read()
        out["pseudo"].append(dict(J=J, S=S, machines=M, gen_seed=7, weight=100.0, population=N, seed=str(seed),
                                  generations=G, archive_objective_trace=trace,
                                  fitness=[hx(v) for v in fit], objective=[hx(v) for v in obj]))
    # whole runs: ffsga::run (solver.cpp:76-198), dual with migrations firing (weight 0 and 100)
    for (J, S, lo, hi, weight, pop, gens, gap, theta, seed) in [(20, 5, 3, 3, 100.0, 64, 30, 10, 1.0, 3),
                                                                 (30, 4, 2, 4, 0.0, 128, 40, 5, 1.0, 5)]:
        M = synthetic_machines(J, S, lo, hi)
        d = ref.generate(J, S, M, weight=weight, seed=7)
        r = ref.instance(d).run(population=pop, generations=gens, gap=gap, theta=theta, seed=seed)
        out["run"].append(dict(J=J, S=S, machines=M, gen_seed=7, weight=weight, population=pop, generations=gens,
                               gap=gap, theta=theta, seed=seed, best_objective=hx(r["best_objective"]),
                               best_chromosome=r["best_chromosome"],
                               trace_combined=[hx(v) for v in r["trace_combined"]],
                               migrations=[dict(generation=m["generation"], beta=hx(m["beta"]),
                                                alpha=hx(m["alpha"]), direction=m["direction"],
                                                migrants=m["migrants"]) for m in r["migrations"]]))
    # test_solver.cpp:227-271: J=8, S=2, M=[2,2], weight 0, population 64, gap 1 -- migrations fire
    found = 0
    for seed in range(1, 51):
        d = ref.generate(8, 2, [2, 2], weight=0.0, seed=seed)
        r = ref.instance(d).run(population=64, generations=30, gap=1, theta=1.0, seed=seed)
        if not r["migrations"]:
            continue
        out["run"].append(dict(J=8, S=2, machines=[2, 2], gen_seed=seed, weight=0.0, population=64, generations=30,
                               gap=1, theta=1.0, seed=seed, best_objective=hx(r["best_objective"]),
                               best_chromosome=r["best_chromosome"],
                               trace_combined=[hx(v) for v in r["trace_combined"]],
                               migrations=[dict(generation=m["generation"], beta=hx(m["beta"]),
                                                alpha=hx(m["alpha"]), direction=m["direction"],
                                                migrants=m["migrants"]) for m in r["migrations"]]))
        found += 1
        if found == 3:
            break
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_vectors.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
