"""The command-line front end (paper_1903_10722_b200/bin/ffsga) against the reference CLI's own
test cases (proj/tests/test_cli.cpp).  Parsing, `generate` and every error path run on the host;
the subcommands that solve are marked gpu."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1903_10722_b200", "bin", "ffsga")


def run_cli(*args):
    assert os.path.exists(CLI), "build the CLI first: python build.py"
    p = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout, p.stderr


def lines_of(path):
    with open(path) as f:
        return f.read().splitlines()


def test_help_and_missing_subcommand():
    # test_cli.cpp:74-83
    assert run_cli("--help")[0] == 0
    assert run_cli("solve", "--help")[0] == 0
    code, _, err = run_cli()
    assert code == 2 and err.startswith("error: ")
    code, _, err = run_cli("solve", "--no-such-flag")
    assert code == 2 and err.startswith("error: ")
    code, _, err = run_cli("no-such-command")
    assert code == 2 and err.startswith("error: ")


def test_generate_reports_shape_and_writes_instance(tmp_path, orc):
    # test_cli.cpp:85-106
    path = tmp_path / "generated.json"
    code, out, _ = run_cli("generate", "--jobs", 6, "--stages", 2, "--machines", 2, "--seed", 5, "--out", path)
    assert code == 0
    assert "instance: 6 jobs, 2 stages, machines 2 2, weight 100" in out
    assert "mean total load: " in out and "due range: [" in out and f"wrote {path}" in out
    doc = json.loads(path.read_text())
    assert doc["num_jobs"] == 6 and doc["num_stages"] == 2 and doc["machines_per_stage"] == [2, 2]
    mixed = tmp_path / "mixed.json"
    assert run_cli("generate", "--jobs", 4, "--stages", 3, "--machines", "2,1,3", "--out", mixed)[0] == 0
    assert json.loads(mixed.read_text())["machines_per_stage"] == [2, 1, 3]
    # the instance is the reference generator's: same arrays as the oracle's restatement
    d = orc.generate(6, 2, [2, 2], seed=5)
    import numpy as np
    assert np.array_equal(np.asarray(doc["release"], dtype=np.float64), d.release)
    assert np.array_equal(np.asarray(doc["due"], dtype=np.float64), d.due)


def test_invalid_generator_parameters(tmp_path):
    # test_cli.cpp:108-115: one line, "error: " prefix, no file written
    never = tmp_path / "never.json"
    code, _, err = run_cli("generate", "--jobs", 0, "--out", never)
    assert code == 2
    assert len(err.splitlines()) == 1 and err.startswith("error: ")
    assert not never.exists()
    code, _, err = run_cli("generate", "--jobs", "six")
    assert code == 2 and "--jobs" in err


def test_missing_instance_file():
    # test_cli.cpp:185-190
    code, _, err = run_cli("solve", "--instance", "/nonexistent/input.json")
    assert code == 2 and err.startswith("error: ") and "/nonexistent/input.json" in err


def test_argument_conflicts(tmp_path):
    # test_cli.cpp:212-216 (--runs 1 for compare) and 236-246 (--instance with --vary-instance)
    code, _, err = run_cli("compare", "--jobs", 6, "--stages", 2, "--machines", 2, "--population", 16,
                           "--generations", 5, "--runs", 1)
    assert code == 2 and "--runs" in err
    inst = tmp_path / "sweep_input.json"
    assert run_cli("generate", "--jobs", 6, "--stages", 2, "--machines", 2, "--out", inst)[0] == 0
    code, _, err = run_cli("sweep-gap", "--instance", inst, "--vary-instance", "--population", 16,
                           "--generations", 5, "--gaps", 2, "--runs", 2)
    assert code == 2 and "--vary-instance" in err


@pytest.mark.gpu
def test_solve_result_and_trace(tmp_path):
    # test_cli.cpp:117-146
    inst = tmp_path / "solve_input.json"
    assert run_cli("generate", "--jobs", 6, "--stages", 2, "--machines", 2, "--seed", 9, "--out", inst)[0] == 0
    out, trace = tmp_path / "solve_result.json", tmp_path / "solve_trace.csv"
    code, text, err = run_cli("solve", "--instance", inst, "--population", 16, "--generations", 10, "--gap", 5,
                              "--seed", 3, "--out", out, "--trace", trace)
    assert code == 0, err
    for s in ("best objective: ", "migrations executed: ", "total seconds: ", f"wrote {out}", f"wrote {trace}"):
        assert s in text
    doc = json.loads(out.read_text())
    assert doc["schema"] == "ffsga-result-v1" and doc["config"]["mode"] == "dual"
    assert doc["config"]["population"] == 16 and doc["config"]["generations"] == 10
    assert isinstance(doc["best"]["objective"], float)
    rows = lines_of(trace)
    assert len(rows) == 11
    assert rows[0] == ("generation,best_objective_combined,best_objective_island_a,best_objective_island_b,"
                       "migration_flag")
    assert rows[1].startswith("1,") and rows[10].startswith("10,")


@pytest.mark.gpu
def test_solve_matches_reference_run(tmp_path, ref):
    """The CLI's result equals the compiled reference's run() on the same instance file."""
    import numpy as np
    from pyoracle import InstanceData
    inst = tmp_path / "in.json"
    assert run_cli("generate", "--jobs", 12, "--stages", 3, "--machines", "2,3,2", "--seed", 4, "--out", inst)[0] == 0
    out = tmp_path / "out.json"
    code, _, err = run_cli("solve", "--instance", inst, "--population", 32, "--generations", 30, "--gap", 10,
                           "--seed", 6, "--out", out)
    assert code == 0, err
    doc = json.loads(out.read_text())
    j = json.loads(inst.read_text())
    proc = np.array([[p for stage in job for p in stage] for job in j["proc_time"]], dtype=np.float64)
    d = InstanceData(j["num_jobs"], j["num_stages"], j["machines_per_stage"], proc, j["release"], j["due"],
                     j["weight"])
    r = ref.instance(d).run(population=32, generations=30, gap=10, seed=6)
    assert doc["best"]["objective"] == r["best_objective"]
    assert doc["best"]["chromosome"] == r["best_chromosome"]


@pytest.mark.gpu
def test_solve_deterministic_across_workers_and_drivers(tmp_path):
    # test_cli.cpp:148-183
    inst = tmp_path / "det_input.json"
    assert run_cli("generate", "--jobs", 8, "--stages", 2, "--machines", 2, "--seed", 21, "--out", inst)[0] == 0
    results, traces = [], []
    for label, flags in (("w1", ["--workers", 1]), ("w4", ["--workers", 4]), ("ser", ["--workers", 4, "--serialized"])):
        out, trace = tmp_path / f"det_{label}.json", tmp_path / f"det_{label}.csv"
        assert run_cli("solve", "--instance", inst, "--population", 16, "--generations", 15, "--gap", 5, "--seed", 2,
                       *flags, "--out", out, "--trace", trace)[0] == 0
        doc = json.loads(out.read_text())
        doc.pop("timings", None)
        results.append(doc)
        traces.append(trace.read_text())
    assert results[0] == results[1] == results[2]
    assert traces[0] == traces[1] == traces[2]


@pytest.mark.gpu
def test_compare_sweep_and_bench_tables(tmp_path):
    # test_cli.cpp:192-234, 248-262
    out = tmp_path / "compare.csv"
    code, text, err = run_cli("compare", "--jobs", 6, "--stages", 2, "--machines", 2, "--instance-seed", 4,
                              "--population", 16, "--generations", 8, "--runs", 2, "--seed", 11, "--out", out)
    assert code == 0, err
    rows = lines_of(out)
    assert rows[0] == "algorithm,best,average,variance" and len(rows) == 4
    assert [r.split(",")[0] for r in rows[1:]] == ["Heterogeneous", "Cellular", "Pseudo"]
    assert "algorithm,best,average,variance" in text
    out = tmp_path / "sweep.csv"
    assert run_cli("sweep-gap", "--jobs", 6, "--stages", 2, "--machines", 2, "--instance-seed", 8, "--population", 16,
                   "--generations", 9, "--gaps", "3,5", "--runs", 2, "--seed", 13, "--out", out)[0] == 0
    rows = lines_of(out)
    assert rows[0] == "gap,mean_objective,std" and rows[1].startswith("3,") and rows[2].startswith("5,")
    out = tmp_path / "bench.csv"
    assert run_cli("bench-time", "--jobs", 6, "--stages", 2, "--machines", 2, "--population", 16, "--generations", 5,
                   "--populations", "8,16", "--out", out)[0] == 0
    rows = lines_of(out)
    assert rows[0] == "population,concurrent_seconds,serialized_seconds,speedup"
    assert rows[1].startswith("8,") and rows[2].startswith("16,")


def _doc_without_timings(text):
    from collections import OrderedDict
    doc = json.loads(text, parse_float=str, object_pairs_hook=OrderedDict)  # numbers keep their text
    doc.pop("timings", None)
    return doc


def test_instance_file_bytes_match_reference(tmp_path, ref):
    """`generate` writes the reference's instance JSON byte for byte (io.cpp save_instance)."""
    import numpy as np
    from pyoracle import InstanceData
    ours = tmp_path / "ours.json"
    assert run_cli("generate", "--jobs", 30, "--stages", 4, "--machines", "2,3,1,4", "--seed", 11, "--wt", 7.5,
                   "--out", ours)[0] == 0
    d = ref.generate(30, 4, [2, 3, 1, 4], weight=7.5, seed=11)
    theirs = tmp_path / "theirs.json"
    ref.instance(d).save(theirs)
    assert ours.read_bytes() == theirs.read_bytes()


@pytest.mark.gpu
def test_result_and_trace_files_match_reference(tmp_path, ref):
    """`solve` writes the reference's result JSON (outside `timings`) and trace CSV byte for byte
    (io.cpp save_result_json / save_trace_csv), migrations included."""
    import numpy as np
    from pyoracle import InstanceData
    for seed in (4, 12):  # tests/golden: runs with migrations at these seeds
        inst = tmp_path / f"in{seed}.json"
        assert run_cli("generate", "--jobs", 8, "--stages", 2, "--machines", 2, "--wt", 0, "--seed", seed,
                       "--out", inst)[0] == 0
        ours, ours_tr = tmp_path / f"ours{seed}.json", tmp_path / f"ours{seed}.csv"
        code, _, err = run_cli("solve", "--instance", inst, "--population", 64, "--generations", 30, "--gap", 1,
                               "--seed", seed, "--out", ours, "--trace", ours_tr)
        assert code == 0, err
        d = ref.generate(8, 2, [2, 2], weight=0.0, seed=seed)
        theirs, theirs_tr = tmp_path / f"theirs{seed}.json", tmp_path / f"theirs{seed}.csv"
        r = ref.instance(d).run(population=64, generations=30, gap=1, seed=seed, result_json=theirs,
                                trace_csv=theirs_tr)
        assert r["migrations"], "the fixture seeds fire migrations"
        assert _doc_without_timings(ours.read_text()) == _doc_without_timings(theirs.read_text())
        assert ours_tr.read_bytes() == theirs_tr.read_bytes()


@pytest.mark.gpu
def test_c2_run_files_match_reference(tmp_path, ref):
    """C2: 100 x 10 x [2, 5], dual, population 4096 (grid 64 x 32 + 1024 pairs),
    migration gap 500, 600 generations so the run crosses a rendezvous: the result JSON (outside
    timings) and the trace CSV byte for byte against the compiled reference's run()
    (proj/src/solver.cpp:58-164, proj/src/io.cpp)."""
    from pyoracle import synthetic_machines
    machines = synthetic_machines(100, 10, 2, 5)
    inst = tmp_path / "c2.json"
    assert run_cli("generate", "--jobs", 100, "--stages", 10, "--machines", ",".join(map(str, machines)),
                   "--seed", 7, "--out", inst)[0] == 0
    ours, ours_tr = tmp_path / "ours.json", tmp_path / "ours.csv"
    code, _, err = run_cli("solve", "--instance", inst, "--population", 4096, "--generations", 600, "--gap", 500,
                           "--seed", 1, "--out", ours, "--trace", ours_tr)
    assert code == 0, err
    d = ref.generate(100, 10, machines, weight=100.0, seed=7)
    theirs, theirs_tr = tmp_path / "theirs.json", tmp_path / "theirs.csv"
    r = ref.instance(d).run(population=4096, generations=600, gap=500, seed=1, workers=os.cpu_count() or 1,
                            result_json=theirs, trace_csv=theirs_tr)
    assert len(r["trace_combined"]) == 600
    assert _doc_without_timings(ours.read_text()) == _doc_without_timings(theirs.read_text())
    assert ours_tr.read_bytes() == theirs_tr.read_bytes()
