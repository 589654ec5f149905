"""Host-side pieces of the product API (pybind `_core` over the C++ API), CPU only: instance
generation, E_max, loads and JSON files, checked against the oracle and the compiled reference.
Mirrors the reference's Python smoke tests (proj/tests/python/test_smoke.py) where no GPU is needed."""
import math

import numpy as np
import pytest

import paper_1903_10722_b200 as ffsga


@pytest.fixture(scope="module")
def instance():
    return ffsga.generate_instance(jobs=6, stages=2, machines=[2], seed=5)


def test_version():
    assert isinstance(ffsga.__version__, str) and ffsga.__version__


def test_generated_instance_shape(instance):  # test_smoke.py:19-36
    assert instance.num_jobs == 6 and instance.num_stages == 2
    assert instance.machines_per_stage == [2, 2] and instance.num_genes == 12
    assert len(instance.release) == 6 and len(instance.due) == 6 and instance.weight == 100.0
    for j in range(6):
        assert instance.release[j] >= 0.0 and instance.due[j] >= instance.release[j]
        for s in range(2):
            for m in range(2):
                assert 1.0 <= instance.proc_time(j, s, m) < 5.0
    assert "6 jobs" in repr(instance)


def test_generator_bitwise_vs_oracle(orc):
    for (J, S, M, seed, it) in [(6, 2, [2, 2], 5, False), (500, 20, [5, 2, 2, 8, 4, 7, 6, 5, 7, 8, 3, 8, 3, 6, 3, 5,
                                                                     5, 2, 5, 2], 7, False),
                                (40, 6, [2, 3, 4, 2, 3, 2], 3, True)]:
        a = ffsga.generate_instance(jobs=J, stages=S, machines=M, seed=seed, integer_times=it)
        b = orc.generate(J, S, M, seed=seed, integer_times=it)
        assert np.array_equal(np.array(a.proc), b.proc)
        assert np.array_equal(np.array(a.release), b.release) and np.array_equal(np.array(a.due), b.due)
        oi = orc.instance(b)
        assert ffsga.estimate_emax(a) == oi.estimate_emax()
        assert ffsga.mean_total_load(a) == oi.mean_total_load()


def test_generator_vs_reference(ref):
    a = ffsga.generate_instance(jobs=100, stages=10, machines=[4, 2, 2, 3, 4, 4, 2, 3, 4, 5], seed=7)
    b = ref.generate(100, 10, [4, 2, 2, 3, 4, 4, 2, 3, 4, 5], seed=7)
    assert np.array_equal(np.array(a.proc), b.proc) and np.array_equal(np.array(a.due), b.due)
    assert ffsga.estimate_emax(a) == ref.instance(b).estimate_emax()


def test_invalid_parameters_raise_value_error():  # test_smoke.py:49-53
    with pytest.raises(ValueError):
        ffsga.generate_instance(jobs=0)
    with pytest.raises(ValueError):
        ffsga.generate_instance(jobs=4, stages=2, machines=[1, 1])


def test_mean_total_load(instance):  # test_smoke.py:80-86
    total = 0.0
    for j in range(instance.num_jobs):
        for s in range(instance.num_stages):
            m = instance.machines_per_stage[s]
            total += sum(instance.proc_time(j, s, k) for k in range(m)) / m
    assert math.isclose(ffsga.mean_total_load(instance), total, rel_tol=1e-12)


def test_files_round_trip(tmp_path, instance):  # test_smoke.py:127-142
    p = tmp_path / "instance.json"
    ffsga.save_instance(instance, str(p))
    back = ffsga.load_instance(str(p))
    assert back.num_jobs == instance.num_jobs and back.release == instance.release and back.due == instance.due
    assert [back.proc_time(2, 1, m) for m in range(2)] == [instance.proc_time(2, 1, m) for m in range(2)]
    text = p.read_text()
    assert text.startswith('{\n  "num_jobs": 6,\n  "num_stages": 2,\n  "machines_per_stage": [')
    with pytest.raises(OSError):
        ffsga.load_instance(str(tmp_path / "missing.json"))
    (tmp_path / "bad.json").write_text('{"num_jobs": 1}')
    with pytest.raises(OSError, match="num_stages"):
        ffsga.load_instance(str(tmp_path / "bad.json"))
