"""Shared fixtures.  The oracle (oracle/pyoracle.py) is test infrastructure: the checker."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (run with -m gpu on a B200)")
    config.addinivalue_line("markers", "slow: long parity sweeps")


@pytest.fixture(scope="session")
def orc():
    from pyoracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from pyoracle import RefLib, have_ref
    if not have_ref():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return RefLib()


def synthetic(orc, jobs, stages, lo=2, hi=8, weight=100.0, seed=7, integer_times=False):
    """SURVEY 8(d) synthetic convention."""
    from pyoracle import synthetic_machines
    m = synthetic_machines(jobs, stages, lo, hi)
    return orc.generate(jobs, stages, m, weight=weight, seed=seed, integer_times=integer_times)


@pytest.fixture(autouse=True)
def _device_checks(request):
    """With FFSGA_CUDA_LIB pointing at the checked build (python build.py --checked), every GPU
    test also asserts that no device-side bounds / invariant check failed during it."""
    yield
    if os.environ.get("FFSGA_CUDA_LIB") and request.node.get_closest_marker("gpu"):
        from paper_1903_10722_b200 import capi
        st = capi.checked_status(reset=True)  # -1: the library is not a checked build
        assert st in (0, -1), f"device check {st >> 48} failed (a={(st >> 24) & 0xFFFFFF}, b={st & 0xFFFFFF})"
