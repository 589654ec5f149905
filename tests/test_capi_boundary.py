"""The C-ABI library loads and exports every symbol include/ffsga_cuda.h declares (CPU only:
no compute call is made without a GPU, except to check that it fails loudly)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    text = open(os.path.join(ROOT, "include", "ffsga_cuda.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ffsga_cuda_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    from paper_1903_10722_b200 import capi
    lib = ctypes.CDLL(capi.LIB_PATH)
    names = declared()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding covers the whole header
    assert sorted(set(capi.exported_symbols())) == names


def test_abi_version():
    from paper_1903_10722_b200 import capi
    assert capi.lib().ffsga_cuda_abi_version() == 1


def test_no_gpu_fails_loudly():
    from paper_1903_10722_b200 import capi
    if capi.device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(capi.CudaError, match="no CUDA device"):
        capi.Instance(2, 2, [2, 1], [2, 3, 4, 2, 3, 1], [0, 0], [10, 10], 100.0, 211.0)
    import paper_1903_10722_b200 as f
    inst = f.generate_instance(jobs=4, stages=2, machines=[2], seed=1)
    with pytest.raises(f.DeviceError):
        f.evaluate_assignment(inst, [0] * inst.num_genes)


def test_product_does_not_import_oracle():
    """The product package never reaches into oracle/ (the checker)."""
    pkg = os.path.join(ROOT, "paper_1903_10722_b200")
    for base, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")):
                src = open(os.path.join(base, fn), errors="ignore").read()
                assert "pyoracle" not in src and "ffsga_oracle" not in src and "liboracle" not in src, fn


def test_device_plane_entry_points_validate_arguments():
    """The device-packet entry points reject bad arguments before touching the device (runs
    without a GPU): the same status codes as the rest of the C ABI."""
    from paper_1903_10722_b200 import capi
    L = capi.lib()
    n = ctypes.c_int64(0)
    assert L.ffsga_cuda_packet_bytes(None, 0, 1, ctypes.byref(n)) == capi.FFSGA_ERR_ARG
    for f in (L.ffsga_cuda_cellular_export_device, L.ffsga_cuda_pseudo_export_device,
              L.ffsga_cuda_cellular_import_device, L.ffsga_cuda_pseudo_import_device):
        assert f(None, 1, None, None) == capi.FFSGA_ERR_ARG
        assert "null island" in L.ffsga_cuda_last_error().decode()
    for f in (L.ffsga_cuda_cellular_state_device, L.ffsga_cuda_pseudo_state_device):
        assert f(None, None, None) == capi.FFSGA_ERR_ARG
    assert L.ffsga_cuda_timing_busy(None, 0, None) == capi.FFSGA_ERR_ARG
    assert L.ffsga_cuda_checked_status(0, None) == capi.FFSGA_ERR_ARG
