"""B200-native (sm_100a) flexible-flow-shop GA hot path with the reference's Python API.

The names below are the reference package's public surface (proj/python/ffsga/__init__.py:1-32),
served by the pybind11 module `_core` over the device-backed C++ API (csrc/host), which calls
the sm_100a kernels through the C ABI (include/ffsga_cuda.h).  Extensions:

* ``evaluate_batch``  -- Evaluator::score over many chromosomes in one K1 launch;
* ``capi``            -- ctypes view of the C ABI (batches, islands, step, migration);
* ``islands``         -- the multi-island / multi-GPU driver (torch.distributed plumbing).

There is no CPU fallback: without an sm_100 GPU every evaluation raises DeviceError.
"""
from types import SimpleNamespace

import numpy as np

from ._core import (
    ConfigError,
    ContractError,
    DeviceError,
    Instance,
    IoError,
    estimate_emax,
    evaluate_assignment,
    evaluate_batch,
    generate_instance,
    load_instance,
    mean_total_load,
    save_instance,
    solve,
)

__version__ = "0.1.0"


def instance_arrays(inst: Instance) -> SimpleNamespace:
    """Plain arrays of an Instance (job-major proc), the form the C ABI takes."""
    return SimpleNamespace(num_jobs=inst.num_jobs, num_stages=inst.num_stages,
                           machines=list(inst.machines_per_stage),
                           proc=np.asarray(inst.proc, dtype=np.float64),
                           release=np.asarray(inst.release, dtype=np.float64),
                           due=np.asarray(inst.due, dtype=np.float64), weight=float(inst.weight))


__all__ = [
    "ConfigError",
    "ContractError",
    "DeviceError",
    "Instance",
    "IoError",
    "estimate_emax",
    "evaluate_assignment",
    "evaluate_batch",
    "generate_instance",
    "instance_arrays",
    "load_instance",
    "mean_total_load",
    "save_instance",
    "solve",
    "__version__",
]
