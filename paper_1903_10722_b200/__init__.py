"""B200-native (sm_100a) flexible-flow-shop GA hot path with the reference's Python API.

The names below are the reference package's public surface (proj/python/ffsga/__init__.py:1-32),
served by the pybind11 module `_core` over the device-backed C++ API (csrc/host), which calls
the sm_100a kernels through the C ABI (include/ffsga_cuda.h).  Extensions:

* ``evaluate_batch``  -- Evaluator::score over many chromosomes in one K1 launch;
* ``evaluate_tensor`` -- the same over a population already on the GPU (a torch CUDA tensor),
  results returned as CUDA tensors, ordered on the tensor's current stream;
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

_device_instances = {}


def _device_instance(inst: Instance, device: int):
    """One C-ABI instance per distinct (device, instance contents), reused across calls."""
    from . import capi
    a = instance_arrays(inst)
    key = (device, a.num_jobs, a.num_stages, tuple(a.machines), a.weight, a.proc.tobytes(), a.release.tobytes(),
           a.due.tobytes())
    h = _device_instances.get(key)
    if h is None:
        if len(_device_instances) >= 4:
            _device_instances.pop(next(iter(_device_instances)))
        h = capi.Instance.from_data(a, estimate_emax(inst), device)
        _device_instances[key] = h
    return h


def evaluate_tensor(inst: Instance, genes, full: bool = False):
    """Evaluator::score over a device-resident population: `genes` is a CUDA tensor of shape
    (n, num_jobs * num_stages), job-major machine indices (any integer dtype; uint8 avoids a
    conversion).  Returns CUDA float64 tensors (objective, fitness[, makespan, tardiness]); the
    work is ordered on torch's current stream.  Out-of-range genes raise ContractError."""
    import torch
    if not (isinstance(genes, torch.Tensor) and genes.is_cuda):
        raise ValueError("evaluate_tensor expects a CUDA tensor")
    L = inst.num_jobs * inst.num_stages
    if genes.dim() != 2 or genes.shape[1] != L:
        raise ValueError("evaluate_tensor: genes must have shape (n, num_jobs * num_stages)")
    if genes.dtype != torch.uint8:  # out-of-range values must stay out of range after narrowing
        genes = torch.where((genes < 0) | (genes > 254), torch.full_like(genes, 255), genes).to(torch.uint8)
    genes = genes.contiguous()
    h = _device_instance(inst, genes.device.index or 0)
    n = genes.shape[0]
    with torch.cuda.device(genes.device):
        out = [torch.empty(n, dtype=torch.float64, device=genes.device) for _ in range(4 if full else 2)]
        stream = torch.cuda.current_stream(genes.device).cuda_stream
        h.evaluate_device(genes.data_ptr(), n, out[0].data_ptr(), out[1].data_ptr(),
                          out[2].data_ptr() if full else None, out[3].data_ptr() if full else None, stream)
    return tuple(out)


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
    "evaluate_tensor",
    "generate_instance",
    "instance_arrays",
    "load_instance",
    "mean_total_load",
    "save_instance",
    "solve",
    "__version__",
]
