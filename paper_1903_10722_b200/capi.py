"""ctypes binding of the C ABI (include/ffsga_cuda.h) -- the thin Python view of the device path.

This is the same binding a reference-side maintainer would add.  It loads the
in-tree ``libffsga_cuda.so`` and fails loudly when it is missing or when no sm_100 device is
present: there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# FFSGA_CUDA_LIB: load another build of the same library (the checked build of
# `python build.py --checked`, paper_1903_10722_b200/checked/libffsga_cuda.so)
LIB_PATH = os.environ.get("FFSGA_CUDA_LIB") or os.path.join(HERE, "libffsga_cuda.so")

FFSGA_OK, FFSGA_ERR_CONTRACT, FFSGA_ERR_CONFIG, FFSGA_ERR_CUDA, FFSGA_ERR_OOM, FFSGA_ERR_ARG = range(6)

_i32, _i64, _u64, _f64, _vp = C.c_int, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
_pi32 = C.POINTER(C.c_int32)
_pd = C.POINTER(C.c_double)
_pu8 = C.POINTER(C.c_uint8)
_pvp = C.POINTER(C.c_void_p)


class FfsgaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class ContractError(FfsgaError, ValueError):
    """Mirrors ffsga::ContractError (errors.hpp:14-16), a ValueError in Python (module.cpp:73)."""


class ConfigError(FfsgaError, ValueError):
    """Mirrors ffsga::ConfigError (errors.hpp:19-21), a ValueError in Python (module.cpp:72)."""


class CudaError(FfsgaError):
    pass


_SIGS = {
    "ffsga_cuda_last_error": (C.c_char_p, []),
    "ffsga_cuda_abi_version": (_i32, []),
    "ffsga_cuda_device_count": (_i32, [C.POINTER(_i32)]),
    "ffsga_cuda_instance_create": (_i32, [_i32, _i32, _i32, _pi32, _pd, _pd, _pd, _f64, _f64, _pvp]),
    "ffsga_cuda_instance_destroy": (_i32, [_vp]),
    "ffsga_cuda_instance_info": (_i32, [_vp, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32)]),
    "ffsga_cuda_evaluate": (_i32, [_vp, _pi32, _i64, _pd, _pd, _pd, _pd]),
    "ffsga_cuda_evaluate_u8": (_i32, [_vp, _pu8, _i64, _pd, _pd, _pd, _pd]),
    "ffsga_cuda_evaluate_device": (_i32, [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "ffsga_cuda_decode": (_i32, [_vp, _pi32, _pi32, _pd, _pd, _pd]),
    "ffsga_cuda_batch_create": (_i32, [_vp, _i64, _pvp]),
    "ffsga_cuda_batch_destroy": (_i32, [_vp]),
    "ffsga_cuda_batch_fill_random": (_i32, [_vp, _u64, _i64, _i64]),
    "ffsga_cuda_batch_upload": (_i32, [_vp, _pi32, _i64]),
    "ffsga_cuda_batch_upload_u8": (_i32, [_vp, _pu8, _i64]),
    "ffsga_cuda_batch_evaluate": (_i32, [_vp, _i64]),
    "ffsga_cuda_batch_results": (_i32, [_vp, _i64, _pd, _pd, _pd, _pd]),
    "ffsga_cuda_batch_device_results": (_i32, [_vp, _pvp, _pvp]),
    "ffsga_cuda_batch_download": (_i32, [_vp, _i64, _i64, _pi32]),
    "ffsga_cuda_batch_sync": (_i32, [_vp]),
    "ffsga_cuda_batch_last_eval_ms": (_i32, [_vp, C.POINTER(C.c_float)]),
    "ffsga_cuda_cellular_create": (_i32, [_vp, _i32, _i32, _i32, _f64, _f64, _u64, _pi32, _pvp]),
    "ffsga_cuda_cellular_destroy": (_i32, [_vp]),
    "ffsga_cuda_cellular_size": (_i32, [_vp, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32)]),
    "ffsga_cuda_cellular_generation": (_i32, [_vp, C.POINTER(_u64)]),
    "ffsga_cuda_cellular_read": (_i32, [_vp, _pd, _pd]),
    "ffsga_cuda_cellular_genes": (_i32, [_vp, _i32, _pi32]),
    "ffsga_cuda_cellular_slots": (_i32, [_vp, _i32, _pi32]),
    "ffsga_cuda_cellular_best": (_i32, [_vp, C.POINTER(_i32), _pd, _pd]),
    "ffsga_cuda_cellular_install": (_i32, [_vp, _i32, _pi32, _f64, _f64]),
    "ffsga_cuda_cellular_candidate": (_i32, [_vp, _i32, _u64, _pi32, _pd, _pd, C.POINTER(_i32), C.POINTER(_u64)]),
    "ffsga_cuda_pseudo_create": (_i32, [_vp, _i32, _f64, _u64, _pvp]),
    "ffsga_cuda_pseudo_destroy": (_i32, [_vp]),
    "ffsga_cuda_pseudo_size": (_i32, [_vp, C.POINTER(_i32), C.POINTER(_i32)]),
    "ffsga_cuda_pseudo_generation": (_i32, [_vp, C.POINTER(_u64)]),
    "ffsga_cuda_pseudo_read": (_i32, [_vp, _pd, _pd]),
    "ffsga_cuda_pseudo_member": (_i32, [_vp, _i32, _pu8]),
    "ffsga_cuda_pseudo_best": (_i32, [_vp, C.POINTER(_i32), _pd, _pd]),
    "ffsga_cuda_pseudo_archive": (_i32, [_vp, _pd, _pd, _pu8]),
    "ffsga_cuda_pseudo_install": (_i32, [_vp, _i32, _pu8, _f64, _f64]),
    "ffsga_cuda_pseudo_archive_genes": (_i32, [_vp, _pi32]),
    "ffsga_cuda_step": (_i32, [_pvp, _i32, _pvp, _i32, _i32, _pd, _pd]),
    "ffsga_cuda_migrate_cellular_to_pseudo": (_i32, [_vp, _vp, _i32]),
    "ffsga_cuda_migrate_pseudo_to_cellular": (_i32, [_vp, _vp, _i32]),
    "ffsga_cuda_cellular_export": (_i32, [_vp, _i32, _pi32, _pd, _pd]),
    "ffsga_cuda_pseudo_export": (_i32, [_vp, _i32, _pu8, _pd, _pd]),
    "ffsga_cuda_cellular_import": (_i32, [_vp, _i32, _pu8, _pd, _pd]),
    "ffsga_cuda_pseudo_import": (_i32, [_vp, _i32, _pi32, _pd, _pd]),
    "ffsga_cuda_packet_bytes": (_i32, [_vp, _i32, _i32, C.POINTER(_i64)]),
    "ffsga_cuda_cellular_export_device": (_i32, [_vp, _i32, _vp, _vp]),
    "ffsga_cuda_pseudo_export_device": (_i32, [_vp, _i32, _vp, _vp]),
    "ffsga_cuda_cellular_import_device": (_i32, [_vp, _i32, _vp, _vp]),
    "ffsga_cuda_pseudo_import_device": (_i32, [_vp, _i32, _vp, _vp]),
    "ffsga_cuda_cellular_state_device": (_i32, [_vp, _vp, _vp]),
    "ffsga_cuda_pseudo_state_device": (_i32, [_vp, _vp, _vp]),
    "ffsga_cuda_last_step_ms": (_i32, [_vp, C.POINTER(C.c_float)]),
    "ffsga_cuda_evaluations": (_i32, [_vp, C.POINTER(_i64)]),
    "ffsga_cuda_set_timing": (_i32, [_vp, _i32]),
    "ffsga_cuda_timing": (_i32, [_vp, _i32, _pd, C.POINTER(_i64)]),
    "ffsga_cuda_timing_busy": (_i32, [_vp, _i32, _pd]),
    "ffsga_cuda_reset_timing": (_i32, [_vp]),
    "ffsga_cuda_launch_count": (_i32, [C.POINTER(_i64)]),
    "ffsga_cuda_checked_status": (_i32, [_i32, C.POINTER(_i64)]),
}

_lib = None


def lib():
    """Load libffsga_cuda.so (raises if the extension was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python build.py` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def _check(status):
    if status == FFSGA_OK:
        return
    msg = lib().ffsga_cuda_last_error().decode()
    cls = {FFSGA_ERR_CONTRACT: ContractError, FFSGA_ERR_CONFIG: ConfigError}.get(status, CudaError)
    raise cls(status, msg)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def device_count():
    n = C.c_int(0)
    _check(lib().ffsga_cuda_device_count(C.byref(n)))
    return n.value


def checked_status(reset=True):
    """First failed device check of a checked build (0 = none), -1 from a normal build."""
    n = C.c_int64(0)
    _check(lib().ffsga_cuda_checked_status(int(reset), C.byref(n)))
    return n.value


def launch_count():
    n = C.c_int64(0)
    _check(lib().ffsga_cuda_launch_count(C.byref(n)))
    return n.value


class Instance:
    """Device copy of one FFS instance (ffsga_cuda_instance)."""

    def __init__(self, num_jobs, num_stages, machines, proc, release, due, weight, emax, device=0):
        self.num_jobs, self.num_stages = int(num_jobs), int(num_stages)
        self.machines = np.ascontiguousarray(machines, dtype=np.int32)
        proc = np.ascontiguousarray(proc, dtype=np.float64)
        release = np.ascontiguousarray(release, dtype=np.float64)
        due = np.ascontiguousarray(due, dtype=np.float64)
        self.emax = float(emax)
        self.device = int(device)
        h = C.c_void_p()
        _check(lib().ffsga_cuda_instance_create(device, self.num_jobs, self.num_stages, _p(self.machines, _pi32),
                                                _p(proc, _pd), _p(release, _pd), _p(due, _pd), float(weight),
                                                self.emax, C.byref(h)))
        self.h = h

    @classmethod
    def from_data(cls, data, emax, device=0):
        return cls(data.num_jobs, data.num_stages, data.machines, data.proc, data.release, data.due,
                   data.weight, emax, device)

    def close(self):
        if getattr(self, "h", None):
            lib().ffsga_cuda_instance_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def num_genes(self):
        return self.num_jobs * self.num_stages

    def info(self):
        a, b, c, d = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(lib().ffsga_cuda_instance_info(self.h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        return dict(row_stride=a.value, group_lanes=b.value, total_bits=c.value, smem_per_group=d.value)

    def evaluate(self, genes, full=False):
        """Evaluator::score over a batch -> (objective, fitness[, makespan, tardiness])."""
        genes = np.asarray(genes)
        if genes.dtype == np.uint8:
            g = np.ascontiguousarray(genes).reshape(-1, self.num_genes)
            fn = lib().ffsga_cuda_evaluate_u8
            gp = _p(g, _pu8)
        else:
            g = np.ascontiguousarray(genes, dtype=np.int32).reshape(-1, self.num_genes)
            fn = lib().ffsga_cuda_evaluate
            gp = _p(g, _pi32)
        n = g.shape[0]
        obj, fit = np.empty(n), np.empty(n)
        mk = np.empty(n) if full else None
        td = np.empty(n) if full else None
        _check(fn(self.h, gp, n, _p(obj, _pd), _p(fit, _pd), _p(mk, _pd), _p(td, _pd)))
        return (obj, fit, mk, td) if full else (obj, fit)

    def evaluate_device(self, genes_ptr, n, obj_ptr, fit_ptr, mk_ptr=None, td_ptr=None, stream=None):
        """Evaluator::score over n device-resident job-major u8 chromosomes; every argument is a
        raw device pointer (int), results land in device memory, ordered on `stream`."""
        _check(lib().ffsga_cuda_evaluate_device(self.h, C.c_void_p(genes_ptr), n, C.c_void_p(obj_ptr),
                                                C.c_void_p(fit_ptr), C.c_void_p(mk_ptr or 0), C.c_void_p(td_ptr or 0),
                                                C.c_void_p(stream or 0)))

    def decode(self, genes):
        """decode + evaluate of one chromosome -> (machine, start, completion, report dict)."""
        g = np.ascontiguousarray(genes, dtype=np.int32).reshape(self.num_genes)
        L = self.num_genes
        m, s, c, r = np.empty(L, dtype=np.int32), np.empty(L), np.empty(L), np.empty(5)
        _check(lib().ffsga_cuda_decode(self.h, _p(g, _pi32), _p(m, _pi32), _p(s, _pd), _p(c, _pd), _p(r, _pd)))
        rep = dict(makespan=r[0], total_tardiness=r[1], objective=r[2], fitness=r[3], emax_used=r[4])
        return m, s, c, rep

    def packet_bytes(self, from_kind, k):
        """Bytes of a migrant packet of k members leaving a cellular (0) or pseudo (1) island."""
        n = C.c_int64()
        _check(lib().ffsga_cuda_packet_bytes(self.h, int(from_kind), int(k), C.byref(n)))
        return n.value

    def last_step_ms(self):
        ms = C.c_float()
        _check(lib().ffsga_cuda_last_step_ms(self.h, C.byref(ms)))
        return ms.value

    def evaluations(self):
        n = C.c_int64()
        _check(lib().ffsga_cuda_evaluations(self.h, C.byref(n)))
        return n.value

    def set_timing(self, on=True):
        _check(lib().ffsga_cuda_set_timing(self.h, int(on)))

    def reset_timing(self):
        _check(lib().ffsga_cuda_reset_timing(self.h))

    def timing_busy(self, which):
        """Milliseconds during which at least one launch of kind `which` ran (interval union)."""
        ms = C.c_double()
        _check(lib().ffsga_cuda_timing_busy(self.h, which, C.byref(ms)))
        return ms.value

    def timing(self, which):
        ms, n = C.c_double(), C.c_int64()
        _check(lib().ffsga_cuda_timing(self.h, which, C.byref(ms), C.byref(n)))
        return ms.value, n.value


class Batch:
    """Device-resident chromosome batch (decoder sweep)."""

    def __init__(self, inst: Instance, capacity):
        self.inst = inst
        self.cap = int(capacity)
        h = C.c_void_p()
        _check(lib().ffsga_cuda_batch_create(inst.h, self.cap, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().ffsga_cuda_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def fill_random(self, base_seed, first, n):
        _check(lib().ffsga_cuda_batch_fill_random(self.h, base_seed, first, n))

    def upload(self, genes):
        genes = np.asarray(genes)
        if genes.dtype == np.uint8:
            g = np.ascontiguousarray(genes).reshape(-1, self.inst.num_genes)
            _check(lib().ffsga_cuda_batch_upload_u8(self.h, _p(g, _pu8), g.shape[0]))
        else:
            g = np.ascontiguousarray(genes, dtype=np.int32).reshape(-1, self.inst.num_genes)
            _check(lib().ffsga_cuda_batch_upload(self.h, _p(g, _pi32), g.shape[0]))

    def evaluate(self, n):
        _check(lib().ffsga_cuda_batch_evaluate(self.h, n))

    def sync(self):
        _check(lib().ffsga_cuda_batch_sync(self.h))

    def last_eval_ms(self):
        ms = C.c_float()
        _check(lib().ffsga_cuda_batch_last_eval_ms(self.h, C.byref(ms)))
        return ms.value

    def results(self, n, full=False):
        obj, fit = np.empty(n), np.empty(n)
        mk = np.empty(n) if full else None
        td = np.empty(n) if full else None
        _check(lib().ffsga_cuda_batch_results(self.h, n, _p(obj, _pd), _p(fit, _pd), _p(mk, _pd), _p(td, _pd)))
        return (obj, fit, mk, td) if full else (obj, fit)

    def download(self, first, n):
        out = np.empty((n, self.inst.num_genes), dtype=np.int32)
        _check(lib().ffsga_cuda_batch_download(self.h, first, n, _p(out, _pi32)))
        return out


class Cellular:
    """Device cellular island (ffsga_cuda_cellular ~ CellGrid)."""

    def __init__(self, inst: Instance, width, height, seed, crossover=1.0, mutation=0.05, radius=1, genes=None):
        self.inst = inst
        g = None if genes is None else np.ascontiguousarray(genes, dtype=np.int32)
        h = C.c_void_p()
        _check(lib().ffsga_cuda_cellular_create(inst.h, width, height, radius, crossover, mutation, seed,
                                                _p(g, _pi32), C.byref(h)))
        self.h = h
        n, w, hh, k = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(lib().ffsga_cuda_cellular_size(h, C.byref(n), C.byref(w), C.byref(hh), C.byref(k)))
        self.size, self.width, self.height, self.neighbors = n.value, w.value, hh.value, k.value

    def close(self):
        if getattr(self, "h", None):
            lib().ffsga_cuda_cellular_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def generation(self):
        g = C.c_uint64()
        _check(lib().ffsga_cuda_cellular_generation(self.h, C.byref(g)))
        return g.value

    def read(self):
        fit, obj = np.empty(self.size), np.empty(self.size)
        _check(lib().ffsga_cuda_cellular_read(self.h, _p(fit, _pd), _p(obj, _pd)))
        return fit, obj

    def genes(self, index=-1):
        rows = self.size if index < 0 else 1
        out = np.empty((rows, self.inst.num_genes), dtype=np.int32)
        _check(lib().ffsga_cuda_cellular_genes(self.h, index, _p(out, _pi32)))
        return out if index < 0 else out[0]

    def slots(self, index):
        out = np.empty(self.neighbors, dtype=np.int32)
        _check(lib().ffsga_cuda_cellular_slots(self.h, index, _p(out, _pi32)))
        return out

    def best(self):
        i, f, o = C.c_int(), C.c_double(), C.c_double()
        _check(lib().ffsga_cuda_cellular_best(self.h, C.byref(i), C.byref(f), C.byref(o)))
        return i.value, f.value, o.value

    def install(self, index, genes, fit, obj):
        g = np.ascontiguousarray(genes, dtype=np.int32)
        _check(lib().ffsga_cuda_cellular_install(self.h, index, _p(g, _pi32), fit, obj))

    def candidate(self, index, stream_state):
        """compute_cell on an explicit stream -> (genes, fitness, objective, replaced, draws_used)."""
        g = np.empty(self.inst.num_genes, dtype=np.int32)
        f, o, r, d = C.c_double(), C.c_double(), C.c_int(), C.c_uint64()
        _check(lib().ffsga_cuda_cellular_candidate(self.h, index, stream_state, _p(g, _pi32), C.byref(f), C.byref(o),
                                                   C.byref(r), C.byref(d)))
        return g, f.value, o.value, bool(r.value), d.value

    def export_best(self, k):
        """k best cells in sort_island order -> (genes [k, L] int32, fitness, objective)."""
        g = np.empty((k, self.inst.num_genes), dtype=np.int32)
        f, o = np.empty(k), np.empty(k)
        _check(lib().ffsga_cuda_cellular_export(self.h, k, _p(g, _pi32), _p(f, _pd), _p(o, _pd)))
        return g, f, o

    def import_worst(self, bits, fit, obj):
        """Install k pseudo migrants (bit chromosomes) over the k worst cells."""
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        f = np.ascontiguousarray(fit, dtype=np.float64)
        o = np.ascontiguousarray(obj, dtype=np.float64)
        _check(lib().ffsga_cuda_cellular_import(self.h, len(f), _p(b, _pu8), _p(f, _pd), _p(o, _pd)))

    # -- device-resident data plane (torch CUDA tensors; ordered on torch's current stream)
    def export_packet(self, k, out=None):
        """k best cells as a device migrant packet (uint8 torch tensor on this island's GPU)."""
        return _export_packet(self, 0, lib().ffsga_cuda_cellular_export_device, k, out)

    def import_packet(self, packet, k):
        """Install a pseudo island's packet over the k worst cells (device to device)."""
        _import_packet(self, lib().ffsga_cuda_cellular_import_device, packet, k)

    def state_device(self, out):
        """{best fitness, best objective, -1, 0} into a float64 CUDA tensor of 4 (device copy)."""
        _state_device(self, lib().ffsga_cuda_cellular_state_device, out)


class Pseudo:
    """Device complementary-pair island (ffsga_cuda_pseudo ~ PairPopulation)."""

    def __init__(self, inst: Instance, population, seed, crossover=0.75):
        self.inst = inst
        h = C.c_void_p()
        _check(lib().ffsga_cuda_pseudo_create(inst.h, population, crossover, seed, C.byref(h)))
        self.h = h
        n, tb = C.c_int(), C.c_int()
        _check(lib().ffsga_cuda_pseudo_size(h, C.byref(n), C.byref(tb)))
        self.size, self.total_bits = n.value, tb.value

    def close(self):
        if getattr(self, "h", None):
            lib().ffsga_cuda_pseudo_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def generation(self):
        g = C.c_uint64()
        _check(lib().ffsga_cuda_pseudo_generation(self.h, C.byref(g)))
        return g.value

    def read(self):
        fit, obj = np.empty(self.size), np.empty(self.size)
        _check(lib().ffsga_cuda_pseudo_read(self.h, _p(fit, _pd), _p(obj, _pd)))
        return fit, obj

    def members(self, index=-1):
        rows = self.size if index < 0 else 1
        out = np.empty((rows, max(self.total_bits, 1)), dtype=np.uint8)
        _check(lib().ffsga_cuda_pseudo_member(self.h, index, _p(out, _pu8)))
        out = out[:, : self.total_bits]
        return out if index < 0 else out[0]

    def best(self):
        i, f, o = C.c_int(), C.c_double(), C.c_double()
        _check(lib().ffsga_cuda_pseudo_best(self.h, C.byref(i), C.byref(f), C.byref(o)))
        return i.value, f.value, o.value

    def archive(self):
        f, o = C.c_double(), C.c_double()
        bits = np.empty(max(self.total_bits, 1), dtype=np.uint8)
        _check(lib().ffsga_cuda_pseudo_archive(self.h, C.byref(f), C.byref(o), _p(bits, _pu8)))
        return bits[: self.total_bits], f.value, o.value

    def archive_genes(self):
        """bits_to_int(archive_chromosome()) computed on the device."""
        out = np.empty(self.inst.num_genes, dtype=np.int32)
        _check(lib().ffsga_cuda_pseudo_archive_genes(self.h, _p(out, _pi32)))
        return out

    def install(self, index, bits, fit, obj):
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        _check(lib().ffsga_cuda_pseudo_install(self.h, index, _p(b, _pu8), fit, obj))

    def export_best(self, k):
        """k best members in sort_island order -> (bits [k, total_bits] uint8, fitness, objective)."""
        b = np.empty((k, max(self.total_bits, 1)), dtype=np.uint8)
        f, o = np.empty(k), np.empty(k)
        _check(lib().ffsga_cuda_pseudo_export(self.h, k, _p(b, _pu8), _p(f, _pd), _p(o, _pd)))
        return b[:, : self.total_bits], f, o

    def import_worst(self, genes, fit, obj):
        """Install k cellular migrants (int genes) over the k worst members; archive absorbs them."""
        g = np.ascontiguousarray(genes, dtype=np.int32)
        f = np.ascontiguousarray(fit, dtype=np.float64)
        o = np.ascontiguousarray(obj, dtype=np.float64)
        _check(lib().ffsga_cuda_pseudo_import(self.h, len(f), _p(g, _pi32), _p(f, _pd), _p(o, _pd)))

    # -- device-resident data plane (torch CUDA tensors; ordered on torch's current stream)
    def export_packet(self, k, out=None):
        """k best members as a device migrant packet (uint8 torch tensor on this island's GPU)."""
        return _export_packet(self, 1, lib().ffsga_cuda_pseudo_export_device, k, out)

    def import_packet(self, packet, k):
        """Install a cellular island's packet over the k worst members; the archive absorbs them."""
        _import_packet(self, lib().ffsga_cuda_pseudo_import_device, packet, k)

    def state_device(self, out):
        """{best fitness, best objective, archive fitness, archive objective} into a float64 CUDA
        tensor of 4 (device copy)."""
        _state_device(self, lib().ffsga_cuda_pseudo_state_device, out)


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _export_packet(isl, kind, fn, k, out):
    import torch
    nbytes = isl.inst.packet_bytes(kind, k)
    if out is None:
        out = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=torch.device("cuda", isl.inst.device))
    if out.numel() < nbytes or not out.is_cuda or not out.is_contiguous():
        raise ValueError("export_packet: out must be a contiguous CUDA uint8 tensor of packet_bytes()")
    _check(fn(isl.h, int(k), C.c_void_p(out.data_ptr()), _stream()))
    return out


def _import_packet(isl, fn, packet, k):
    if not packet.is_cuda or not packet.is_contiguous():
        raise ValueError("import_packet: packet must be a contiguous CUDA tensor")
    _check(fn(isl.h, int(k), C.c_void_p(packet.data_ptr()), _stream()))


def _state_device(isl, fn, out):
    import torch
    if not out.is_cuda or out.dtype != torch.float64 or out.numel() < 4 or not out.is_contiguous():
        raise ValueError("state_device: out must be a contiguous float64 CUDA tensor of >= 4 elements")
    _check(fn(isl.h, C.c_void_p(out.data_ptr()), _stream()))


def step(cells=(), pseudos=(), generations=1, traces=True):
    """Advance every listed island `generations` times in one fused launch sequence per generation.
    Returns (trace_cellular [nc, G], trace_pseudo [np, G])."""
    nc, np_ = len(cells), len(pseudos)
    ch = (C.c_void_p * max(nc, 1))(*[c.h.value for c in cells])
    ph = (C.c_void_p * max(np_, 1))(*[p.h.value for p in pseudos])
    tc = np.empty((nc, generations)) if (traces and nc) else None
    tp = np.empty((np_, generations)) if (traces and np_) else None
    _check(lib().ffsga_cuda_step(ch, nc, ph, np_, generations, _p(tc, _pd), _p(tp, _pd)))
    return tc, tp


def migrate_cellular_to_pseudo(cell: Cellular, pseudo: Pseudo, k):
    _check(lib().ffsga_cuda_migrate_cellular_to_pseudo(cell.h, pseudo.h, k))


def migrate_pseudo_to_cellular(pseudo: Pseudo, cell: Cellular, k):
    _check(lib().ffsga_cuda_migrate_pseudo_to_cellular(pseudo.h, cell.h, k))
