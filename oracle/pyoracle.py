"""ctypes front-end for the CPU checkers (TEST INFRASTRUCTURE ONLY).

Two checkers sit behind one Python surface:

* ``Oracle``  -- ``oracle/liboracle.so``, the C restatement (``oracle/ffsga_oracle.c``);
* ``RefLib``  -- ``oracle/_ref/libffsga_ref.so``, the unmodified reference sources compiled
  by ``oracle/Makefile`` behind ``oracle/ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline / ``--impl
reference``) may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libffsga_ref.so")

_u64, _i32, _f64, _vp = C.c_uint64, C.c_int, C.c_double, C.c_void_p
_pi = C.POINTER(C.c_int)
_pd = C.POINTER(C.c_double)
_pu8 = C.POINTER(C.c_uint8)
_pu64 = C.POINTER(C.c_uint64)


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


def synthetic_machines(jobs: int, stages: int, lo: int = 2, hi: int = 8) -> list:
    """M[s] = lo + Rng(1000 + J*S).next_index(hi - lo + 1)."""
    st = np.array([1000 + jobs * stages], dtype=np.uint64)
    out = []
    for _ in range(stages):
        u = _splitmix_next(st)
        unit = float(u >> np.uint64(11)) * 2.0 ** -53
        v = int(unit * float(hi - lo + 1))
        out.append(lo + min(v, hi - lo))
    return out


def _splitmix_next(state):
    with np.errstate(over="ignore"):
        state[0] = state[0] + np.uint64(0x9E3779B97F4A7C15)
        z = state[0]
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return np.uint64(z ^ (z >> np.uint64(31)))


class _OrcInstance(C.Structure):
    _fields_ = [("num_jobs", _i32), ("num_stages", _i32), ("machines_per_stage", _pi),
                ("stage_offset", _pi), ("machines_total", _i32), ("proc", _pd),
                ("release", _pd), ("due", _pd), ("weight", _f64)]


class _OrcReport(C.Structure):
    _fields_ = [("makespan", _f64), ("total_tardiness", _f64), ("objective", _f64),
                ("fitness", _f64), ("emax_used", _f64)]


class _OrcLayout(C.Structure):
    _fields_ = [("num_jobs", _i32), ("num_stages", _i32), ("bits_per_stage", _i32 * 256),
                ("stage_bit_offset", _i32 * 257), ("bits_per_job", _i32), ("total_bits", _i32)]


class _OrcCellular(C.Structure):
    _fields_ = [("inst", _vp), ("emax", _f64), ("width", _i32), ("height", _i32), ("size", _i32),
                ("radius", _i32), ("neighbors_per_cell", _i32), ("crossover_rate", _f64),
                ("mutation_rate", _f64), ("island_seed", _u64), ("generation", _u64),
                ("genes", _pi), ("fitness", _pd), ("objective", _pd), ("slots", _pi)]


class _OrcPseudo(C.Structure):
    _fields_ = [("inst", _vp), ("emax", _f64), ("layout", _OrcLayout), ("size", _i32),
                ("crossover_rate", _f64), ("island_seed", _u64), ("generation", _u64),
                ("members", _pu8), ("fitness", _pd), ("objective", _pd), ("archive", _pu8),
                ("archive_fitness", _f64), ("archive_objective", _f64)]


class _OrcRunConfig(C.Structure):
    _fields_ = [("population", _i32), ("generations", _i32), ("migration_gap", _i32),
                ("theta", _f64), ("cellular_crossover", _f64), ("cellular_mutation", _f64),
                ("radius", _i32), ("pseudo_crossover", _f64), ("mode", _i32), ("seed", _u64),
                ("grid_w", _i32), ("grid_h", _i32), ("pseudo_fit_from_archive", _i32)]


class _OrcRunResult(C.Structure):
    _fields_ = [("best_objective", _f64), ("best_fitness", _f64), ("best_makespan", _f64),
                ("best_tardiness", _f64), ("emax", _f64), ("best_chromosome", _pi),
                ("trace_combined", _pd), ("trace_a", _pd), ("trace_b", _pd),
                ("num_migrations", _i32), ("mig_generation", _pu64), ("mig_beta", _pd),
                ("mig_alpha", _pd), ("mig_direction", _pi), ("mig_migrants", _pi)]


MODES = {"dual": 0, "cellular": 1, "cellular-only": 1, "pseudo": 2, "pseudo-only": 2}


class InstanceData:
    """Plain arrays of one instance (job-major proc as the reference stores it)."""

    def __init__(self, jobs, stages, machines, proc, release, due, weight):
        self.num_jobs = int(jobs)
        self.num_stages = int(stages)
        self.machines = [int(m) for m in machines]
        self.proc = np.ascontiguousarray(proc, dtype=np.float64)
        self.release = np.ascontiguousarray(release, dtype=np.float64)
        self.due = np.ascontiguousarray(due, dtype=np.float64)
        self.weight = float(weight)

    @property
    def num_genes(self):
        return self.num_jobs * self.num_stages

    @property
    def machines_total(self):
        return sum(self.machines)

    def stage_offset(self):
        return np.concatenate([[0], np.cumsum(self.machines)]).astype(np.int64)


class Oracle:
    """The C restatement, oracle/ffsga_oracle.c."""

    def __init__(self, path: str = ORACLE_SO):
        self.lib = L = C.CDLL(path)
        L.orc_rng_next_u64.restype = _u64
        L.orc_rng_next_u64.argtypes = [_pu64]
        L.orc_rng_next_unit.restype = _f64
        L.orc_rng_next_unit.argtypes = [_pu64]
        L.orc_rng_next_uniform.restype = _f64
        L.orc_rng_next_uniform.argtypes = [_pu64, _f64, _f64]
        L.orc_rng_next_index.restype = _i32
        L.orc_rng_next_index.argtypes = [_pu64, _i32]
        L.orc_rng_next_coin.restype = _i32
        L.orc_rng_next_coin.argtypes = [_pu64, _f64]
        L.orc_derive_seed.restype = _u64
        L.orc_derive_seed.argtypes = [_u64, _u64]
        L.orc_instance_new.restype = C.POINTER(_OrcInstance)
        L.orc_instance_new.argtypes = [_i32, _i32, _pi, _pd, _pd, _pd, _f64]
        L.orc_generate.restype = C.POINTER(_OrcInstance)
        L.orc_generate.argtypes = [_i32, _i32, _pi, _f64, _u64, _i32]
        L.orc_instance_free.argtypes = [_vp]
        L.orc_instance_export.argtypes = [_vp, _pd, _pd, _pd]
        L.orc_estimate_emax.restype = _f64
        L.orc_estimate_emax.argtypes = [_vp]
        L.orc_mean_total_load.restype = _f64
        L.orc_mean_total_load.argtypes = [_vp]
        L.orc_mean_job_load.restype = _f64
        L.orc_mean_job_load.argtypes = [_vp, _i32]
        L.orc_release_order.argtypes = [_vp, _pi]
        L.orc_score.restype = _i32
        L.orc_score.argtypes = [_vp, _pi, _f64, C.POINTER(_OrcReport), _pi, _pd, _pd, _pi, _pi]
        L.orc_simulate_selection.argtypes = [_vp, _pi, C.POINTER(_OrcReport)]
        L.orc_bit_layout_for.restype = _i32
        L.orc_bit_layout_for.argtypes = [_vp, C.POINTER(_OrcLayout)]
        L.orc_int_to_bits.argtypes = [C.POINTER(_OrcLayout), _pi, _pi, _pu8]
        L.orc_bits_to_int.argtypes = [C.POINTER(_OrcLayout), _pi, _pu8, _pi]
        L.orc_random_int_chromosome.argtypes = [_vp, _pu64, _pi]
        L.orc_grid_shape_for.restype = _i32
        L.orc_grid_shape_for.argtypes = [_i32, _pi, _pi]
        L.orc_neighborhood_slots.restype = _i32
        L.orc_neighborhood_slots.argtypes = [_i32, _i32, _i32, _i32, _i32, _pi]
        L.orc_sort_island.argtypes = [_pd, _i32, _pi]
        L.orc_cellular_new.restype = C.POINTER(_OrcCellular)
        L.orc_cellular_new.argtypes = [_vp, _f64, _i32, _i32, _i32, _f64, _f64, _u64, _pi]
        L.orc_cellular_free.argtypes = [_vp]
        L.orc_cellular_candidate.restype = _i32
        L.orc_cellular_candidate.argtypes = [_vp, _i32, _u64, _pi, _pd, _pd]
        L.orc_cellular_candidate_draws.restype = _i32
        L.orc_cellular_candidate_draws.argtypes = [_vp, _i32, _u64, _pi, _pd, _pd, _pu64]
        L.orc_cellular_step.argtypes = [_vp]
        L.orc_cellular_best_index.restype = _i32
        L.orc_cellular_best_index.argtypes = [_vp]
        L.orc_cellular_install.argtypes = [_vp, _i32, _pi, _f64, _f64]
        L.orc_pair_step.restype = _i32
        L.orc_pair_step.argtypes = [_pu8, _pu8, _i32, _pu64, _f64, _pu8, _pu8]
        L.orc_pseudo_new.restype = C.POINTER(_OrcPseudo)
        L.orc_pseudo_new.argtypes = [_vp, _f64, _i32, _f64, _u64]
        L.orc_pseudo_free.argtypes = [_vp]
        L.orc_pseudo_step.argtypes = [_vp]
        L.orc_pseudo_best_index.restype = _i32
        L.orc_pseudo_best_index.argtypes = [_vp]
        L.orc_pseudo_install.argtypes = [_vp, _i32, _pu8, _f64, _f64]
        L.orc_compute_beta.restype = _f64
        L.orc_compute_beta.argtypes = [_f64, _f64]
        L.orc_compute_alpha.restype = _f64
        L.orc_compute_alpha.argtypes = [_f64, _f64]
        L.orc_decide.argtypes = [_f64, _f64, _f64, _i32, _pd, _pd, _pi, _pi]
        L.orc_migrate_cellular_to_pseudo.argtypes = [_vp, _vp, _i32]
        L.orc_migrate_pseudo_to_cellular.argtypes = [_vp, _vp, _i32]
        L.orc_run.restype = _i32
        L.orc_run.argtypes = [C.POINTER(_OrcRunConfig), _vp, C.POINTER(_OrcRunResult)]
        L.orc_run_result_free.argtypes = [C.POINTER(_OrcRunResult)]

    # -- rng -------------------------------------------------------------------------
    def rng(self, seed):
        return OracleRng(self, seed)

    def derive_seed(self, base, key):
        return int(self.lib.orc_derive_seed(_u64(base), _u64(key)))

    # -- instances -------------------------------------------------------------------
    def instance(self, data: InstanceData):
        return OracleInstance(self, data)

    def generate(self, jobs, stages, machines, weight=100.0, seed=1, integer_times=False):
        m = np.ascontiguousarray(machines, dtype=np.int32)
        p = self.lib.orc_generate(jobs, stages, _ptr(m, _pi), weight, _u64(seed), int(integer_times))
        mt = int(m.sum())
        proc = np.empty(jobs * mt)
        rel = np.empty(jobs)
        due = np.empty(jobs)
        self.lib.orc_instance_export(p, _ptr(proc, _pd), _ptr(rel, _pd), _ptr(due, _pd))
        self.lib.orc_instance_free(p)
        return InstanceData(jobs, stages, list(m), proc, rel, due, weight)


class OracleRng:
    def __init__(self, orc, seed):
        self.lib = orc.lib
        self.state = C.c_uint64(seed)

    def next_u64(self):
        return int(self.lib.orc_rng_next_u64(C.byref(self.state)))

    def next_unit(self):
        return float(self.lib.orc_rng_next_unit(C.byref(self.state)))

    def next_uniform(self, lo, hi):
        return float(self.lib.orc_rng_next_uniform(C.byref(self.state), lo, hi))

    def next_index(self, n):
        return int(self.lib.orc_rng_next_index(C.byref(self.state), n))

    def next_coin(self, p):
        return bool(self.lib.orc_rng_next_coin(C.byref(self.state), p))


class OracleInstance:
    def __init__(self, orc: Oracle, data: InstanceData):
        self.orc, self.data = orc, data
        self._m = np.ascontiguousarray(data.machines, dtype=np.int32)
        self.ptr = orc.lib.orc_instance_new(data.num_jobs, data.num_stages, _ptr(self._m, _pi),
                                            _ptr(data.proc, _pd), _ptr(data.release, _pd),
                                            _ptr(data.due, _pd), data.weight)
        self.layout = _OrcLayout()
        orc.lib.orc_bit_layout_for(self.ptr, C.byref(self.layout))

    def __del__(self):
        try:
            self.orc.lib.orc_instance_free(self.ptr)
        except Exception:
            pass

    def estimate_emax(self):
        return float(self.orc.lib.orc_estimate_emax(self.ptr))

    def mean_total_load(self):
        return float(self.orc.lib.orc_mean_total_load(self.ptr))

    def mean_job_load(self, j):
        return float(self.orc.lib.orc_mean_job_load(self.ptr, j))

    def release_order(self):
        out = np.empty(self.data.num_jobs, dtype=np.int32)
        self.orc.lib.orc_release_order(self.ptr, _ptr(out, _pi))
        return out

    def score(self, genes, emax, schedule=False):
        """Evaluator::score; returns dict (+ schedule arrays).  Raises ValueError on a bad gene."""
        g = np.ascontiguousarray(genes, dtype=np.int32)
        rep = _OrcReport()
        L = self.data.num_genes
        sm = np.empty(L, dtype=np.int32) if schedule else None
        ss = np.empty(L) if schedule else None
        sc = np.empty(L) if schedule else None
        bj, bs = C.c_int(-1), C.c_int(-1)
        st = self.orc.lib.orc_score(self.ptr, _ptr(g, _pi), emax, C.byref(rep), _ptr(sm, _pi),
                                    _ptr(ss, _pd), _ptr(sc, _pd), C.byref(bj), C.byref(bs))
        if st != 0:
            raise ValueError(f"decode: machine index out of range at job {bj.value} stage {bs.value}")
        out = dict(makespan=rep.makespan, total_tardiness=rep.total_tardiness,
                   objective=rep.objective, fitness=rep.fitness, emax_used=rep.emax_used)
        if schedule:
            out.update(machine=sm, start=ss, completion=sc)
        return out

    def score_batch(self, genes, emax):
        genes = np.ascontiguousarray(genes, dtype=np.int32).reshape(-1, self.data.num_genes)
        n = genes.shape[0]
        obj, fit, mk, td = np.empty(n), np.empty(n), np.empty(n), np.empty(n)
        rep = _OrcReport()
        for i in range(n):
            st = self.orc.lib.orc_score(self.ptr, _ptr(genes[i], _pi), emax, C.byref(rep), None,
                                        None, None, None, None)
            if st != 0:
                raise ValueError("decode: machine index out of range")
            obj[i], fit[i], mk[i], td[i] = rep.objective, rep.fitness, rep.makespan, rep.total_tardiness
        return obj, fit, mk, td

    def simulate_selection(self, genes):
        g = np.ascontiguousarray(genes, dtype=np.int32)
        rep = _OrcReport()
        self.orc.lib.orc_simulate_selection(self.ptr, _ptr(g, _pi), C.byref(rep))
        return dict(makespan=rep.makespan, total_tardiness=rep.total_tardiness,
                    objective=rep.objective)

    def total_bits(self):
        return int(self.layout.total_bits)

    def int_to_bits(self, genes):
        g = np.ascontiguousarray(genes, dtype=np.int32)
        out = np.empty(self.total_bits(), dtype=np.uint8)
        self.orc.lib.orc_int_to_bits(C.byref(self.layout), _ptr(self._m, _pi), _ptr(g, _pi), _ptr(out, _pu8))
        return out

    def bits_to_int(self, bits):
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        out = np.empty(self.data.num_genes, dtype=np.int32)
        self.orc.lib.orc_bits_to_int(C.byref(self.layout), _ptr(self._m, _pi), _ptr(b, _pu8), _ptr(out, _pi))
        return out

    def random_chromosome(self, rng: OracleRng):
        out = np.empty(self.data.num_genes, dtype=np.int32)
        self.orc.lib.orc_random_int_chromosome(self.ptr, C.byref(rng.state), _ptr(out, _pi))
        return out

    def random_population(self, base_seed, first, n):
        """chromosome i = random_int_chromosome(inst, Rng(derive_seed(base, first + i)))."""
        out = np.empty((n, self.data.num_genes), dtype=np.int32)
        st = C.c_uint64(0)
        for i in range(n):
            st.value = self.orc.derive_seed(base_seed, first + i)
            self.orc.lib.orc_random_int_chromosome(self.ptr, C.byref(st), _ptr(out[i], _pi))
        return out

    # -- islands ---------------------------------------------------------------------
    def cellular(self, emax, width, height, seed, crossover=1.0, mutation=0.05, radius=1, genes=None):
        return OracleCellular(self, emax, width, height, seed, crossover, mutation, radius, genes)

    def pseudo(self, emax, population, seed, crossover=0.75):
        return OraclePseudo(self, emax, population, seed, crossover)

    def run(self, population=512, generations=2000, gap=500, theta=1.0, mode="dual", seed=1,
            cellular_crossover=1.0, cellular_mutation=0.05, pseudo_crossover=0.75, radius=1,
            grid_shape=None, pseudo_fit_from_archive=False):
        cfg = _OrcRunConfig(population, generations, gap, theta, cellular_crossover,
                            cellular_mutation, radius, pseudo_crossover, MODES[mode], seed,
                            grid_shape[0] if grid_shape else 0, grid_shape[1] if grid_shape else 0,
                            int(pseudo_fit_from_archive))
        res = _OrcRunResult()
        if self.orc.lib.orc_run(C.byref(cfg), self.ptr, C.byref(res)) != 0:
            raise ValueError("invalid run configuration")
        G, L = generations, self.data.num_genes
        m = MODES[mode]
        out = dict(
            best_objective=res.best_objective, best_fitness=res.best_fitness,
            best_makespan=res.best_makespan, best_total_tardiness=res.best_tardiness,
            emax=res.emax, best_chromosome=[res.best_chromosome[i] for i in range(L)],
            trace_combined=[res.trace_combined[i] for i in range(G)],
            trace_island_a=[res.trace_a[i] for i in range(G)] if m != 2 else [],
            trace_island_b=[res.trace_b[i] for i in range(G)] if m != 1 else [],
            migrations=[dict(generation=int(res.mig_generation[i]), beta=res.mig_beta[i],
                             alpha=res.mig_alpha[i],
                             direction={1: "a_to_b", 2: "b_to_a"}[res.mig_direction[i]],
                             migrants=res.mig_migrants[i]) for i in range(res.num_migrations)])
        self.orc.lib.orc_run_result_free(C.byref(res))
        return out


class OracleCellular:
    def __init__(self, inst: OracleInstance, emax, width, height, seed, crossover, mutation, radius, genes):
        self.inst, self.lib = inst, inst.orc.lib
        g = None if genes is None else np.ascontiguousarray(genes, dtype=np.int32)
        self.ptr = self.lib.orc_cellular_new(inst.ptr, emax, width, height, radius, crossover,
                                             mutation, _u64(seed), _ptr(g, _pi))
        self.size = width * height

    def __del__(self):
        try:
            self.lib.orc_cellular_free(self.ptr)
        except Exception:
            pass

    def step(self):
        self.lib.orc_cellular_step(self.ptr)

    @property
    def generation(self):
        return int(self.ptr.contents.generation)

    def fitness(self):
        return np.ctypeslib.as_array(self.ptr.contents.fitness, (self.size,)).copy()

    def objective(self):
        return np.ctypeslib.as_array(self.ptr.contents.objective, (self.size,)).copy()

    def genes(self):
        L = self.inst.data.num_genes
        return np.ctypeslib.as_array(self.ptr.contents.genes, (self.size * L,)).reshape(self.size, L).copy()

    def slots(self):
        n = self.ptr.contents.neighbors_per_cell
        return np.ctypeslib.as_array(self.ptr.contents.slots, (self.size * n,)).reshape(self.size, n).copy()

    def best_index(self):
        return int(self.lib.orc_cellular_best_index(self.ptr))

    def candidate(self, index, stream_seed, with_draws=False):
        child = np.empty(self.inst.data.num_genes, dtype=np.int32)
        fit, obj, dr = C.c_double(), C.c_double(), C.c_uint64()
        r = self.lib.orc_cellular_candidate_draws(self.ptr, index, _u64(stream_seed), _ptr(child, _pi),
                                                  C.byref(fit), C.byref(obj), C.byref(dr))
        if with_draws:
            return child, fit.value, obj.value, bool(r), dr.value
        return child, fit.value, obj.value, bool(r)

    def install(self, index, genes, fit, obj):
        g = np.ascontiguousarray(genes, dtype=np.int32)
        self.lib.orc_cellular_install(self.ptr, index, _ptr(g, _pi), fit, obj)


class OraclePseudo:
    def __init__(self, inst: OracleInstance, emax, population, seed, crossover):
        self.inst, self.lib = inst, inst.orc.lib
        self.ptr = self.lib.orc_pseudo_new(inst.ptr, emax, population, crossover, _u64(seed))
        if not self.ptr:
            raise ValueError("pseudo island population must be even and >= 2")
        self.size = population
        self.nbits = inst.total_bits()

    def __del__(self):
        try:
            self.lib.orc_pseudo_free(self.ptr)
        except Exception:
            pass

    def step(self):
        self.lib.orc_pseudo_step(self.ptr)

    @property
    def generation(self):
        return int(self.ptr.contents.generation)

    def fitness(self):
        return np.ctypeslib.as_array(self.ptr.contents.fitness, (self.size,)).copy()

    def objective(self):
        return np.ctypeslib.as_array(self.ptr.contents.objective, (self.size,)).copy()

    def members(self):
        return np.ctypeslib.as_array(self.ptr.contents.members, (self.size * self.nbits,)).reshape(
            self.size, self.nbits).copy()

    def archive(self):
        c = self.ptr.contents
        bits = np.ctypeslib.as_array(c.archive, (max(self.nbits, 1),))[: self.nbits].copy()
        return bits, c.archive_fitness, c.archive_objective

    def best_index(self):
        return int(self.lib.orc_pseudo_best_index(self.ptr))

    def install(self, index, bits, fit, obj):
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        self.lib.orc_pseudo_install(self.ptr, index, _ptr(b, _pu8), fit, obj)


# ----------------------------------------------------------------------------------------
class RefLib:
    """The reference itself, compiled from /root/reference by oracle/Makefile."""

    def __init__(self, path: str = REF_SO):
        self.lib = L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_generate.restype = _vp
        L.ref_generate.argtypes = [_i32, _i32, _pi, _f64, _u64, _i32]
        L.ref_instance_new.restype = _vp
        L.ref_instance_new.argtypes = [_i32, _i32, _pi, _pd, _pd, _pd, _f64]
        L.ref_instance_validate.restype = _i32
        L.ref_instance_validate.argtypes = [_vp]
        L.ref_instance_machines_total.restype = _i32
        L.ref_instance_machines_total.argtypes = [_vp]
        L.ref_instance_export.argtypes = [_vp, _pd, _pd, _pd]
        L.ref_instance_free.argtypes = [_vp]
        L.ref_estimate_emax.restype = _f64
        L.ref_estimate_emax.argtypes = [_vp]
        L.ref_mean_total_load.restype = _f64
        L.ref_mean_total_load.argtypes = [_vp]
        L.ref_score_batch.restype = _i32
        L.ref_score_batch.argtypes = [_vp, _f64, _pi, C.c_int64, _pd, _pd, _pd, _pd, _i32]
        L.ref_decode.restype = _i32
        L.ref_decode.argtypes = [_vp, _pi, _pi, _pd, _pd]
        L.ref_oracle_simulate.restype = _f64
        L.ref_oracle_simulate.argtypes = [_vp, _pi]
        L.ref_random_chromosomes.argtypes = [_vp, _u64, C.c_int64, C.c_int64, _pi]
        L.ref_derive_seed.restype = _u64
        L.ref_derive_seed.argtypes = [_u64, _u64]
        L.ref_cellular_new.restype = _vp
        L.ref_cellular_new.argtypes = [_vp, _f64, _i32, _i32, _i32, _i32, _f64, _f64, _u64]
        L.ref_cellular_new_explicit.restype = _vp
        L.ref_cellular_new_explicit.argtypes = [_vp, _f64, _pi, _i32, _i32, _i32, _f64, _f64, _u64]
        L.ref_cellular_free.argtypes = [_vp]
        L.ref_cellular_step.argtypes = [_vp, _i32]
        for f in ("size", "width", "height", "best_index"):
            getattr(L, "ref_cellular_" + f).restype = _i32
            getattr(L, "ref_cellular_" + f).argtypes = [_vp]
        L.ref_cellular_generation.restype = _u64
        L.ref_cellular_generation.argtypes = [_vp]
        L.ref_cellular_read.argtypes = [_vp, _pd, _pd, _pi]
        L.ref_cellular_slots.argtypes = [_vp, _i32, _pi, _pi]
        L.ref_cellular_candidate.restype = _i32
        L.ref_cellular_candidate.argtypes = [_vp, _i32, _u64, _pi, _pd, _pd]
        L.ref_cellular_install.argtypes = [_vp, _i32, _pi, _f64, _f64]
        L.ref_pseudo_new.restype = _vp
        L.ref_pseudo_new.argtypes = [_vp, _f64, _i32, _f64, _u64]
        L.ref_pseudo_free.argtypes = [_vp]
        L.ref_pseudo_step.argtypes = [_vp, _i32]
        for f in ("size", "total_bits", "best_index"):
            getattr(L, "ref_pseudo_" + f).restype = _i32
            getattr(L, "ref_pseudo_" + f).argtypes = [_vp]
        L.ref_pseudo_generation.restype = _u64
        L.ref_pseudo_generation.argtypes = [_vp]
        L.ref_pseudo_read.argtypes = [_vp, _pd, _pd, _pu8]
        L.ref_pseudo_archive.argtypes = [_vp, _pd, _pd, _pu8]
        L.ref_pseudo_install.argtypes = [_vp, _i32, _pu8, _f64, _f64]
        L.ref_pair_step.restype = _i32
        L.ref_pair_step.argtypes = [_pu8, _pu8, _i32, _u64, _f64, _pu8, _pu8]
        L.ref_decide.argtypes = [_f64, _f64, _f64, _i32, _pd, _pd, _pi, _pi]
        L.ref_migrate_c2p.argtypes = [_vp, _vp, _i32]
        L.ref_migrate_p2c.argtypes = [_vp, _vp, _i32]
        L.ref_run.restype = _vp
        L.ref_run.argtypes = [_vp, _i32, _i32, _i32, _f64, _i32, _u64, _i32, _i32, _f64, _f64, _f64, _i32]
        L.ref_run_scalars.argtypes = [_vp, _pd]
        L.ref_run_num_migrations.restype = _i32
        L.ref_run_num_migrations.argtypes = [_vp]
        L.ref_run_migration.argtypes = [_vp, _i32, _pu64, _pd, _pd, _pi, _pi]
        L.ref_run_traces.argtypes = [_vp, _pd, _pd, _pd, _pi]
        L.ref_run_free.argtypes = [_vp]
        for f in ("ref_save_result_json", "ref_save_trace_csv", "ref_save_instance"):
            if hasattr(L, f):  # io.cpp (file formats); absent from older builds
                getattr(L, f).restype = _i32
                getattr(L, f).argtypes = [_vp, C.c_char_p]

    def generate(self, jobs, stages, machines, weight=100.0, seed=1, integer_times=False):
        m = np.ascontiguousarray(machines, dtype=np.int32)
        h = self.lib.ref_generate(jobs, stages, _ptr(m, _pi), weight, _u64(seed), int(integer_times))
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        mt = int(m.sum())
        proc, rel, due = np.empty(jobs * mt), np.empty(jobs), np.empty(jobs)
        self.lib.ref_instance_export(h, _ptr(proc, _pd), _ptr(rel, _pd), _ptr(due, _pd))
        self.lib.ref_instance_free(h)
        return InstanceData(jobs, stages, list(m), proc, rel, due, weight)

    def instance(self, data: InstanceData):
        return RefInstance(self, data)


class RefInstance:
    def __init__(self, ref: RefLib, data: InstanceData):
        self.ref, self.lib, self.data = ref, ref.lib, data
        self._m = np.ascontiguousarray(data.machines, dtype=np.int32)
        self.h = self.lib.ref_instance_new(data.num_jobs, data.num_stages, _ptr(self._m, _pi),
                                           _ptr(data.proc, _pd), _ptr(data.release, _pd),
                                           _ptr(data.due, _pd), data.weight)

    def __del__(self):
        try:
            self.lib.ref_instance_free(self.h)
        except Exception:
            pass

    def estimate_emax(self):
        return float(self.lib.ref_estimate_emax(self.h))

    def mean_total_load(self):
        return float(self.lib.ref_mean_total_load(self.h))

    def score_batch(self, genes, emax, workers=1):
        genes = np.ascontiguousarray(genes, dtype=np.int32).reshape(-1, self.data.num_genes)
        n = genes.shape[0]
        obj, fit, mk, td = np.empty(n), np.empty(n), np.empty(n), np.empty(n)
        st = self.lib.ref_score_batch(self.h, emax, _ptr(genes, _pi), n, _ptr(obj, _pd),
                                      _ptr(fit, _pd), _ptr(mk, _pd), _ptr(td, _pd), workers)
        if st != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return obj, fit, mk, td

    def decode(self, genes):
        g = np.ascontiguousarray(genes, dtype=np.int32)
        L = self.data.num_genes
        m, s, c = np.empty(L, dtype=np.int32), np.empty(L), np.empty(L)
        if self.lib.ref_decode(self.h, _ptr(g, _pi), _ptr(m, _pi), _ptr(s, _pd), _ptr(c, _pd)) != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return m, s, c

    def random_population(self, base_seed, first, n):
        out = np.empty((n, self.data.num_genes), dtype=np.int32)
        self.lib.ref_random_chromosomes(self.h, _u64(base_seed), first, n, _ptr(out, _pi))
        return out

    def cellular(self, emax, population, seed, width=0, height=0, crossover=1.0, mutation=0.05, radius=1):
        h = self.lib.ref_cellular_new(self.h, emax, population, width, height, radius, crossover,
                                      mutation, _u64(seed))
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        return RefCellular(self, h)

    def cellular_explicit(self, emax, genes, width, height, seed, crossover=1.0, mutation=0.05, radius=1):
        g = np.ascontiguousarray(genes, dtype=np.int32)
        h = self.lib.ref_cellular_new_explicit(self.h, emax, _ptr(g, _pi), width, height, radius,
                                               crossover, mutation, _u64(seed))
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        return RefCellular(self, h)

    def pseudo(self, emax, population, seed, crossover=0.75):
        h = self.lib.ref_pseudo_new(self.h, emax, population, crossover, _u64(seed))
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        return RefPseudo(self, h)

    def save(self, path):
        """ffsga::save_instance (io.cpp) -- the reference's instance JSON bytes."""
        if self.lib.ref_save_instance(self.h, str(path).encode()) != 0:
            raise OSError(self.lib.ref_last_error().decode())

    def run(self, population=512, generations=2000, gap=500, theta=1.0, mode="dual", seed=1,
            workers=1, serialized=False, cellular_crossover=1.0, cellular_mutation=0.05,
            pseudo_crossover=0.75, pseudo_fit_from_archive=False, result_json=None, trace_csv=None):
        r = self.lib.ref_run(self.h, population, generations, gap, theta, MODES[mode], _u64(seed),
                             workers, int(serialized), cellular_crossover, cellular_mutation,
                             pseudo_crossover, int(pseudo_fit_from_archive))
        if not r:
            raise ValueError(self.lib.ref_last_error().decode())
        if result_json is not None:  # ffsga::save_result_json / save_trace_csv (io.cpp)
            self.lib.ref_save_result_json(r, str(result_json).encode())
        if trace_csv is not None:
            self.lib.ref_save_trace_csv(r, str(trace_csv).encode())
        sc = np.empty(5)
        self.lib.ref_run_scalars(r, _ptr(sc, _pd))
        G, L = generations, self.data.num_genes
        m = MODES[mode]
        comb, a, b = np.empty(G), np.empty(G), np.empty(G)
        chrom = np.empty(L, dtype=np.int32)
        self.lib.ref_run_traces(r, _ptr(comb, _pd), _ptr(a, _pd), _ptr(b, _pd), _ptr(chrom, _pi))
        migs = []
        for i in range(self.lib.ref_run_num_migrations(r)):
            gen, beta, alpha, d, k = C.c_uint64(), C.c_double(), C.c_double(), C.c_int(), C.c_int()
            self.lib.ref_run_migration(r, i, C.byref(gen), C.byref(beta), C.byref(alpha), C.byref(d), C.byref(k))
            migs.append(dict(generation=gen.value, beta=beta.value, alpha=alpha.value,
                             direction={1: "a_to_b", 2: "b_to_a"}[d.value], migrants=k.value))
        self.lib.ref_run_free(r)
        return dict(best_objective=sc[0], best_fitness=sc[1], best_makespan=sc[2],
                    best_total_tardiness=sc[3], emax=sc[4], best_chromosome=chrom.tolist(),
                    trace_combined=comb.tolist(), trace_island_a=a.tolist() if m != 2 else [],
                    trace_island_b=b.tolist() if m != 1 else [], migrations=migs)


class RefCellular:
    def __init__(self, inst: RefInstance, h):
        self.inst, self.lib, self.h = inst, inst.lib, h
        self.size = self.lib.ref_cellular_size(h)

    def __del__(self):
        try:
            self.lib.ref_cellular_free(self.h)
        except Exception:
            pass

    def step(self, workers=1):
        self.lib.ref_cellular_step(self.h, workers)

    def read(self, genes=False):
        fit, obj = np.empty(self.size), np.empty(self.size)
        g = np.empty((self.size, self.inst.data.num_genes), dtype=np.int32) if genes else None
        self.lib.ref_cellular_read(self.h, _ptr(fit, _pd), _ptr(obj, _pd), _ptr(g, _pi))
        return (fit, obj, g) if genes else (fit, obj)

    def best_index(self):
        return int(self.lib.ref_cellular_best_index(self.h))

    def install(self, index, genes, fit, obj):
        g = np.ascontiguousarray(genes, dtype=np.int32)
        self.lib.ref_cellular_install(self.h, index, _ptr(g, _pi), fit, obj)


class RefPseudo:
    def __init__(self, inst: RefInstance, h):
        self.inst, self.lib, self.h = inst, inst.lib, h
        self.size = self.lib.ref_pseudo_size(h)
        self.nbits = self.lib.ref_pseudo_total_bits(h)

    def __del__(self):
        try:
            self.lib.ref_pseudo_free(self.h)
        except Exception:
            pass

    def step(self, workers=1):
        self.lib.ref_pseudo_step(self.h, workers)

    def read(self, bits=False):
        fit, obj = np.empty(self.size), np.empty(self.size)
        b = np.empty((self.size, self.nbits), dtype=np.uint8) if bits else None
        self.lib.ref_pseudo_read(self.h, _ptr(fit, _pd), _ptr(obj, _pd), _ptr(b, _pu8))
        return (fit, obj, b) if bits else (fit, obj)

    def archive(self):
        f, o = C.c_double(), C.c_double()
        b = np.zeros(max(self.nbits, 1), dtype=np.uint8)
        self.lib.ref_pseudo_archive(self.h, C.byref(f), C.byref(o), _ptr(b, _pu8))
        return b[: self.nbits], f.value, o.value

    def best_index(self):
        return int(self.lib.ref_pseudo_best_index(self.h))


def have_ref() -> bool:
    return os.path.exists(REF_SO)
