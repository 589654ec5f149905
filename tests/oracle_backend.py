"""CPU stand-in for the capi device backend, built on the C restatement (TEST INFRASTRUCTURE).

IslandModel (paper_1903_10722_b200/islands.py) takes a `backend` with the capi.py surface; this
one lets the multi-rank driver logic (segments, rendezvous, cross-rank migrant rows, champion)
run under gloo on CPU.  Never used by the product.
"""
import numpy as np

from paper_1903_10722_b200.capi import ConfigError, ContractError  # noqa: F401  (exception types only)
from pyoracle import Oracle

_orc = Oracle()


class Instance:
    def __init__(self, data, emax):
        self.data = data
        self.oi = _orc.instance(data)
        self.emax = emax
        self.num_genes = data.num_jobs * data.num_stages

    @classmethod
    def from_data(cls, data, emax, device=0):
        return cls(data, emax)

    def info(self):
        return {"total_bits": self.oi.total_bits()}

    def decode(self, genes):
        r = self.oi.score(np.asarray(genes, dtype=np.int32), self.emax, schedule=True)
        rep = {k: r[k] for k in ("makespan", "total_tardiness", "objective", "fitness", "emax_used")}
        return r["machine"], r["start"], r["completion"], rep


def _sort(f):
    return sorted(range(len(f)), key=lambda i: (-f[i], i))


class Cellular:
    def __init__(self, inst, w, h, seed, crossover=1.0, mutation=0.05, radius=1):
        self.inst = inst
        self.o = inst.oi.cellular(inst.emax, w, h, seed, crossover, mutation, radius)
        self.size = w * h

    def best(self):
        i = self.o.best_index()
        return i, float(self.o.fitness()[i]), float(self.o.objective()[i])

    def genes(self, i=-1):
        g = self.o.genes()
        return g if i < 0 else g[i]

    def export_best(self, k):
        f, o, g = self.o.fitness(), self.o.objective(), self.o.genes()
        best = _sort(f)[:k]
        return g[best], f[best], o[best]

    def import_worst(self, bits, fit, obj):
        order = _sort(self.o.fitness())
        for i in range(len(fit)):
            self.o.install(order[self.size - 1 - i], self.inst.oi.bits_to_int(bits[i]), fit[i], obj[i])


class Pseudo:
    def __init__(self, inst, n, seed, crossover=0.75):
        self.inst = inst
        self.o = inst.oi.pseudo(inst.emax, n, seed, crossover)
        self.size = n

    def best(self):
        i = self.o.best_index()
        return i, float(self.o.fitness()[i]), float(self.o.objective()[i])

    def archive(self):
        return self.o.archive()

    def archive_genes(self):
        return self.inst.oi.bits_to_int(self.o.archive()[0])

    def export_best(self, k):
        f, o, m = self.o.fitness(), self.o.objective(), self.o.members()
        best = _sort(f)[:k]
        return m[best], f[best], o[best]

    def import_worst(self, genes, fit, obj):
        order = _sort(self.o.fitness())
        for i in range(len(fit)):
            self.o.install(order[self.size - 1 - i], self.inst.oi.int_to_bits(genes[i]), fit[i], obj[i])


def step(cells=(), pseudos=(), generations=1, traces=True):
    tc = np.empty((len(cells), generations))
    tp = np.empty((len(pseudos), generations))
    for g in range(generations):
        for i, c in enumerate(cells):
            c.o.step()
            tc[i, g] = c.o.objective()[c.o.best_index()]
        for i, p in enumerate(pseudos):
            p.o.step()
            tp[i, g] = p.o.archive()[2]
    return tc, tp


def migrate_cellular_to_pseudo(c, p, k):
    _orc.lib.orc_migrate_cellular_to_pseudo(c.o.ptr, p.o.ptr, k)


def migrate_pseudo_to_cellular(p, c, k):
    _orc.lib.orc_migrate_pseudo_to_cellular(p.o.ptr, c.o.ptr, k)
