"""Island-model driver: the reference's drive() (proj/src/solver.cpp:76-198) generalised to C
couples of (cellular, pseudo) islands, sharded over the ranks of one node.

Extension contract: island i has seed derive_seed(seed, i); even islands
are cellular, odd islands pseudo; couple c = (2c, 2c+1) runs the reference migration policy
(decide, migration.cpp:21-36) at every rendezvous.  With one couple this is exactly run():
island seeds derive_seed(seed, 0|1) (solver.cpp:93,96), the same segments, rendezvous,
trace refresh, combined trace and champion rule (cellular wins ties, solver.cpp:179).

All population work runs in the CUDA kernels behind capi.py; this module only sequences
segments, evaluates the scalar migration policy and moves the (rare) migrant rows between
ranks.  Islands are owned by rank floor(i * world / n_islands): couples stay on one GPU
whenever world <= C, so migration is a device-local copy; only when world > C is a couple
split, and then the k migrant rows travel over torch.distributed (NCCL over NVLink on a GPU
node, gloo in the CPU tests).  No data-path collective exists between rendezvous.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
MASK = (1 << 64) - 1


def splitmix_next(state: int):
    """One SplitMix64 step (rng.hpp:18-23) -> (new_state, output)."""
    state = (state + GAMMA) & MASK
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return state, z ^ (z >> 31)


def derive_seed(base: int, key: int) -> int:
    """rng.hpp:55-58."""
    return splitmix_next((base + key * GAMMA) & MASK)[1]


def grid_shape_for(population: int):
    """Most-square factorisation, width >= height (cellular.cpp:38-48)."""
    from .capi import ConfigError
    if population < 4:
        raise ConfigError(2, "cellular island needs a population of at least 4")
    best = 1
    d = 1
    while d * d <= population:
        if population % d == 0:
            best = d
        d += 1
    if best < 2:
        raise ConfigError(2, f"cellular population {population} has no grid factorization with both sides >= 2")
    return population // best, best


def compute_beta(fit_a: float, fit_b: float) -> float:
    """migration.cpp:9-14."""
    from .capi import ContractError
    if fit_a < 0.0 or fit_b < 0.0:
        raise ContractError(1, "compute_beta: fitness values must be non-negative")
    if fit_a == fit_b:
        return 1.0
    return fit_a / fit_b if fit_a < fit_b else fit_b / fit_a


def compute_alpha(beta: float, theta: float) -> float:
    """migration.cpp:16-19."""
    rate = 1.0 - beta
    return rate if rate < theta else 0.0


def decide(fit_a: float, fit_b: float, theta: float, island_population: int):
    """migration.cpp:21-36 -> (beta, alpha, direction, migrants); direction in
    {"none", "a_to_b", "b_to_a"}."""
    from .capi import ContractError
    if island_population < 1:
        raise ContractError(1, "decide: island population must be positive")
    beta = compute_beta(fit_a, fit_b)
    alpha = compute_alpha(beta, theta)
    migrants = int(math.floor(alpha * island_population))
    if migrants <= 0 or fit_a == fit_b:
        return beta, alpha, "none", 0
    return beta, alpha, ("a_to_b" if fit_a > fit_b else "b_to_a"), migrants


# ----------------------------------------------------------------------------------- comms
class LocalComm:
    """Single process, every island local."""

    rank = 0
    world = 1

    def allgather(self, vec: np.ndarray) -> np.ndarray:
        return vec[None, :].copy()

    def send(self, arr: np.ndarray, dst: int):
        raise RuntimeError("LocalComm has no peers")

    def recv(self, shape, dtype, src: int) -> np.ndarray:
        raise RuntimeError("LocalComm has no peers")

    def barrier(self):
        pass


class TorchComm:
    """torch.distributed plumbing.  Only island statistics (all_gather, 32 B per island) and
    migrant packets (point-to-point, k rows) ever move.

    With NCCL (`device_tensors`) the data plane is device memory end to end: island statistics
    are copied on the GPU into a tensor that NCCL all-gathers over NVLink, and migrant packets are
    exported into a CUDA tensor, sent GPU to GPU and installed from it (capi export_packet /
    import_packet).  With gloo (the CPU tests) the same exchanges go through host arrays."""

    def __init__(self, device: Optional[str] = None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        backend = dist.get_backend()
        self.device = device or ("cuda" if backend == "nccl" else "cpu")
        self.device_tensors = backend == "nccl"

    # device-tensor plane (NCCL)
    def allgather_tensor(self, t):
        out = self.torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, t.contiguous())
        return out

    def send_tensor(self, t, dst: int):
        self.dist.send(t, dst)

    def recv_tensor(self, t, src: int):
        self.dist.recv(t, src)

    def broadcast_tensor(self, t, src: int):
        self.dist.broadcast(t, src)

    def _t(self, arr):
        return self.torch.from_numpy(np.ascontiguousarray(arr)).to(self.device)

    def allgather(self, vec: np.ndarray) -> np.ndarray:
        t = self._t(vec.astype(np.float64))
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t)
        return np.stack([o.cpu().numpy() for o in out])

    def send(self, arr: np.ndarray, dst: int):
        self.dist.send(self._t(arr), dst)

    def recv(self, shape, dtype, src: int) -> np.ndarray:
        t = self.torch.empty(tuple(shape), dtype=getattr(self.torch, np.dtype(dtype).name), device=self.device)
        self.dist.recv(t, src)
        return t.cpu().numpy()

    def barrier(self):
        self.dist.barrier()


# ------------------------------------------------------------------------------- config
@dataclass
class IslandConfig:
    couples: int = 1
    island_population: int = 256
    generations: int = 2000
    migration_gap: int = 500
    theta: float = 1.0
    cellular_crossover: float = 1.0
    cellular_mutation: float = 0.05
    radius: int = 1
    pseudo_crossover: float = 0.75
    seed: int = 1
    mode: str = "dual"  # dual | cellular | pseudo  (one couple only for the single-island modes)
    grid_shape: Optional[tuple] = None
    pseudo_fit_from_archive: bool = False

    @property
    def n_islands(self):
        return 2 * self.couples if self.mode == "dual" else self.couples

    def kind(self, i: int) -> str:
        if self.mode == "dual":
            return "cellular" if i % 2 == 0 else "pseudo"
        return self.mode

    def island_seed(self, i: int) -> int:
        # reference: cellular derive_seed(seed, 0), pseudo derive_seed(seed, 1) (solver.cpp:93,96)
        if self.mode == "dual":
            return derive_seed(self.seed, i)
        return derive_seed(self.seed, 2 * i + (0 if self.mode == "cellular" else 1))

    def validate(self):
        """RunConfig::validate (solver.cpp:39-70) for the per-island shape."""
        from .capi import ConfigError
        if self.generations < 1:
            raise ConfigError(2, "generations must be at least 1")
        if self.migration_gap < 1:
            raise ConfigError(2, "migration gap must be at least 1")
        if not (0.0 <= self.theta <= 1.0):
            raise ConfigError(2, "theta must lie in [0, 1]")
        for name, v in (("cellular crossover", self.cellular_crossover), ("cellular mutation", self.cellular_mutation),
                        ("pseudo crossover", self.pseudo_crossover)):
            if not (0.0 <= v <= 1.0):
                raise ConfigError(2, f"{name} rate must lie in [0, 1]")
        if self.mode not in ("dual", "cellular", "pseudo"):
            raise ConfigError(2, f"unknown mode '{self.mode}' (expected dual, cellular or pseudo)")
        if self.couples < 1:
            raise ConfigError(2, "at least one island couple is required")


def owner(i: int, n_islands: int, world: int) -> int:
    return (i * world) // n_islands


@dataclass
class MigrationEvent:
    generation: int
    beta: float
    alpha: float
    direction: str
    migrants: int
    couple: int = 0


@dataclass
class IslandResult:
    traces: np.ndarray                  # [n_islands, generations]
    trace_combined: np.ndarray          # [generations]
    best_island: int
    best_chromosome: np.ndarray
    best_report: dict
    migrations: List[MigrationEvent] = field(default_factory=list)
    seconds: dict = field(default_factory=dict)


class IslandModel:
    """Owns this rank's islands on one device and runs the segment / rendezvous loop."""

    def __init__(self, data, emax: float, cfg: IslandConfig, comm=None, device: int = 0, backend=None):
        """`backend` provides Instance / Cellular / Pseudo / step / migrate_* with the signatures of
        capi.py; it defaults to the device path (capi).  The CPU tests plug the oracle in here to
        exercise the multi-rank logic without a GPU."""
        if backend is None:
            from . import capi as backend
        capi = backend
        cfg.validate()
        self.capi = capi
        self.cfg = cfg
        self.comm = comm or LocalComm()
        self.emax = float(emax)
        self.inst = capi.Instance.from_data(data, emax, device)
        self.total_bits = self.inst.info()["total_bits"]
        n = cfg.n_islands
        self.local = {}
        t0 = time.perf_counter()
        for i in range(n):
            if owner(i, n, self.comm.world) != self.comm.rank:
                continue
            if cfg.kind(i) == "cellular":
                w, h = cfg.grid_shape if cfg.grid_shape else grid_shape_for(cfg.island_population)
                if w * h != cfg.island_population:
                    raise capi.ConfigError(2, "cellular grid shape does not match island population")
                if w < 2 or h < 2:
                    raise capi.ConfigError(2, "cellular grid sides must both be >= 2")
                self.local[i] = capi.Cellular(self.inst, w, h, cfg.island_seed(i), cfg.cellular_crossover,
                                              cfg.cellular_mutation, cfg.radius)
            else:
                self.local[i] = capi.Pseudo(self.inst, cfg.island_population, cfg.island_seed(i), cfg.pseudo_crossover)
        self.init_seconds = time.perf_counter() - t0
        self.generation = 0
        self.traces = {i: [] for i in self.local}
        # device-resident exchanges when the comm moves CUDA tensors and the backend exports
        # device packets (capi); host arrays otherwise (gloo tests, the oracle backend)
        self.device_plane = bool(getattr(self.comm, "device_tensors", False)) and \
            hasattr(capi.Cellular, "export_packet")
        self.device = device
        if self.comm.world == 1 and hasattr(capi.Cellular, "state_device"):
            import torch  # torch's CUDA state, used by the rendezvous statistics, set up here
            torch.zeros(1, dtype=torch.float64, device=torch.device("cuda", device))

    # -- pieces -------------------------------------------------------------------------
    def _cells(self):
        return [self.local[i] for i in sorted(self.local) if self.cfg.kind(i) == "cellular"]

    def _pseudos(self):
        return [self.local[i] for i in sorted(self.local) if self.cfg.kind(i) == "pseudo"]

    def advance(self, generations: int):
        """Every local island advances `generations` in one joint launch sequence."""
        cells, pseudos = self._cells(), self._pseudos()
        if not cells and not pseudos:  # a rank that owns no island (world > islands)
            self.generation += generations
            return
        tc, tp = self.capi.step(cells, pseudos, generations)
        ci = pi = 0
        for i in sorted(self.local):
            if self.cfg.kind(i) == "cellular":
                self.traces[i].append(tc[ci])
                ci += 1
            else:
                self.traces[i].append(tp[pi])
                pi += 1
        self.generation += generations

    def _policy_fitness(self, i):
        isl = self.local[i]
        if self.cfg.kind(i) == "cellular":
            return isl.best()[1]
        return isl.archive()[1] if self.cfg.pseudo_fit_from_archive else isl.best()[1]

    def _trace_value(self, i):
        isl = self.local[i]
        return isl.best()[2] if self.cfg.kind(i) == "cellular" else isl.archive()[2]

    def _gather_states(self):
        """{best fitness, best objective, archive fitness, archive objective} of every island
        (global order), gathered over the ranks.  Device plane: each island's statistics are
        copied on its GPU into one tensor that NCCL all-gathers; the host then reads the n x 4
        values the (host-side, solver.cpp:142-163) policy needs."""
        n, comm = self.cfg.n_islands, self.comm
        # one process with the device backend: the same device copies and a single read-back
        # (per-island host reads cost a synchronisation each: 64 islands ~ 5 ms per rendezvous)
        local_dev = comm.world == 1 and hasattr(self.capi.Cellular, "state_device")
        if self.device_plane or local_dev:
            import torch
            vec = torch.zeros((n, 4), dtype=torch.float64, device=torch.device("cuda", self.device))
            vec[:, 2] = -1.0
            for i, isl in self.local.items():
                isl.state_device(vec[i])
            allv = comm.allgather_tensor(vec).cpu().numpy() if self.device_plane else vec.cpu().numpy()[None]
        else:
            vec = np.zeros((n, 4))
            vec[:, 2] = -1.0
            for i, isl in self.local.items():
                _, bf, bo = isl.best()
                if self.cfg.kind(i) == "pseudo":
                    _, af, ao = isl.archive()
                else:
                    af, ao = -1.0, 0.0
                vec[i] = (bf, bo, af, ao)
            allv = comm.allgather(vec.reshape(-1)).reshape(comm.world, n, 4)
        return np.stack([allv[owner(i, n, comm.world), i] for i in range(n)])

    def _move_migrants(self, src, dst, k, direction):
        """Rows of a split couple: export on the source's GPU, point-to-point, import on the
        destination's GPU (migration.cpp:47-69 split at the wire)."""
        comm, n = self.comm, self.cfg.n_islands
        osrc, odst = owner(src, n, comm.world), owner(dst, n, comm.world)
        if self.device_plane:
            import torch
            if osrc == comm.rank:
                comm.send_tensor(self.local[src].export_packet(k), odst)
            elif odst == comm.rank:
                kind = 0 if direction == "a_to_b" else 1
                pk = torch.empty(self.inst.packet_bytes(kind, k), dtype=torch.uint8,
                                 device=torch.device("cuda", self.device))
                comm.recv_tensor(pk, osrc)
                self.local[dst].import_packet(pk, k)
            return
        if osrc == comm.rank:
            rows, f, o = self.local[src].export_best(k)
            comm.send(np.ascontiguousarray(rows), odst)
            comm.send(np.stack([f, o]), odst)
        elif odst == comm.rank:
            L = self.inst.num_genes
            width = L if direction == "a_to_b" else self.total_bits
            dtype = np.int32 if direction == "a_to_b" else np.uint8
            rows = comm.recv((k, width), dtype, osrc)
            fo = comm.recv((2, k), np.float64, osrc)
            self.local[dst].import_worst(rows, fo[0], fo[1])

    def rendezvous(self, done: int) -> List[MigrationEvent]:
        """solver.cpp:142-163 for every couple."""
        cfg, comm, n = self.cfg, self.comm, self.cfg.n_islands
        st = self._gather_states()
        fit = np.array([st[i, 2] if (cfg.kind(i) == "pseudo" and cfg.pseudo_fit_from_archive) else st[i, 0]
                        for i in range(n)])
        events = []
        for c in range(cfg.couples):
            a, b = 2 * c, 2 * c + 1
            beta, alpha, direction, k = decide(float(fit[a]), float(fit[b]), cfg.theta, cfg.island_population)
            if direction == "none":
                continue
            src, dst = (a, b) if direction == "a_to_b" else (b, a)
            osrc, odst = owner(src, n, comm.world), owner(dst, n, comm.world)
            if osrc == odst == comm.rank:
                if direction == "a_to_b":
                    self.capi.migrate_cellular_to_pseudo(self.local[a], self.local[b], k)
                else:
                    self.capi.migrate_pseudo_to_cellular(self.local[b], self.local[a], k)
            elif comm.rank in (osrc, odst):
                self._move_migrants(src, dst, k, direction)
            events.append(MigrationEvent(done, beta, alpha, direction, k, c))
            # the entries already written for this generation are refreshed (solver.cpp:156-160)
            for i in (a, b):
                if i in self.local:
                    self.traces[i][-1][-1] = self._trace_value(i)
        return events

    def run(self) -> IslandResult:
        """The segment loop of solver.cpp:128-164, then traces + champion (166-189)."""
        cfg = self.cfg
        budget, gap = cfg.generations, cfg.migration_gap
        both = cfg.mode == "dual"
        done = 0
        events: List[MigrationEvent] = []
        t0 = time.perf_counter()
        t_mig = 0.0
        while done < budget:
            stop = min(budget, (done // gap + 1) * gap)
            self.advance(stop - done)
            done = stop
            if both and done < budget and done % gap == 0:
                tm = time.perf_counter()
                events += self.rendezvous(done)
                t_mig += time.perf_counter() - tm
        t_islands = time.perf_counter() - t0 - t_mig
        return self.finish(events, dict(islands=t_islands, migration=t_mig, init=self.init_seconds))

    def finish(self, events, seconds) -> IslandResult:
        cfg, comm, n = self.cfg, self.comm, self.cfg.n_islands
        G = self.generation  # every rank advanced the same budget, islands or not
        local_tr = np.zeros((n, G))
        for i in self.local:
            local_tr[i] = np.concatenate(self.traces[i]) if self.traces[i] else np.zeros(0)
        st = self._gather_states()
        # champion fitness: cellular best, pseudo archive (solver.cpp:175-183)
        champ = np.array([st[i, 0] if cfg.kind(i) == "cellular" else st[i, 2] for i in range(n)])
        if comm.world > 1:
            if self.device_plane:
                import torch
                t = torch.from_numpy(local_tr).to(torch.device("cuda", self.device))
                tr_all = comm.allgather_tensor(t).cpu().numpy()
            else:
                tr_all = comm.allgather(local_tr.reshape(-1)).reshape(comm.world, n, G)
            traces = np.stack([tr_all[owner(i, n, comm.world), i] for i in range(n)])
        else:
            traces = local_tr
        # combined = fold of std::min in island order (solver.cpp:166-173)
        comb = traces[0].copy()
        for i in range(1, n):
            comb = np.where(traces[i] < comb, traces[i], comb)
        # champion: max fitness, ties to the lower island index (cellular wins, solver.cpp:175-183)
        best = 0
        for i in range(1, n):
            if champ[i] > champ[best]:
                best = i
        chrom, rep = None, None
        ob = owner(best, n, comm.world)
        if ob == comm.rank:
            isl = self.local[best]
            chrom = isl.genes(isl.best()[0]) if cfg.kind(best) == "cellular" else isl.archive_genes()
            _, _, _, rep = self.inst.decode(chrom)  # decode + evaluate on the device (K7)
        if comm.world > 1:
            L = self.inst.num_genes
            buf = np.zeros(L + 5)
            if ob == comm.rank:
                buf[:L] = chrom
                buf[L:] = [rep["makespan"], rep["total_tardiness"], rep["objective"], rep["fitness"], rep["emax_used"]]
            if self.device_plane:
                import torch
                t = torch.from_numpy(buf).to(torch.device("cuda", self.device))
                comm.broadcast_tensor(t, ob)
                buf = t.cpu().numpy()
            else:
                buf = comm.allgather(buf)[ob]
            chrom = buf[:L].astype(np.int32)
            rep = dict(makespan=buf[L], total_tardiness=buf[L + 1], objective=buf[L + 2], fitness=buf[L + 3],
                       emax_used=buf[L + 4])
        return IslandResult(traces, comb, best, np.asarray(chrom, dtype=np.int32), rep, events, seconds)
