#!/usr/bin/env python3
"""Benchmark of the FFS hot path on B200: GA generations/s and makespan evaluations/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload ga|decoder]

Workload (default "ga", BASELINE.json configs[2] = SURVEY 8(d) C3): synthetic 500 jobs x 20 stages,
machines per stage in [2, 8] (M[s] = 2 + Rng(1000 + J*S).next_index(7)), generator seed 7,
weight 100; 8 islands = 4 couples of (cellular 128x64, pseudo 8192), total population 65536,
gap 500, theta 1, seed 1.  One step = one GA generation of every island (all selection,
crossover, mutation, decode/evaluate, replacement, archive and trace work).  Under torchrun the
8 islands are sharded over the ranks (couples kept together while ranks <= 4): total work is
fixed, so scaling is "strong"; value = generations/s of the whole job (the same generation on
every island, device time max over ranks).

"decoder" workload: 1M random chromosomes of the 500x20 instance evaluated per
launch; one step = one launch.

--impl reference times the reference's own CPU implementation (oracle/_ref, the unmodified
reference sources compiled by oracle/Makefile) on this box's host cores with all of them as
workers, same config and metric.  Under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FFS makespan evals/sec & GA generations/sec at 1/2/4/8 B200 vs CPU ref"
J, S, LO, HI, GEN_SEED, WEIGHT = 500, 20, 2, 8, 7, 100.0
COUPLES, ISLAND_POP, GRID = 4, 8192, (128, 64)
RUN_SEED, GAP, THETA = 1, 500, 1.0
E2E_RUNS = 3
SWEEP_N = 1 << 20


def synthetic_machines(jobs, stages, lo=LO, hi=HI):
    """M[s] = lo + Rng(1000 + J*S).next_index(hi - lo + 1) (plain Python, so that
    neither arm imports the other's code to build its config)."""
    g, mask = 0x9E3779B97F4A7C15, (1 << 64) - 1
    st = 1000 + jobs * stages
    out = []
    for _ in range(stages):
        st = (st + g) & mask
        z = st
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & mask
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & mask
        u = z ^ (z >> 31)
        v = int(float(u >> 11) * 2.0 ** -53 * float(hi - lo + 1))
        out.append(lo + min(v, hi - lo))
    return out


def cpu_info():
    """Host CPU model, current clock and thread count (nproc, CPU model, clocks)."""
    model, mhz = None, []
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                k, _, v = line.partition(":")
                k = k.strip()
                if k == "model name" and model is None:
                    model = v.strip()
                elif k == "cpu MHz":
                    mhz.append(float(v))
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"cpu_model": model, "cpu_mhz_mean": (sum(mhz) / len(mhz)) if mhz else None,
            "cpu_mhz_max": max(mhz) if mhz else None, "nproc": os.cpu_count(), "usable_threads": usable}


def make_instance():
    """Synthetic C3 instance through the product's host generator."""
    from paper_1903_10722_b200 import generate_instance, estimate_emax
    inst = generate_instance(jobs=J, stages=S, machines=synthetic_machines(J, S), weight=WEIGHT, seed=GEN_SEED)
    return inst, estimate_emax(inst)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """SM clock and throttle reasons sampled (NVML, every 20 ms) during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None

    def _poll(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while True:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((sm, rs))
                if self._stop.wait(0.02):
                    break
        except Exception as e:  # NVML missing: record why
            self.rows.append((None, str(e)))

    def __enter__(self):
        self._t = threading.Thread(target=self._poll, daemon=True)
        self._t.start()
        time.sleep(0.05)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        sm = [r[0] for r in self.rows if isinstance(r[0], (int, float))]
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        reasons = sorted({n for _, rs in self.rows if isinstance(rs, int) for n, bit in self.REASONS.items()
                          if rs & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm)}


def _ref_islands(ri, emax, derive):
    """The 8 C3 islands on the reference (oracle/_ref): island i seed derive_seed(seed, i), even =
    CellGrid 128x64, odd = PairPopulation 8192 (bench.py's island set, islands.py extension)."""
    isl = []
    for i in range(2 * COUPLES):
        if i % 2 == 0:
            isl.append(ri.cellular(emax, ISLAND_POP, derive(RUN_SEED, i), width=GRID[0], height=GRID[1]))
        else:
            isl.append(ri.pseudo(emax, ISLAND_POP, derive(RUN_SEED, i)))
    return isl


def _ref_island_objectives(isl):
    """Per island: cellular objective at best_index, pseudo archive objective (the trace values,
    solver.cpp:113,121)."""
    out = []
    for i, x in enumerate(isl):
        if i % 2 == 0:
            out.append(float(x.read()[1][x.best_index()]))
        else:
            out.append(float(x.archive()[2]))
    return out


def cpu_baseline_ga(inst_data, emax, workers):
    """The reference's CPU generation (oracle/_ref: the unmodified reference sources) on the full
    C3 island set, timed on this box's host cores: one warm-up generation, then 2 timed ones."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import RefLib, have_ref
    if not have_ref():
        return None
    ref = RefLib()
    ri = ref.instance(inst_data)
    isl = _ref_islands(ri, emax, lambda b, k: int(ref.lib.ref_derive_seed(b, k)))
    for x in isl:
        x.step(workers)
    reps = 2
    t0 = time.perf_counter()
    for _ in range(reps):
        for x in isl:
            x.step(workers)
    dt = (time.perf_counter() - t0) / reps
    out = {"value": 1.0 / dt, "unit": "generations/s", "cores": workers, "kind": "reference",
           "sample": f"{reps} timed generations (after 1 warm-up) of the full C3 island set: 4 CellGrid 128x64 + "
                     f"4 PairPopulation 8192 steps, oracle/_ref, workers={workers}"}
    out.update(cpu_info())
    return out


def reference_arm(args):
    """The reference's own CPU implementation (oracle/_ref) -- nothing of the product package is
    imported here."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import RefLib, have_ref
    if not have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libffsga_ref.so not built"}))
        return 0
    if args.workload == "c4":
        print(json.dumps({"impl": "reference", "unavailable": "the reference arm times the headline C3 step "
                          "(default) and the C5 decoder sweep; C4 is a secondary GPU workload"}))
        return 0
    workers = os.cpu_count() or 1
    ref = RefLib()
    m = synthetic_machines(J, S)
    data = ref.generate(J, S, m, weight=WEIGHT, seed=GEN_SEED)
    ri = ref.instance(data)
    emax = ri.estimate_emax()
    extra = {}
    if args.workload == "decoder":
        n = 20000
        pop = ri.random_population(99, 0, n)
        for _ in range(args.warmup):
            ri.score_batch(pop[:2000], emax, workers)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ri.score_batch(pop, emax, workers)
        dt = time.perf_counter() - t0
        val = n * args.steps / dt
        unit = "evals/s"
        sample = f"{n} chromosomes per step (of the 1M launch), Evaluator::score via parallel_chunks"
        cfg = {"workload": "C5 decoder sweep 500x20, M in [2,8]", "n_per_step_sampled": n}
    else:
        isl = _ref_islands(ri, emax, lambda b, k: int(ref.lib.ref_derive_seed(b, k)))
        for _ in range(args.warmup):
            for x in isl:
                x.step(workers)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            for x in isl:
                x.step(workers)
        dt = time.perf_counter() - t0
        val = args.steps / dt
        unit = "generations/s"
        sample = (f"full C3 generation per step: 4 CellGrid 128x64 + 4 PairPopulation 8192 steps, "
                  f"workers={workers}")
        cfg = ga_config(world, m)
        extra["island_best_objectives"] = _ref_island_objectives(isl)
        extra["generations_done"] = args.warmup + args.steps
    cpu = {"value": val, "unit": unit, "cores": workers, "kind": "reference", "sample": sample}
    cpu.update(cpu_info())
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg, "cpu_baseline": cpu,
        "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    line.update(extra)
    print(json.dumps(line), flush=True)
    return 0


def ga_config(world, machines):
    return {"workload": "C3: FFS 500 jobs x 20 stages x 2-8 machines/stage, 8 islands (4 cellular 128x64 + "
                        "4 pseudo 8192), pop 65536",
            "jobs": J, "stages": S, "machines": list(machines), "islands": 2 * COUPLES,
            "population": 2 * COUPLES * ISLAND_POP, "gap": GAP, "theta": THETA, "seed": RUN_SEED,
            "ranks": world, "islands_per_rank": 2 * COUPLES // world if world <= 2 * COUPLES else None,
            "l2": "inputs larger than L2 (resident population 0.77 GB > 126 MB)"}


PROFILE = os.path.join(ROOT, "profiles", "r2_k1_profile.json")


def load_profile():
    """The committed ncu numbers of this library's K1 inside the C3 step (profiles/r2_k1_profile.json,
    written by profiles/tools/summarize_ncu.py from an `ncu --set full` capture of bench.py)."""
    try:
        with open(PROFILE) as f:
            d = json.load(f)
        d["source"] = os.path.relpath(PROFILE, ROOT)
        return d
    except Exception:
        return {}


def island_objectives(model, comm):
    """Per island (global order): cellular objective at best_index, pseudo archive objective --
    the reference arm prints the same list for the same generations."""
    n = model.cfg.n_islands
    vec = np.full(n, np.nan)
    for i, isl in model.local.items():
        vec[i] = isl.best()[2] if model.cfg.kind(i) == "cellular" else isl.archive()[2]
    if comm is not None:
        from paper_1903_10722_b200.islands import owner
        allv = comm.allgather(vec)
        vec = np.array([allv[owner(i, n, comm.world), i] for i in range(n)])
    return [float(x) for x in vec]


def sweep_traffic(n):
    """DRAM bytes per sweep launch of n chromosomes, from the committed ncu capture (per-evaluation
    figure of profiles/r1_sweep_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1_sweep_traffic.json")) as f:
            return json.load(f)["traffic_bytes_per_eval"] * n
    except Exception:
        return None


def decoder_sweep(inst_data, emax, device, steps, warmup):
    """C5: 1M random chromosomes per launch (K2 fill, then K1 launches timed with events)."""
    from paper_1903_10722_b200 import capi
    ci = capi.Instance.from_data(inst_data, emax, device)
    b = capi.Batch(ci, SWEEP_N)
    b.fill_random(99, 0, SWEEP_N)
    for _ in range(max(1, warmup)):
        b.evaluate(SWEEP_N)
    b.sync()
    ms = []
    for _ in range(max(1, steps)):
        b.evaluate(SWEEP_N)
        ms.append(b.last_eval_ms())
    avg = float(np.mean(ms))
    L = J * S
    bytes_per = SWEEP_N * (L + 16)
    obj, _ = b.results(SWEEP_N)
    return {"evals_per_s": SWEEP_N / (avg / 1e3), "n_per_launch": SWEEP_N, "ms_per_launch": avg,
            "dispatches_per_s": SWEEP_N * L / (avg / 1e3),
            "roofline": {"bound": "hbm", "achieved": bytes_per / (avg / 1e3) / 1e9, "unit": "GB/s",
                         "traffic": sweep_traffic(SWEEP_N), "algorithmic_bytes_per_launch": bytes_per},
            "checksum_objective_sum": float(np.sum(obj))}


def c4_workload(args, comm, local, world, rank):
    """C4: 1000 x 20 x [2, 8], 64 islands (32 couples of CellGrid 32x32 +
    PairPopulation 1024), weight 0, a rendezvous every 10 generations -- so the timed region
    crosses rendezvous (policy all-gather, decide, migrant packets when k > 0).  Wall clock with
    the device synchronised on both sides (the rendezvous is host policy + collectives), max over
    ranks."""
    import torch
    from paper_1903_10722_b200 import capi, generate_instance, estimate_emax, instance_arrays
    from paper_1903_10722_b200.islands import IslandConfig, IslandModel
    J4, S4, gap = 1000, 20, 10
    m4 = synthetic_machines(J4, S4)
    inst = generate_instance(jobs=J4, stages=S4, machines=m4, weight=0.0, seed=GEN_SEED)
    emax = estimate_emax(inst)
    cfg = IslandConfig(couples=32, island_population=1024, generations=args.warmup + args.steps, migration_gap=gap,
                       theta=THETA, seed=RUN_SEED, grid_shape=(32, 32))
    model = IslandModel(instance_arrays(inst), emax, cfg, comm, device=local)

    def barrier():
        if comm is not None:
            comm.barrier()

    def segment(n, done):  # n generations from `done`, rendezvous at the gap boundaries (solver.cpp:128-164)
        events, t_mig, crossed = [], 0.0, 0
        end = done + n
        while done < end:
            stop = min(end, (done // gap + 1) * gap)
            model.advance(stop - done)
            done = stop
            if done % gap == 0 and done < cfg.generations:
                tm = time.perf_counter()
                events += model.rendezvous(done)
                t_mig += time.perf_counter() - tm
                crossed += 1
        return done, events, t_mig, crossed

    done, _, _, _ = segment(args.warmup, 0)
    torch.cuda.synchronize()
    barrier()
    ev0 = model.inst.evaluations()
    l0 = capi.launch_count()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        done, events, t_mig, crossed = segment(args.steps, done)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    barrier()
    l1 = capi.launch_count()
    evals = model.inst.evaluations() - ev0
    if comm is not None:
        agg = comm.allgather(np.array([dt, t_mig, evals], dtype=np.float64))
        dt, t_mig, evals_all = float(agg[:, 0].max()), float(agg[:, 1].max()), float(agg[:, 2].sum())
    else:
        evals_all = float(evals)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": args.steps / dt, "unit": "generations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY 8(d) generator convention, random-init populations)",
            "config": {"workload": "C4: FFS 1000 jobs x 20 stages x 2-8 machines/stage, 64 islands (32 cellular 32x32 "
                                   "+ 32 pseudo 1024), weight 0, rendezvous every 10 generations",
                       "jobs": J4, "stages": S4, "machines": m4, "islands": 64, "population": 65536, "gap": gap,
                       "weight": 0.0, "ranks": world},
            "evals_per_s": evals_all / dt, "rendezvous_in_timed_region": crossed,
            "migrations_in_timed_region": [[e.generation, e.couple, e.direction, e.migrants] for e in events],
            "rendezvous_s": t_mig,
            "timing": "wall clock, device synchronised on both sides, max over ranks",
            "gpu_launches": int(l1 - l0), "clocks": clk.summary()}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="ga", choices=["ga", "decoder", "c4"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    comm = None
    if os.environ.get("FFSGA_BENCH_DEVICE") is not None:  # test hook: all ranks on one GPU
        local = int(os.environ["FFSGA_BENCH_DEVICE"])
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        backend = os.environ.get("FFSGA_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        from paper_1903_10722_b200.islands import TorchComm
        comm = TorchComm(device=f"cuda:{local}" if backend == "nccl" else "cpu")

    if args.workload == "c4":
        rc = c4_workload(args, comm, local, world, rank)
        if comm is not None:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return rc
    from paper_1903_10722_b200 import capi
    from paper_1903_10722_b200.islands import IslandConfig, IslandModel
    inst, emax = make_instance()
    from paper_1903_10722_b200 import instance_arrays
    data = instance_arrays(inst)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"

    def barrier():
        if comm is not None:
            comm.barrier()

    cfg = IslandConfig(couples=COUPLES, island_population=ISLAND_POP, generations=args.steps, migration_gap=GAP,
                       theta=THETA, seed=RUN_SEED, grid_shape=GRID)
    model = IslandModel(data, emax, cfg, comm, device=local)
    L = J * S
    if args.workload == "ga":
        model.advance(args.warmup)
        model.inst.set_timing(True)
        model.inst.reset_timing()
        ev0 = model.inst.evaluations()
        torch.cuda.synchronize()
        barrier()
        l0 = capi.launch_count()
        with ClockSampler(local) as clk:
            model.advance(args.steps)
            dev_ms = model.inst.last_step_ms()
        l1 = capi.launch_count()
        evals = model.inst.evaluations() - ev0
        eval_ms, eval_n = model.inst.timing(0)
        eval_busy_ms = model.inst.timing_busy(0)
        island_obj = island_objectives(model, comm)
        breed_ms, _ = model.inst.timing(1)
        commit_ms, _ = model.inst.timing(2)
        model.inst.set_timing(False)
        barrier()
        if comm is not None:
            agg = comm.allgather(np.array([dev_ms, evals, eval_ms, eval_n], dtype=np.float64))
            ms_max = float(agg[:, 0].max())
            evals_all = float(agg[:, 1].sum())
        else:
            ms_max, evals_all = dev_ms, float(evals)
        gens_per_s = args.steps / (ms_max / 1e3)
        algo_bytes = evals * (L + 16)
        prof = load_profile()
        traffic = None  # DRAM bytes per K1 launch from the committed ncu capture, scaled per evaluation
        if prof.get("traffic_bytes_per_eval"):
            traffic = prof["traffic_bytes_per_eval"] * (evals / max(1, eval_n))
        # K1 of the cellular and the pseudo chain run concurrently on two streams: the kernel's
        # time is the union of its launch intervals (timing_busy), not the per-stream sum
        achieved = algo_bytes / (eval_busy_ms / 1e3) / 1e9 if eval_busy_ms > 0 else 0.0
        issue = None  # K1 is issue/latency bound: the issue roofline from the committed capture
        if prof.get("issue_active") is not None:
            issue = {"bound": "issue", "frac": prof["issue_active"], "unit": "warp instructions/cycle/SMSP",
                     "achieved": prof["issue_active"], "peak": 1.0, "warps_per_sm": prof.get("warps_per_sm"),
                     "threads_per_inst": prof.get("threads_per_inst"), "kernel": prof.get("kernel"),
                     "source": prof.get("source")}

        # e2e: the public API call a user makes (instance upload, island init, K generations,
        # traces + champion back to the host), wall clock; median of E2E_RUNS independent runs
        # one untimed end-to-end run first: the process's first model pays one-time costs (lazy
        # kernel-module loading, growth of the stream-ordered memory pool to the model's 0.8 GB)
        # that a serving process does not pay per request
        runs = []
        for it in range(E2E_RUNS + 1):
            barrier()
            t0 = time.perf_counter()
            inst2, emax2 = make_instance()
            cfg2 = IslandConfig(couples=COUPLES, island_population=ISLAND_POP, generations=args.steps,
                                migration_gap=GAP, theta=THETA, seed=RUN_SEED, grid_shape=GRID)
            model2 = IslandModel(instance_arrays(inst2), emax2, cfg2, comm, device=local)
            t1 = time.perf_counter()
            res = model2.run()
            barrier()
            t2 = time.perf_counter()
            if it > 0:
                runs.append((t2 - t0, t1 - t0, t2 - t1, model2.inst.last_step_ms() / 1e3))
            del model2
            if os.environ.get("FFSGA_BENCH_DEBUG") and runs:
                print("e2e run", runs[-1], file=sys.stderr, flush=True)
        if comm is not None:  # max over ranks, per run
            agg = comm.allgather(np.array([r[0] for r in runs]))
            runs = [(float(agg[:, i].max()),) + runs[i][1:] for i in range(len(runs))]
        runs.sort()
        e2e_s = runs[len(runs) // 2][0]
        e2e_parts = {"instance_and_init_s": runs[len(runs) // 2][1], "run_s": runs[len(runs) // 2][2],
                     "run_device_s": runs[len(runs) // 2][3], "runs_total_s": [r[0] for r in runs]}
        # instance upload: proc (J x sum M fp64) + release + due (fp64) + machines per stage (int32)
        h2d = J * sum(synthetic_machines(J, S)) * 8 + 16 * J + 4 * S
        d2h = 2 * COUPLES * args.steps * 8 + L * 4 + 5 * 8

        sweep = None
        if world == 1 and not args.no_sweep:
            sweep = decoder_sweep(data, emax, local, 3, 1)
            sweep["roofline"]["peak"] = hbm_peak
            sweep["roofline"]["frac"] = sweep["roofline"]["achieved"] / hbm_peak
        cpu = None
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline_ga(data, emax, os.cpu_count() or 1)
        if rank == 0:
            line = {
                "metric": METRIC, "value": gens_per_s, "unit": "generations/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (SURVEY 8(d) generator convention, random-init populations)",
                "config": ga_config(world, synthetic_machines(J, S)),
                "evals_per_s": evals_all / (ms_max / 1e3),
                "evals_per_step": evals_all / args.steps,
                "kernel_ms_per_step": {"eval": eval_ms / args.steps, "eval_busy": eval_busy_ms / args.steps,
                                       "breed": breed_ms / args.steps, "commit": commit_ms / args.steps,
                                       "note": "eval/breed/commit summed per stream (the cellular and pseudo "
                                               "chains overlap); eval_busy = union of the K1 intervals"},
                "island_best_objectives": island_obj,
                "generations_done": args.warmup + args.steps,
                "roofline": {"bound": "hbm", "kernel": "k_eval (K1 decoder)", "achieved": achieved,
                             "peak": hbm_peak, "peak_source": peak_src, "unit": "GB/s",
                             "frac": achieved / hbm_peak, "traffic": traffic,
                             "traffic_unit": "bytes per launch (ncu dram read+write, %s)" % prof.get("source"),
                             "time_basis": "union of the K1 launch intervals (CUDA events on both step streams)",
                             "launches": eval_n,
                             "algorithmic_bytes_per_launch": algo_bytes / max(1, eval_n),
                             "algorithmic_bytes_per_eval": L + 16,
                             "issue_roofline": issue,
                             "note": "decoder is latency/issue bound (fp64 max/add chains + smem list "
                                     "merges); see profiles/ for issue-active and DRAM counters"},
                "e2e": {"value": args.steps / e2e_s, "unit": "generations/s",
                        "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
                        "what": "generate instance + IslandModel init + run(K generations) + traces/champion D2H; "
                                "median of %d runs in one process after one untimed run" % E2E_RUNS,
                        "parts": e2e_parts,
                        "best_objective": res.best_report["objective"]},
                "gpu_launches": int(l1 - l0),
                "clocks": clk.summary(),
                "cpu_baseline": cpu,
                "decoder_sweep": sweep,
            }
            print(json.dumps(line), flush=True)
    else:  # decoder workload
        ci = model.inst
        b = capi.Batch(ci, SWEEP_N)
        b.fill_random(99, 0, SWEEP_N)
        for _ in range(args.warmup):
            b.evaluate(SWEEP_N)
        b.sync()
        barrier()
        l0 = capi.launch_count()
        ms = []
        with ClockSampler(local) as clk:
            for _ in range(args.steps):
                b.evaluate(SWEEP_N)
                ms.append(b.last_eval_ms())
        l1 = capi.launch_count()
        tot = float(np.sum(ms))
        if comm is not None:
            tot = float(comm.allgather(np.array([tot]))[:, 0].max())
        val = world * SWEEP_N * args.steps / (tot / 1e3)
        # e2e: host u8 genes -> device -> evaluate -> results back, through the C ABI
        host = b.download(0, 4096).astype(np.uint8)
        n_e2e = 65536
        import torch
        # the batch in page-locked host memory (the contract's e2e input): the copy engine reads
        # it in place; a pageable batch goes through the library's pinned staging pair instead
        pinned = torch.empty((n_e2e, L), dtype=torch.uint8, pin_memory=True).numpy()
        pinned[:] = np.tile(host, (n_e2e // 4096, 1))
        pageable = np.array(pinned, copy=True)

        def e2e_rate(buf):
            ci.evaluate(buf)  # untimed: the first call sizes the device (and staging) buffers
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                ci.evaluate(buf)
                ts.append(time.perf_counter() - t0)
            return n_e2e / float(np.median(ts))

        e2e = e2e_rate(pinned)
        e2e_pageable = e2e_rate(pageable)
        if rank == 0:
            achieved = SWEEP_N * (L + 16) / (tot / args.steps / 1e3) / 1e9
            print(json.dumps({
                "metric": METRIC, "value": val, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": tot / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "C5 decoder sweep: 1M random chromosomes per launch, 500x20, M in [2,8]",
                           "l2": "inputs larger than L2 (10.7 GB of genes per launch)"},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                             "frac": achieved / hbm_peak, "traffic": None},
                "e2e": {"value": e2e, "unit": "evals/s", "h2d_bytes_per_step": n_e2e * L,
                        "d2h_bytes_per_step": n_e2e * 16, "input": "page-locked host batch (u8)",
                        "pageable_value": e2e_pageable},
                "gpu_launches": int(l1 - l0), "clocks": clk.summary()}), flush=True)
    if comm is not None:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
