"""The device-resident cross-GPU data plane (VERDICT r1 "Next round" 6).

* Migrant packets: export on one island, import on another, device to device, equal to the
  device-local migrate_* (migration.cpp:47-69) -- including the archive (pseudo.cpp:98-113).
* The island driver with a comm that moves CUDA tensors (the NCCL code path of islands.py):
  two ranks as two threads on one GPU exchanging device tensors through an in-process hub (no
  kernel waits on another rank), against the single-process run.  Split couples make the
  migrant packets cross ranks.
* With >= 2 GPUs visible: the same over NCCL, one process per GPU (skipped on a 1-GPU box).
"""
import os
import queue
import subprocess
import sys
import threading

import numpy as np
import pytest

import paper_1903_10722_b200 as ffsga
from paper_1903_10722_b200 import capi, instance_arrays
from paper_1903_10722_b200 import islands as isl

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def as_data(inst):
    from pyoracle import InstanceData
    a = instance_arrays(inst)
    return InstanceData(a.num_jobs, a.num_stages, a.machines, a.proc, a.release, a.due, a.weight)


def test_packets_equal_local_migration():
    import torch
    inst = ffsga.generate_instance(jobs=10, stages=3, machines=[2, 3, 2], weight=0.0, seed=2)
    d = as_data(inst)
    emax = ffsga.estimate_emax(inst)
    ci = capi.Instance.from_data(d, emax)
    a1, b1 = capi.Cellular(ci, 8, 4, 1), capi.Pseudo(ci, 32, 2)
    a2, b2 = capi.Cellular(ci, 8, 4, 1), capi.Pseudo(ci, 32, 2)
    capi.step([a1, a2], [b1, b2], 3)
    capi.migrate_cellular_to_pseudo(a1, b1, 7)
    pk = a2.export_packet(7)
    assert pk.is_cuda and pk.numel() == ci.packet_bytes(0, 7)
    b2.import_packet(pk.clone(), 7)
    torch.cuda.synchronize()
    assert np.array_equal(b1.members(), b2.members()) and np.array_equal(b1.read()[0], b2.read()[0])
    assert b1.archive()[1] == b2.archive()[1] and np.array_equal(b1.archive()[0], b2.archive()[0])
    capi.step([a1, a2], [b1, b2], 2)
    capi.migrate_pseudo_to_cellular(b1, a1, 5)
    pk = b2.export_packet(5)
    assert pk.numel() == ci.packet_bytes(1, 5)
    a2.import_packet(pk, 5)
    assert np.array_equal(a1.genes(), a2.genes()) and np.array_equal(a1.read()[0], a2.read()[0])
    assert a1.best() == a2.best()
    st = torch.empty(4, dtype=torch.float64, device="cuda")
    a2.state_device(st)
    i, f, o = a2.best()
    assert st[0].item() == f and st[1].item() == o
    b2.state_device(st)
    _, af, ao = b2.archive()
    assert st[2].item() == af and st[3].item() == ao
    # host halves ride the same packets
    g, f, o = a1.export_best(4)
    b1.import_worst(g, f, o)
    b2.import_packet(a2.export_packet(4), 4)
    assert np.array_equal(b1.members(), b2.members()) and b1.archive()[1] == b2.archive()[1]


class _Hub:
    def __init__(self, world):
        self.world = world
        self.slots = [None] * world
        self.bar = threading.Barrier(world)
        self.q = {(s, t): queue.Queue() for s in range(world) for t in range(world)}


class ThreadComm:
    """A comm whose ranks are threads of one process, moving CUDA tensors (device_tensors: the
    islands.py NCCL path).  Test double only."""

    device_tensors = True

    def __init__(self, hub, rank):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def allgather_tensor(self, t):
        import torch
        self.hub.slots[self.rank] = t.clone()
        self.hub.bar.wait()
        out = torch.stack(list(self.hub.slots))
        self.hub.bar.wait()
        return out

    def send_tensor(self, t, dst):
        self.hub.q[(self.rank, dst)].put(t.clone())

    def recv_tensor(self, t, src):
        t.copy_(self.hub.q[(src, self.rank)].get(timeout=120))

    def broadcast_tensor(self, t, src):
        if self.rank == src:
            self.hub.slots[src] = t.clone()
        self.hub.bar.wait()
        if self.rank != src:
            t.copy_(self.hub.slots[src])
        self.hub.bar.wait()

    def allgather(self, vec):
        self.hub.slots[self.rank] = np.array(vec, copy=True)
        self.hub.bar.wait()
        out = np.stack(self.hub.slots)
        self.hub.bar.wait()
        return out

    def barrier(self):
        self.hub.bar.wait()


@pytest.mark.parametrize("couples,world,gap", [(1, 2, 2), (3, 2, 3), (2, 4, 2)])
def test_island_driver_device_plane_equals_single_process(couples, world, gap):
    # weight 0 on a small instance: the policy moves rows (k >= 1) at several rendezvous
    inst = ffsga.generate_instance(jobs=8, stages=2, machines=[2, 2], weight=0.0, seed=12)
    d = as_data(inst)
    emax = ffsga.estimate_emax(inst)
    cfg = isl.IslandConfig(couples=couples, island_population=32, generations=24, migration_gap=gap, seed=12)
    want = isl.IslandModel(d, emax, cfg).run()
    assert want.migrations, "the instance must make migrations fire"
    hub = _Hub(world)
    res, errs = [None] * world, []

    def rank(r):
        try:
            m = isl.IslandModel(d, emax, cfg, comm=ThreadComm(hub, r))
            assert m.device_plane
            res[r] = m.run()
        except BaseException as e:  # surfaced below
            errs.append(e)
            hub.bar.abort()

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errs, errs
    for r in range(world):
        got = res[r]
        assert np.array_equal(got.traces, want.traces) and np.array_equal(got.trace_combined, want.trace_combined)
        assert list(got.best_chromosome) == list(want.best_chromosome)
        assert got.best_report == want.best_report
        assert [(e.generation, e.couple, e.direction, e.migrants) for e in got.migrations] == \
               [(e.generation, e.couple, e.direction, e.migrants) for e in want.migrations]


NCCL_SCRIPT = r"""
import os, sys, json
import numpy as np
import torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "oracle"))
import paper_1903_10722_b200 as ffsga
from paper_1903_10722_b200 import instance_arrays, islands as isl
from pyoracle import InstanceData
r = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(r)
dist.init_process_group("nccl", device_id=torch.device("cuda", r))
inst = ffsga.generate_instance(jobs=8, stages=2, machines=[2, 2], weight=0.0, seed=12)
a = instance_arrays(inst)
d = InstanceData(a.num_jobs, a.num_stages, a.machines, a.proc, a.release, a.due, a.weight)
cfg = isl.IslandConfig(couples=1, island_population=32, generations=24, migration_gap=2, seed=12)
comm = isl.TorchComm(device=f"cuda:{r}")
m = isl.IslandModel(d, ffsga.estimate_emax(inst), cfg, comm=comm, device=r)
assert m.device_plane
res = m.run()
if r == 0:
    print(json.dumps({"comb": list(res.trace_combined), "chrom": [int(x) for x in res.best_chromosome],
                      "mig": len(res.migrations)}))
dist.destroy_process_group()
"""


def test_island_driver_over_nccl_two_gpus(tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (NCCL cannot put two ranks on one device)")
    script = tmp_path / "nccl_islands.py"
    script.write_text(NCCL_SCRIPT)
    env = dict(os.environ, ROOT=ROOT)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29541", str(script)],
                       capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    import json
    got = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    inst = ffsga.generate_instance(jobs=8, stages=2, machines=[2, 2], weight=0.0, seed=12)
    cfg = isl.IslandConfig(couples=1, island_population=32, generations=24, migration_gap=2, seed=12)
    want = isl.IslandModel(as_data(inst), ffsga.estimate_emax(inst), cfg).run()
    assert got["comb"] == list(want.trace_combined) and got["chrom"] == list(want.best_chromosome)
    assert got["mig"] == len(want.migrations) > 0


def test_packet_argument_errors():
    import torch
    inst = ffsga.generate_instance(jobs=6, stages=2, machines=[2, 2], seed=3)
    ci = capi.Instance.from_data(as_data(inst), ffsga.estimate_emax(inst))
    c, p = capi.Cellular(ci, 4, 4, 1), capi.Pseudo(ci, 8, 2)
    with pytest.raises(ValueError, match="exceeds an island population"):
        c.export_packet(17)
    with pytest.raises(ValueError, match="exceeds an island population"):
        p.import_packet(torch.zeros(ci.packet_bytes(0, 9), dtype=torch.uint8, device="cuda"), 9)
    with pytest.raises(ValueError):
        c.export_packet(3, out=torch.zeros(4, dtype=torch.uint8, device="cuda"))  # too small
    assert ci.packet_bytes(0, 0) == 0 and c.export_packet(0).numel() == 1  # k = 0: nothing moves
    assert ci.packet_bytes(1, 3) == 3 * (16 + 8 * ((ci.info()["total_bits"] + 63) // 64))
