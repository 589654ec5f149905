"""Turn the ncu outputs of one GPU session into the committed profile files.

    python profiles/tools/summarize_ncu.py LAUNCHES_CSV REPORT.ncu-rep [REPORT ...] --tag r1

LAUNCHES_CSV: `ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ...`
of `bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep` (per-launch times, cold-cache,
serialised: only the SHARES are meaningful).  REPORTs: `ncu --set full --clock-control none`
captures of single launches of the GA step.  Writes profiles/<tag>_summary.txt,
profiles/<tag>_ncu.json and profiles/<tag>_traffic.json (K1 DRAM bytes per evaluation).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.per_cycle_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__occupancy_limit_shared_mem",
]


def short(name):
    return name.split("(")[0].replace("ffsga_dev::", "").replace("<unnamed>::", "").strip()


def launches(path):
    txt = open(path).read()
    txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in csv.DictReader(io.StringIO(txt)):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
        k = short(r["Kernel Name"])
        tot[k] += ms
        cnt[k] += 1
    return tot, cnt


def raw(rep):
    """rep: an .ncu-rep, or its `ncu -i REP --page raw --csv` export (.csv)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for row in data:
        d = {"kernel": row[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = row[i].replace(",", "")
                try:
                    x = float(v)
                except ValueError:
                    d[m] = v
                    continue
                u = units[i].strip()
                if m == "gpu__time_duration.sum":  # -> ms
                    x *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                          "second": 1e3, "s": 1e3}.get(u, 1.0)
                elif m.startswith("dram__bytes"):  # -> bytes
                    x *= {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
                d[m] = x
        d["stalls"] = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                key = h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
                try:
                    d["stalls"][key] = float(row[i])
                except ValueError:
                    pass
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("launches")
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--command", default="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep")
    ap.add_argument("--cell-items", type=int, default=32768,
                    help="items of the cellular K1 launch (C3: 4 x 8192 children); the captured K1 launch "
                         "with the most instructions is that one (the pseudo list holds ~24.6k)")
    a = ap.parse_args()
    tot, cnt = launches(a.launches)
    s = sum(tot.values())
    shares = {k: v / s for k, v in sorted(tot.items(), key=lambda x: -x[1])}
    kernels = []
    for rep in a.reports:
        kernels += raw(rep)
    lines = [f"# {a.tag}: launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)",
             f"# command: {a.command}  (includes island init)"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k:34s} launches {cnt[k]:4d}  total {v:10.3f} ms  share {v / s * 100:5.1f}%")
    lines += ["", f"# {a.tag}: ncu --set full --clock-control none (one capture per kernel, inside the GA step)"]
    for d in kernels:
        lines += ["", f"## {d['kernel']}"]
        for m in METRICS:
            if m in d:
                unit = {"gpu__time_duration.sum": " ms", "dram__bytes_read.sum": " B", "dram__bytes_write.sum": " B"}.get(m, "")
                lines.append(f"  {m:64s} {d[m]}{unit}")
        lines.append("  stalls (warps per issue-active cycle):")
        for k, v in sorted(d["stalls"].items(), key=lambda x: -x[1])[:8]:
            lines.append(f"    {k:24s} {v:.3f}")
    with open(os.path.join(HERE, f"{a.tag}_summary.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(HERE, f"{a.tag}_ncu.json"), "w") as f:
        json.dump({"shares": shares, "kernels": kernels}, f, indent=1)
    evals = [d for d in kernels if "k_eval<8, 0" in d["kernel"]]
    if evals:
        d = max(evals, key=lambda x: x["smsp__inst_executed.sum"])
        rd, wr = d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
        scale = 1.0
        tr = {"kernel": "k_eval<8,0> (cellular work list of one C3 generation, 4 x 8192 children; joint-step CTAs)",
              "items_in_captured_launch": a.cell_items,
              "dram_read_bytes": rd * scale, "dram_write_bytes": wr * scale,
              "traffic_bytes_per_eval": (rd + wr) * scale / a.cell_items,
              "algorithmic_bytes_per_eval": 10016,
              "source": f"profiles/{a.tag}_summary.txt (ncu --set full --clock-control none, bench.py GA step)"}
        with open(os.path.join(HERE, f"{a.tag}_traffic.json"), "w") as f:
            json.dump(tr, f, indent=1)
        # what bench.py reads (roofline.traffic, roofline.issue_roofline): one file per round
        prof = {"kernel": d["kernel"], "items_in_captured_launch": a.cell_items,
                "launch_ms": d["gpu__time_duration.sum"],
                "traffic_bytes_per_eval": (rd + wr) / a.cell_items,
                "algorithmic_bytes_per_eval": 10016,
                "achieved_gbs_ncu": 10016 * a.cell_items / (d["gpu__time_duration.sum"] / 1e3) / 1e9,
                "issue_active": d["smsp__issue_active.avg.pct_of_peak_sustained_active"] / 100.0,
                "warps_per_sm": d["sm__warps_active.avg.per_cycle_active"],
                "threads_per_inst": d["smsp__thread_inst_executed_per_inst_executed.ratio"],
                "smem_bank_conflicts": d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
                "capture": f"profiles/{a.tag}_summary.txt"}
        with open(os.path.join(HERE, f"{a.tag}_k1_profile.json"), "w") as f:
            json.dump(prof, f, indent=1)
    print("\n".join(lines[:20]))


if __name__ == "__main__":
    main()
