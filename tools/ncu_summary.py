#!/usr/bin/env python3
"""Summarise gpurun ncu outputs for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches <launches.csv>        per-kernel share of a launch list
  python tools/ncu_summary.py full <report.ncu-rep> [...]     SOL / occupancy / stalls / DRAM bytes
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("GPU Speed Of Light Throughput", ["Duration", "Elapsed Cycles", "SM Active Cycles", "SM Frequency",
                                       "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
                                       "L2 Cache Throughput", "L1/TEX Cache Throughput"]),
    ("Compute Workload Analysis", ["Issue Slots Busy", "Executed Ipc Active"]),
    ("Occupancy", ["Theoretical Occupancy", "Achieved Occupancy", "Achieved Active Warps Per SM"]),
    ("Launch Statistics", ["Registers Per Thread", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block"]),
    ("Scheduler Statistics", ["Issued Warp Per Scheduler", "No Eligible", "Eligible Warps Per Scheduler"]),
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def ncu_csv(rep, page, *extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(rep):
    """One table per profiled launch: SOL / occupancy / launch / scheduler
    sections, DRAM and instruction counters, and the stall breakdown."""
    rows = ncu_csv(rep, "details")
    h = rows[0]
    per = collections.OrderedDict()   # launch ID -> (kernel, lines)
    for r in rows[1:]:
        d = dict(zip(h, r))
        lid = d.get("ID")
        if lid not in per:
            per[lid] = (d.get("Kernel Name"), [])
        for sec, names in KEYS:
            if d.get("Section Name") == sec and d.get("Metric Name") in names:
                per[lid][1].append("| %s | %s | %s %s |" % (sec.split()[0], d["Metric Name"], d["Metric Value"],
                                                             d["Metric Unit"]))
    raw = ncu_csv(rep, "raw")
    rh, units = raw[0], raw[1]
    for i, rv in enumerate(raw[2:]):
        lid = list(per.keys())[i] if i < len(per) else None
        if lid is None:
            break
        lines = per[lid][1]
        stalls = []
        for name, u, v in zip(rh, units, rv):
            if name in RAW:
                lines.append("| raw | %s | %s %s |" % (name, v, u))
            if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
                try:
                    if float(v) >= 0.05:
                        stalls.append((float(v), name[len("smsp__average_warps_issue_stalled_"):
                                                      -len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        lines.append("| stalls | per issued instruction | %s |" % ", ".join("%s %.2f" % (n, v) for v, n in stalls))
    for lid, (kern, lines) in per.items():
        print("### %s, launch %s\n\n`%s`\n\n| section | metric | value |\n|---|---|---|" % (rep.split("/")[-1], lid,
                                                                                              kern))
        print("\n".join(lines))
        print()


def launches(path, traffic_out=None):
    """Per-kernel time share; with dram__bytes_{read,write}.sum in the list
    (ncu --cache-control none), also the warm-L2 DRAM traffic per kernel."""
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    with open(path) as f:
        txt = [l for l in f if l.startswith('"')]
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    for r in csv.DictReader(io.StringIO("".join(txt))):
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        if r.get("Metric Name") == "gpu__time_duration.sum":
            agg[k][0] += 1
            agg[k][1] += v * scale.get(r["Metric Unit"], 1.0)
        elif r.get("Metric Name", "").startswith("dram__bytes_"):
            agg[k][2] += v * bscale.get(r["Metric Unit"], 1.0)
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | total us | share | avg us | DRAM bytes (warm) |\n|---|---|---|---|---|---|")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print("| `%s` | %d | %.1f | %.1f%% | %.2f | %s |" % (k, n, t, 100 * t / tot, t / n,
                                                          "%.3g" % b if b else "-"))
    print("\nTotal %.1f us over %d launches (serialised by ncu: compare shares)." %
          (tot, sum(a[0] for a in agg.values())))
    if traffic_out:
        corr = sum(b for k, (n, t, b) in agg.items() if k.startswith("k_corr"))
        with open(traffic_out, "w") as f:
            json.dump({"corr_dram_bytes_per_step": corr, "source": path,
                       "note": "sum of dram__bytes_read.sum + dram__bytes_write.sum over the correlation "
                               "launches of one bench step, ncu --cache-control none (warm L2)"}, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        for rep in sys.argv[2:]:
            full(rep)
