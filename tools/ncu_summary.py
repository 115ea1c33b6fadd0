"""Summarise ncu outputs for profiles/: a launch list (gpu__time_duration.sum
CSV) as per-kernel shares of the step, and a --set full report's key metrics
and stall reasons.

    python tools/ncu_summary.py --launches gpurun_out/launches.csv --steps 2 \
        --report gpurun_out/prof_raster.ncu-rep > profiles/r1_config3.md
"""

import argparse
import collections
import csv
import subprocess
import sys

KEYS = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy",
        "Achieved Occupancy", "Waves Per SM", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler"]


def launches(path, steps):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        us = v / 1000 if u == "nsecond" else v * 1000 if u == "msecond" else v if u == "usecond" else v / 1000
        name = d["Kernel Name"].split("(")[0][:80]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    out = [f"Launch list ({path}), {steps} profiled steps, serialised cold-cache times "
           f"(compare shares, not absolutes). Total {tot / steps:.1f} us/step.", "",
           "| kernel | launches/step | us/step | share |", "|---|---|---|---|"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{n}` | {c / steps:g} | {t / steps:.1f} | {100 * t / tot:.1f} % |")
    return "\n".join(out)


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                              "Metric Unit"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        k = r[ki].split("(")[0]
        if r[mi] in KEYS:
            per.setdefault(k, {}).setdefault(r[mi], f"{r[vi]} {r[ui]}".strip())
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    stalls = {}
    dram = {}
    if rr:
        h = rr[0]
        for r in rr[2:]:
            k = r[h.index("Kernel Name")].split("(")[0]
            items = []
            for i, col in enumerate(h):
                if col.startswith("smsp__average_warps_issue_stalled_") and col.endswith(
                        "_per_issue_active.ratio"):
                    try:
                        items.append((float(r[i]), col[len("smsp__average_warps_issue_stalled_"):
                                                       -len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
                if col in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    dram.setdefault(k, {})[col] = (r[i], rr[1][i])
            items.sort(reverse=True)
            stalls.setdefault(k, items[:6])
    out = [f"Full ncu capture ({path}):", ""]
    for k, m in per.items():
        out.append(f"### `{k}`")
        out.append("")
        for key in KEYS:
            if key in m:
                out.append(f"- {key}: {m[key]}")
        if k in dram:
            out.append("- DRAM bytes: " + ", ".join(f"{c} = {v} {u}" for c, (v, u) in dram[k].items()))
        if stalls.get(k):
            out.append("- top stalls (cycles per issued instruction): " +
                       ", ".join(f"{n} {v:.2f}" for v, n in stalls[k]))
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--report")
    a = ap.parse_args()
    if a.launches:
        print(launches(a.launches, a.steps))
        print()
    if a.report:
        print(report(a.report))
