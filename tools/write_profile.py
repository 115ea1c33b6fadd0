"""Write profiles/<round>_config3.md and profiles/<round>_traffic.json from the
ncu outputs of one profiling session (see the commands in the generated
markdown):

    python tools/write_profile.py --round r1 --launches gpurun_out/launches.csv \
        --raster gpurun_out/prof_raster2.ncu-rep [--extra gpurun_out/prof_scatter.ncu-rep ...]

The raster report must hold one raster_fwd and one raster_bwd launch.
"""

import argparse
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tools"))
import ncu_summary  # noqa: E402

UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
PIPES = ["smsp__issue_active.avg.pct_of_peak_sustained_active",
         "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
         "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
         "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
         "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
         "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
         "gpu__time_duration.sum",
         "sm__throughput.avg.pct_of_peak_sustained_elapsed",
         "lts__throughput.avg.pct_of_peak_sustained_elapsed",
         "l1tex__throughput.avg.pct_of_peak_sustained_active",
         "lts__t_sector_hit_rate.pct",
         "sm__warps_active.avg.pct_of_peak_sustained_active"]


def raster_sha16():
    import hashlib

    src = ROOT / "paper_2409_07759_b200" / "csrc" / "raster.cu"
    return hashlib.sha256(src.read_bytes()).hexdigest()[:16]


def kernel_table(rep, peak_gbs):
    """Per-kernel DRAM bytes / duration / achieved GB/s / fraction of the
    measured HBM peak and issue utilisation from a --set full report."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]

    def val(r, w):
        i = hdr.index(w)
        try:
            return float(r[i]) * UNITS.get(units[i], 1.0)
        except ValueError:
            return float("nan")

    out = ["| kernel | time (us) | DRAM read+write (MB) | achieved DRAM GB/s | frac of "
           f"{peak_gbs:.0f} GB/s | issue busy % | SM throughput % | occupancy % |",
           "|---|---|---|---|---|---|---|---|"]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").replace("ss::", "")[:40]
        us = val(r, "gpu__time_duration.sum")
        b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        gbs = b / (us * 1e-6) / 1e9
        out.append(f"| `{short}` | {us:.1f} | {b / 1e6:.1f} | {gbs:.0f} | {gbs / peak_gbs:.3f} | "
                   f"{val(r, PIPES[0]):.0f} | {val(r, PIPES[9]):.0f} | {val(r, PIPES[13]):.0f} |")
    return "\n".join(out)


def raw_metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        key = "raster_fwd" if "raster_fwd" in name else "raster_bwd" if "raster_bwd" in name else name
        m = {}
        for w in PIPES:
            if w in hdr:
                i = hdr.index(w)
                try:
                    m[w] = float(r[i]) * UNITS.get(units[i], 1.0)
                except ValueError:
                    pass
        out[key] = m
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r1")
    ap.add_argument("--launches", required=True)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--raster", required=True)
    ap.add_argument("--extra", nargs="*", default=[])
    ap.add_argument("--k-used", type=float, default=None,
                    help="K_used of the profiled view (bench --profile-steps prints it)")
    ap.add_argument("--peak", type=float, default=6553.6)
    a = ap.parse_args()
    prof = ROOT / "profiles"
    shutil.copy(a.launches, prof / f"{a.round}_config3_launches.csv")
    m = raw_metrics(a.raster)
    f, b = m["raster_fwd"], m["raster_bwd"]
    sha = raster_sha16()
    traffic = {k: {"dram_bytes_read": v["dram__bytes_read.sum"],
                   "dram_bytes_write": v["dram__bytes_write.sum"],
                   "duration_us": v["gpu__time_duration.sum"],
                   "issue_active_pct": v["smsp__issue_active.avg.pct_of_peak_sustained_active"],
                   "warp_instructions": v["smsp__inst_executed.sum"],
                   "sm_throughput_pct": v.get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                   "l2_throughput_pct": v.get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                   "l1_throughput_pct": v.get("l1tex__throughput.avg.pct_of_peak_sustained_active"),
                   "l2_hit_rate_pct": v.get("lts__t_sector_hit_rate.pct"),
                   "occupancy_pct": v.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
                   **({"k_used": a.k_used,
                       "warp_instructions_per_k_used_entry": v["smsp__inst_executed.sum"] / a.k_used}
                      if a.k_used else {})}
               for k, v in (("raster_fwd", f), ("raster_bwd", b))}
    traffic["raster_cu_sha16"] = sha
    traffic["source"] = (f"ncu --set full --clock-control none, config 3 (bench.py --profile-steps 1), "
                         f"round {a.round[1:]}; bytes converted from the raw page's units")
    (prof / f"{a.round}_traffic.json").write_text(json.dumps(traffic, indent=1))

    def row(name, v):
        return (f"| {name} | {v[PIPES[0]]:.0f} | {v[PIPES[1]]:.0f} | {v[PIPES[2]]:.0f} | "
                f"{v[PIPES[3]]:.0f} | {v[PIPES[4]]:.0f} | {v[PIPES[5]] / 1e6:.0f} M |")

    def row2(name, v):
        g = lambda k: v.get(k, float("nan"))  # noqa: E731
        return (f"| {name} | {g(PIPES[9]):.0f} | {g(PIPES[10]):.0f} | {g(PIPES[11]):.0f} | "
                f"{g(PIPES[12]):.0f} | {g(PIPES[13]):.0f} |")

    reports = "\n".join(ncu_summary.report(r) for r in [a.raster] + a.extra)
    tables = "\n\n".join(kernel_table(r, a.peak) for r in [a.raster] + a.extra)
    md = f"""# Round {a.round[1:]} — config 3 profile (DyNeRF-shaped, 300k splats, 1352x1014, B200)

Commands (one B200; each ncu command ran after the same command exited 0 without ncu):

    python bench.py --warmup 3 --profile-steps 2 --no-cpu-baseline --no-e2e
    ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \\
        --csv --log-file launches.csv python bench.py --warmup 3 --profile-steps 2 --no-cpu-baseline --no-e2e
    ncu --set full --clock-control none --import-source on --profile-from-start off \\
        -k regex:raster_ -c 2 -o prof_raster python bench.py --warmup 3 --profile-steps 1 --no-cpu-baseline --no-e2e

`bench.py --profile-steps N` runs N training views between cudaProfilerStart/Stop
after warm-up (window [1, 11)).  Raw launch list: `profiles/{a.round}_config3_launches.csv`;
per-launch DRAM bytes and issue utilisation of the raster kernels:
`profiles/{a.round}_traffic.json` (bench.py reports them in `roofline`).
Regenerate with `python tools/write_profile.py`.

{ncu_summary.launches(a.launches, a.steps)}

## Where the raster kernels sit

Both raster kernels are instruction-issue bound, not HBM bound: DRAM traffic is
{(f['dram__bytes_read.sum'] + f['dram__bytes_write.sum']) / 1e6:.1f} MB (fwd) and {(b['dram__bytes_read.sum'] + b['dram__bytes_write.sum']) / 1e6:.1f} MB (bwd) per launch, a few % of
the HBM roofline, while the SM issue slots are busy {f[PIPES[0]]:.0f} % (fwd) and {b[PIPES[0]]:.0f} % (bwd)
of active cycles.  Pipe shares (percent of peak, active cycles):

| kernel | issue | fma | alu | xu (MUFU) | lsu | warp instructions |
|---|---|---|---|---|---|---|
{row("raster_fwd", f)}
{row("raster_bwd", b)}

Throughput against B200 peak (ncu, percent): SM is busy, the memory
hierarchy is not -- L2 a few %, DRAM ~1 % (the tile lists' 36-B records are
re-read from L1/L2, hit rate below).

| kernel | SM throughput | L2 throughput | L1 throughput | L2 hit rate | achieved occupancy |
|---|---|---|---|---|---|
{row2("raster_fwd", f)}
{row2("raster_bwd", b)}

## Per-kernel DRAM roofline (ncu --set full, one launch each, config 3)

Achieved DRAM GB/s = (dram__bytes_read + dram__bytes_write) / duration, over
the measured HBM copy peak (MEASURED_PEAKS.json).  Serialised, cold-cache
replays: read the fractions, not the absolute times.

{tables}

{reports}
"""
    (prof / f"{a.round}_config3.md").write_text(md)
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
