#!/usr/bin/env python
"""Summarise ncu outputs (gpurun_out/) into tracked files under profiles/.

  python scripts/summarize_ncu.py --round r01 [--launches gpurun_out/launches.csv]
                                   [--full gpurun_out/prof_full.ncu-rep]

Writes profiles/<round>_launches.json (per-kernel launch count, total and
average device time, share of the launch list) and
profiles/<round>_<kernel>_full.json (the key --set full metrics of the top
kernel: duration, DRAM bytes, throughput, occupancy, issue, stall reasons),
plus profiles/traffic_<round>.json (dram bytes per launch) read by bench.py.
"""
import argparse
import collections
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_static", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def to_us(v, unit):
    v = float(str(v).replace(",", ""))
    return {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}.get(unit, v)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += to_us(r[vi], r[ui])
        cnt[name] += 1
    T = sum(tot.values())
    return [{"kernel": k, "launches": cnt[k], "total_ms": tot[k] / 1e3, "avg_us": tot[k] / cnt[k],
             "share": tot[k] / T} for k in sorted(tot, key=lambda k: -tot[k])]


def full(path):
    # a .csv is the raw page already exported on the GPU box (ncu -i X.ncu-rep --page raw --csv)
    out = (open(path).read() if path.endswith(".csv") else
           subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            d[h] = {"value": v, "unit": u}
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                d.setdefault("stall_per_issue", {})[h[len("smsp__average_warps_issue_stalled_"):-len(
                    "_per_issue_active.ratio")]] = float(v)
            except ValueError:
                pass
    d["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--launches", default=os.path.join(ROOT, "gpurun_out", "launches.csv"))
    ap.add_argument("--full", default=os.path.join(ROOT, "gpurun_out", "prof_full.ncu-rep"))
    ap.add_argument("--cr", default=os.path.join(ROOT, "gpurun_out", "prof_cr.ncu-rep"),
                    help="--set full capture of cr_kernel (config 2)")
    ap.add_argument("--gz", default=os.path.join(ROOT, "gpurun_out", "prof_gz_raw.csv"),
                    help="--set full capture of gz_kernel (config 3 fp32)")
    ap.add_argument("--f64", default=os.path.join(ROOT, "gpurun_out", "prof_tb_f64_raw.csv"),
                    help="raw page of the --set full capture of tb_kernel<double> on the config-4 grid")
    ap.add_argument("--cmd", default="")
    ap.add_argument("--workload", default="c4_roofline", help="bench workload tag of the --full capture")
    ap.add_argument("--kernel-tag", default="tb_kernel<float,K=4>", help="bench.py's kernel name")
    ap.add_argument("--cells", type=float, default=16384.0 * 16384 * 4, help="cell-updates per captured launch")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if os.path.exists(a.launches):
        L = launches(a.launches)
        json.dump({"source": "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: "
                             "compare shares, not absolutes)", "command": a.cmd, "kernels": L},
                  open(os.path.join(PROF, f"{a.round}_launches.json"), "w"), indent=1)
        for r in L:
            print(f"{r['kernel'][:70]:70s} n={r['launches']:5d} avg={r['avg_us']:10.1f} us share={r['share']*100:6.2f}%")
    if os.path.exists(a.full):
        F = full(a.full)
        json.dump(F, open(os.path.join(PROF, f"{a.round}_tb_kernel_full.json"), "w"), indent=1)
        rb = float(F["dram__bytes_read.sum"]["value"]) * (1e9 if F["dram__bytes_read.sum"]["unit"] == "Gbyte" else 1e6 if F["dram__bytes_read.sum"]["unit"] == "Mbyte" else 1)
        wb = float(F["dram__bytes_write.sum"]["value"]) * (1e9 if F["dram__bytes_write.sum"]["unit"] == "Gbyte" else 1e6 if F["dram__bytes_write.sum"]["unit"] == "Mbyte" else 1)
        # bench.py uses an entry only for this exact workload / kernel / launch size
        ent = {"workload": a.workload, "kernel": a.kernel_tag, "cell_updates_per_launch": a.cells,
               "dram_bytes_per_launch": rb + wb, "read": rb, "write": wb, "ncu_kernel": F["kernel"],
               "source": f"ncu --set full capture ({os.path.basename(a.full)}), profiles/{a.round}_tb_kernel_full.json"}
        json.dump({"what": "DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) from one ncu "
                           "--set full capture, with the workload, kernel and cell-updates per launch it was "
                           "measured on", "entries": [ent]},
                  open(os.path.join(PROF, f"traffic_{a.round}.json"), "w"), indent=1)
        for k, v in F.items():
            print(k, v)
    if os.path.exists(a.cr):
        F = full(a.cr)
        F["source"] = f"ncu --set full capture ({os.path.basename(a.cr)}), config 3 fp32 (scripts/gpu_round2_base.sh)"
        json.dump(F, open(os.path.join(PROF, f"{a.round}_cr_kernel_full.json"), "w"), indent=1)
        print("cr_kernel:", {k: F[k] for k in ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active") if k in F})
    gz_summary(a)
    if os.path.exists(a.f64):
        F = full(a.f64)
        F["source"] = (f"ncu --set full capture ({os.path.basename(a.f64)}), tb_kernel<double, K=4> (LEAN) on the "
                       "config-4 grid in fp64 (bench.config4_fp64, scripts/gpu_round2_base.sh)")
        json.dump(F, open(os.path.join(PROF, f"{a.round}_tb_kernel_f64_full.json"), "w"), indent=1)
        print("tb_kernel fp64:", {k: F[k] for k in ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active") if k in F})


def gz_summary(a):
    if os.path.exists(a.gz):
        F = full(a.gz)
        F["source"] = f"ncu --set full capture ({os.path.basename(a.gz)}), config 3 fp32 (2 x 200x600, 20000 steps)"
        json.dump(F, open(os.path.join(PROF, f"{a.round}_gz_kernel_full.json"), "w"), indent=1)
        print("gz_kernel:", {k: F[k] for k in ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active") if k in F})


if __name__ == "__main__":
    main()
