#!/usr/bin/env python
"""gpurun_out/kt_<K>.{json,csv} (scripts/gpu_ktable.sh) -> profiles/<round>_ktable.json:
per temporal-blocking depth K on config 4, the device-timed rate, and from
ncu the DRAM bytes and thread-instructions per cell-update of one tb_kernel
launch (SURVEY.md §8(d) effective-bytes model)."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
H = W = 16384
rows = []
# KT_TAG of scripts/gpu_ktable.sh: "s" = RD_TB_UPHI=0 (phi plane streamed), "u" = the default
# (config 4's one-valued phi as a kernel parameter, K <= 4), "" = untagged.
for tag, K in [(t, k) for t in ("s", "u", "") for k in range(1, 9)]:
    jf, cf = (os.path.join(ROOT, "gpurun_out", f"kt{tag}_{K}.{x}") for x in ("json", "csv"))
    if not (os.path.exists(jf) and os.path.exists(cf)):
        continue
    line = json.loads(open(jf).read().strip().splitlines()[-1])
    m = {}
    with open(cf) as fh:
        body = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(body):
        if "tb_kernel" in r["Kernel Name"]:
            m.setdefault(r["Metric Name"], []).append((r["Metric Unit"], float(r["Metric Value"].replace(",", ""))))

    def avg(name):
        v = m.get(name, [])
        if not v:
            return None
        f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "ns": 1e-9, "usecond": 1e-6,
             "nsecond": 1e-9, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "%": 1, "Ghz": 1e9, "hz": 1}.get(v[0][0], 1)
        return sum(x for _, x in v) / len(v) * f

    cells = H * W * K  # one launch = K steps over the whole grid
    dram = (avg("dram__bytes_read.sum") or 0) + (avg("dram__bytes_write.sum") or 0)
    inst = avg("smsp__inst_executed.sum")
    # SURVEY §8(d) B_eff(k) for 120 output columns per strip: u, v (and phi when streamed) read with the
    # 2K-column halo, u', v' written once
    # (K = 5, 6 run 116 output columns per 128-column strip, K = 4 120, K <= 3 120 with HX = 4)
    wo = 116 if K in (5, 6) else 120
    model = ((8 if line.get("phi_uniform") else 12) * 128 / wo + 8) / K
    rows.append({"K": K, "phi": {"s": "streamed", "u": "parameter when uniform (fp32: K <= 7)", "": "default"}[tag],
                 "phi_uniform_path": line.get("phi_uniform"), "gcell_per_s": line["value"], "sm_mhz": line["clocks"]["sm_mhz"],
                 "ncu_launch_s": avg("gpu__time_duration.sum"),
                 "dram_bytes_per_launch": dram, "dram_bytes_per_cell_update": dram / cells,
                 "model_bytes_per_cell_update": model,
                 "thread_inst_per_cell_update": inst * 32 / cells if inst else None,
                 "issue_active_pct": avg("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 "launches_averaged": len(m.get("dram__bytes_read.sum", []))})
out = {"what": "tb_kernel<float,K> on config 4 (16384^2 fp32): rate from a plain bench run "
               "(--timesteps 60 --steps 3), DRAM bytes / instructions per cell-update from ncu over three "
               "launches of the same command (--clock-control none); cell-updates per launch = 16384^2 x K. "
               "Re-measured on the final round-2 kernel (row-triple rings, UPHI up to K = 7, 6-column halos at "
               "K = 5 and 6); the short runs stay under the power cap, so sm_mhz is the maximum",
       "command": "bash scripts/gpu_ktable.sh", "rows": rows}
dst = os.path.join(ROOT, "profiles", f"{rnd}_ktable.json")
json.dump(out, open(dst, "w"), indent=1)
for r in rows:
    print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()})
