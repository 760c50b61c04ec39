#!/usr/bin/env python
"""Throughput of the engine on every BASELINE.json configuration that fits one
GPU (informational; bench.py is the contract line). For each config it runs
the full configured step count through rd_step and reports device time,
Gcell-updates/s, launches and the probe outcomes. Prints one JSON per config.

  python scripts/bench_configs.py [--configs 1,2,3,4] [--dtype f32|f64|both]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1901_06535_b200 as rd  # noqa: E402
from rdinputs import config  # noqa: E402


def hbm_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


def run(n, dtype, tb):
    w = config(n, dtype=dtype)
    if n in (4, 5):
        # large grids are built on the device (phi paint + seeded noise)
        sim = rd.Sim(None, shape=(1, w.H, w.W), dtype=dtype, tb_depth=tb)
        sim.paint_phi(0.054)
        for rect in w.meta.get("obstacles", []):
            sim.paint_phi(0.2, rect)
        sim.fill_noise(seed=1)
    else:
        phi = np.stack([w.phi_plane(b).astype(dtype) for b in range(w.B)])
        sim = rd.Sim(phi, dtype=dtype, tb_depth=tb)
        if w.init is not None:
            for b in range(w.B):
                u0, v0 = w.init_planes(b)
                sim.write(b, u0, v0)
    for b in range(w.B):
        for shape, val, at in w.events[b]:
            sim.stimulate(shape, val, at, b=b)
    pids = [[sim.probe_latch(b, r, t, s) for (r, t, s) in w.probes[b]] for b in range(w.B)] if w.probes else []
    stream = torch.cuda.current_stream()
    sim.set_stream(stream)
    rd.rd_reset_stats(sim.h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(stream)
    sim.step(w.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    st = sim.stats()
    fires = [[sim.probe_result(p) for p in ps] for ps in pids]
    cells = w.B * w.H * w.W * w.steps
    sim.close()
    gcells = cells / (ms / 1e3) / 1e9
    # one-step HBM roofline: read u, v, phi + write u, v = 20 B (fp32) / 40 B
    # (fp64) per cell-update at the measured copy bandwidth
    roof = hbm_gbs() / (20 if np.dtype(dtype).itemsize == 4 else 40)
    return {"config": w.name, "dtype": np.dtype(dtype).name, "B": w.B, "H": w.H, "W": w.W, "steps": w.steps,
            "device_ms": ms, "wall_s": wall, "gcell_updates_per_s": gcells,
            "frac_of_one_step_hbm_roofline": gcells / roof, "stencil_kernel": ["tb", "lp", "cr", "gz"][st["kernel"]],
            "launches": st["launches"], "step_launches": st["step_launches"], "tb_depth": st["tb_depth"],
            "first_fire": fires, "expect": w.expect.get("fires")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--dtype", default="both")
    ap.add_argument("--tb", type=int, default=0)
    ap.add_argument("--repeat", type=int, default=2, help="runs per config; the last is reported (the first "
                    "warms clocks, caches and graph captures)")
    a = ap.parse_args()
    dts = {"f32": [np.float32], "f64": [np.float64], "both": [np.float32, np.float64]}[a.dtype]
    for n in map(int, a.configs.split(",")):
        for dt in dts:
            if n in (4, 5) and dt == np.float64:
                continue
            for _ in range(a.repeat - 1):
                run(n, dt, a.tb)
            print(json.dumps(run(n, dt, a.tb)), flush=True)


if __name__ == "__main__":
    main()
