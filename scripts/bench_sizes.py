#!/usr/bin/env python
"""Throughput against grid size (informational): one instance of side n (or a
batch), uniform phi, seeded noise, a few stimuli, `--steps` time steps through
rd_step with the default kernel choice. Shows where gz_kernel hands over to
tb_kernel and what the sizes in between reach. One JSON line per size.

  python scripts/bench_sizes.py [--sizes 128,256,8192x65536,...] [--dtype f32|f64] [--kernel auto|tb|gz|cr]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1901_06535_b200 as rd  # noqa: E402


def run(n, dtype, steps, batch, obstacles=0):
    h, w = (int(x) for x in n.split("x")) if "x" in n else (int(n), int(n))
    n = h
    sim = rd.Sim(None, shape=(batch, h, w), dtype=dtype)
    sim.paint_phi(0.054)
    rng = np.random.default_rng(3)
    for _ in range(obstacles):  # config-5 style sub-excitable rectangles, sides 32..1024
        hh, ww = (int(x) for x in rng.integers(32, 1025, 2))
        y, x = int(rng.integers(0, max(1, h - hh))), int(rng.integers(0, max(1, w - ww)))
        sim.paint_phi(0.2, (y, x, min(h, y + hh), min(w, x + ww)))
    sim.fill_noise(seed=1)
    sim.stimulate({"kind": "disc", "cy2": h, "cx2": w, "r": 6, "mask_phi": 0.054}, 1.0, 0)
    stream = torch.cuda.current_stream()
    sim.set_stream(stream)
    ms = None
    from bench import Clocks
    for it in range(4):  # the last run is reported (segment graph captured on the 2nd call, clocks up)
        rd.rd_reset_stats(sim.h)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with Clocks(torch.cuda.current_device()) as clk:
            e0.record(stream)
            sim.step(steps)
            e1.record(stream)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    st = sim.stats()
    sim.close()
    mhz = clk.summary()["sm_mhz"]
    rate = batch * h * w * steps / (ms / 1e3) / 1e9
    return {"sm_mhz": mhz, "gcell_per_s_per_ghz": rate / (mhz / 1e3) if mhz else None,"side": n, "width": w, "batch": batch, "dtype": np.dtype(dtype).name, "steps": steps, "device_ms": ms,
            "us_per_step": ms * 1e3 / steps, "gcell_updates_per_s": batch * h * w * steps / (ms / 1e3) / 1e9,
            "stencil_kernel": ["tb", "lp", "cr", "gz"][st["kernel"]], "tb_depth": st["tb_depth"],
            "phi_uniform": st["phi_uniform"], "obstacles": obstacles,
            "launches": st["launches"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="128,256,384,512,768,1024,1536,2048,3072,4096,8192")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--obstacles", type=int, default=0, help="phi = 0.2 rectangles painted into the map")
    a = ap.parse_args()
    os.environ["RD_KERNEL"] = a.kernel
    dt = np.float32 if a.dtype == "f32" else np.float64
    for n in a.sizes.split(","):
        cells = int(n.split("x")[0]) * int(n.split("x")[-1])
        steps = a.steps if cells <= 4096 * 4096 else max(200, a.steps // 4)
        print(json.dumps(run(n, dt, steps, a.batch, a.obstacles)), flush=True)


if __name__ == "__main__":
    main()
