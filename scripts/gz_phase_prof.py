#!/usr/bin/env python
"""Phase timing of gz_kernel from a measurement build (-DRD_GZ_PROF): runs a
config through the library, then prints per-exchange-block cycle averages
(compute, publish, slowest fetch, post-exchange barrier) over the CTAs.
Development tool: python scripts/gz_phase_prof.py --config 3 --dtype f32"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1901_06535_b200 as rd  # noqa: E402
from rdinputs import config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--dtype", default="f32")
a = ap.parse_args()
dt = np.float32 if a.dtype == "f32" else np.float64
w = config(a.config, dtype=dt)
sim = rd.Sim(np.stack([w.phi_plane(b).astype(dt) for b in range(w.B)]), dtype=dt)
for b in range(w.B):
    if w.init is not None:
        sim.write(b, *w.init_planes(b))
    for s, val, at in w.events[b]:
        sim.stimulate(s, val, at, b=b)
lib = rd.load()
buf = (ctypes.c_ulonglong * (2048 * 8))()
lib.rd_gz_prof_dump(buf, 2048 * 8)  # clear
sim.step(w.steps)
sim.stats()
lib.rd_gz_prof_dump(buf, 2048 * 8)
arr = np.frombuffer(buf, dtype=np.uint64).reshape(2048, 8).astype(np.float64)
used = arr[:, 4] > 0
blocks = arr[used, 4]
ph = arr[used, :7] / blocks[:, None]
print(f"{used.sum()} CTAs, {blocks.mean():.0f} exchange blocks each; cycles per block (mean / max over CTAs):")
for i, name in [(0, "compute"), (1, "publish"), (2, "slowest fetch"), (3, "post barrier"),
                (5, "poll passes (max thread)"), (6, "fetch loop (max thread)")]:
    print(f"  {name:14s} {ph[:, i].mean():9.0f} {ph[:, i].max():9.0f}")
sim.close()
