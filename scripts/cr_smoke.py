#!/usr/bin/env python
"""Quick GPU check of the kernel choice and oracle parity on a few ragged
small grids (development helper; the tests are the gate)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1901_06535_b200 as rd  # noqa: E402
from rdinputs import noise_plane  # noqa: E402

for dt in (np.float32, np.float64):
    for (H, W) in [(64, 64), (37, 131), (301, 29), (9, 700), (128, 128)]:
        u0 = noise_plane(H, W, 0, seed=4, dtype=dt)
        v0 = noise_plane(H, W, 1, seed=4, dtype=dt)
        phi = np.full((H, W), 0.054, dt)
        ev = [({"kind": "disc", "cy2": H, "cx2": W, "r": 3}, 1.0, 0)]
        sim = rd.Sim(phi[None], dtype=dt)
        k0 = sim.stats()["kernel"]
        sim.write(0, u0, v0)
        for s, val, at in ev:
            sim.stimulate(s, val, at)
        sim.step(20)
        u, v = sim.read(0)
        st = sim.stats()
        sim.close()
        ref = oracle.run(u0, v0, phi, 20, events=ev)
        print(np.dtype(dt).name, H, W, "kernel", k0, st["kernel"], "step_launches", st["step_launches"],
              "equal", np.array_equal(u, ref.u), np.array_equal(v, ref.v), float(np.abs(u - ref.u).max()), flush=True)
