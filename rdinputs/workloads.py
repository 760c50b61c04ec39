"""The five BASELINE.json configurations as seeded synthetic workloads.

A Workload is plain data: grid shape, dtype, per-instance phi planes (fp64,
rounded once by the consumer), initial u/v (None = zeros) and per-instance
events (shape, value, at_step) and probes (rect, threshold, stride). Both the
oracle and the CUDA path consume the same Workload. Recipe: DESIGN.md §4.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from .gen import half_discs, noise_plane, obstacles
from .geometry import and_gate, diode, phi_from_rects

PROBE_THRESHOLD = 0.1  # SPEC.md:269 (R-16)
PROBE_STRIDE = 50


@dataclass
class Workload:
    name: str
    H: int
    W: int
    B: int
    dtype: type
    steps: int
    phi: list                      # B planes (H, W) fp64, or a callable(row0, rows) -> plane
    events: list = field(default_factory=list)   # per instance: [(shape, value, at_step)]
    probes: list = field(default_factory=list)   # per instance: [((y0,x0,y1,x1), thr, stride)]
    init: Callable | None = None   # init(b, row0, rows) -> (u, v) in dtype, or None for zeros
    expect: dict = field(default_factory=dict)   # the paper's outcome for each instance
    meta: dict = field(default_factory=dict)
    rest_init: bool = False        # start from the quiescent rest state u=v=u*(phi) (computed by each side)

    def phi_plane(self, b: int, row0: int = 0, rows: int | None = None) -> np.ndarray:
        rows = self.H if rows is None else rows
        p = self.phi[b]
        if callable(p):
            return p(row0, rows)
        return p[row0:row0 + rows]

    def init_planes(self, b: int, row0: int = 0, rows: int | None = None):
        rows = self.H if rows is None else rows
        if self.init is None:
            z = np.zeros((rows, self.W), dtype=self.dtype)
            return z, z.copy()
        return self.init(b, row0, rows)


def _cfg1(dtype=np.float64, steps=1000, **kw) -> Workload:
    """configs[0]: 128x128, uniform phi=0.054, u=v=0, disc r=4 at the grid
    centre (63.5, 63.5) -> 52 cells (R-14), 1000 steps."""
    H = W = 128
    phi = np.full((H, W), 0.054)
    disc = {"kind": "disc", "cy2": H - 1, "cx2": W - 1, "r": 4}
    return Workload("c1_disc128", H, W, 1, dtype, steps, [phi], events=[[(disc, 1.0, 0)]])


def _cfg2(dtype=np.float32, steps=20000, phi_passive=0.119, **kw) -> Workload:
    """configs[1]: AND gate, batch of 4 truth-table rows (00, 01, 10, 11) on
    400x300, 20000 steps; output probe fires only for 11."""
    g = and_gate(phi_passive=phi_passive)
    a, b = g["inputs"]
    rows = [(), (b,), (a,), (a, b)]  # 00, 01, 10, 11 (input A = left arm)
    events = [[(s, 1.0, 0) for s in r] for r in rows]
    probes = [[(g["probe"], PROBE_THRESHOLD, PROBE_STRIDE)] for _ in rows]
    return Workload("c2_and_gate", g["H"], g["W"], 4, dtype, steps, [g["phi"]] * 4, events, probes,
                    expect={"fires": [False, False, False, True]}, meta={"geometry": g})


def _cfg3(dtype=np.float32, steps=20000, **kw) -> Workload:
    """configs[2]: chemical diode, 600x200, run L (anode->cathode) and run R
    (cathode->anode), 20000 steps; only run L crosses."""
    d = diode()
    events = [[(d["stim_L"], 1.0, 0)], [(d["stim_R"], 1.0, 0)]]
    probes = [[(d["probe_L"], PROBE_THRESHOLD, PROBE_STRIDE)], [(d["probe_R"], PROBE_THRESHOLD, PROBE_STRIDE)]]
    return Workload("c3_diode", d["H"], d["W"], 2, dtype, steps, [d["phi"]] * 2, events, probes,
                    expect={"fires": [True, False]}, meta={"geometry": d})


def _noise_init(H_global: int, W: int, dtype):
    def init(b, row0, rows):
        u = noise_plane(rows, W, 0, seed=1, dtype=dtype, row0=row0, W_global=W)
        v = noise_plane(rows, W, 1, seed=1, dtype=dtype, row0=row0, W_global=W)
        return u, v
    return init


def _cfg4(dtype=np.float32, steps=10000, H=16384, W=16384, **kw) -> Workload:
    """configs[3]: 16384^2 fp32, uniform phi=0.054, u,v ~ U[0,0.1) (seed 1) plus
    64 u:=1 half-discs of radius 8 (seed 2) at step 0, 10000 steps."""
    phi = lambda row0, rows: np.full((rows, W), 0.054)  # noqa: E731
    events = [[(s, 1.0, 0) for s in half_discs(H, W, 64, seed=2)]]
    return Workload("c4_roofline", H, W, 1, dtype, steps, [phi], events, init=_noise_init(H, W, dtype))


def _cfg5(dtype=np.float32, steps=2000, H=65536, W=65536, n_obstacles=256, **kw) -> Workload:
    """configs[4]: 65536^2 fp32 (or the weak-scaling 16384 x 16384G grid), the
    config-4 initial state plus 256 rectangles of phi=0.2; half-disc writes
    masked to phi_active cells (R-22), 2000 steps."""
    rects = obstacles(H, W, n_obstacles, seed=3)

    def phi(row0, rows):
        p = np.full((rows, W), 0.054)
        for (y0, x0, y1, x1) in rects:
            a, b = max(y0, row0), min(y1, row0 + rows)
            if a < b:
                p[a - row0:b - row0, x0:x1] = 0.2
        return p
    events = [[(s, 1.0, 0) for s in half_discs(H, W, 64, seed=2, mask_phi=0.054)]]
    return Workload("c5_multigpu", H, W, 1, dtype, steps, [phi], events, init=_noise_init(H, W, dtype),
                    meta={"obstacles": rects})


def spiral_seed(dtype=np.float64, steps=40000, H=160, W=160, delay=3500, offset=22, radius=5,
                staggered=True) -> Workload:
    """f4: "starting a simple target wave, then starting another
    wave inside the target wave shortly afterwards ... slightly to one side
    of the centre" on a quiescent medium. With the second stimulus
    `offset` cells right of the centre at step `delay`, the broken wave
    re-enters and activity is sustained; a single target wave (staggered=False)
    leaves the domain."""
    phi = np.full((H, W), 0.054)
    ev = [({"kind": "disc", "cy2": H - 1, "cx2": W - 1, "r": radius}, 1.0, 0)]
    if staggered:
        ev.append(({"kind": "disc", "cy2": H - 1, "cx2": W - 1 + 2 * offset, "r": radius}, 1.0, delay))
    return Workload("f4_spiral" if staggered else "f4_target", H, W, 1, dtype, steps, [phi], [ev], rest_init=True)


PRESET_PX = {"permeable": 2, "semi_permeable": 3, "impermeable": 8}


def preset_cells(px: int) -> int:
    """Barrier width in cells for a preset in display pixels: the 400x300
    simulation is shown at 800x600, so px/2 cells, a half cell
    rounded up (R-21): 2 px -> 1, 3 px -> 2, 8 px -> 4."""
    return (px + 1) // 2


def barrier(preset: str, incidence: str, dtype=np.float64, steps=16000, H=120, W=200, x0=100, cap=30,
            phi_passive=0.0975) -> Workload:
    """f3: a straight line of inhibitive substrate
    (phi_passive, Table 1) of the preset's width along the whole height at
    column x0, in an otherwise active medium.
      incidence="perpendicular": a plane wave launched from the left edge hits
        the line head-on; the probe sits 30 columns past it.
      incidence="parallel": a plane wave launched along the top rows travels
        down, sliding along the line (front perpendicular to it); the first
        `cap` rows of the line are made impermeable (12 cells of phi=0.2) so
        the launch itself does not touch the line; the probe watches the far
        side below the cap.
      preset=None: no line (the control)."""
    w = preset_cells(PRESET_PX[preset]) if preset else 0
    phi = np.full((H, W), 0.054)
    if w:
        phi[:, x0:x0 + w] = phi_passive
    if incidence == "perpendicular":
        ev = [({"kind": "rect", "y0": 0, "x0": 0, "y1": H, "x1": 4}, 1.0, 0)]
        pr = [((H // 2 - 10, x0 + 30, H // 2 + 10, x0 + 32), PROBE_THRESHOLD, PROBE_STRIDE)]
    else:
        if w:
            phi[:cap, x0:x0 + 12] = 0.2
        ev = [({"kind": "rect", "y0": 0, "x0": 0, "y1": 4, "x1": x0}, 1.0, 0)]
        pr = [((cap + 10, x0 + 14, H, x0 + 16), PROBE_THRESHOLD, PROBE_STRIDE)]
    return Workload(f"f3_{preset or 'control'}_{incidence}", H, W, 1, dtype, steps, [phi], [ev], [pr],
                    meta={"width_cells": w})


_CFGS = {1: _cfg1, 2: _cfg2, 3: _cfg3, 4: _cfg4, 5: _cfg5}


def config(n: int, **kw) -> Workload:
    """Build BASELINE.json configs[n-1] (n = 1..5); keyword overrides allowed
    (dtype, steps, H, W, ...) for reduced parity cases."""
    return _CFGS[n](**kw)


__all__ = ["Workload", "config", "phi_from_rects", "spiral_seed", "barrier", "preset_cells", "PRESET_PX"]
