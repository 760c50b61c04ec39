"""Synthetic circuit geometries standing in for the paper's hand-drawn circuits.

The paper gives no dimensions ("drawn by hand"); these are
the parametric stand-ins of DESIGN.md §4 (readings R-11, R-12, R-13), verified
against the paper's outcomes by the oracle (tests/test_circuits.py).

Cell (i, j) has its centre at (y=i, x=j). Every map is a two-level phi field
(active 0.054 / passive phi_p, Table 1) returned in fp64; the
caller rounds it once to its working precision.
"""
from __future__ import annotations

import math

import numpy as np


def _capsule(H: int, W: int, p0, p1, radius: float) -> np.ndarray:
    """Cells whose centre is within `radius` of segment p0-p1."""
    (y0, x0), (y1, x1) = p0, p1
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    dy, dx = y1 - y0, x1 - x0
    L2 = dy * dy + dx * dx
    t = ((yy - y0) * dy + (xx - x0) * dx) / L2
    t = np.clip(t, 0.0, 1.0)
    py, px = y0 + t * dy, x0 + t * dx
    return (yy - py) ** 2 + (xx - px) ** 2 <= radius * radius


def phi_from_rects(H: int, W: int, rects, background: float, value: float) -> np.ndarray:
    """phi = value on each [y0,y1) x [x0,x1), background elsewhere."""
    phi = np.full((H, W), background, dtype=np.float64)
    for (y0, x0, y1, x1) in rects:
        phi[y0:y1, x0:x1] = value
    return phi


def and_gate(H: int = 300, W: int = 400, phi_active: float = 0.054, phi_passive: float = 0.119,
             arm_len: float = 120.0, half_angle_deg: float = 60.0, arm_radius: float = 8.0,
             junction_y: float = 130.0, gap: int = 1, out_half_width: float = 8.0) -> dict:
    """Coincidence detector: two active input arms meet at a
    junction; a 1-row passive gap separates the junction from the output
    channel, so one wave dies at the gap and two colliding waves cross it.

    Mirror-symmetric about x_a = (W-1)/2 (the left arm is built, then mirrored,
    so the map is exactly symmetric: pin P-10). Each arm is a capsule of radius
    8 (16 cells wide, BASELINE.json configs[1]) meeting the output axis at 60
    degrees (R-12). Returns phi (fp64), the two input stimuli
    (10x10 blocks at the arms' outer ends), the probe rect and the mirror axis.
    """
    xa = (W - 1) / 2.0
    J = (junction_y, xa)
    a = math.radians(half_angle_deg)
    A = (junction_y - arm_len * math.cos(a), xa - arm_len * math.sin(a))
    left = _capsule(H, W, A, J, arm_radius)
    active = left | left[:, ::-1]
    # lowest active row of the arm union on the axis columns -> gap -> output
    axis_cols = [int(math.floor(xa)), int(math.ceil(xa))]
    rows = np.nonzero(active[:, axis_cols].any(axis=1))[0]
    junction_bottom = int(rows.max())
    out_top = junction_bottom + 1 + gap
    cols = np.abs(np.arange(W) - xa) < out_half_width
    active[out_top:H - 5, :] |= cols[None, :]
    phi = np.where(active, phi_active, phi_passive)
    ay, ax = int(round(A[0])), int(math.floor(A[1]))
    stim_a = {"kind": "rect", "y0": ay - 5, "x0": ax - 5, "y1": ay + 5, "x1": ax + 5}
    stim_b = {"kind": "rect", "y0": ay - 5, "x0": W - (ax + 5), "y1": ay + 5, "x1": W - (ax - 5)}
    c0, c1 = int(np.nonzero(cols)[0].min()), int(np.nonzero(cols)[0].max()) + 1
    probe = (out_top + 40, c0, out_top + 42, c1)
    return {"phi": phi, "inputs": (stim_a, stim_b), "probe": probe, "junction_bottom": junction_bottom,
            "out_top": out_top, "H": H, "W": W}


def diode(H: int = 200, W: int = 600, phi_active: float = 0.054, phi_passive: float = 0.0975,
          ch_y0: int = 90, ch_w: int = 20, gap_x0: int = 300, gap: int = 2, tip_len: int = 8,
          stim_offset: int = 120, probe_offset: int = 50) -> dict:
    """Chemical diode: a channel cut by a passive gap with a
    flat interface on the anode side (left, columns < gap_x0) and a pointed
    interface on the cathode side (right): a triangular tip of length
    `tip_len` whose apex column is gap_x0+gap; a cell in the tip columns is
    active iff |y - yc| <= (ch_w/2) * (x - (apex - 0.5)) / tip_len.

    Run L (anode -> cathode, must cross) stimulates a 10-column
    block `stim_offset` cells left of the gap; run R (cathode -> anode, must be
    blocked) the mirror position right of the tip. Probes sit `probe_offset`
    cells past the gap on the far side (R-13).
    """
    yc = ch_y0 + (ch_w - 1) / 2.0
    apex = gap_x0 + gap
    phi = np.full((H, W), phi_passive, dtype=np.float64)
    y = np.arange(H)
    in_ch = (y >= ch_y0) & (y < ch_y0 + ch_w)
    phi[in_ch, :gap_x0] = phi_active
    for x in range(apex, apex + tip_len):
        half = (ch_w / 2.0) * (x - (apex - 0.5)) / tip_len
        phi[(np.abs(y - yc) <= half) & in_ch, x] = phi_active
    phi[in_ch, apex + tip_len:] = phi_active
    sl = gap_x0 - stim_offset - 10
    stim_L = {"kind": "rect", "y0": ch_y0, "x0": sl, "y1": ch_y0 + ch_w, "x1": sl + 10}
    sr = apex + stim_offset
    stim_R = {"kind": "rect", "y0": ch_y0, "x0": sr, "y1": ch_y0 + ch_w, "x1": sr + 10}
    probe_L = (ch_y0, apex + probe_offset, ch_y0 + ch_w, apex + probe_offset + 2)
    probe_R = (ch_y0, gap_x0 - probe_offset - 2, ch_y0 + ch_w, gap_x0 - probe_offset)
    return {"phi": phi, "stim_L": stim_L, "stim_R": stim_R, "probe_L": probe_L, "probe_R": probe_R,
            "H": H, "W": W}
