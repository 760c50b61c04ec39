"""The paper's qualitative verification results, reproduced by the oracle.

PAPER.md §4.1 (AND gate / coincidence detector, Fig. 4 captions PAPER.md:280-285)
and §4.2 (chemical diode, Fig. 6 captions PAPER.md:323-329),
on the synthetic geometries of rdinputs.geometry (R-11..R-13), in
fp64 and in the fp32 mode. Also SPEC.md:99/:641 boundedness along the runs and
SPEC.md:264 mirror symmetry of the gate (DESIGN.md pin P-10).
"""
import numpy as np
import pytest

import oracle
from rdinputs import config
from helpers import golden

CHUNK = 2000


def _run_chunked(w, b):
    """Run instance b of workload w in chunks, recording the latched probe
    result and the field extrema after every chunk."""
    dt = w.dtype
    u, v = w.init_planes(b)
    phi = w.phi_plane(b).astype(dt)
    fire = [-1] * len(w.probes[b])
    ext = []
    s = 0
    while s < w.steps:
        n = min(CHUNK, w.steps - s)
        r = oracle.run(u, v, phi, n, events=w.events[b], probes=w.probes[b], step0=s)
        assert r.status == 0
        fire = [f if f >= 0 else g for f, g in zip(fire, r.first_fire)]
        u, v = r.u, r.v
        ext.append((float(u.min()), float(u.max()), float(v.min()), float(v.max())))
        s += n
    return u, v, fire, ext


@pytest.fixture(scope="module", params=[np.float64, np.float32], ids=["f64", "f32"])
def and_runs(request):
    w = config(2, dtype=request.param)
    return w, [_run_chunked(w, b) for b in range(w.B)]


@pytest.fixture(scope="module", params=[np.float64, np.float32], ids=["f64", "f32"])
def diode_runs(request):
    w = config(3, dtype=request.param)
    return w, [_run_chunked(w, b) for b in range(w.B)]


def test_and_gate_truth_table(and_runs):
    """00 -> 0, 01 -> 0, 10 -> 0, 11 -> 1."""
    w, runs = and_runs
    expect = golden("paper_outcomes.json")["and_gate"]["fires"]
    fired = [r[2][0] >= 0 for r in runs]
    assert fired == expect == w.expect["fires"]


def test_and_gate_mirror_symmetry(and_runs):
    """the gate is mirror-symmetric, so run (0,1) is the bitwise
    mirror image of run (1,0) at every step (checked at the last one)."""
    w, runs = and_runs
    u01, v01 = runs[1][0], runs[1][1]
    u10, v10 = runs[2][0], runs[2][1]
    assert np.array_equal(u01, u10[:, ::-1]) and np.array_equal(v01, v10[:, ::-1])


def test_and_gate_bounded(and_runs):
    """u in (-0.1, 1.1), v in (-0.01, 1.1) along the runs."""
    _, runs = and_runs
    for r in runs:
        for (umin, umax, vmin, vmax) in r[3]:
            assert -0.1 < umin and umax < 1.1 and -0.01 < vmin and vmax < 1.1


def test_diode_directionality(diode_runs):
    """Anode -> cathode crosses; cathode -> anode is blocked for 20000 steps
    (PAPER.md:316-318, :323-329)."""
    w, runs = diode_runs
    expect = golden("paper_outcomes.json")["diode"]["fires"]
    fired = [r[2][0] >= 0 for r in runs]
    assert fired == expect == w.expect["fires"]
    for r in runs:
        for (umin, umax, vmin, vmax) in r[3]:
            assert -0.1 < umin and umax < 1.1 and -0.01 < vmin and vmax < 1.1


def test_staggered_stimuli_sustain_activity():
    """f4 / PAPER.md:343-347: on a quiescent medium a second stimulus
    placed beside the first target wave after a delay breaks it into a
    re-entrant (spiral) wave: activity is sustained at step 40000, while a
    single target wave has left the domain by step 12000."""
    from rdinputs import spiral_seed
    w = spiral_seed()
    u, v = oracle.rest_fill(w.phi_plane(0))
    r = oracle.run(u, v, w.phi_plane(0), w.steps, events=w.events[0])
    assert (r.u > 0.1).mean() > 0.05
    c = spiral_seed(staggered=False, steps=12000)
    r1 = oracle.run(u, v, c.phi_plane(0), c.steps, events=c.events[0])
    assert r1.u.max() < 0.01


@pytest.fixture(scope="module")
def barrier_runs():
    from rdinputs import barrier
    out = {}
    for preset in (None, "permeable", "semi_permeable", "impermeable"):
        for inc in ("perpendicular", "parallel"):
            if preset is None and inc == "parallel":
                continue
            w = barrier(preset, inc)
            z = np.zeros((w.H, w.W))
            out[(preset, inc)] = oracle.run(z, z, w.phi_plane(0), w.steps, events=w.events[0],
                                            probes=w.probes[0]).first_fire[0]
    return out


def test_permeability_presets(barrier_runs):
    """f3: with Table 1's phi_passive and the preset widths
    read as display pixels at 2x (R-21: 1, 2, 4 cells), a permeable line slows
    a perpendicular wave and lets both through; a semi-permeable line passes
    the perpendicular wave and blocks the parallel one; an impermeable line
    blocks both."""
    want = golden("paper_outcomes.json")["permeability_presets"]
    ctrl = barrier_runs[(None, "perpendicular")]
    assert ctrl > 0
    for preset in ("permeable", "semi_permeable", "impermeable"):
        perp = barrier_runs[(preset, "perpendicular")]
        par = barrier_runs[(preset, "parallel")]
        assert (perp >= 0) == want[preset]["perpendicular"], preset
        assert (par >= 0) == want[preset]["parallel"], preset
        if want[preset].get("delayed"):
            assert perp > ctrl
