"""Pins of the CPU oracle against what the paper and mathematics fix.

Each test pins the oracle (oracle/) to something other than itself: the
SPEC/PAPER worked examples (tests/golden), closed forms (the homogeneous fixed
point cubic, Euler linearisation eigenvalues, the discrete-cosine eigenmodes of
the no-flux Laplacian), an exact rational evaluation of Eq. 1 on tiny grids, a
library routine (scipy.ndimage.laplace), invariants (conservation, maximum
principle, homogeneity, D4 symmetry, determinism) and first-order convergence.
"""
import hashlib
import math
from fractions import Fraction as Fr

import numpy as np
import pytest
import scipy.ndimage

import oracle
from rdinputs import config
from helpers import golden

P = oracle.Params()
DTYPES = [np.float64, np.float32]


# ---------------------------------------------------------------- SPEC examples

def test_table1_defaults(table1):
    """Params() defaults are Table 1."""
    for k in ("eps", "f", "q", "Du", "dt", "dx"):
        assert getattr(P, k) == table1[k]


@pytest.mark.parametrize("dtype", DTYPES)
def test_laplacian_spec_examples(dtype):
    """uniform -> 0; unit impulse -> -64 centre, +16 neighbours;
    x^2 sampled at dx=0.25 -> 2.0 in the interior."""
    g = golden("spec_examples.json")["laplacian"]
    u = np.full((7, 9), g["uniform_value"], dtype=dtype)
    assert np.all(oracle.laplacian(u) == g["uniform_expected"])
    u = np.zeros((7, 9), dtype=dtype)
    u[3, 4] = 1.0
    L = oracle.laplacian(u)
    assert L[3, 4] == g["impulse_center_expected"]
    for (i, j) in ((2, 4), (4, 4), (3, 3), (3, 5)):
        assert L[i, j] == g["impulse_neighbour_expected"]
    mask = np.ones_like(L, dtype=bool)
    for (i, j) in ((3, 4), (2, 4), (4, 4), (3, 3), (3, 5)):
        mask[i, j] = False
    assert np.all(L[mask] == 0)
    x = np.arange(12) * 0.25
    u = np.tile(x * x, (5, 1)).astype(dtype)
    L = oracle.laplacian(u)
    np.testing.assert_allclose(L[:, 1:-1], 2.0, rtol=0, atol=1e-3 if dtype == np.float32 else 1e-12)


@pytest.mark.parametrize("dtype", DTYPES)
def test_laplacian_matches_library_routine(dtype):
    """Special case reducing to a library routine: the five-node stencil with
    ghost = edge is scipy.ndimage.laplace(mode='nearest'), times 1/dx^2 = 16."""
    rng = np.random.default_rng(5)
    u = rng.random((17, 23))
    ref = scipy.ndimage.laplace(u, mode="nearest") * 16.0
    got = oracle.laplacian(u.astype(dtype)).astype(np.float64)
    tol = 1e-12 if dtype == np.float64 else 2e-4
    np.testing.assert_allclose(got, ref, rtol=0, atol=tol)


@pytest.mark.parametrize("dtype", DTYPES)
def test_reaction_spec_examples(dtype):
    """SPEC.md:55-57 reaction_terms worked examples of Eq. 1."""
    cases = golden("spec_examples.json")["reaction"]["cases"]
    env = {"q": P.q, "eps": P.eps, "phi": 0.054}
    rtol = 1e-14 if dtype == np.float64 else 1e-6
    for c in cases:
        du, dv = oracle.reaction(c["u"], c["v"], c["phi"], dtype=dtype)
        edu = c["du"] if "du" in c else eval(c["du_expr"], {}, env)
        edv = c["dv"] if "dv" in c else eval(c["dv_expr"], {}, env)
        assert du == pytest.approx(edu, rel=rtol, abs=1e-14)
        assert dv == pytest.approx(edv, rel=rtol, abs=1e-7)


@pytest.mark.parametrize("dtype", DTYPES)
def test_one_step_from_zero(dtype):
    """u=v=0, phi=0.054 -> after one step u = dt*phi/eps = 1/450,
    v = 0, within a few ulp of the exact value."""
    H, W = 5, 6
    z = np.zeros((H, W), dtype=dtype)
    phi = np.full((H, W), 0.054, dtype=dtype)
    u1, v1 = oracle.step(z, z, phi)
    exact = float(Fr("0.001") * Fr("0.054") / Fr("0.0243"))
    ulp = np.spacing(dtype(exact))
    assert np.all(np.abs(u1.astype(np.float64) - exact) <= 4 * float(ulp))
    assert np.all(u1 == u1[0, 0]) and np.all(v1 == 0)


def test_stimulus_spec_examples():
    """r=0 -> one pixel; r=2 at (10,10) -> 13 pixels; an
    off-grid disc farther than r from the grid -> nothing. The centred r=4 disc
    of config 1 at (63.5, 63.5) holds the 52 lattice points a brute-force
    Euclidean count gives."""
    for c in golden("spec_examples.json")["stimulus"]["cases"]:
        u = np.zeros((c["H"], c["W"]))
        s = {"kind": "disc", "cy2": 2 * c["cy"], "cx2": 2 * c["cx"], "r": c["r"]}
        assert oracle.stamp(u, u, s, 1.0) == c["count"]
        assert int(u.sum()) == c["count"]
    brute = sum(1 for i in range(128) for j in range(128) if (i - 63.5) ** 2 + (j - 63.5) ** 2 <= 16)
    u = np.zeros((128, 128))
    assert oracle.stamp(u, u, {"kind": "disc", "cy2": 127, "cx2": 127, "r": 4}) == brute == 52


def test_rect_stamp_is_half_open():
    """A RECT stimulus covers [y0, y1) x [x0, x1), clipped to the grid
    (rd.h RD_RECT; SPEC rect regions are half-open): the stamped cells equal
    numpy slicing of the same box, including boxes that cross every edge."""
    H, W = 17, 23
    for (y0, x0, y1, x1) in [(3, 4, 9, 11), (0, 0, 1, 1), (-5, -2, 4, 30), (12, 20, 40, 25), (16, 22, 17, 23)]:
        u = np.zeros((H, W))
        n = oracle.stamp(u, u, {"kind": "rect", "y0": y0, "x0": x0, "y1": y1, "x1": x1}, 1.0)
        want = np.zeros((H, W))
        want[max(y0, 0):max(min(y1, H), 0), max(x0, 0):max(min(x1, W), 0)] = 1.0
        assert np.array_equal(u, want) and n == int(want.sum())


def test_half_disc_and_mask():
    """Half-disc of radius 8 facing +x: brute-force lattice count; the phi mask
    restricts writes to cells whose phi equals mask_phi (R-22)."""
    H = W = 40
    u = np.zeros((H, W))
    s = {"kind": "half_disc", "cy2": 40, "cx2": 40, "r": 8, "dir": 0}
    brute = sum(1 for i in range(H) for j in range(W) if (i - 20) ** 2 + (j - 20) ** 2 <= 64 and j - 20 >= 0)
    assert oracle.stamp(u, u, s) == brute
    phi = np.full((H, W), 0.054)
    phi[:, 25:] = 0.2
    u = np.zeros((H, W))
    n = oracle.stamp(u, phi, dict(s, mask_phi=0.054))
    brute_m = sum(1 for i in range(H) for j in range(W)
                  if (i - 20) ** 2 + (j - 20) ** 2 <= 64 and j - 20 >= 0 and j < 25)
    assert n == brute_m and np.all(u[:, 25:] == 0)


# ------------------------------------------------- exact arithmetic, tiny grids

def _exact_step(u, v, phi):
    """Eq. 1 + forward Euler + five-node no-flux Laplacian in EXACT rational
    arithmetic (Table-1 decimals as exact fractions) on the fp64 inputs."""
    eps, f, q, Du, dt, dx = (Fr(str(x)) for x in (P.eps, P.f, P.q, P.Du, P.dt, P.dx))
    H, W = u.shape
    U = [[Fr(float(u[i, j])) for j in range(W)] for i in range(H)]
    uo = np.empty((H, W))
    vo = np.empty((H, W))
    for i in range(H):
        for j in range(W):
            c = U[i][j]
            n = U[max(i - 1, 0)][j]
            s = U[min(i + 1, H - 1)][j]
            w = U[i][max(j - 1, 0)]
            e = U[i][min(j + 1, W - 1)]
            lap = (n + s + e + w - 4 * c) / (dx * dx)
            vv, pp = Fr(float(v[i, j])), Fr(float(phi[i, j]))
            du = (c - c * c - (f * vv + pp) * (c - q) / (c + q)) / eps + Du * lap
            uo[i, j] = float(c + dt * du)
            vo[i, j] = float(vv + dt * (c - vv))
    return uo, vo


def test_step_matches_exact_rational_evaluation():
    """The exact result within rounding: on random tiny grids (edges included,
    so the no-flux boundary is exercised) the fp64 oracle step equals Eq. 1's
    forward-Euler step evaluated in exact rational arithmetic to ~1e-15.
    A dropped term, wrong sign, wrong neighbour or transposed operand fails."""
    rng = np.random.default_rng(11)
    for trial in range(4):
        H, W = 3 + trial, 4 + (trial % 2)
        u = rng.random((H, W)) * 0.9
        v = rng.random((H, W)) * 0.3
        phi = np.where(rng.random((H, W)) < 0.5, 0.054, 0.0975)
        uo, vo = oracle.step(u, v, phi)
        eu, ev = _exact_step(u, v, phi)
        np.testing.assert_allclose(uo, eu, rtol=0, atol=2e-15)
        np.testing.assert_allclose(vo, ev, rtol=0, atol=1e-16)
        uo32, vo32 = oracle.step(u.astype(np.float32), v.astype(np.float32), phi.astype(np.float32))
        eu32, ev32 = _exact_step(u.astype(np.float32), v.astype(np.float32), phi.astype(np.float32))
        np.testing.assert_allclose(uo32, eu32, rtol=0, atol=2e-6)


# ------------------------------------------------------------- closed forms

def _fixed_point(phi):
    """Smallest positive root of u^3 + (f+q-1)u^2 + (phi-q-fq)u - phi q = 0,
    the homogeneous rest state of Eq. 1 (v* = u*; derived from PAPER.md:91-92)."""
    f, q = P.f, P.q
    roots = np.roots([1.0, f + q - 1.0, phi - q - f * q, -phi * q])
    pos = sorted(r.real for r in roots if abs(r.imag) < 1e-14 and r.real > 0)
    assert len(pos) == 1  # Descartes: exactly one sign change
    return pos[0]


@pytest.mark.parametrize("phi", [0.054, 0.0975])
def test_homogeneous_fixed_point(phi):
    """A uniform medium relaxes to the closed-form fixed point u* = v*, where
    the reaction residual vanishes (SPEC.md:85-93 steady state)."""
    us = _fixed_point(phi)
    du, dv = oracle.reaction(us, us, phi)
    assert abs(du) < 1e-10 and abs(dv) == 0
    z = np.zeros((3, 4))
    r = oracle.run(z, z, np.full((3, 4), phi), 30000)
    assert np.all(r.u == r.u[0, 0]) and np.all(r.v == r.v[0, 0])
    assert abs(r.u[0, 0] - us) < 1e-9 and abs(r.v[0, 0] - us) < 1e-9


def _jacobian(us, phi):
    """Jacobian of the reaction part of Eq. 1 at (u*, v*=u*), closed form."""
    f, q, eps = P.f, P.q, P.eps
    a = (1 - 2 * us - (f * us + phi) * 2 * q / (us + q) ** 2) / eps
    b = -(f / eps) * (us - q) / (us + q)
    return np.array([[a, b], [1.0, -1.0]])


@pytest.mark.parametrize("phi", [0.054, 0.0975, 0.2])
def test_euler_linearisation_eigenvalues(phi):
    """A small uniform perturbation along an eigenvector of I + dt J is scaled
    by its eigenvalue in one oracle step. At phi=0.2 the fast eigenvalue is
    below -1 (period-2 instability of the Euler rest state, R-19)."""
    us = _fixed_point(phi)
    M = np.eye(2) + P.dt * _jacobian(us, phi)
    lam, vec = np.linalg.eig(M)
    for k in range(2):
        d = vec[:, k] / np.max(np.abs(vec[:, k])) * 1e-7
        u = np.full((3, 3), us + d[0])
        v = np.full((3, 3), us + d[1])
        uo, vo = oracle.step(u, v, np.full((3, 3), phi))
        ratio_u = (uo[0, 0] - us) / d[0]
        assert ratio_u == pytest.approx(lam[k].real, rel=2e-4, abs=2e-4)
    if phi == 0.2:
        assert min(lam.real) < -1.0
    else:
        assert np.all(np.abs(lam) < 1.0)


@pytest.mark.parametrize("k,l", [(1, 0), (3, 2), (7, 5)])
def test_diffusion_cosine_eigenmode(k, l):
    """With the reaction off, cos(pi k (j+1/2)/W) cos(pi l (i+1/2)/H) is an
    eigenvector of the no-flux five-node Laplacian with eigenvalue
    -(4/dx^2)[sin^2(pi k/2W) + sin^2(pi l/2H)], so one Euler step multiplies
    it by 1 + dt Du lambda (pins stencil, BC and dt*Du)."""
    H, W = 24, 32
    j = np.arange(W)
    i = np.arange(H)
    mode = np.outer(np.cos(np.pi * l * (i + 0.5) / H), np.cos(np.pi * k * (j + 0.5) / W))
    lam = -(4 / P.dx ** 2) * (math.sin(math.pi * k / (2 * W)) ** 2 + math.sin(math.pi * l / (2 * H)) ** 2)
    uo, vo = oracle.step(mode, mode, np.zeros_like(mode), reaction_off=True)
    np.testing.assert_allclose(uo, mode * (1 + P.dt * P.Du * lam), rtol=0, atol=1e-14)
    assert np.all(vo == mode)


# ------------------------------------------------------------------ invariants

@pytest.mark.parametrize("dtype", DTYPES)
def test_diffusion_only_conservation_and_maximum_principle(dtype):
    """Reaction off: sum(u) is conserved (discrete divergence theorem with
    flux-free edges) and min/max never expand (dt Du 4/dx^2 < 1)."""
    rng = np.random.default_rng(3)
    u = rng.random((40, 50)).astype(dtype)
    z = np.zeros_like(u)
    s0, lo, hi = u.astype(np.float64).sum(), u.min(), u.max()
    r = oracle.run(u, z, z, 1000, reaction_off=True)
    drift = abs(r.u.astype(np.float64).sum() - s0) / s0
    assert drift < (1e-13 if dtype == np.float64 else 1e-6)
    assert r.u.min() >= lo and r.u.max() <= hi


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("phi", [0.054, 0.2])
def test_homogeneity_10000_steps(dtype, phi):
    """A spatially uniform state with uniform phi stays bit-exactly uniform
    for 10,000 steps."""
    z = np.zeros((5, 7), dtype=dtype)
    r = oracle.run(z, z, np.full((5, 7), phi, dtype=dtype), 10000)
    assert np.all(r.u == r.u[0, 0]) and np.all(r.v == r.v[0, 0])
    assert np.isfinite(r.u[0, 0])


@pytest.mark.parametrize("dtype", DTYPES)
def test_centred_disc_d4_symmetry(dtype):
    """Config 1 (centred r=4 disc): u and v are exactly invariant under the 8
    symmetries of the square at step 1000 (north star: 'symmetry of a centred
    stimulus')."""
    w = config(1, dtype=dtype)
    u, v = w.init_planes(0)
    r = oracle.run(u, v, w.phi_plane(0).astype(dtype), 1000, events=w.events[0])
    for a in (r.u, r.v):
        for t in (a[::-1], a[:, ::-1], a.T, a[::-1, ::-1], a.T[::-1], a.T[:, ::-1], a.T[::-1, ::-1]):
            assert np.array_equal(a, t)
    assert r.u.max() > 0.5  # a target wave is travelling


def test_determinism_and_thread_independence():
    """Bit-identical results on repeated runs and with 1 vs 8 threads
    (SPEC.md:96, :638)."""
    w = config(1, dtype=np.float32, steps=300)
    u, v = w.init_planes(0)
    phi = w.phi_plane(0).astype(np.float32)
    n0 = oracle.num_threads()
    try:
        oracle.set_num_threads(1)
        a = oracle.run(u, v, phi, 300, events=w.events[0])
        oracle.set_num_threads(max(2, n0))
        b = oracle.run(u, v, phi, 300, events=w.events[0])
    finally:
        oracle.set_num_threads(n0)
    assert np.array_equal(a.u, b.u) and np.array_equal(a.v, b.v)


@pytest.mark.parametrize("dtype", DTYPES)
def test_run_split_and_event_timing(dtype):
    """run(a) then run(b) == run(a+b) (stride neutrality); an
    event at step s applies after s steps, before step s+1."""
    w = config(1, dtype=dtype)
    u, v = w.init_planes(0)
    phi = w.phi_plane(0).astype(dtype)
    ev = w.events[0] + [({"kind": "rect", "y0": 5, "x0": 5, "y1": 9, "x1": 12}, 1.0, 37)]
    full = oracle.run(u, v, phi, 120, events=ev)
    a = oracle.run(u, v, phi, 37, events=ev)
    b = oracle.run(a.u, a.v, phi, 83, events=ev, step0=37)
    assert np.array_equal(full.u, b.u) and np.array_equal(full.v, b.v)
    # manual: 37 steps, stamp, 83 steps
    m = oracle.run(u, v, phi, 37, events=w.events[0])
    oracle.stamp(m.u, phi, ev[-1][0], 1.0)
    m2 = oracle.run(m.u, m.v, phi, 83)
    assert np.array_equal(full.u, m2.u)


def test_probe_latch_semantics():
    """Probes are sampled after steps that are multiples of stride and latch
    the first such step with max u >= threshold."""
    H, W = 20, 20
    z = np.zeros((H, W))
    phi = np.full((H, W), 0.054)
    ev = [({"kind": "rect", "y0": 8, "x0": 8, "y1": 12, "x1": 12}, 1.0, 0)]
    r = oracle.run(z, z, phi, 100, events=ev, probes=[((9, 9, 11, 11), 0.1, 50), ((0, 0, 1, 1), 0.1, 50),
                                                      ((9, 9, 11, 11), 0.1, 7)])
    assert r.first_fire == [50, -1, 7]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_probe_max_is_the_rect_maximum(dtype):
    """a probe reads the maximum of u over [y0,y1)x[x0,x1).
    Pinned to numpy's max / nanmax (library routines) on a seeded random field,
    on ragged, single-cell, single-row and full-grid rects; NaN cells never
    win (R-23)."""
    rng = np.random.default_rng(11)
    u = rng.uniform(-1.0, 1.0, (23, 37)).astype(dtype)
    rects = [(0, 0, 23, 37), (3, 5, 4, 6), (7, 0, 8, 37), (0, 30, 23, 37), (11, 13, 19, 29), (22, 36, 23, 37)]
    for rect in rects:
        y0, x0, y1, x1 = rect
        assert oracle.probe_max(u, rect) == float(u[y0:y1, x0:x1].max())
    un = u.copy()
    un[12, 14] = np.nan
    un[11, 13] = np.nan
    assert oracle.probe_max(un, (11, 13, 19, 29)) == float(np.nanmax(un[11:19, 13:29]))


def test_probe_threshold_is_inclusive():
    """SPEC.md:243-247 "fired iff max >= threshold": a threshold equal to the
    rect's maximum after the sampled step fires, the next double above it does
    not."""
    rng = np.random.default_rng(5)
    u0 = rng.uniform(0.0, 0.5, (12, 12))
    v0 = rng.uniform(0.0, 0.5, (12, 12))
    phi = np.full((12, 12), 0.054)
    u1, _ = oracle.step(u0, v0, phi)
    rect = (2, 3, 9, 10)
    m = float(u1[2:9, 3:10].max())
    r = oracle.run(u0, v0, phi, 1, probes=[(rect, m, 1), (rect, np.nextafter(m, np.inf), 1)])
    assert r.first_fire == [1, -1]


def test_fault_reports_first_step_and_cell():
    """S:62 stop at the first non-finite cell, reporting its step and (row,
    column). Closed form: u = 1e200 at (3, 5) makes C*C overflow, so
    u' = C + dt*((C - inf)/eps + ...) = -inf after step 1. Each neighbour only
    receives Du*dt*16*1e200 = 7.2e197 through the Laplacian, finite. So the run
    stops at step 1 with the fault at row 3, column 5, and u holds that state."""
    u0 = np.zeros((9, 11))
    u0[3, 5] = 1e200
    r = oracle.run(u0, np.zeros((9, 11)), np.full((9, 11), 0.054), 10)
    assert r.status != 0 and r.fault == (1, 3, 5)
    assert np.isneginf(r.u[3, 5]) and np.isfinite(np.delete(r.u.ravel(), 3 * 11 + 5)).all()


def test_rest_state_never_fires():
    """a quiescent medium never reaches the 0.1 threshold; zeros
    relax to the rest state without firing (R-10)."""
    z = np.zeros((10, 10))
    r = oracle.run(z, z, np.full((10, 10), 0.054), 2000, probes=[((0, 0, 10, 10), 0.1, 50)])
    assert r.first_fire == [-1] and r.u.max() < 0.01


# --------------------------------------------------------- convergence, waves

def test_euler_first_order_convergence():
    """on a stimulated 100x100 medium integrated to t=1.0,
    max-norm differences between dt, dt/2, dt/4 shrink by a factor in
    [1.5, 2.5] (first-order forward Euler)."""
    H = W = 100
    z = np.zeros((H, W))
    phi = np.full((H, W), 0.054)
    ev = [({"kind": "disc", "cy2": 99, "cx2": 99, "r": 5}, 1.0, 0)]
    sols = []
    for m in (1, 2, 4):
        p = oracle.Params(dt=0.001 / m)
        sols.append(oracle.run(z, z, phi, 1000 * m, events=ev, params=p).u)
    d1 = np.abs(sols[0] - sols[1]).max()
    d2 = np.abs(sols[1] - sols[2]).max()
    assert 1.5 <= d1 / d2 <= 2.5


def test_plane_wave_speed_constant():
    """a plane wave's front (u >= 0.1 crossing) advances at
    constant speed (+-5%) over two disjoint intervals."""
    H, W = 4, 400
    z = np.zeros((H, W))
    phi = np.full((H, W), 0.054)
    ev = [({"kind": "rect", "y0": 0, "x0": 0, "y1": H, "x1": 6}, 1.0, 0)]
    u, v = z, z
    fronts = []
    step = 0
    for n in (2000, 2000, 2000, 2000):
        r = oracle.run(u, v, phi, n, events=ev, step0=step)
        step += n
        u, v = r.u, r.v
        fronts.append(int(np.nonzero((u[0] >= 0.1))[0].max()))
    s1 = fronts[2] - fronts[1]
    s2 = fronts[3] - fronts[2]
    assert s1 > 10 and abs(s1 - s2) <= 0.05 * s1 + 1


# ------------------------------------------------------------ non-finite path

def test_nonfinite_reproducer_reports_first_cell():
    """T5 (R-22): uniform phi=0.2, u,v ~ U[0,0.1), one unmasked u:=1
    half-disc: Euler diverges past u=-q; the run stops at the first step with
    a non-finite cell and reports its row-major first (i, j).
    The same stimulus masked to phi_active cells (here: none) stays finite."""
    from rdinputs import noise_plane
    H = W = 128
    u = noise_plane(H, W, 0, seed=7, dtype=np.float64)
    v = noise_plane(H, W, 1, seed=7, dtype=np.float64)
    phi = np.full((H, W), 0.2)
    s = {"kind": "half_disc", "cy2": 128, "cx2": 128, "r": 8, "dir": 0}
    r = oracle.run(u, v, phi, 400, events=[(s, 1.0, 0)])
    assert r.status == -4 and r.fault is not None
    st, i, j = r.fault
    assert 1 <= st <= 400
    bad = ~(np.isfinite(r.u) & np.isfinite(r.v))
    first = np.argwhere(bad)[0]
    assert (i, j) == tuple(first)
    prev = oracle.run(u, v, phi, st - 1, events=[(s, 1.0, 0)])
    assert prev.status == 0
    ok = oracle.run(u, v, phi, 400, events=[(dict(s, mask_phi=0.054), 1.0, 0)])
    assert ok.status == 0


# ------------------------------------------------ cross-implementation (survey)

@pytest.mark.parametrize("sfx,dtype", [("f64", np.float64), ("f32", np.float32)])
def test_survey_cross_implementation_digest(sfx, dtype):
    """two independent survey programs of the same canonical
    tree produced these config-1 digests at step 1000; ours must agree
    bit-for-bit (cross-check of tree, constants, BC and disc readings)."""
    g = golden("survey_cross_impl.json")[sfx]
    w = config(1, dtype=dtype)
    u, v = w.init_planes(0)
    r = oracle.run(u, v, w.phi_plane(0).astype(dtype), 1000, events=w.events[0])
    assert hashlib.sha256(r.u.astype("<" + r.u.dtype.str[1:]).tobytes()).hexdigest() == g["u_sha256"]
    assert hashlib.sha256(r.v.astype("<" + r.v.dtype.str[1:]).tobytes()).hexdigest() == g["v_sha256"]


# ------------------------------------------------------ f2: timelapse max-u

def test_timelapse_record_spec_examples():
    """recording u=0.2 then u=0.5 gives 0.5; recording the same
    state twice leaves the accumulator unchanged; NaN never replaces a value."""
    m = np.full((2, 3), -np.inf)
    oracle.timelapse_record(np.full((2, 3), 0.2), m)
    oracle.timelapse_record(np.full((2, 3), 0.5), m)
    assert np.all(m == 0.5)
    oracle.timelapse_record(np.full((2, 3), 0.3), m)
    assert np.all(m == 0.5)
    x = np.full((2, 3), 0.7)
    x[0, 1] = np.nan
    oracle.timelapse_record(x, m)
    assert m[0, 1] == 0.5 and m[1, 2] == 0.7


def test_timelapse_run_equals_brute_force_max():
    """The run's timelapse equals the pointwise max of u over the sampled
    steps, computed from separately recorded snapshots, and a fresh
    accumulator on a quiescent medium holds the rest state."""
    w = config(1, dtype=np.float64, steps=300)
    u, v = w.init_planes(0)
    phi = w.phi_plane(0)
    r = oracle.run(u, v, phi, 300, events=w.events[0], timelapse_stride=25)
    snaps = []
    uu, vv = u, v
    for s in range(0, 300, 25):
        rr = oracle.run(uu, vv, phi, 25, events=w.events[0], step0=s)
        uu, vv = rr.u, rr.v
        snaps.append(uu)
    assert np.array_equal(r.max_u, np.max(np.stack(snaps), axis=0))
    assert np.array_equal(r.u, uu)
    z = np.zeros((6, 6))
    q = oracle.run(z, z, np.full((6, 6), 0.054), 30000, timelapse_stride=30000)
    assert np.allclose(q.max_u, _fixed_point(0.054), atol=1e-9)


# ------------------------------------------------------- f4: rest-state init

@pytest.mark.parametrize("phi", [0.054, 0.0975, 0.119, 0.2])
def test_rest_state_bisection_is_the_cubic_root(phi):
    """the bisection's u* is the closed-form cubic root
    (numpy.roots) to ~1 ulp, its reaction residual vanishes, and it is
    invariant under scaling eps."""
    us = oracle.rest_state(phi)
    assert us == pytest.approx(_fixed_point(phi), rel=1e-13, abs=0)
    du, _ = oracle.reaction(us, us, phi)
    assert abs(du) < 1e-10
    assert oracle.rest_state(phi, oracle.Params(eps=2 * 0.0243)) == us


def test_rest_fill_is_stationary():
    """A quiescent medium filled with u*(phi) per cell stays at rest: uniform
    regions stay bitwise uniform and nothing fires over 2000 steps."""
    phi = np.full((30, 40), 0.054)
    phi[10:20, :] = 0.0975
    u, v = oracle.rest_fill(phi)
    assert np.all(u == v) and u[0, 0] == oracle.rest_state(0.054) and u[15, 0] == oracle.rest_state(0.0975)
    r = oracle.run(u, v, phi, 2000, probes=[((0, 0, 30, 40), 0.1, 50)])
    assert r.first_fire == [-1] and np.abs(r.u - u).max() < 1e-4
    u32, _ = oracle.rest_fill(phi.astype(np.float32))
    assert u32.dtype == np.float32 and u32[0, 0] == np.float32(oracle.rest_state(float(np.float32(0.054))))


# ------------------------------------------------------------ P-6 nullclines

def _u_nullcline_v(u, phi, p=oracle.Params()):
    """Eq. 1: du/dt = 0 <=> v = [(u - u^2)(u + q)/(u - q) - phi] / f."""
    return ((u - u * u) * (u + p.q) / (u - p.q) - phi) / p.f


@pytest.mark.parametrize("u", [0.01, 0.0563, 0.2, 0.5, 0.9396])
def test_reaction_vanishes_on_the_u_nullcline(u):
    """SURVEY P-6: the oracle's reaction du/dt is zero (to rounding) on the
    closed-form u-nullcline, and dv/dt = u - v vanishes on v = u."""
    phi = 0.054
    v = _u_nullcline_v(u, phi)
    du, dv = oracle.reaction(u, v, phi)
    scale = (u + u * u + abs(v) + phi) / oracle.Params().eps
    assert abs(du) <= 1e-13 * scale
    assert oracle.reaction(u, u, phi)[1] == 0.0


def test_excitability_threshold_between_the_nullcline_crossings():
    """SURVEY P-6: at v = v* (the rest level) the u-nullcline crosses at the
    threshold u ~= 0.0563 and the excited branch u ~= 0.9396 (phi = 0.054).
    A homogeneous medium (no diffusion, so the grid is the ODE) started just
    below the threshold relaxes to rest; just above it, u jumps to the
    excited branch (u > 0.5)."""
    phi = 0.054
    ustar = oracle.rest_state(phi)
    # the crossings of the u-nullcline with v = v*: bracket and bisect the
    # closed form, then check the documented values
    def cross(lo, hi):
        f = lambda x: _u_nullcline_v(x, phi) - ustar  # noqa: E731
        for _ in range(200):
            m = 0.5 * (lo + hi)
            if (f(lo) > 0) == (f(m) > 0):
                lo = m
            else:
                hi = m
        return 0.5 * (lo + hi)
    th, ex = cross(0.01, 0.3), cross(0.5, 0.999)
    assert abs(th - 0.0563) < 5e-4 and abs(ex - 0.9396) < 5e-4
    n = 3
    phi_p = np.full((n, n), phi)
    peaks = []
    for u0 in (th - 0.01, th + 0.01):
        u = np.full((n, n), u0)
        v = np.full((n, n), ustar)
        peak = u0
        for _ in range(30):
            r = oracle.run(u, v, phi_p, 100)
            u, v = r.u, r.v
            peak = max(peak, float(u.max()))
        peaks.append(peak)
    # below: back to rest without crossing the threshold; above: a jump onto
    # the excited branch (its peak sits below the v = v* crossing because v
    # rises during the excursion: eps is small, not zero)
    assert peaks[0] < th and peaks[1] > 0.5
