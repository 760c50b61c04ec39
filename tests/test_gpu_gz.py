"""gz_kernel (whole-chip tiles, border exchange through L2 every k steps):
bitwise equal to the oracle (oracle/) over tilings, block depths, ragged
shapes, mirrored edges, batches with per-instance parameters, stimuli inside
a run, fused probes and the timelapse record. GPU only."""
import numpy as np
import pytest

import oracle
import paper_1901_06535_b200 as rd
from rdinputs import config, noise_plane

pytestmark = pytest.mark.gpu

GZ = 3  # rd_stats.kernel of gz_kernel


def _case(H, W, dt, seed):
    u0 = noise_plane(H, W, 0, seed=seed, dtype=dt)
    v0 = noise_plane(H, W, 1, seed=seed, dtype=dt)
    phi = np.full((H, W), 0.054, dt)
    phi[H // 3:H // 2, W // 4:W // 2] = 0.0975
    ev = [({"kind": "disc", "cy2": H, "cx2": W, "r": 3}, 1.0, 0),
          ({"kind": "rect", "y0": 0, "x0": 0, "y1": min(3, H), "x1": W}, 1.0, 17)]
    return u0, v0, phi, ev


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("H,W", [(8, 16), (9, 17), (37, 131), (64, 64), (150, 150), (301, 29), (200, 602),
                                 (33, 1021)])
@pytest.mark.parametrize("k", [1, 2, 3, 5, 8, 12])
def test_tilings_and_depths(dtype, H, W, k, monkeypatch):
    """Every tiling the geometry picker chooses for these shapes (ragged last
    tiles, W not a multiple of the vector width, one-tile instances), block
    depths 1..12 (ghost zones narrower and wider than a vector), 45 steps
    split unevenly with a stimulus at step 17: bitwise equal to the oracle."""
    dt = np.float32 if dtype == "f32" else np.float64
    monkeypatch.setenv("RD_KERNEL", "gz")
    monkeypatch.setenv("RD_GZ_K", str(k))
    u0, v0, phi, ev = _case(H, W, dt, seed=H * 7 + W)
    ref = oracle.run(u0, v0, phi, 45, events=ev)
    sim = rd.Sim(phi[None], dtype=dt)
    try:
        vec = 16 // np.dtype(dt).itemsize
        gx = (k + vec - 1) // vec * vec
        applies = H >= 2 * k and W >= 2 * gx + vec  # mirrored ghosts stay inside the grid
        assert sim.stats()["kernel"] == (GZ if applies else 0), (H, W, k)
        sim.write(0, u0, v0)
        for s, val, at in ev:
            sim.stimulate(s, val, at)
        for n in (7, 1, 30, 7):
            sim.step(n)
        u, v = sim.read(0)
    finally:
        sim.close()
    assert np.array_equal(u, ref.u), (H, W, k)
    assert np.array_equal(v, ref.v), (H, W, k)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_batch_params_probes_timelapse(dtype, monkeypatch):
    """A batch of three instances with their own Eq.-1 parameters (f1), fused
    probes of several strides (some due inside a launch, some at its end) and
    the timelapse record: bitwise the oracle's fields, latches and max_u."""
    dt = np.float32 if dtype == "f32" else np.float64
    monkeypatch.setenv("RD_KERNEL", "gz")
    monkeypatch.setenv("RD_GZ_K", "6")
    H, W, steps = 90, 140, 120
    prm = [None, dict(eps=0.03, f=1.0, q=0.002, Du=0.45, dt=0.001, dx=0.25),
           dict(eps=0.0243, f=2.0, q=0.005, Du=0.45, dt=0.001, dx=0.25)]
    cases = [_case(H, W, dt, seed=50 + b) for b in range(3)]
    probes = [[((40, 60, 50, 80), 0.3, 7), ((0, 0, 10, 10), 0.05, 20)], [((80, 100, 90, 140), 0.1, 3)],
              [((45, 70, 46, 71), 0.2, 11)]]
    sim = rd.Sim(np.stack([c[2] for c in cases]), dtype=dt)
    try:
        assert sim.stats()["kernel"] == GZ
        for b, (u0, v0, phi, ev) in enumerate(cases):
            if prm[b] is not None:
                p = rd.rd_params_default()
                for k_, v_ in prm[b].items():
                    setattr(p, k_, v_)
                sim.set_params(b, p)
            sim.write(b, u0, v0)
            for s, val, at in ev:
                sim.stimulate(s, val, at, b=b)
        pids = [[sim.probe_latch(b, r, t, st) for (r, t, st) in probes[b]] for b in range(3)]
        sim.timelapse(10)
        for n in (33, 40, 47):
            sim.step(n)
        for b, (u0, v0, phi, ev) in enumerate(cases):
            p = oracle.Params(**prm[b]) if prm[b] is not None else oracle.Params()
            ref = oracle.run(u0, v0, phi, steps, events=ev, probes=probes[b], params=p, timelapse_stride=10)
            u, v = sim.read(b)
            assert np.array_equal(u, ref.u), b
            assert np.array_equal(v, ref.v), b
            assert [sim.probe_result(q) for q in pids[b]] == ref.first_fire, b
            assert np.array_equal(sim.read_timelapse(b), ref.max_u), b
    finally:
        sim.close()


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("n", [2, 3])
def test_paper_configs_short(dtype, n, monkeypatch):
    """The AND-gate (config 2) and diode (config 3) batches for 400 steps on
    gz_kernel: bitwise the oracle, and the same as tb_kernel."""
    dt = np.float32 if dtype == "f32" else np.float64
    w = config(n, dtype=dt, steps=400)
    out = {}
    for kern in ("gz", "tb"):
        monkeypatch.setenv("RD_KERNEL", kern)
        sim = rd.Sim(np.stack([w.phi_plane(b).astype(dt) for b in range(w.B)]), dtype=dt)
        try:
            assert sim.stats()["kernel"] == (GZ if kern == "gz" else 0)
            for b in range(w.B):
                sim.write(b, *w.init_planes(b))
                for s, val, at in w.events[b]:
                    sim.stimulate(s, val, at, b=b)
            sim.step(w.steps)
            out[kern] = [sim.read(b) for b in range(w.B)]
        finally:
            sim.close()
    for b in range(w.B):
        ref = oracle.run(*w.init_planes(b), w.phi_plane(b).astype(dt), w.steps, events=w.events[b])
        assert np.array_equal(out["gz"][b][0], ref.u) and np.array_equal(out["gz"][b][1], ref.v), b
        assert np.array_equal(out["gz"][b][0], out["tb"][b][0]), b
