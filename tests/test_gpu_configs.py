"""GPU parity on the BASELINE.json configurations 2-5.

Configs 2/3 (the paper's AND gate and diode shapes, §4) run in full
(20000 steps) in fp32 and fp64, bitwise against the oracle, with the paper's
outcomes. Configs 4/5 run at full size in the launch configuration bench.py
times: bitwise vs the oracle over the first steps of the full grid, and by
properties (blocking-depth invariance, determinism, boundedness) at full
length where the oracle cannot follow.
"""
import numpy as np
import pytest

from gpu_util import assert_bitwise, gpu_run, oracle_run
from helpers import golden
from rdinputs import config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
def test_and_gate_batched_truth_table(dtype, kernel):
    """configs[1]: 4 truth-table rows in one batched launch; fields and probe
    latches bitwise equal to the oracle; output fires only for 11
    (PAPER.md:280-285)."""
    w = config(2, dtype=dtype)
    U, V, fire, _ = gpu_run(w)
    expect = golden("paper_outcomes.json")["and_gate"]["fires"]
    assert [f[0] >= 0 for f in fire] == expect
    for b in range(w.B):
        r = oracle_run(w, b)
        assert fire[b] == r.first_fire
        assert_bitwise(U[b], r.u, f"u row {b}")
        assert_bitwise(V[b], r.v, f"v row {b}")
    assert np.array_equal(U[1], U[2][:, ::-1])  # P-10 mirror symmetry


@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
def test_diode_batched(dtype, kernel):
    """configs[2]: both directions in one batched launch; anode->cathode
    crosses, cathode->anode does not."""
    w = config(3, dtype=dtype)
    U, V, fire, _ = gpu_run(w)
    assert [f[0] >= 0 for f in fire] == golden("paper_outcomes.json")["diode"]["fires"]
    for b in range(w.B):
        r = oracle_run(w, b)
        assert fire[b] == r.first_fire
        assert_bitwise(U[b], r.u, f"u run {b}")
        assert_bitwise(V[b], r.v, f"v run {b}")


def test_config4_full_grid_first_steps_bitwise():
    """configs[3] at full size (16384^2 fp32, noise + 64 half-discs) in the
    bench launch configuration: the first 20 steps equal the oracle bitwise
    on every cell of the full grid."""
    w = config(4, steps=20)
    U, V, _, st = gpu_run(w)
    assert st["tb_depth"] >= 1
    r = oracle_run(w, 0)
    assert_bitwise(U[0], r.u, "u")
    assert_bitwise(V[0], r.v, "v")


def test_config4_full_length_properties():
    """configs[3] for the full 10000 steps: the auto depth (6) and depth 4 give
    bit-identical fields (T2), and the fields are finite and bounded."""
    w = config(4)
    Ua, Va, _, _ = gpu_run(w)
    Ub, Vb, _, _ = gpu_run(w, tb_depth=4)
    assert_bitwise(Ua, Ub, "u auto vs k=4")
    assert_bitwise(Va, Vb, "v auto vs k=4")
    assert np.isfinite(Ua).all() and np.isfinite(Va).all()
    assert Ua.min() > -0.1 and Ua.max() < 1.1


@pytest.mark.xfail(strict=False, reason="KNOWN DEFECT (DESIGN.md 5.2): tb_kernel at depth 1 on config 4 at full length "
                                        "differs from the other depths in about one run in three (a few rows, tens of "
                                        "columns, 1e-8): 10000 one-step launches; depths 4-7 never differ in 74 runs")
def test_config4_full_length_depth1_known_intermittent():
    w = config(4)
    Ua, Va, _, _ = gpu_run(w, tb_depth=4)
    Ub, Vb, _, _ = gpu_run(w, tb_depth=1)
    assert_bitwise(Ua, Ub, "u k=4 vs k=1")
    assert_bitwise(Va, Vb, "v k=4 vs k=1")


def test_config5_crop_bitwise():
    """configs[4] inputs (noise, 256 obstacles of phi=0.2, masked half-discs)
    on a 4096^2 crop of the global grid, 40 steps, bitwise vs the oracle."""
    w = config(5, H=4096, W=4096, steps=40, n_obstacles=16)
    U, V, _, _ = gpu_run(w)
    r = oracle_run(w, 0)
    assert_bitwise(U[0], r.u, "u")
    assert_bitwise(V[0], r.v, "v")


@pytest.mark.parametrize("path", ["handle", "slab"])
def test_config5_full_size_sampled_blocks(path):
    """configs[4] at its full 65536^2 (120 GB resident, built on the device as
    `bench.py --scaling strong` builds it), 24 steps. Sampled 16x16 blocks --
    the four corners, obstacle corners, stimulus centres, seeded interior
    points -- equal the oracle run on each block's dependency cone, bitwise.
    After n steps a cell depends only on cells within n of it, so a window
    n cells wider than the block on every side is exact at the block. Where
    the window reaches a global edge it stops there, and the real no-flux
    boundary applies on both sides. The GPU blocks are read straight from the
    device rows (rd_row_ptr). path "slab" is the launch configuration the
    strong-scaling bench line times at N = 1 (SlabSim, halo 4, block protocol);
    "handle" is a plain rd_create handle."""
    import torch
    import paper_1901_06535_b200 as rd
    import oracle
    from slab_protocol import SlabSim, _dev_rows
    n, S = 24, 16
    w = config(5, steps=n)
    H, W = w.H, w.W
    sim = (rd.Sim(None, shape=(1, H, W), dtype=np.float32) if path == "handle" else
           SlabSim(W, H, 0, 1, None, dtype=np.float32, halo=4))
    try:
        rd.rd_paint_phi(sim.h, -1, None, 0.054)
        for rect in w.meta["obstacles"]:
            rd.rd_paint_phi(sim.h, -1, rect, 0.2)
        sim.fill_noise(seed=1)
        for s, val, at in w.events[0]:
            sim.stimulate(s, val, at)
        sim.step(n)
        torch.cuda.synchronize()
        rng = np.random.default_rng(9)
        corners = [(0, 0), (0, W - S), (H - S, 0), (H - S, W - S)]
        obst = [(y0 - S // 2, x0 - S // 2) for (y0, x0, _, _) in w.meta["obstacles"][:3]]
        stim = [(s["cy2"] // 2 - S // 2, s["cx2"] // 2 - S // 2) for s, _, _ in w.events[0][:3]]
        rand = [(int(rng.integers(0, H - S)), int(rng.integers(0, W - S))) for _ in range(3)]
        for (by0, bx0) in corners + obst + stim + rand:
            by0, bx0 = min(max(by0, 0), H - S), min(max(bx0, 0), W - S)
            by1, bx1 = by0 + S, bx0 + S
            wy0, wy1, wx0, wx1 = max(0, by0 - n), min(H, by1 + n), max(0, bx0 - n), min(W, bx1 + n)
            u0, v0 = w.init_planes(0, wy0, wy1 - wy0)
            phi = w.phi_plane(0, wy0, wy1 - wy0)[:, wx0:wx1].astype(np.float32)
            ev = []
            for s, val, at in w.events[0]:
                t = dict(s)
                t["cy2"] -= 2 * wy0
                t["cx2"] -= 2 * wx0
                ev.append((t, val, at))
            r = oracle.run(u0[:, wx0:wx1].astype(np.float32), v0[:, wx0:wx1].astype(np.float32), phi, n, events=ev)
            for plane, ref in ((0, r.u), (1, r.v)):
                rows = _dev_rows(sim.h, 0, plane, by0, by1).view(torch.float32).view(S, -1)
                got = rows[:, 8 + bx0:8 + bx1].cpu().numpy()
                assert_bitwise(got, ref[by0 - wy0:by1 - wy0, bx0 - wx0:bx1 - wx0], f"plane {plane} block ({by0}, {bx0})")
    finally:
        sim.close()


def test_config5_device_built_crop_bitwise():
    """configs[4] built on the device (rd_paint_phi background + obstacles,
    rd_fill_noise, masked half-discs) on a 2048^2 crop equals the oracle on
    the rdinputs host inputs, bitwise, after 30 steps."""
    import paper_1901_06535_b200 as rd
    import oracle
    w = config(5, H=2048, W=2048, steps=30, n_obstacles=24)
    sim = rd.Sim(None, shape=(1, w.H, w.W), dtype=np.float32)
    sim.paint_phi(0.054)
    for (y0, x0, y1, x1) in w.meta["obstacles"]:
        sim.paint_phi(0.2, (y0, x0, y1, x1))
    sim.fill_noise(seed=1)
    for s, val, at in w.events[0]:
        sim.stimulate(s, val, at)
    sim.step(w.steps)
    u, v = sim.read(0)
    sim.close()
    r = oracle_run(w, 0)
    assert_bitwise(u, r.u, "u")
    assert_bitwise(v, r.v, "v")


@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
def test_permeability_presets_batched(dtype):
    """f3: the seven barrier runs (control + 3 presets x 2 incidences) as ONE
    batched handle (per-instance phi maps); fields and probe latches bitwise
    equal to the oracle, outcomes as P:163-168 describes."""
    import oracle
    from helpers import golden
    from rdinputs import barrier
    from rdinputs.workloads import Workload
    runs = [(None, "perpendicular")] + [(p, i) for p in ("permeable", "semi_permeable", "impermeable")
                                        for i in ("perpendicular", "parallel")]
    ws = [barrier(p, i, dtype=dtype) for p, i in runs]
    w = Workload("f3_batch", ws[0].H, ws[0].W, len(ws), dtype, ws[0].steps, [x.phi[0] for x in ws],
                 [x.events[0] for x in ws], [x.probes[0] for x in ws])
    U, V, fire, _ = gpu_run(w)
    res = {}
    for b, (p, i) in enumerate(runs):
        r = oracle_run(w, b)
        assert fire[b] == r.first_fire
        assert_bitwise(U[b], r.u, f"u {p} {i}")
        res[(p, i)] = fire[b][0]
    want = golden("paper_outcomes.json")["permeability_presets"]
    for p in ("permeable", "semi_permeable", "impermeable"):
        assert (res[(p, "perpendicular")] >= 0) == want[p]["perpendicular"]
        assert (res[(p, "parallel")] >= 0) == want[p]["parallel"]
    assert res[("permeable", "perpendicular")] > res[(None, "perpendicular")]
