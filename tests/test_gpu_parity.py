"""GPU parity: the CUDA path through the C ABI against the oracle, element by
element on the same seeded inputs.

Bar: bitwise equality in fp64 AND fp32 (the canonical tree is reproduced
exactly; readings R-17/R-18 — this implies the north star's 1e-10 (fp64) and
2e-3 (fp32-vs-fp32) tolerances). Self-consistency at sizes the oracle cannot
reach: every temporal-blocking depth, batching and rd_step splitting gives
bit-identical results.
"""
import numpy as np
import pytest

import oracle
import paper_1901_06535_b200 as rd
from gpu_util import assert_bitwise, gpu_run, oracle_run
from rdinputs import config, half_discs, noise_plane
from rdinputs.workloads import Workload

pytestmark = pytest.mark.gpu
DT = [np.float64, np.float32]
IDS = ["f64", "f32"]


def _noise_workload(H, W, dtype, steps, B=1, phi=None, n_discs=6, seed=1, mask=None):
    def init(b, row0, rows):
        return (noise_plane(rows, W, 0, seed=seed + b, dtype=dtype, row0=row0),
                noise_plane(rows, W, 1, seed=seed + b, dtype=dtype, row0=row0))
    phis = []
    for b in range(B):
        p = np.full((H, W), 0.054) if phi is None else phi
        phis.append(p)
    ev = [[(s, 1.0, 0) for s in half_discs(H, W, n_discs, seed=2 + b, mask_phi=mask)] for b in range(B)]
    return Workload(f"noise{H}x{W}", H, W, B, dtype, steps, phis, ev, [], init=init)


# ------------------------------------------------------------- config 1

@pytest.mark.parametrize("dtype", DT, ids=IDS)
def test_config1_bitwise(dtype, kernel):
    """configs[0]: 128x128 centred disc, 1000 steps, fields bitwise equal to
    the oracle (fp64: max|du|,|dv| = 0 <= 1e-10)."""
    w = config(1, dtype=dtype)
    U, V, _, st = gpu_run(w)
    r = oracle_run(w, 0)
    assert st["step_launches"] > 0
    assert_bitwise(U[0], r.u, "u")
    assert_bitwise(V[0], r.v, "v")
    a = U[0]
    assert np.array_equal(a, a.T) and np.array_equal(a, a[::-1])  # P-9 on the GPU result


def test_config1_fp32_vs_fp64_oracle_early():
    """Reading R-17 (ii): the fp32 GPU path is within 2e-3 of the fp64 oracle
    up to step 300 (beyond it the refractory-wake instability amplifies any
    fp32 rounding, R-17; reported by bench, not gated)."""
    w32 = config(1, dtype=np.float32, steps=300)
    U, V, _, _ = gpu_run(w32)
    r = oracle_run(config(1, dtype=np.float64, steps=300), 0)
    assert np.abs(U[0] - r.u).max() <= 2e-3 and np.abs(V[0] - r.v).max() <= 2e-3


# -------------------------------------------- blocking depth, ragged shapes

@pytest.mark.parametrize("dtype", DT, ids=IDS)
@pytest.mark.parametrize("H,W", [(3, 3), (37, 131), (130, 250), (64, 517), (301, 29)])
def test_ragged_shapes_all_depths(dtype, H, W, kernel):
    """Ragged grids (W not a multiple of the vector width or strip, tiny and
    tall/narrow) spanning several strips and row blocks: every tb_depth 1..8
    equals the oracle bitwise from a noisy initial state with stimuli."""
    w = _noise_workload(H, W, dtype, 41)
    r = oracle_run(w, 0)
    for k in range(1, rd._lib.RD_MAX_TB + 1):
        U, V, _, st = gpu_run(w, tb_depth=k)
        assert st["tb_depth"] == k
        assert_bitwise(U[0], r.u, f"u k={k}")
        assert_bitwise(V[0], r.v, f"v k={k}")


@pytest.mark.parametrize("dtype", DT, ids=IDS)
def test_batched_equals_unbatched_and_oracle(dtype, kernel):
    """a8: a batch of 3 different instances (own phi, init and stimuli) equals
    each instance run alone and the oracle."""
    H, W = 90, 140
    phi = np.full((H, W), 0.054)
    phi[30:60, 40:100] = 0.0975
    w = _noise_workload(H, W, dtype, 60, B=3, phi=phi)
    U, V, _, _ = gpu_run(w)
    for b in range(3):
        r = oracle_run(w, b)
        assert_bitwise(U[b], r.u, f"u b={b}")
        assert_bitwise(V[b], r.v, f"v b={b}")
        U1, V1, _, _ = gpu_run(w, batch=[b])
        assert_bitwise(U1[0], U[b], f"unbatched b={b}")


@pytest.mark.parametrize("dtype", DT, ids=IDS)
def test_step_splitting_and_events(dtype, kernel):
    """rd_step(a); rd_step(b) == rd_step(a+b) with events at
    steps inside, at and across the split points."""
    H, W = 70, 90
    w = _noise_workload(H, W, dtype, 97)
    w.events[0] += [({"kind": "rect", "y0": 10, "x0": 3, "y1": 14, "x1": 30}, 1.0, 13),
                    ({"kind": "disc", "cy2": 81, "cx2": 100, "r": 5}, 0.7, 50),
                    ({"kind": "rect", "y0": 60, "x0": 60, "y1": 80, "x1": 95}, 1.0, 50)]
    r = oracle_run(w, 0)
    for splits in ([97], [13, 84], [1, 12, 37, 47], [50, 47], [3] * 32 + [1]):
        U, V, _, _ = gpu_run(w, splits=splits)
        assert_bitwise(U[0], r.u, f"u splits={splits[:5]}")
        assert_bitwise(V[0], r.v, f"v splits={splits[:5]}")


@pytest.mark.parametrize("dtype", DT, ids=IDS)
def test_reaction_off(dtype):
    """RD_REACTION_OFF: u' = u + dt Du L, v' = v, bitwise vs the oracle."""
    w = _noise_workload(50, 77, dtype, 100)
    U, V, _, _ = gpu_run(w, flags=rd.RD_REACTION_OFF)
    r = oracle_run(w, 0, reaction_off=True)
    assert_bitwise(U[0], r.u, "u")
    assert_bitwise(V[0], r.v, "v")


@pytest.mark.parametrize("dtype", DT, ids=IDS)
def test_masked_half_discs(dtype):
    """Half-disc stimuli masked to phi_active cells (R-22) over a
    two-level phi map with obstacles."""
    H, W = 120, 160
    phi = np.full((H, W), 0.054)
    phi[20:70, 30:90] = 0.2
    phi[80:110, 100:150] = 0.2
    w = _noise_workload(H, W, dtype, 30, phi=phi, n_discs=20, mask=0.054)
    U, V, _, _ = gpu_run(w)
    r = oracle_run(w, 0)
    assert_bitwise(U[0], r.u, "u")
    assert_bitwise(V[0], r.v, "v")


# ------------------------------------------------------------ probes, faults

@pytest.mark.parametrize("dtype", DT, ids=IDS)
def test_probes_latch_and_immediate(dtype):
    H, W = 40, 300
    w = _noise_workload(H, W, dtype, 2500, n_discs=0)
    w.init = None
    w.events = [[({"kind": "rect", "y0": 0, "x0": 0, "y1": H, "x1": 5}, 1.0, 0)]]
    w.probes = [[((0, 10, H, 12), 0.1, 50), ((5, 25, 9, 27), 0.1, 7), ((0, 290, H, 300), 0.1, 50)]]
    U, V, fire, _ = gpu_run(w)
    r = oracle_run(w, 0)
    assert fire[0] == r.first_fire
    assert fire[0][0] > 0 and fire[0][2] == -1
    sim = rd.Sim(w.phi_plane(0).astype(dtype), dtype=dtype)
    sim.stimulate({"kind": "rect", "y0": 3, "x0": 4, "y1": 5, "x1": 9}, 1.0, 0)
    sim.step(1)
    ref = oracle.run(np.zeros((H, W), dtype), np.zeros((H, W), dtype), w.phi_plane(0).astype(dtype), 1,
                     events=[({"kind": "rect", "y0": 3, "x0": 4, "y1": 5, "x1": 9}, 1.0, 0)])
    fired, m = sim.probe(0, (0, 0, 10, 20), 0.1)
    assert fired and m == oracle.probe_max(ref.u, (0, 0, 10, 20))
    with pytest.raises(rd.RDError):
        sim.probe(0, (0, 0, 0, 5), 0.1)
    sim.close()


@pytest.mark.parametrize("dtype", DT, ids=IDS)
@pytest.mark.parametrize("splits", [None, [90, 7, 203, 2200]], ids=["one_call", "split"])
def test_probe_strides_inside_and_at_launch_ends(dtype, splits, kernel):
    """a6 with strides 30 and 45 in one instance: cr_kernel tests the due steps
    inside a launch in its step loop (every gcd = 15 steps) and the step that
    ends a launch in its write-back. rd_step splits end before, on and after
    due steps. Latched steps and fields equal the oracle's under every kernel."""
    H, W = 64, 256
    w = _noise_workload(H, W, dtype, 2500, B=2, n_discs=0)
    w.init = None
    w.events = [[({"kind": "rect", "y0": 0, "x0": 0, "y1": H, "x1": 4}, 1.0, 0)],
                [({"kind": "rect", "y0": 20, "x0": 0, "y1": 44, "x1": 4}, 1.0, 0)]]
    w.probes = [[((0, 6, H, 8), 0.1, 30), ((0, 10, H, 12), 0.1, 45), ((0, 14, 9, 16), 0.1, 45), ((0, 250, H, 256), 0.1, 30)],
                [((30, 8, 34, 10), 0.1, 45), ((0, 12, 2, 14), 0.1, 30)]]
    U, V, fire, _ = gpu_run(w, splits=splits)
    for b in range(2):
        r = oracle_run(w, b)
        assert fire[b] == r.first_fire, (b, fire[b], r.first_fire)
        assert_bitwise(U[b], r.u, f"u[{b}]")
        assert_bitwise(V[b], r.v, f"v[{b}]")
    assert fire[0][0] > 0 and fire[0][1] > 0 and fire[0][0] != fire[0][1] and fire[0][3] == -1


@pytest.mark.parametrize("dtype", DT, ids=IDS)
@pytest.mark.parametrize("tb", [1, 4, 8])
def test_nonfinite_fault_matches_oracle(dtype, tb, kernel):
    """T5: uniform phi=0.2, noisy u,v, an unmasked u:=1 half-disc -> Euler
    diverges. rd_step returns RD_ENONFINITE, the handle stops at the oracle's
    failing step with the oracle's first (i, j) and identical fields."""
    H = W = 128
    u0 = noise_plane(H, W, 0, seed=7, dtype=dtype)
    v0 = noise_plane(H, W, 1, seed=7, dtype=dtype)
    phi = np.full((H, W), 0.2, dtype=dtype)
    s = {"kind": "half_disc", "cy2": 128, "cx2": 128, "r": 8, "dir": 0}
    ref = oracle.run(u0, v0, phi, 400, events=[(s, 1.0, 0)])
    assert ref.status == -4
    sim = rd.Sim(phi, dtype=dtype, tb_depth=tb)
    sim.write(0, u0, v0)
    sim.stimulate(s, 1.0, 0)
    with pytest.raises(rd.RDError) as e:
        sim.step(400)
    assert e.value.code == rd.RD_ENONFINITE
    st, b, i, j = sim.fault()
    assert (st, b, i, j) == (ref.fault[0], 0, ref.fault[1], ref.fault[2])
    assert sim.step_count == ref.fault[0]
    u, v = sim.read(0)
    assert_bitwise(u, ref.u, "u at fault")
    assert_bitwise(v, ref.v, "v at fault")
    sim.close()


def test_write_fields_rejects_nonfinite():
    sim = rd.Sim(np.full((8, 8), 0.054, np.float32))
    bad = np.zeros((8, 8), np.float32)
    bad[3, 4] = np.nan
    with pytest.raises(rd.RDError) as e:
        sim.write(0, bad, None)
    assert e.value.code == rd.RD_ENONFINITE
    with pytest.raises(rd.RDError) as e:
        sim.stimulate({"kind": "disc", "cy2": 0, "cx2": 0, "r": 1}, 1.0, -1)
    assert e.value.code == rd._lib.RD_ERANGE
    sim.close()
    phi = np.full((8, 8), 0.054, np.float32)
    phi[0, 0] = np.inf
    with pytest.raises(rd.RDError) as e:
        rd.Sim(phi)
    assert e.value.code == rd.RD_ENONFINITE


@pytest.mark.parametrize("tb", [1, 4])
@pytest.mark.parametrize("qv,mode", [(0.002, 4), (2.0 ** -40, None)], ids=["q=0.002", "q=2^-40"])
def test_fast_division_guard_replay(tb, kernel, qv, mode):
    """Cells where the fast division is not certified make the rd_step replay
    precisely from its checkpoint (stats.replays); the result equals the
    oracle bitwise (finite or at the first fault).
    q = 0.002 (guard-free mode 4): C = -q gives C + q == 0, so the fast
    sequence yields NaN and the non-finite check triggers the replay (C one
    ulp above -q gives C + q = 2^-32, inside the certified range).
    q = 2^-40 (guarded modes): C = -q + ulp gives 0 < C + q = 2^-63 < 2^-60,
    which the min|C+q| guard catches."""
    H, W = 24, 40
    dtype = np.float32
    q = np.float32(qv)
    u0 = noise_plane(H, W, 0, seed=9, dtype=dtype)
    v0 = noise_plane(H, W, 1, seed=9, dtype=dtype)
    if mode == 4:
        u0[5, 7] = np.nextafter(-q, np.float32(0))
        u0[12, 30] = -q
    else:
        u0[5, 7] = np.nextafter(-q, np.float32(0))
        assert 0 < np.float32(u0[5, 7] + q) < np.float32(2.0 ** -60)
    phi = np.full((H, W), 0.054, dtype)
    ref = oracle.run(u0, v0, phi, 6, params=oracle.Params(q=float(q)))
    p = rd.rd_params_default()
    p.q = float(q)
    sim = rd.Sim(phi, dtype=dtype, tb_depth=tb, params=p)
    if mode is not None:
        assert sim.stats()["arith_mode"] == mode
    else:
        assert sim.stats()["arith_mode"] in (2, 3)
    sim.write(0, u0, v0)
    try:
        sim.step(6)
        assert ref.status == 0
    except rd.RDError as e:
        assert e.code == rd.RD_ENONFINITE and ref.status == -4
        st, b, i, j = sim.fault()
        assert (st, i, j) == ref.fault
    u, v = sim.read(0)
    assert sim.stats()["replays"] >= 1
    assert_bitwise(u, ref.u, "u")
    assert_bitwise(v, ref.v, "v")
    sim.close()


@pytest.mark.parametrize("dtype", DT, ids=IDS)
@pytest.mark.parametrize("stride,tb", [(25, 4), (7, 4), (50, 1), (3, 8)])
def test_timelapse_matches_oracle(dtype, stride, tb, kernel):
    """f2: the fused timelapse max_u, recorded after
    every multiple of stride, equals the oracle's bitwise; splitting rd_step
    calls does not change it."""
    w = _noise_workload(60, 90, dtype, 140)
    u0, v0 = w.init_planes(0)
    ref = oracle.run(u0, v0, w.phi_plane(0).astype(dtype), 140, events=w.events[0], timelapse_stride=stride)
    for splits in ([140], [13, 50, 77]):
        sim = rd.Sim(w.phi_plane(0).astype(dtype), dtype=dtype, tb_depth=tb)
        sim.write(0, u0, v0)
        for s, val, at in w.events[0]:
            sim.stimulate(s, val, at)
        sim.timelapse(stride)
        for n in splits:
            sim.step(n)
        assert_bitwise(sim.read_timelapse(0), ref.max_u, f"max_u splits={splits}")
        assert_bitwise(sim.read(0)[0], ref.u, "u")
        sim.close()


@pytest.mark.parametrize("dtype", DT, ids=IDS)
def test_rest_init_and_spiral_seeding(dtype):
    """f4: rd_init_rest gives the oracle's quiescent planes bitwise (per-cell
    u*(phi) on a two-level phi map), and the staggered spiral-seeding run
     equals the oracle bitwise at step 40000 with sustained
    activity."""
    from rdinputs import spiral_seed
    phi = np.full((50, 70), 0.054)
    phi[20:30, 10:60] = 0.119
    sim = rd.Sim(phi.astype(dtype), dtype=dtype)
    sim.init_rest()
    u, v = sim.read(0)
    ru, rv = oracle.rest_fill(phi.astype(dtype))
    assert_bitwise(u, ru, "u*")
    assert_bitwise(v, rv, "v*")
    sim.close()
    w = spiral_seed(dtype=dtype)
    sim = rd.Sim(w.phi_plane(0).astype(dtype), dtype=dtype)
    sim.init_rest()
    for s, val, at in w.events[0]:
        sim.stimulate(s, val, at)
    sim.step(w.steps)
    u, v = sim.read(0)
    sim.close()
    u0, v0 = oracle.rest_fill(w.phi_plane(0).astype(dtype))
    ref = oracle.run(u0, v0, w.phi_plane(0).astype(dtype), w.steps, events=w.events[0])
    assert_bitwise(u, ref.u, "u")
    assert_bitwise(v, ref.v, "v")
    assert (u > 0.1).mean() > 0.05


@pytest.mark.parametrize("dtype", DT, ids=IDS)
def test_graph_replay_equals_direct_launches(dtype, monkeypatch):
    """CUDA-graph replay of rd_step segments (default) and direct launches
    (RD_NO_GRAPH) give bitwise identical fields and probe latches (tb_kernel:
    cr_kernel segments are single launches and are not captured)."""
    from rdinputs import config
    monkeypatch.setenv("RD_KERNEL", "tb")
    w = config(2, dtype=dtype, steps=1500)
    Ug, Vg, Fg, sg = gpu_run(w)
    Ud, Vd, Fd, sd = gpu_run(w, flags=rd.RD_NO_GRAPH)
    assert_bitwise(Ug, Ud, "u")
    assert_bitwise(Vg, Vd, "v")
    assert Fg == Fd
    assert sg["step_launches"] == sd["step_launches"]


@pytest.mark.parametrize("dtype", DT, ids=IDS)
def test_device_noise_equals_rdinputs(dtype):
    """rd_fill_noise (device SplitMix64) equals rdinputs.noise_plane bitwise,
    for a full grid and for a slab with a global row offset."""
    H, W = 77, 301
    sim = rd.Sim(np.full((H, W), 0.054, dtype=dtype), dtype=dtype)
    sim.fill_noise(seed=1)
    u, v = sim.read(0)
    sim.close()
    assert_bitwise(u, noise_plane(H, W, 0, seed=1, dtype=dtype), "u")
    assert_bitwise(v, noise_plane(H, W, 1, seed=1, dtype=dtype), "v")
    h = rd.rd_create_slab(W, 20, np.full((28, W), 0.054, dtype=dtype), 40, H, 4, dtype=dtype)
    rd.rd_fill_noise(h, -1, 3, 9, 0.1)
    us = np.empty((20, W), dtype)
    vs = np.empty((20, W), dtype)
    rd.rd_read_fields(h, 0, us, vs)
    rd.rd_destroy(h)
    assert_bitwise(us, noise_plane(20, W, 0, seed=9, dtype=dtype, row0=40, W_global=W), "u slab")
    assert_bitwise(vs, noise_plane(20, W, 1, seed=9, dtype=dtype, row0=40, W_global=W), "v slab")
