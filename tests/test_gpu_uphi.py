"""tb_kernel's uniform-phi variants (UPHI): when the phi map is one value the
kernel takes it as a parameter instead of streaming the plane. The handle
re-derives that on the device after every change of phi, and the results are
bitwise those of the oracle (and of the streaming path) either way."""
import numpy as np
import pytest

import oracle
import paper_1901_06535_b200 as rd
from gpu_util import assert_bitwise
from rdinputs import noise_plane

pytestmark = pytest.mark.gpu

DISC = {"kind": "disc", "cy2": 60, "cx2": 200, "r": 6}


@pytest.fixture(autouse=True)
def _tb(monkeypatch):
    monkeypatch.setenv("RD_KERNEL", "tb")


@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
@pytest.mark.parametrize("depth", [1, 2, 3, 4, 6, 7, 8])
@pytest.mark.parametrize("shape", [(67, 131), (40, 517), (131, 250)])
def test_uniform_map_runs_the_parameter_variant_and_equals_the_oracle(shape, depth, dtype):
    """Ragged shapes (one strip, several strips, W % V != 0) at depths the
    variant exists for (fp32: 1-7, fp64: 1-4) and some it does not (the plane
    is streamed)."""
    H, W = shape
    phi = np.full((1, H, W), 0.054, dtype=dtype)
    u0 = noise_plane(H, W, 0, seed=7, dtype=dtype)
    v0 = noise_plane(H, W, 1, seed=7, dtype=dtype)
    with rd.Sim(phi, dtype=dtype, tb_depth=depth) as sim:
        sim.write(0, u0, v0)
        sim.stimulate(DISC, 1.0, 3)
        sim.step(11)
        sim.step(18)
        st = sim.stats()
        u, v = sim.read(0)
    assert st["kernel"] == 0 and st["phi_uniform"] == 1
    ref = oracle.run(u0, v0, phi[0], 29, events=[(DISC, 1.0, 3)])
    assert_bitwise(u, ref.u, "u")
    assert_bitwise(v, ref.v, "v")


@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
def test_class_follows_every_change_of_phi(dtype):
    """uniform -> an obstacle painted between steps -> painted over again: the
    handle switches variants (captured graphs included) and stays on the oracle."""
    H, W = 90, 300
    u0 = noise_plane(H, W, 0, seed=9, dtype=dtype)
    v0 = noise_plane(H, W, 1, seed=9, dtype=dtype)
    phi = np.full((H, W), 0.054, dtype=dtype)
    with rd.Sim(None, shape=(1, H, W), dtype=dtype) as sim:
        sim.paint_phi(0.054)
        sim.write(0, u0, v0)
        sim.stimulate(DISC, 1.0, 0)
        for _ in range(3):  # the same segment shape three times: replayed from a graph
            sim.step(8)
        assert sim.stats()["phi_uniform"] == 1
        r1 = oracle.run(u0, v0, phi, 24, events=[(DISC, 1.0, 0)])
        u, v = sim.read(0)
        assert_bitwise(u, r1.u, "u uniform")
        sim.paint_phi(0.2, (20, 40, 50, 120))
        phi2 = phi.copy()
        phi2[20:50, 40:120] = dtype(0.2)
        for _ in range(3):
            sim.step(8)
        assert sim.stats()["phi_uniform"] == 0
        r2 = oracle.run(r1.u, r1.v, phi2, 24, step0=24)
        u, v = sim.read(0)
        assert_bitwise(u, r2.u, "u with obstacle")
        assert_bitwise(v, r2.v, "v with obstacle")
        sim.paint_phi(0.0975)  # the whole grid: one value again, a different one
        phi3 = np.full((H, W), 0.0975, dtype=dtype)
        for _ in range(3):
            sim.step(8)
        assert sim.stats()["phi_uniform"] == 1
        r3 = oracle.run(r2.u, r2.v, phi3, 24, step0=48)
        u, v = sim.read(0)
        assert_bitwise(u, r3.u, "u repainted")
        assert_bitwise(v, r3.v, "v repainted")


def test_instances_with_different_values_stream_the_plane():
    """One value per instance is not one value: the general kernel runs."""
    dtype = np.float32
    H, W = 50, 140
    phi = np.stack([np.full((H, W), 0.054, dtype), np.full((H, W), 0.0975, dtype)])
    u0 = noise_plane(H, W, 0, seed=4, dtype=dtype)
    v0 = noise_plane(H, W, 1, seed=4, dtype=dtype)
    with rd.Sim(phi, dtype=dtype) as sim:
        for b in range(2):
            sim.write(b, u0, v0)
        sim.step(20)
        assert sim.stats()["phi_uniform"] == 0
        for b in range(2):
            ref = oracle.run(u0, v0, phi[b], 20)
            u, v = sim.read(b)
            assert_bitwise(u, ref.u, f"u b={b}")
            assert_bitwise(v, ref.v, f"v b={b}")


def test_handing_out_phi_disables_the_variant():
    """After rd_field_ptr(plane 2) the caller may write phi behind the handle's
    back: the handle streams the plane from then on, and sees such writes."""
    dtype = np.float32
    H, W = 48, 136
    phi = np.full((1, H, W), 0.054, dtype=dtype)
    u0 = noise_plane(H, W, 0, seed=5, dtype=dtype)
    v0 = noise_plane(H, W, 1, seed=5, dtype=dtype)
    with rd.Sim(phi, dtype=dtype) as sim:
        sim.write(0, u0, v0)
        sim.step(8)
        assert sim.stats()["phi_uniform"] == 1
        ptr, pitch = rd.rd_field_ptr(sim.h, 0, 2)
        assert ptr and pitch >= W
        sim.step(8)
        assert sim.stats()["phi_uniform"] == 0
        ref = oracle.run(u0, v0, phi[0], 16)
        u, v = sim.read(0)
        assert_bitwise(u, ref.u, "u")
