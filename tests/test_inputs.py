"""The seeded input generators (rdinputs): reference vectors and invariants."""
import numpy as np

from rdinputs import and_gate, diode, half_discs, noise_plane, obstacles, splitmix64


def test_splitmix64_reference_vectors():
    """SplitMix64 (Steele, Lea & Flood 2014) seeded with 0 yields the published
    sequence e220a8397b1dcdaf, 6e789e6aa1b965f4, 06c45d188009454f."""
    g = 0x9E3779B97F4A7C15
    got = [int(splitmix64(np.uint64((k * g) % 2 ** 64))) for k in range(3)]
    assert got == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_noise_range_and_slab_independence():
    """U[0, 0.1) values; a row slab generated on its own equals the same rows
    of the full grid (inputs independent of the GPU count)."""
    full = noise_plane(64, 48, 0, seed=1, dtype=np.float64)
    assert full.min() >= 0 and full.max() < 0.1
    assert abs(full.mean() - 0.05) < 0.005
    slab = noise_plane(16, 48, 0, seed=1, dtype=np.float64, row0=32, W_global=48)
    assert np.array_equal(slab, full[32:48])
    other = noise_plane(64, 48, 1, seed=1, dtype=np.float64)
    assert not np.array_equal(full, other)
    f32 = noise_plane(64, 48, 0, seed=1, dtype=np.float32)
    assert np.array_equal(f32, full.astype(np.float32))


def test_half_discs_and_obstacles():
    hd = half_discs(1000, 800, 64, seed=2)
    assert len(hd) == 64 and hd == half_discs(1000, 800, 64, seed=2)
    assert all(0 <= s["cy2"] // 2 < 1000 and 0 <= s["cx2"] // 2 < 800 and 0 <= s["dir"] < 4 for s in hd)
    ob = obstacles(65536, 65536, 256, seed=3)
    assert len(ob) == 256
    for (y0, x0, y1, x1) in ob:
        assert 0 < y1 - y0 <= 1024 and 0 < x1 - x0 <= 1024 and y1 <= 65536 and x1 <= 65536


def test_and_gate_geometry():
    """Mirror-symmetric two-level map, 1-row gap under the junction, the two
    input blocks mirror images of each other."""
    g = and_gate()
    phi = g["phi"]
    assert np.array_equal(phi, phi[:, ::-1])
    assert set(np.unique(phi)) == {0.054, 0.119}
    assert g["out_top"] == g["junction_bottom"] + 2
    assert np.all(phi[g["junction_bottom"] + 1] == 0.119)
    a, b = g["inputs"]
    assert (a["x0"], a["x1"]) == (400 - b["x1"], 400 - b["x0"])


def test_diode_geometry():
    """Flat anode wall, 2-column gap, triangular cathode tip widths 2..18."""
    d = diode()
    phi = d["phi"]
    widths = [int((phi[:, x] == 0.054).sum()) for x in range(298, 312)]
    assert widths == [20, 20, 0, 0, 2, 4, 6, 8, 12, 14, 16, 18, 20, 20]
