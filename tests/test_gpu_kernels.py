"""Kernel-level checks that need a GPU but no oracle: the fast fp32 division
(rdk::div_fast_f32) is bit-identical to IEEE div.rn on the whole input domain
the reaction can produce, for Table-1 q and other q values."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def divcheck(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cuda") / "divcheck")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-o", exe,
                    os.path.join(HERE, "cuda", "divcheck.cu")], check=True)
    return exe


@pytest.mark.parametrize("q", ["0.002", "0.5", "1e-12", "0.999"])
def test_fast_division_exhaustive(divcheck, q):
    out = subprocess.run([divcheck, q], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout)
    assert r["tested"] > 4_000_000_000
    assert r["mismatch_guarded"] == 0, r


def test_certified_four_op_division_selected_for_table1_q():
    """For Table-1 q the 4-op division is certified exhaustively at rd_create
    and selected without the min|C+q| guard (arith_mode 4: q >= 2^-35); a q
    where it is not exact keeps the 6-op sequence (arith_mode 2); results are
    bitwise the oracle's either way."""
    import numpy as np
    import oracle
    import paper_1901_06535_b200 as rd
    from rdinputs import config
    for q, mode in ((0.002, 4), (0.1, 2)):
        p = rd.rd_params_default()
        p.q = q
        w = config(1, dtype=np.float32, steps=200)
        sim = rd.Sim(w.phi_plane(0).astype(np.float32), dtype=np.float32, params=p)
        assert sim.stats()["arith_mode"] == mode
        for s, val, at in w.events[0]:
            sim.stimulate(s, val, at)
        sim.step(200)
        u, v = sim.read(0)
        sim.close()
        u0, v0 = w.init_planes(0)
        ref = oracle.run(u0, v0, w.phi_plane(0).astype(np.float32), 200, events=w.events[0],
                         params=oracle.Params(q=q))
        assert np.array_equal(u, ref.u) and np.array_equal(v, ref.v)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_cluster_resident_kernel_selection_and_parity(dtype, monkeypatch):
    """a8: configs 1-3 run on gz_kernel by default (rd_stats.kernel == 3);
    cr_kernel (forced) on instances that fit a cluster's shared memory is
    bitwise equal to the oracle and to tb_kernel, over row splits with and
    without a ragged remainder (H % cs != 0), narrow W (< one block of
    threads) and a segment cut by a mid-run stimulus."""
    import numpy as np
    import oracle
    import paper_1901_06535_b200 as rd
    from rdinputs import config, noise_plane
    dt = np.float32 if dtype == "f32" else np.float64
    monkeypatch.delenv("RD_KERNEL", raising=False)
    # the default choice on configs 1-3 is now gz_kernel (whole-chip tiles,
    # its model beats cr_kernel's on every one); cr_kernel
    # is forced below
    for n in (1, 2, 3):
        w = config(n, dtype=dt)
        sim = rd.Sim(np.stack([w.phi_plane(b).astype(dt) for b in range(w.B)]), dtype=dt)
        assert sim.stats()["kernel"] == 3, n
        sim.close()
    for (H, W) in [(64, 64), (37, 131), (301, 29), (9, 700), (150, 150)]:
        u0 = noise_plane(H, W, 0, seed=4, dtype=dt)
        v0 = noise_plane(H, W, 1, seed=4, dtype=dt)
        phi = np.full((H, W), 0.054, dt)
        phi[H // 3:H // 2, W // 4:W // 2] = 0.0975
        ev = [({"kind": "disc", "cy2": H, "cx2": W, "r": 3}, 1.0, 0),
              ({"kind": "rect", "y0": 0, "x0": 0, "y1": 3, "x1": W}, 1.0, 17)]
        ref = oracle.run(u0, v0, phi, 40, events=ev)
        out = {}
        for kern in ("cr", "tb"):
            monkeypatch.setenv("RD_KERNEL", kern)
            sim = rd.Sim(phi[None], dtype=dt)
            assert sim.stats()["kernel"] == (2 if kern == "cr" else 0), (H, W, kern)
            sim.write(0, u0, v0)
            for s, val, at in ev:
                sim.stimulate(s, val, at)
            sim.step(40)
            out[kern] = sim.read(0)
            sim.close()
            assert np.array_equal(out[kern][0], ref.u), (H, W, kern)
            assert np.array_equal(out[kern][1], ref.v), (H, W, kern)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("H,W", [(4, 3), (5, 3), (33, 3), (4, 5), (17, 8), (6, 4), (64, 2048), (40, 1021)])
def test_cluster_resident_edge_shapes(dtype, H, W, monkeypatch):
    """cr_kernel at its shape limits: bands of one or two rows (H = 4, 5 with
    2-CTA clusters), the narrowest grids the API accepts (W = 3: the ghost
    column W inside the only vector), exact multiples of the vector width
    (ghost column W in the pad vector) and wide rows (one thread per vector,
    up to 512 vectors) -- bitwise equal to the oracle, with a mid-segment
    event and uneven rd_step splits."""
    import numpy as np
    import oracle
    import paper_1901_06535_b200 as rd
    from rdinputs import noise_plane
    dt = np.float32 if dtype == "f32" else np.float64
    monkeypatch.setenv("RD_KERNEL", "cr")
    u0 = noise_plane(H, W, 0, seed=11, dtype=dt)
    v0 = noise_plane(H, W, 1, seed=11, dtype=dt)
    phi = np.full((H, W), 0.054, dt)
    phi[:, W // 2:] = 0.0975
    ev = [({"kind": "disc", "cy2": H, "cx2": W, "r": 2}, 1.0, 0),
          ({"kind": "rect", "y0": H - 1, "x0": 0, "y1": H, "x1": W}, 1.0, 13)]
    ref = oracle.run(u0, v0, phi, 30, events=ev)
    sim = rd.Sim(phi[None], dtype=dt)
    vec = 16 // np.dtype(dt).itemsize
    fits = (W + vec - 1) // vec <= 512
    assert sim.stats()["kernel"] == (2 if fits else 0)
    sim.write(0, u0, v0)
    for s, val, at in ev:
        sim.stimulate(s, val, at)
    for n in (7, 6, 17):
        sim.step(n)
    u, v = sim.read(0)
    sim.close()
    assert np.array_equal(u, ref.u) and np.array_equal(v, ref.v)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_cluster_resident_palette_layout(dtype, monkeypatch):
    """cr_kernel with phi as palette indices (the layout that fits fp64
    configs 2/3): a device-painted handle (phi = 0 plus painted values, the
    palette tracked from rd_paint_phi, repainted between rd_step calls) and
    a config-3-sized diode batch are bitwise equal to the oracle; a phi map
    with more than 256 distinct values per instance falls back to tb_kernel
    and stays exact."""
    import numpy as np
    import oracle
    import paper_1901_06535_b200 as rd
    from rdinputs import config, noise_plane
    dt = np.float32 if dtype == "f32" else np.float64
    monkeypatch.setenv("RD_KERNEL", "cr")
    H, W = 300, 400  # config-2 instances: fp64 fits only with the palette layout
    sim = rd.Sim(None, shape=(1, H, W), dtype=dt)
    sim.paint_phi(0.054)
    sim.paint_phi(0.0975, (100, 200, 140, 380))
    assert sim.stats()["kernel"] == 2
    u0 = noise_plane(H, W, 0, seed=5, dtype=dt)
    v0 = noise_plane(H, W, 1, seed=5, dtype=dt)
    sim.write(0, u0, v0)
    sim.stimulate({"kind": "disc", "cy2": H, "cx2": 200, "r": 6}, 1.0, 0)
    sim.step(25)
    sim.paint_phi(0.2, (10, 10, 30, 60))   # a third value mid-run
    sim.step(15)
    u, v = sim.read(0)
    st = sim.stats()
    sim.close()
    phi = np.full((H, W), 0.054, dt)
    phi[100:140, 200:380] = dt(0.0975)
    r1 = oracle.run(u0, v0, phi, 25, events=[({"kind": "disc", "cy2": H, "cx2": 200, "r": 6}, 1.0, 0)])
    phi2 = phi.copy()
    phi2[10:30, 10:60] = dt(0.2)
    r2 = oracle.run(r1.u, r1.v, phi2, 15, step0=25)
    assert st["kernel"] == 2
    assert np.array_equal(u, r2.u) and np.array_equal(v, r2.v)
    # AND-gate batch at config-2 size in this dtype (palette layout in fp64)
    w = config(2, dtype=dt, steps=300)
    phis = np.stack([w.phi_plane(b).astype(dt) for b in range(w.B)])
    s2 = rd.Sim(phis, dtype=dt)
    assert s2.stats()["kernel"] == 2
    for b in range(w.B):
        for sh, val, at in w.events[b]:
            s2.stimulate(sh, val, at, b=b)
    s2.step(w.steps)
    for b in range(w.B):
        ub, vb = s2.read(b)
        u0b, v0b = w.init_planes(b)
        ref = oracle.run(u0b, v0b, w.phi_plane(b).astype(dt), w.steps, events=w.events[b])
        assert np.array_equal(ub, ref.u) and np.array_equal(vb, ref.v), b
    s2.close()
    # > 256 distinct phi values: no palette; fp64 does not fit otherwise
    rough = (0.05 + 0.01 * noise_plane(H, W, 0, seed=6, dtype=np.float64)).astype(dt)
    s3 = rd.Sim(rough[None], dtype=dt)
    assert s3.stats()["kernel"] == (2 if dt == np.float32 else 0)
    s3.write(0, u0, v0)
    s3.step(12)
    u3, v3 = s3.read(0)
    s3.close()
    ref3 = oracle.run(u0, v0, rough, 12)
    assert np.array_equal(u3, ref3.u) and np.array_equal(v3, ref3.v)


def test_c_abi_from_plain_c(tmp_path):
    """The boundary used from C, without Python: tests/c/abi_c_demo.c links
    librd.so (and, as a test, the oracle's C library), runs a two-instance
    fp64 and fp32 batch through rd_create / rd_stimulate / rd_step /
    rd_read_fields / rd_probe and compares with the oracle bitwise, plus
    error codes (RD_EINVAL, RD_ERANGE)."""
    import subprocess
    root = os.path.dirname(HERE)
    exe = str(tmp_path / "abi_c_demo")
    lib, orc = os.path.join(root, "paper_1901_06535_b200"), os.path.join(root, "oracle")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(root, "include"), "-I", orc,
                    os.path.join(HERE, "c", "abi_c_demo.c"), "-L", lib, "-lrd", "-L", orc, "-lorc",
                    f"-Wl,-rpath,{lib}:{orc}", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "C ABI ok" in out.stdout


def test_c_dist_abi_from_plain_c(tmp_path):
    """The multi-GPU calls from C (tests/c/dist_c_demo.c): two forked rank
    processes over rd_dist_shm_id (CUDA IPC push, no NCCL, no Python),
    rd_dist_unique_id + rd_create_dist at world 1 over NCCL, and two
    in-process ranks (rd_dist_local_id, pthreads) on one device, in fp32 and
    fp64 -- each bitwise equal to the oracle's C library on the whole grid."""
    root = os.path.dirname(HERE)
    exe = str(tmp_path / "dist_c_demo")
    lib, orc = os.path.join(root, "paper_1901_06535_b200"), os.path.join(root, "oracle")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(root, "include"), "-I", orc,
                    os.path.join(HERE, "c", "dist_c_demo.c"), "-L", lib, "-lrd", "-L", orc, "-lorc", "-lpthread",
                    f"-Wl,-rpath,{lib}:{orc}", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "C dist ABI ok" in out.stdout


@pytest.fixture(scope="module")
def divcheck64(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cuda64") / "divcheck64")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-o", exe,
                    os.path.join(HERE, "cuda", "divcheck64.cu")], check=True)
    return exe


@pytest.mark.parametrize("q", ["0.002", "0.5", "1e-12", "0.999"])
def test_fast_division_f64_matches_ddiv_rn(divcheck64, q):
    """The inline fp64 fast path (rdk::div_fast_f64) equals __ddiv_rn bitwise
    wherever its guard passes, on 2^32 seeded reaction operands a = C - q,
    b = C + q (any finite bit pattern, U[-2, 2], and C within 2^-40 of -q and
    +q); a tripped guard means a PRECISE replay, never a wrong quotient."""
    out = subprocess.run([divcheck64, q, str(1 << 32)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout)
    assert r["tested"] > 3_000_000_000
    assert r["mismatch_guarded"] == 0, r


def test_default_depth_and_balanced_segment_cuts(monkeypatch):
    """auto depth (DESIGN.md §5.2 "Depth"): fp32 handles of >= 2^22 cells take
    depth 6, smaller ones and fp64 keep 4; a segment is cut into launches of
    nearly equal depth (50 steps at depth 6: nine launches 6 6 6 6 6 5 5 5 5,
    at depth 4: thirteen), and the cuts do not change the result."""
    import numpy as np
    import paper_1901_06535_b200 as rd
    monkeypatch.setenv("RD_KERNEL", "tb")
    monkeypatch.delenv("RD_TB_DEPTH", raising=False)
    monkeypatch.delenv("RD_TB_DEEP", raising=False)

    def stats(shape, dtype, steps, depth=0):
        with rd.Sim(None, shape=shape, dtype=dtype, tb_depth=depth, flags=rd.RD_NO_GRAPH) as sim:
            sim.paint_phi(0.054)
            sim.fill_noise(seed=3)
            rd.rd_reset_stats(sim.h)
            sim.step(steps)
            st = sim.stats()
            return st, sim.read(0)

    st, _ = stats((1, 2048, 2048), np.float32, 50, depth=6)
    assert st["tb_depth"] == 6 and st["step_launches"] == 9
    st, _ = stats((1, 2048, 2047), np.float32, 8)
    assert st["tb_depth"] == 4
    st, _ = stats((1, 4096, 16384), np.float64, 8)
    assert st["tb_depth"] == 4
    st6, (u6, v6) = stats((1, 300, 500), np.float32, 50, depth=6)
    st4, (u4, v4) = stats((1, 300, 500), np.float32, 50, depth=4)
    assert st6["step_launches"] == 9 and st4["step_launches"] == 13
    assert np.array_equal(u6, u4) and np.array_equal(v6, v4)
