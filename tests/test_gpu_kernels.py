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
    """a8: instances that fit a cluster's shared memory run on cr_kernel by
    default (rd_stats.kernel == 2) -- configs 1-3 in fp32, config 1 in fp64 --
    bitwise equal to the oracle and to tb_kernel, over row splits with and
    without a ragged remainder (H % cs != 0), narrow W (< one block of
    threads) and a segment cut by a mid-run stimulus."""
    import numpy as np
    import oracle
    import paper_1901_06535_b200 as rd
    from rdinputs import config, noise_plane
    dt = np.float32 if dtype == "f32" else np.float64
    monkeypatch.delenv("RD_KERNEL", raising=False)
    fits = {1: True, 2: dt == np.float32, 3: dt == np.float32}
    for n, want in fits.items():
        w = config(n, dtype=dt)
        sim = rd.Sim(np.stack([w.phi_plane(b).astype(dt) for b in range(w.B)]), dtype=dt)
        assert sim.stats()["kernel"] == (2 if want else 0), n
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
