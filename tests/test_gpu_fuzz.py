"""Seeded randomized parity: every feature of the hot path at once, against
the oracle, bitwise.

Each case draws (from a fixed seed) a dtype, a batch of 1-3 instances with
ragged shapes (one in eight up to 300x400: cr_kernel's palette layout), two-level phi maps with obstacles, noisy u/v, stimuli of every
kind (disc, rect, half-disc, with and without the phi mask) at random steps,
latched probes, a timelapse stride, sometimes per-instance Eq.-1 parameters
(including a non-power-of-two dx, which forces the PRECISE mode), a temporal
blocking depth, a stencil kernel (auto / tb / lp / cr) and a random split of
the run into rd_step calls. Fields, probe latches and the timelapse record
must equal the oracle's exactly; a non-finite fault must stop at the oracle's
step and cell.
"""
import os

import numpy as np
import pytest

import oracle
import paper_1901_06535_b200 as rd
from rdinputs import noise_plane

pytestmark = pytest.mark.gpu
N_CASES = int(os.environ.get("RD_FUZZ_CASES", "96"))  # more seeds on demand


def _case(seed):
    g = np.random.default_rng(1000 + seed)
    dt = np.float32 if g.random() < 0.6 else np.float64
    B = int(g.integers(1, 4))
    H, W = int(g.integers(3, 160)), int(g.integers(3, 260))
    if g.random() < 0.125:  # large instances: cr_kernel's palette layout in fp64
        B, H, W = int(g.integers(1, 3)), int(g.integers(200, 301)), int(g.integers(300, 401))
    steps = int(g.integers(1, 90))
    phis, inits, evs, prs, params = [], [], [], [], []
    for b in range(B):
        lv = [0.054, float(g.choice([0.0975, 0.119, 0.0, round(float(g.uniform(0.0, 0.15)), 4)]))]
        phi = np.full((H, W), lv[0])
        for _ in range(int(g.integers(0, 4))):
            y0, x0 = int(g.integers(0, H)), int(g.integers(0, W))
            phi[y0:y0 + int(g.integers(1, H + 1)), x0:x0 + int(g.integers(1, W + 1))] = lv[1]
        phis.append(phi.astype(dt))
        inits.append((noise_plane(H, W, 0, seed=seed * 7 + b, dtype=dt),
                      noise_plane(H, W, 1, seed=seed * 7 + b, dtype=dt)))
        ev = []
        for _ in range(int(g.integers(0, 6))):
            kind = g.choice(["disc", "rect", "half_disc"])
            if kind == "rect":
                y0, x0 = int(g.integers(-2, H)), int(g.integers(-2, W))
                s = {"kind": "rect", "y0": y0, "x0": x0, "y1": y0 + int(g.integers(1, 20)),
                     "x1": x0 + int(g.integers(1, 20))}
            else:
                s = {"kind": kind, "cy2": int(g.integers(-4, 2 * H + 4)), "cx2": int(g.integers(-4, 2 * W + 4)),
                     "r": int(g.integers(1, 9))}
                if kind == "half_disc":
                    s["dir"] = int(g.integers(0, 4))
            if g.random() < 0.3:
                s["mask_phi"] = lv[int(g.integers(0, 2))]
            ev.append((s, float(g.choice([1.0, 0.5])), int(g.integers(0, steps))))
        evs.append(ev)
        pr = []
        for _ in range(int(g.integers(0, 3))):
            y0, x0 = int(g.integers(0, H)), int(g.integers(0, W))
            pr.append(((y0, x0, min(H, y0 + int(g.integers(1, 8))), min(W, x0 + int(g.integers(1, 8)))),
                       float(g.choice([0.05, 0.1, 0.3])), int(g.integers(1, 12))))
        prs.append(pr)
        if g.random() < 0.3:
            params.append(dict(eps=float(g.choice([0.0243, 0.03, 0.05])), f=float(g.choice([1.4, 1.0, 2.0])),
                               q=float(g.choice([0.002, 0.001, 0.005])), Du=0.45, dt=0.001,
                               dx=float(g.choice([0.25, 0.25, 0.3]))))
        else:
            params.append(None)
    splits, left = [], steps
    while left:
        n = int(g.integers(1, left + 1))
        splits.append(n)
        left -= n
    return dict(dt=dt, B=B, H=H, W=W, steps=steps, phis=phis, inits=inits, evs=evs, prs=prs, params=params,
                tb=int(g.integers(0, 9)), kernel=str(g.choice(["auto", "tb", "lp", "cr", "gz"])),
                tl=int(g.choice([0, 0, 1, 5, 13])), splits=splits)


@pytest.mark.parametrize("seed", range(N_CASES))
def test_randomized_parity(seed, monkeypatch):
    c = _case(seed)
    monkeypatch.setenv("RD_KERNEL", c["kernel"])
    monkeypatch.setenv("RD_GZ_K", str(1 + seed % 12))  # gz_kernel: steps per border exchange
    dt = c["dt"]
    sim = rd.Sim(np.stack(c["phis"]), dtype=dt, tb_depth=c["tb"])
    try:
        for b in range(c["B"]):
            if c["params"][b] is not None:
                p = rd.rd_params_default()
                for k_, v_ in c["params"][b].items():
                    setattr(p, k_, v_)
                sim.set_params(b, p)
            sim.write(b, *c["inits"][b])
            for s, val, at in c["evs"][b]:
                sim.stimulate(s, val, at, b=b)
        pids = [[sim.probe_latch(b, r, t, st) for (r, t, st) in c["prs"][b]] for b in range(c["B"])]
        if c["tl"]:
            sim.timelapse(c["tl"])
        err = None
        try:
            for n in c["splits"]:
                sim.step(n)
        except rd.RDError as e:
            assert e.code == rd.RD_ENONFINITE, e
            err = e
        refs = []
        for b in range(c["B"]):
            prm = oracle.Params(**c["params"][b]) if c["params"][b] is not None else oracle.Params()
            refs.append(oracle.run(*c["inits"][b], c["phis"][b], c["steps"], events=c["evs"][b], probes=c["prs"][b],
                                   params=prm, timelapse_stride=c["tl"]))
        if err is not None or any(r.status != 0 for r in refs):
            # the first fault over the batch: same step, instance and cell
            assert err is not None and any(r.status != 0 for r in refs), "fault on one side only"
            st, fb, fi, fj = sim.fault()
            first = min((r.fault[0], b, r.fault[1], r.fault[2]) for b, r in enumerate(refs) if r.status != 0)
            assert (st, fb, fi, fj) == first
            return
        for b in range(c["B"]):
            u, v = sim.read(b)
            assert np.array_equal(u, refs[b].u), f"u b={b} {c['kernel']} tb={c['tb']}"
            assert np.array_equal(v, refs[b].v), f"v b={b}"
            assert [sim.probe_result(p) for p in pids[b]] == refs[b].first_fire, f"probes b={b}"
            if c["tl"]:
                assert np.array_equal(sim.read_timelapse(b), refs[b].max_u), f"timelapse b={b}"
    finally:
        sim.close()
