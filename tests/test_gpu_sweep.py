"""f1: per-instance parameters and batched calibration sweeps on the GPU."""
import numpy as np
import pytest

import oracle
import paper_1901_06535_b200 as rd
from gpu_util import assert_bitwise
from paper_1901_06535_b200.sweep import Instance, bisect
from rdinputs import and_gate, noise_plane

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
def test_per_instance_params_match_oracle(dtype):
    """Three instances with different (eps, f, q, Du) in one batched handle:
    each equals the oracle run with its own parameters, bitwise."""
    H, W, n = 40, 70, 60
    sets = [dict(), dict(eps=0.03, f=1.2), dict(q=0.1, Du=0.3)]
    phi = np.full((3, H, W), 0.054, dtype=dtype)
    sim = rd.Sim(phi, dtype=dtype)
    u0 = noise_plane(H, W, 0, seed=5, dtype=dtype)
    v0 = noise_plane(H, W, 1, seed=5, dtype=dtype)
    for b, kw in enumerate(sets):
        p = rd.rd_params_default()
        for k, val in kw.items():
            setattr(p, k, val)
        sim.set_params(b, p)
        sim.write(b, u0, v0)
    sim.stimulate({"kind": "disc", "cy2": 40, "cx2": 70, "r": 5}, 1.0, 0)
    sim.step(n)
    for b, kw in enumerate(sets):
        ref = oracle.run(u0, v0, phi[b], n, events=[({"kind": "disc", "cy2": 40, "cx2": 70, "r": 5}, 1.0, 0)],
                         params=oracle.Params(**kw))
        u, v = sim.read(b)
        assert_bitwise(u, ref.u, f"u b={b}")
        assert_bitwise(v, ref.v, f"v b={b}")
    sim.close()


def test_and_gate_calibration_bisection_confirmed_by_oracle():
    """SPEC.md:268 calibration as a batched GPU sweep: bisect phi_passive for
    (i) a single input passing the gate's gap and (ii) two colliding inputs
    passing it. The gate works between the two thresholds; the shipped
    phi_p = 0.119 (R-11) lies inside, and the oracle confirms both
    brackets' end points."""
    steps = 20000

    def make(kind):
        def mk(x):
            g = and_gate(phi_passive=x)
            a, b = g["inputs"]
            ev = [(a, 1.0, 0)] if kind == "single" else [(a, 1.0, 0), (b, 1.0, 0)]
            return [Instance(g["phi"], ev, [(g["probe"], 0.1, 50)])]
        return mk

    fired = lambda fires: fires[0][0] >= 0  # noqa: E731
    single = bisect(make("single"), fired, 0.10, 0.13, steps, rounds=3, width=8)
    dual = bisect(make("dual"), fired, 0.10, 0.13, steps, rounds=3, width=8)
    assert single.hi <= 0.119 < dual.lo
    # the oracle (fp32 mode) agrees on the bracket end points of the dual sweep
    for x, expect in ((dual.lo, True), (dual.hi, False)):
        inst = make("dual")(x)[0]
        z = np.zeros(inst.phi.shape, np.float32)
        r = oracle.run(z, z, inst.phi.astype(np.float32), steps, events=inst.events, probes=inst.probes)
        assert (r.first_fire[0] >= 0) == expect
