#!/usr/bin/env python
"""f1 demo/measurement: calibrate the AND gate's phi_passive window with
batched GPU bisection and report the brackets and wall time."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1901_06535_b200.sweep import Instance, bisect  # noqa: E402
from rdinputs import and_gate  # noqa: E402


def make(kind):
    def mk(x):
        g = and_gate(phi_passive=x)
        a, b = g["inputs"]
        ev = [(a, 1.0, 0)] if kind == "single" else [(a, 1.0, 0), (b, 1.0, 0)]
        return [Instance(g["phi"], ev, [(g["probe"], 0.1, 50)])]
    return mk


out = {}
for kind in ("single", "dual"):
    t = time.perf_counter()
    br = bisect(make(kind), lambda f: f[0][0] >= 0, 0.10, 0.13, 20000, rounds=4, width=16)
    out[kind] = {"pass_up_to": br.lo, "blocked_from": br.hi, "seconds": time.perf_counter() - t,
                 "instances_per_round": 16, "rounds": 4, "steps": 20000}
print(json.dumps({"and_gate_phi_passive_window": out,
                  "gate_works_for": [out["single"]["blocked_from"], out["dual"]["pass_up_to"]]}))
