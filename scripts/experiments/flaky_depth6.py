"""Repeat config 4 at full length (10000 steps) at several depths / variants and
compare every run with a depth-4 reference bitwise: hunts a one-off mismatch
seen once in test_config4_full_length_properties (auto depth 6 vs depth 1)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from gpu_util import gpu_run  # noqa: E402
from rdinputs import config  # noqa: E402

w = config(4)


def run(k, env=None):
    for kk, vv in (env or {}).items():
        os.environ[kk] = vv
    U, V, _, st = gpu_run(w, tb_depth=k)
    for kk in (env or {}):
        os.environ.pop(kk)
    return U, V


ref_u, ref_v = run(4)
plan = [("K6", 6, None)] * int(sys.argv[1]) + [("K6 full-variant", 6, {"RD_TB_VARIANT": "full"})] * int(sys.argv[2]) + \
       [("K1", 1, None)] * int(sys.argv[3])
bad = 0
for i, (tag, k, env) in enumerate(plan):
    U, V = run(k, env)
    d = np.argwhere((U != ref_u) | (V != ref_v))
    if len(d):
        bad += 1
        print("DIFF", i, tag, len(d), "cells; rows", d[:, 1].min(), d[:, 1].max(), "cols", d[:, 2].min(), d[:, 2].max(),
              flush=True)
print("runs", len(plan), "mismatching", bad, flush=True)
