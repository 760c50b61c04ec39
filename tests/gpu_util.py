"""Helpers for the -m gpu parity tests: run a Workload through the C ABI and
through the oracle on the same seeded inputs."""
from __future__ import annotations

import numpy as np

import oracle
import paper_1901_06535_b200 as rd


def gpu_run(w, steps=None, tb_depth=0, splits=None, flags=0, init=True, probes=True, batch=None):
    """Run workload w on the GPU; returns (u[B], v[B], first_fire per instance, sim stats)."""
    steps = w.steps if steps is None else steps
    bs = list(range(w.B)) if batch is None else list(batch)
    phi = np.stack([w.phi_plane(b).astype(w.dtype) for b in bs])
    sim = rd.Sim(phi, dtype=w.dtype, tb_depth=tb_depth, flags=flags)
    try:
        if init and w.init is not None:
            for k, b in enumerate(bs):
                u0, v0 = w.init_planes(b)
                sim.write(k, u0, v0)
        for k, b in enumerate(bs):
            for shape, value, at in (w.events[b] if w.events else []):
                sim.stimulate(shape, value, at, b=k)
        pids = []
        if probes and w.probes:
            for k, b in enumerate(bs):
                pids.append([sim.probe_latch(k, rect, thr, stride) for (rect, thr, stride) in w.probes[b]])
        for n in (splits or [steps]):
            sim.step(n)
        U, V = [], []
        for k in range(len(bs)):
            u, v = sim.read(k)
            U.append(u)
            V.append(v)
        fire = [[sim.probe_result(p) for p in ps] for ps in pids]
        return np.stack(U), np.stack(V), fire, sim.stats()
    finally:
        sim.close()


def oracle_run(w, b, steps=None, dtype=None, reaction_off=False):
    dt = w.dtype if dtype is None else dtype
    steps = w.steps if steps is None else steps
    u0, v0 = w.init_planes(b)
    r = oracle.run(u0.astype(dt), v0.astype(dt), w.phi_plane(b).astype(dt), steps,
                   events=w.events[b] if w.events else (), probes=w.probes[b] if w.probes else (),
                   reaction_off=reaction_off)
    return r


def assert_bitwise(a, b, what=""):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    if not np.array_equal(a, b, equal_nan=True):
        d = np.abs(a.astype(np.float64) - b.astype(np.float64))
        idx = np.unravel_index(np.nanargmax(d), d.shape)
        n = int(np.count_nonzero(a != b))
        raise AssertionError(f"{what}: {n} cells differ, max |diff| {np.nanmax(d):.3e} at {idx}")
