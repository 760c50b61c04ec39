"""Batched parameter / geometry sweeps.

The paper's circuits were hand-drawn; SPEC.md:268 fixes their
dimensions by "a documented calibration sweep (gap length swept until
single-input decays and dual-input passes)". That sweep is hundreds of
400x300 x 20000-step runs: here every round of a bisection is ONE batched
rd_step over `width` candidate values (each instance its own phi map, or its
own Eq.-1 parameters via rd_set_params), so the search is a handful of GPU
launches sequences instead of hundreds of serial runs.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import Sim


@dataclass
class Instance:
    """One sweep point: phi map (H, W), stimuli [(shape, value, at_step)],
    probes [(rect, threshold, stride)], optional Eq.-1 parameter set."""
    phi: np.ndarray
    events: list
    probes: list
    params: object | None = None


def run_batch(instances: list[Instance], steps: int, dtype=np.float32, tb_depth: int = 0):
    """Run every instance for `steps` in one batched handle; returns the list
    of first-fire steps (one list per instance, -1 = never)."""
    phi = np.stack([np.asarray(i.phi, dtype=dtype) for i in instances])
    sim = Sim(phi, dtype=dtype, tb_depth=tb_depth)
    try:
        for b, inst in enumerate(instances):
            if inst.params is not None:
                sim.set_params(b, inst.params)
            for shape, value, at in inst.events:
                sim.stimulate(shape, value, at, b=b)
        pids = [[sim.probe_latch(b, r, t, s) for (r, t, s) in inst.probes] for b, inst in enumerate(instances)]
        sim.step(steps)
        return [[sim.probe_result(p) for p in ps] for ps in pids]
    finally:
        sim.close()


@dataclass
class Bracket:
    lo: float           # largest value where the predicate held
    hi: float           # smallest value where it failed
    evaluations: list = field(default_factory=list)  # (x, outcome) pairs, all rounds


def bisect(make: Callable[[float], list[Instance]], predicate: Callable[[list], bool], lo: float, hi: float,
           steps: int, rounds: int = 4, width: int = 8, dtype=np.float32) -> Bracket:
    """Find the threshold of a predicate that holds at `lo` and fails at `hi`
    (monotone in x). make(x) returns the instance(s) evaluating point x;
    predicate(first_fire_lists_of_those_instances) -> bool. Each round runs
    `width` interior points in ONE batched launch and keeps the sub-interval
    where the predicate flips (width+1 fold narrowing per round)."""
    br = Bracket(lo, hi)
    for _ in range(rounds):
        xs = [br.lo + (br.hi - br.lo) * (k + 1) / (width + 1) for k in range(width)]
        groups = [make(x) for x in xs]
        flat = [i for g in groups for i in g]
        fires = run_batch(flat, steps, dtype=dtype)
        outcomes, at = [], 0
        for g in groups:
            outcomes.append(predicate(fires[at:at + len(g)]))
            at += len(g)
        br.evaluations.extend(zip(xs, outcomes))
        new_lo, new_hi = br.lo, br.hi
        for x, ok in zip(xs, outcomes):
            if ok:
                new_lo = max(new_lo, x)
        for x, ok in zip(xs, outcomes):
            if not ok and x > new_lo:
                new_hi = min(new_hi, x)
        br.lo, br.hi = new_lo, new_hi
    return br
