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


MAX_PARAM_SETS = 32  # rd_set_params: per-instance parameters need batch <= 32


def shard(n: int, world: int, rank: int) -> list[int]:
    """Instances of an n-instance batch that rank `rank` of `world` runs:
    round-robin (the batched mode is replicas only, no
    exchange between GPUs)."""
    return list(range(rank, n, world))


def _run_local(instances: list[Instance], steps: int, dtype, tb_depth: int) -> list:
    if not instances:
        return []
    # one handle per chunk; chunks only when per-instance parameters exceed
    # what one handle carries
    per = MAX_PARAM_SETS if any(i.params is not None for i in instances) else len(instances)
    out = []
    for c0 in range(0, len(instances), per):
        chunk = instances[c0:c0 + per]
        phi = np.stack([np.asarray(i.phi, dtype=dtype) for i in chunk])
        sim = Sim(phi, dtype=dtype, tb_depth=tb_depth)
        try:
            for b, inst in enumerate(chunk):
                if inst.params is not None:
                    sim.set_params(b, inst.params)
                for shape, value, at in inst.events:
                    sim.stimulate(shape, value, at, b=b)
            pids = [[sim.probe_latch(b, r, t, s) for (r, t, s) in inst.probes] for b, inst in enumerate(chunk)]
            sim.step(steps)
            out += [[sim.probe_result(p) for p in ps] for ps in pids]
        finally:
            sim.close()
    return out


def run_batch(instances: list[Instance], steps: int, dtype=np.float32, tb_depth: int = 0, group=None):
    """Run every instance for `steps` (batched handles); returns the list of
    first-fire steps (one list per instance, -1 = never).

    group: a torch.distributed process group (e.g. dist.group.WORLD) to spread
    the instances round-robin over its ranks (one GPU each); every rank
    returns the full list, in instance order. None: this process runs all."""
    if group is None:
        return _run_local(instances, steps, dtype, tb_depth)
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = shard(len(instances), world, rank)
    res = _run_local([instances[i] for i in mine], steps, dtype, tb_depth)
    gathered = [None] * world
    dist.all_gather_object(gathered, (mine, res), group=group)
    out = [None] * len(instances)
    for idx, rs in gathered:
        for i, r in zip(idx, rs):
            out[i] = r
    return out


@dataclass
class Bracket:
    lo: float           # largest value where the predicate held
    hi: float           # smallest value where it failed
    evaluations: list = field(default_factory=list)  # (x, outcome) pairs, all rounds


def bisect(make: Callable[[float], list[Instance]], predicate: Callable[[list], bool], lo: float, hi: float,
           steps: int, rounds: int = 4, width: int = 8, dtype=np.float32, group=None) -> Bracket:
    """Find the threshold of a predicate that holds at `lo` and fails at `hi`
    (monotone in x). make(x) returns the instance(s) evaluating point x;
    predicate(first_fire_lists_of_those_instances) -> bool. Each round runs
    `width` interior points in ONE batched launch and keeps the sub-interval
    where the predicate flips (width+1 fold narrowing per round). With a
    process group the points of a round are spread over its ranks."""
    br = Bracket(lo, hi)
    for _ in range(rounds):
        xs = [br.lo + (br.hi - br.lo) * (k + 1) / (width + 1) for k in range(width)]
        groups = [make(x) for x in xs]
        flat = [i for g in groups for i in g]
        fires = run_batch(flat, steps, dtype=dtype, group=group)
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
