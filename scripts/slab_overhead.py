#!/usr/bin/env python
"""Kernel-side cost of the row-slab decomposition on one GPU (development
evidence for DESIGN.md §7; no NCCL involved).

A middle slab (rank 1 of 3: ghost rows on both sides) of bench.py's N > 1
workload (16384 rows x 16384 columns per rank, fp32) is stepped through
SlabSim's block protocol -- post exchange, rd_step_begin (interior rows),
wait, rd_step_finish (edge bands) -- with a transport whose exchange does
nothing, and compared with the N = 1 handle of the same size (one plain
launch per block). The ratio bounds the per-GPU efficiency of the N > 1
line from the kernel side: the split launches, the ghost rows, the host
protocol. The NCCL transfer itself (~0.5 MB per side per 4-step block) runs
on NCCL's stream beside the interior launch.

  python scripts/slab_overhead.py [--timesteps 1000] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1901_06535_b200 as rd  # noqa: E402
from paper_1901_06535_b200.dist import SlabSim  # noqa: E402


class NullTransport:
    """Virtual neighbours that never send: the exchange is a no-op."""

    def register(self, slab):
        pass

    def exchange(self, slab):
        pass


def timed(fn, T, reps):
    import torch
    fn(T)  # warm-up: graphs, clocks
    torch.cuda.synchronize()
    best = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn(T)
        torch.cuda.synchronize()
        best.append(time.perf_counter() - t0)
    return sorted(best)[len(best) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--timesteps", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    torch.cuda.init()
    n = 16384
    one = rd.Sim(None, shape=(1, n, n), dtype=np.float32)
    one.paint_phi(0.054)
    one.fill_noise(seed=1)
    t1 = timed(one.step, a.timesteps, a.reps)
    st1 = one.stats()
    one.close()
    slab = SlabSim(n, 3 * n, 1, 3, None, dtype=np.float32, halo=4, transport=NullTransport())
    rd.rd_paint_phi(slab.h, -1, None, 0.054)
    slab.fill_noise(seed=1)
    def slab_step(T):  # SlabSim.step without the cross-rank flag all-reduce (no process group here)
        rd.rd_checkpoint(slab.h)
        slab._step_exchange(T)
        rd.rd_read_flags(slab.h)

    ts = timed(slab_step, a.timesteps, a.reps)
    sts = slab.stats()
    slab.close()
    cells = n * n * a.timesteps
    print(json.dumps({
        "what": "middle row slab (rank 1 of 3, ghosts both sides) vs the N = 1 handle, 16384^2 fp32 per GPU, "
                "exchange replaced by a no-op (kernel-side cost of the decomposition)",
        "timesteps": a.timesteps,
        "n1_gcells": cells / t1 / 1e9, "slab_gcells": cells / ts / 1e9, "slab_over_n1": t1 / ts,
        "n1_launches": st1["launches"], "slab_launches": sts["launches"]}))


if __name__ == "__main__":
    main()
