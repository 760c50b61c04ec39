"""The multi-process slab path end to end on ONE GPU: two real ranks
(torch.distributed, gloo backend with host-staged halo exchange, since NCCL
needs one GPU per rank) run SlabSim.step -- super-steps, exchanges from
rd_row_ptr row storage, OR-reduced flags -- and the assembled owned rows equal
the single-grid oracle bitwise. Kernels of the two processes never wait on
each other (the hosts synchronise), so sharing the device is safe."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from gpu_util import assert_bitwise
from rdinputs import half_discs, noise_plane

pytestmark = pytest.mark.gpu
H, W, STEPS = 90, 130, 37


def _phi(b, row0, rows):
    p = np.full((rows, W), 0.054)
    for r in range(rows):
        if 30 <= row0 + r < 50:
            p[r, 40:90] = 0.0975
    return p


def _events():
    return [(s, 1.0, 0) for s in half_discs(H, W, 6, seed=4)] + [
        ({"kind": "rect", "y0": 40, "x0": 3, "y1": 60, "x1": 8}, 1.0, 9)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1901_06535_b200.dist import SlabSim
        sl = SlabSim(W, H, rank, world, _phi, dtype=np.float32, halo=4)
        sl.fill_noise(seed=2)
        for s, val, at in _events():
            sl.stimulate(s, val, at)
        sl.step(STEPS)
        u, v = sl.read_owned(0)
        q.put((rank, sl.row0, u, v))
        sl.close()
    finally:
        dist.destroy_process_group()


def test_two_process_slabs_equal_single_grid():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    U = np.empty((H, W), np.float32)
    V = np.empty((H, W), np.float32)
    for _, row0, u, v in parts:
        U[row0:row0 + u.shape[0]] = u
        V[row0:row0 + v.shape[0]] = v
    ref = oracle.run(noise_plane(H, W, 0, seed=2), noise_plane(H, W, 1, seed=2), _phi(0, 0, H).astype(np.float32),
                     STEPS, events=_events())
    assert_bitwise(U, ref.u, "u")
    assert_bitwise(V, ref.v, "v")


def _sweep_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1901_06535_b200.sweep import Instance, run_batch
        from rdinputs import config
        w = config(2)
        inst = [Instance(w.phi_plane(b), w.events[b], w.probes[b]) for b in range(w.B)]
        q.put((rank, run_batch(inst, w.steps, group=dist.group.WORLD)))
    finally:
        dist.destroy_process_group()


def test_two_process_sweep_replicas_equal_one_process():
    """SURVEY.md §8(e) replicas: the AND-gate batch (config 2) spread over two
    ranks (round-robin, results all-gathered in instance order) gives the
    same first-fire steps on every rank as one process running the whole
    batch, and the paper's truth table 0001."""
    from paper_1901_06535_b200.sweep import Instance, run_batch
    from rdinputs import config
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_sweep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = config(2)
    one = run_batch([Instance(w.phi_plane(b), w.events[b], w.probes[b]) for b in range(w.B)], w.steps)
    for _, fires in got:
        assert fires == one
    assert [f[0] >= 0 for f in one] == w.expect["fires"]
