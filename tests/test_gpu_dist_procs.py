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
        from slab_protocol import SlabSim
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


def _ipc_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_1901_06535_b200 as rd
        from slab_protocol import SlabSim
        H2, W2, halo = 64, 100, 4
        sl = SlabSim(W2, H2, rank, world, lambda b, r0, n: np.full((n, W2), 0.054), dtype=np.float32, halo=halo,
                     p2p=True)  # maps the neighbour's plane allocation (CUDA IPC)
        sl.fill_noise(seed=6)
        torch.cuda.synchronize()
        dist.barrier()
        rd.rd_push_ghosts(sl.h)  # my send rows -> the neighbour's ghost rows, through the mapping
        for f in sl.peer_flags.values():
            rd.rd_stream_signal(sl.h, f, 41 + rank)  # into the neighbour's flag word
        torch.cuda.synchronize()
        dist.barrier()  # the hosts order the two processes: no GPU work waits on the other
        from slab_protocol import _DevRows, _dev_rows
        r0 = -halo if rank == 1 else sl.rows
        ghost = _dev_rows(sl.h, 0, 0, r0, r0 + halo).cpu().numpy()  # row storage, ghost columns included
        rows = ghost.view(np.float32).reshape(halo, -1)
        side = 0 if rank == 1 else 1
        flag = torch.as_tensor(_DevRows(rd.rd_flag_ptr(sl.h, side), 4), device="cuda").cpu().numpy()
        q.put((rank, sl.row0 + r0, rows, int(flag.view(np.uint32)[0])))
        dist.barrier()
        sl.close()
    finally:
        dist.destroy_process_group()


def test_two_process_ipc_push_lands_in_ghost_rows():
    """The peer-memory exchange's cross-process plumbing on one GPU, with the
    hosts ordering the ranks (no GPU work waits on the other process): each
    rank maps the other's plane allocation by CUDA IPC (SlabSim(p2p=True)),
    rd_push_ghosts stores its send rows through the mapping and
    rd_stream_signal writes the neighbour's flag word. Each rank's ghost
    rows then hold exactly the neighbour's rows (seeded noise in global
    coordinates), mirrored columns included, and its flag word the value."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    W2, halo = 100, 4
    for rank, grow, rows, flag in got:
        want = noise_plane(halo, W2, 0, seed=6, dtype=np.float32, row0=grow)
        col0 = 8  # the row storage starts 8 mirrored columns left of column 0
        assert_bitwise(rows[:, col0:col0 + W2], want, f"ghost rows of rank {rank}")
        assert np.array_equal(rows[:, col0 - 1], want[:, 0]) and np.array_equal(rows[:, col0 + W2], want[:, -1])
        assert flag == 41 + (1 - rank)
