"""Multi-rank row-slab decomposition on CPU (gloo, world sizes 2 and 3).

Each rank keeps its slab plus ghost rows as numpy arrays, advances them with
the oracle (test infrastructure standing in for the per-rank GPU kernel) for
k <= halo steps, and refreshes its ghosts with the PRODUCT's exchange logic
(paper_1901_06535_b200.dist: slab_rows, ghost_extent, exchange_plan,
exchange over torch.distributed). The assembled owned rows must equal the
single-grid oracle run bitwise: this pins the partition, the exchange
plan (which rows go to which peer) and the global-coordinate event handling.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1901_06535_b200.dist import exchange_plan, ghost_extent, slab_rows
from slab_protocol import exchange
from rdinputs import half_discs, noise_plane

H, W, STEPS = 37, 53, 23


def _shift(shape, lo):
    s = dict(shape)
    if s["kind"] == "rect":
        s["y0"] -= lo
        s["y1"] -= lo
    else:
        s["cy2"] -= 2 * lo
    return s


def _events():
    ev = [(s, 1.0, 0) for s in half_discs(H, W, 5, seed=4)]
    ev.append(({"kind": "rect", "y0": 10, "x0": 2, "y1": 27, "x1": 9}, 1.0, 7))
    ev.append(({"kind": "disc", "cy2": 2 * 18, "cx2": 2 * 30, "r": 4}, 0.8, 11))
    return ev


def _phi():
    p = np.full((H, W), 0.054)
    p[5:20, 20:40] = 0.0975
    return p


def _worker(rank, world, port, halo, dtype, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        row0, rows = slab_rows(H, world, rank)
        lo, hi = ghost_extent(H, row0, rows, halo)
        u = noise_plane(hi - lo, W, 0, seed=3, dtype=dtype, row0=lo)
        v = noise_plane(hi - lo, W, 1, seed=3, dtype=dtype, row0=lo)
        phi = _phi()[lo:hi].astype(dtype)
        ev = [(_shift(s, lo), val, at) for (s, val, at) in _events()]
        off = row0 - lo  # array index of local row 0
        plan = exchange_plan(world, rank, rows, halo)
        done = 0
        while done < STEPS:
            k = min(halo, STEPS - done)
            # product exchange on CPU tensors viewing the numpy slab
            tu, tv = torch.from_numpy(u), torch.from_numpy(v)
            ops = []
            for peer, (s0, s1), (r0, r1) in plan:
                ops.append((peer, [tu[off + s0:off + s1].contiguous(), tv[off + s0:off + s1].contiguous()],
                            [tu[off + r0:off + r1], tv[off + r0:off + r1]]))
            recv_bufs = [(peer, sends, [torch.empty_like(r) for r in recvs], recvs) for peer, sends, recvs in ops]
            exchange([(p, s, rb) for p, s, rb, _ in recv_bufs])
            for _, _, rb, dst in recv_bufs:
                for a, b in zip(rb, dst):
                    b.copy_(a)
            r = oracle.run(u, v, phi, k, events=ev, step0=done)
            u, v = r.u, r.v
            done += k
        owned = (u[off:off + rows].copy(), v[off:off + rows].copy())
        q.put((rank, row0, owned))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,halo", [(2, 1), (2, 4), (3, 3)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
def test_slab_exchange_equals_single_grid(world, halo, dtype):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, halo, dtype, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    u0 = noise_plane(H, W, 0, seed=3, dtype=dtype)
    v0 = noise_plane(H, W, 1, seed=3, dtype=dtype)
    ref = oracle.run(u0, v0, _phi().astype(dtype), STEPS, events=_events())
    U = np.empty_like(ref.u)
    V = np.empty_like(ref.v)
    for rank, row0, (u, v) in parts:
        U[row0:row0 + u.shape[0]] = u
        V[row0:row0 + v.shape[0]] = v
    assert np.array_equal(U, ref.u) and np.array_equal(V, ref.v)


def test_partition_covers_grid():
    for Hh in (7, 64, 65536):
        for G in (1, 2, 3, 8):
            rows = [slab_rows(Hh, G, r) for r in range(G)]
            assert rows[0][0] == 0 and sum(n for _, n in rows) == Hh
            for (a, n), (b, _) in zip(rows, rows[1:]):
                assert a + n == b


def test_sweep_shard_round_robin_covers_every_instance():
    """batched instances are replicas, spread round-robin;
    every instance runs on exactly one rank, loads differ by at most one."""
    from paper_1901_06535_b200.sweep import shard
    for n in (0, 1, 5, 8, 33):
        for world in (1, 2, 3, 8):
            parts = [shard(n, world, r) for r in range(world)]
            flat = sorted(i for p in parts for i in p)
            assert flat == list(range(n))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
