"""rd_create_dist between PROCESSES on one GPU (rd_dist_shm_id): the ranks'
arenas are mapped into each other by CUDA IPC, halos travel by copy-engine
cudaMemcpyAsync into the neighbour's ghost rows, and the grant / landed
counters are cuStreamWriteValue32 into the mapped arena and
cuStreamWaitValue32 on the rank's own words -- the code path `bench.py --gpus
N` runs with one process per GPU, which NCCL cannot host on a single device.
The control plane is the shared-memory group instead of NCCL. Assembled owned
rows equal the single-grid oracle bitwise."""
import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from gpu_util import assert_bitwise
from rdinputs import half_discs, noise_plane

pytestmark = pytest.mark.gpu
H, W = 90, 130


def _phi(b, row0, rows):
    p = np.full((rows, W), 0.054)
    for r in range(rows):
        if 30 <= row0 + r < 50:
            p[r, 40:90] = 0.0975
    return p


def _events():
    return [(s, 1.0, 0) for s in half_discs(H, W, 6, seed=4)] + [
        ({"kind": "rect", "y0": 40, "x0": 3, "y1": 60, "x1": 8}, 1.0, 9)]


def _worker(rank, world, uid, dtype, depth, steps, q):
    try:
        import torch
        torch.cuda.set_device(0)
        from paper_1901_06535_b200.dist import DistSim
        sl = DistSim(W, H, rank, world, _phi, uid=uid, dtype=dtype, tb_depth=depth)
        sl.fill_noise(seed=2)
        for s, val, at in _events():
            sl.stimulate(s, val, at)
        pid = sl.probe_latch(0, (40, 20, 60, 30), 0.1, 5)
        for n in steps:
            sl.step(n)
        fired = sl.probe_result(pid)
        u, v = sl.read_owned(0)
        q.put((rank, sl.row0, u, v, sl.geometry(), fired))
        sl.close()
    except Exception as e:  # noqa: BLE001 - reported to the parent
        q.put((rank, repr(e)))
        raise


def _run(world, dtype, depth, steps):
    from paper_1901_06535_b200.dist import shm_id
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    uid = shm_id()
    procs = [ctx.Process(target=_worker, args=(r, world, uid, dtype, depth, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        parts = [q.get(timeout=240) for _ in range(world)]
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for part in parts:
        assert len(part) == 6, f"rank {part[0]} failed: {part[1]}"
    for p in procs:
        assert p.exitcode == 0
    return parts


@pytest.mark.parametrize("world,depth", [(2, 4), (3, 2), (2, 1)])
@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
def test_process_ranks_equal_oracle(world, depth, dtype):
    steps = [17, 20]
    parts = _run(world, dtype, depth, steps)
    U = np.empty((H, W), dtype)
    V = np.empty((H, W), dtype)
    for _, row0, u, v, geo, _ in parts:
        U[row0:row0 + u.shape[0]] = u
        V[row0:row0 + v.shape[0]] = v
        assert geo["transport"] == "p2p" and geo["flag_selftest"] == 1 and geo["world"] == world
        assert geo["exchanges"] >= sum(steps) // depth
    ref = oracle.run(noise_plane(H, W, 0, seed=2, dtype=dtype), noise_plane(H, W, 1, seed=2, dtype=dtype),
                     _phi(0, 0, H).astype(dtype), sum(steps), events=_events(),
                     probes=[((40, 20, 60, 30), 0.1, 5)])
    assert_bitwise(U, ref.u, "u")
    assert_bitwise(V, ref.v, "v")
    assert {p[5] for p in parts} == {ref.first_fire[0]}


def _fault_worker(rank, world, uid, steps, q):
    try:
        import torch
        torch.cuda.set_device(0)
        import paper_1901_06535_b200 as rd
        from paper_1901_06535_b200.dist import DistSim
        dtype = np.float32
        s = DistSim(128, 96, rank, world, lambda b, r0, n: np.full((n, 128), 0.2, dtype), uid=uid, dtype=dtype)
        s.write(0, lambda b, r0, n: noise_plane(n, 128, 0, seed=7, dtype=dtype, row0=r0),
                lambda b, r0, n: noise_plane(n, 128, 1, seed=7, dtype=dtype, row0=r0))
        s.stimulate(_FAULT_SHAPE, 1.0, 0)
        code = 0
        try:
            s.step(steps)
        except rd.RDError as e:
            code = e.code
        q.put((rank, s.row0, s.read_owned(0)[0], code, tuple(rd.rd_get_fault(s.h)), rd.rd_get_step(s.h)))
        s.close()
    except Exception as e:  # noqa: BLE001 - reported to the parent
        q.put((rank, repr(e)))
        raise


_FAULT_SHAPE = {"kind": "half_disc", "cy2": 2 * 31, "cx2": 128, "r": 8, "dir": 1}  # straddles the rank 0/1 edge


def test_process_ranks_fault_replay_stops_at_oracle_step():
    """The collective PRECISE replay between processes: an unmasked stimulus
    in a phi = 0.2 medium on noisy fields diverges; every rank process
    restores, replays step by step (one exchange and one shared-memory
    reduction per step) and stops at the oracle's step and global first cell
    with the oracle's field."""
    from paper_1901_06535_b200.dist import shm_id
    import paper_1901_06535_b200 as rd
    H, W, steps, world = 96, 128, 400, 3
    dtype = np.float32
    ref = oracle.run(noise_plane(H, W, 0, seed=7, dtype=dtype), noise_plane(H, W, 1, seed=7, dtype=dtype),
                     np.full((H, W), 0.2, dtype), steps, events=[(_FAULT_SHAPE, 1.0, 0)])
    assert ref.status == -4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    uid = shm_id()
    procs = [ctx.Process(target=_fault_worker, args=(r, world, uid, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        parts = [q.get(timeout=240) for _ in range(world)]
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for part in parts:
        assert len(part) == 6, f"rank {part[0]} failed: {part[1]}"
    parts.sort(key=lambda x: x[1])
    for _, _, _, code, fault, step in parts:
        assert code == rd.RD_ENONFINITE
        assert (fault[0], fault[2], fault[3]) == ref.fault and step == ref.fault[0]
    assert_bitwise(np.concatenate([p[2] for p in parts]), ref.u, "u at fault")


def test_missing_rank_fails_the_group_instead_of_hanging(monkeypatch):
    """A rank whose peers never arrive gives up after RD_DIST_TIMEOUT_S with
    RD_ENCCL (and marks the group failed, so late arrivals fail at once)."""
    import time
    import paper_1901_06535_b200 as rd
    from paper_1901_06535_b200.dist import shm_id
    monkeypatch.setenv("RD_DIST_TIMEOUT_S", "1.5")
    uid = shm_id()
    t = time.perf_counter()
    with pytest.raises(rd.RDError) as e:
        rd.rd_create_dist(64, 64, None, 0, 2, uid)
    assert e.value.code == rd.RD_ENCCL and 1.0 < time.perf_counter() - t < 30
    t = time.perf_counter()
    with pytest.raises(rd.RDError) as e:
        rd.rd_create_dist(64, 64, None, 1, 2, uid)  # the late rank: the segment is marked failed
    assert e.value.code == rd.RD_ENCCL and time.perf_counter() - t < 10
    with pytest.raises(rd.RDError) as e:
        rd.rd_create_dist(64, 64, None, 0, 2, uid)  # every rank has been and gone: the segment's name is unlinked
    assert e.value.code == rd.RD_EINVAL
