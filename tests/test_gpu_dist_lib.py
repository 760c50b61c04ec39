"""rd_create_dist: the multi-GPU row-slab path run INSIDE librd (SURVEY.md
§8(b) rd_dist_unique_id / rd_create_dist, §8(e)).

On one GPU the ranks are host threads of this process sharing an in-process
rendezvous id (rd_dist_local_id): every rank's kernels run on the one device,
its halo rows travel by cudaMemcpyAsync straight into the neighbours' ghost
rows, ordered by stream-ordered counters (no kernel ever waits on another
rank). The assembled owned rows must equal the oracle on the whole grid
bitwise, at any rank count and depth, through stimuli straddling slab edges,
probes, timelapse-free multi-call stepping and the fault replay. A world = 1
handle over a real NCCL communicator (rd_dist_unique_id) covers the NCCL
rendezvous and all-reduce on one GPU.
"""
import threading

import numpy as np
import pytest

import oracle
import paper_1901_06535_b200 as rd
from gpu_util import assert_bitwise
from paper_1901_06535_b200.dist import DistSim, local_id
from rdinputs import half_discs, noise_plane, obstacles

pytestmark = pytest.mark.gpu


def run_ranks(world, fn, timeout=180):
    """fn(rank) on `world` daemon threads (one rank each); re-raise the first
    error. A rank blocked in a collective cannot hang the test process."""
    out, errs = [None] * world, []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001 -- surfaced below
            errs.append((r, e))

    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    assert not any(t.is_alive() for t in ts), "a rank did not finish (collective mismatch?)"
    if errs:
        raise errs[0][1]
    return out


def _inputs(H, W, dtype, seed=1):
    rects = obstacles(H, W, 6, seed=3)

    def phi_fn(b, row0, rows):
        p = np.full((rows, W), 0.054)
        for (y0, x0, y1, x1) in rects:
            a, c = max(y0, row0), min(y1, row0 + rows)
            if a < c:
                p[a - row0:c - row0, x0:x1] = 0.2
        return p.astype(dtype)

    def u_fn(b, row0, rows):
        return noise_plane(rows, W, 0, seed=seed, dtype=dtype, row0=row0)

    def v_fn(b, row0, rows):
        return noise_plane(rows, W, 1, seed=seed, dtype=dtype, row0=row0)

    return phi_fn, u_fn, v_fn


@pytest.mark.parametrize("G,depth", [(1, 4), (2, 1), (2, 4), (3, 4), (4, 8), (3, 3)])
@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
def test_dist_ranks_equal_oracle(G, depth, dtype):
    H, W = 203, 300
    phi_fn, u_fn, v_fn = _inputs(H, W, dtype)
    shapes = half_discs(H, W, 12, seed=2, mask_phi=0.054)
    late = {"kind": "rect", "y0": 60, "x0": 10, "y1": 150, "x1": 14}  # spans every slab edge, due mid-block
    probe = (96, 200, 110, 230)
    uid = local_id()

    def rank(r):
        s = DistSim(W, H, r, G, phi_fn, uid=uid, dtype=dtype, tb_depth=depth)
        try:
            s.write(0, u_fn, v_fn)
            for sh in shapes:
                s.stimulate(sh, 1.0, 0)
            s.stimulate(late, 1.0, 5)
            pid = s.probe_latch(0, probe, 0.1, 7)
            for n in (17, 20):
                s.step(n)
            u, v = s.read_owned(0)
            geo = s.geometry()
            fired = s.probe_result(pid)
            m = s.probe(0, probe, 0.1)[1]
            return s.row0, u, v, geo, fired, m
        finally:
            s.close()

    res = run_ranks(G, rank)
    U = np.concatenate([x[1] for x in sorted(res, key=lambda x: x[0])])
    V = np.concatenate([x[2] for x in sorted(res, key=lambda x: x[0])])
    ev = [(sh, 1.0, 0) for sh in shapes] + [(late, 1.0, 5)]
    ref = oracle.run(u_fn(0, 0, H), v_fn(0, 0, H), phi_fn(0, 0, H), 37, events=ev, probes=[(probe, 0.1, 7)])
    assert_bitwise(U, ref.u, "u")
    assert_bitwise(V, ref.v, "v")
    for row0, _, _, geo, fired, m in res:
        assert geo["world"] == G and geo["halo"] == depth
        assert geo["transport"] == "local"
        if G > 1:
            assert geo["exchanges"] >= -(-37 // depth)  # one exchange per block at least
        assert fired == ref.first_fire[0]  # collective: the same on every rank
        assert m == oracle.probe_max(ref.u, probe)


def test_dist_fault_replay_stops_every_rank_at_oracle_step():
    """An unmasked stimulus inside a phi = 0.2 obstacle on noisy u, v diverges;
    every rank restores, replays step by step with an exchange per step and
    stops at the oracle's failing step, naming the oracle's first cell in
    global coordinates, with the oracle's fields at that step."""
    H, W, steps, G = 96, 128, 400, 3
    dtype = np.float32

    def phi_fn(b, row0, rows):
        return np.full((rows, W), 0.2, dtype)

    def u_fn(b, row0, rows):
        return noise_plane(rows, W, 0, seed=7, dtype=dtype, row0=row0)

    def v_fn(b, row0, rows):
        return noise_plane(rows, W, 1, seed=7, dtype=dtype, row0=row0)

    shape = {"kind": "half_disc", "cy2": 2 * 31, "cx2": 128, "r": 8, "dir": 1}  # straddles the rank 0/1 edge
    ref = oracle.run(u_fn(0, 0, H), v_fn(0, 0, H), phi_fn(0, 0, H), steps, events=[(shape, 1.0, 0)],
                     probes=[((0, 0, H, W), 0.5, 10)])
    assert ref.status == -4
    uid = local_id()

    def rank(r):
        s = DistSim(W, H, r, G, phi_fn, uid=uid, dtype=dtype)
        try:
            s.write(0, u_fn, v_fn)
            s.stimulate(shape, 1.0, 0)
            pid = s.probe_latch(0, (0, 0, H, W), 0.5, 10)
            with pytest.raises(rd.RDError) as e:
                s.step(steps)
            assert e.value.code == rd.RD_ENONFINITE
            return s.row0, s.read_owned(0)[0], rd.rd_get_fault(s.h), rd.rd_get_step(s.h), s.probe_result(pid)
        finally:
            s.close()

    res = sorted(run_ranks(G, rank), key=lambda x: x[0])
    U = np.concatenate([x[1] for x in res])
    for _, _, fault, step, fired in res:
        assert (fault[0], fault[2], fault[3]) == ref.fault
        assert step == ref.fault[0]
        assert fired == ref.first_fire[0]  # the failing step is not sampled (oracle order)
    assert_bitwise(U, ref.u, "u at fault")


def test_dist_world1_nccl_equals_oracle():
    """world = 1 over a real NCCL communicator: rd_dist_unique_id,
    ncclCommInitRank, the flag all-reduce of every rd_step."""
    H, W, dtype = 131, 257, np.float64
    phi_fn, u_fn, v_fn = _inputs(H, W, dtype, seed=5)
    s = DistSim(W, H, 0, 1, phi_fn, uid=rd.rd_dist_unique_id(), dtype=dtype)
    try:
        s.write(0, u_fn, v_fn)
        s.stimulate({"kind": "disc", "cy2": H, "cx2": W, "r": 5}, 1.0, 3)
        s.step(10)
        s.step(21)
        u, v = s.read_owned(0)
        assert s.geometry()["world"] == 1
    finally:
        s.close()
    ref = oracle.run(u_fn(0, 0, H), v_fn(0, 0, H), phi_fn(0, 0, H), 31,
                     events=[({"kind": "disc", "cy2": H, "cx2": W, "r": 5}, 1.0, 3)])
    assert_bitwise(u, ref.u, "u")
    assert_bitwise(v, ref.v, "v")


def test_dist_control_state_must_agree():
    """Stimuli are collective: a stimulus given to one rank only changes that
    rank's launch sequence; rd_step detects the digest mismatch on every rank."""
    H, W, G = 64, 96, 2
    uid = local_id()

    def rank(r):
        s = DistSim(W, H, r, G, lambda b, r0, n: np.full((n, W), 0.054, np.float32), uid=uid)
        try:
            if r == 1:
                s.stimulate({"kind": "rect", "y0": 40, "x0": 3, "y1": 50, "x1": 9}, 1.0, 2)
            with pytest.raises(rd.RDError) as e:
                s.step(8)
            return e.value.code
        finally:
            s.close()

    assert run_ranks(G, rank) == [rd.RD_EINVAL] * G


def test_dist_refuses_low_level_slab_calls():
    H, W = 32, 40
    s = DistSim(W, H, 0, 1, None, uid=local_id())
    try:
        for call in (lambda: rd.rd_step_unchecked(s.h, 1), lambda: rd.rd_checkpoint(s.h),
                     lambda: rd.rd_step_begin(s.h, 1)):
            with pytest.raises(rd.RDError) as e:
                call()
            assert e.value.code == rd.RD_EINVAL
    finally:
        s.close()


def test_device_arena_handle_equals_oracle():
    """rd_create_device over a torch-allocated arena, phi from a torch CUDA
    tensor; zero-copy views of u and phi through rd_field_ptr."""
    import torch
    H, W, dtype = 77, 130, np.float32
    phi_fn, u_fn, v_fn = _inputs(H, W, dtype, seed=9)
    nbytes = rd.rd_arena_bytes(W, H, dtype=dtype)
    arena = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    phi_t = torch.from_numpy(phi_fn(0, 0, H)).cuda()
    h = rd.rd_create_device(W, H, arena.data_ptr(), nbytes, phi_t.data_ptr(), dtype=dtype)
    try:
        rd.rd_write_fields(h, 0, u_fn(0, 0, H), v_fn(0, 0, H))
        rd.rd_stimulate(h, -1, {"kind": "disc", "cy2": H, "cx2": W, "r": 6}, 1.0, 0)
        rd.rd_step(h, 25)
        u = np.empty((H, W), dtype)
        rd.rd_read_fields(h, 0, u, None)
        ptr, pitch = rd.rd_field_ptr(h, 0, 0)
        torch.cuda.synchronize()
        off = (ptr - arena.data_ptr()) // 4
        view = arena.view(torch.float32).as_strided((H, W), (pitch, 1), off)
        assert_bitwise(view.cpu().numpy(), u, "zero-copy u view")
        pptr, _ = rd.rd_field_ptr(h, 0, 2)
        pview = arena.view(torch.float32).as_strided((H, W), (pitch, 1), (pptr - arena.data_ptr()) // 4)
        assert_bitwise(pview.cpu().numpy(), phi_fn(0, 0, H), "phi view")
    finally:
        rd.rd_destroy(h)
    ref = oracle.run(u_fn(0, 0, H), v_fn(0, 0, H), phi_fn(0, 0, H), 25,
                     events=[({"kind": "disc", "cy2": H, "cx2": W, "r": 6}, 1.0, 0)])
    assert_bitwise(u, ref.u, "u")
    with pytest.raises(rd.RDError):
        rd.rd_create_device(W, H, arena.data_ptr() + 8, nbytes - 8, None, dtype=dtype)  # misaligned


def test_binding_validates_host_buffers():
    """a short, mistyped or non-contiguous host array is refused
    before the C side copies H*W elements."""
    sim = rd.Sim(np.full((1, 20, 30), 0.054, np.float32))
    try:
        with pytest.raises(ValueError):
            rd.rd_read_fields(sim.h, 0, np.empty((20, 29), np.float32), None)
        with pytest.raises(ValueError):
            rd.rd_write_fields(sim.h, 0, np.zeros((20, 30), np.float64), None)
        with pytest.raises(ValueError):
            rd.rd_write_fields(sim.h, 0, np.zeros((30, 20), np.float32).T, None)
        # a rejected non-finite write leaves the handle untouched
        sim.write(0, np.full((20, 30), 0.01, np.float32), np.zeros((20, 30), np.float32))
        bad = np.full((20, 30), 0.02, np.float32)
        bad[3, 4] = np.nan
        with pytest.raises(rd.RDError):
            rd.rd_write_fields(sim.h, 0, np.full((20, 30), 0.5, np.float32), bad)
        u, v = sim.read(0)
        assert np.all(u == np.float32(0.01)) and np.all(v == 0)
    finally:
        sim.close()
