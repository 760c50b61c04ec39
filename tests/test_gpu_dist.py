"""Row-slab decomposition on ONE GPU with virtual ranks (LoopbackGroup): the
G-slab result (kernels clamp only at global edges, ghosts come from the
neighbour slab) is bitwise identical to the single-grid result and to the
oracle (SURVEY.md §8(e) invariant)."""
import numpy as np
import pytest

import oracle
import paper_1901_06535_b200 as rd
from gpu_util import assert_bitwise
from slab_protocol import LoopbackGroup, SlabSim
from rdinputs import half_discs, noise_plane, obstacles

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p2p", [False, True], ids=["nccl-style", "p2p-push"])
@pytest.mark.parametrize("G,halo", [(2, 1), (2, 4), (3, 4), (4, 8)])
@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
def test_virtual_slabs_equal_single_grid(G, halo, dtype, kernel, p2p):
    H, W, steps = 203, 300, 37
    rects = obstacles(H, W, 6, seed=3)

    def phi_fn(b, row0, rows):
        p = np.full((rows, W), 0.054)
        for (y0, x0, y1, x1) in rects:
            a, c = max(y0, row0), min(y1, row0 + rows)
            if a < c:
                p[a - row0:c - row0, x0:x1] = 0.2
        return p

    def u_fn(b, row0, rows):
        return noise_plane(rows, W, 0, seed=1, dtype=dtype, row0=row0)

    def v_fn(b, row0, rows):
        return noise_plane(rows, W, 1, seed=1, dtype=dtype, row0=row0)

    shapes = half_discs(H, W, 12, seed=2, mask_phi=0.054)
    grp = LoopbackGroup(G, p2p=p2p)
    slabs = [SlabSim(W, H, r, G, phi_fn, dtype=dtype, halo=halo, transport=grp) for r in range(G)]
    for s in slabs:
        s.write(0, u_fn, v_fn)
        for sh in shapes:
            s.stimulate(sh, 1.0, 0)
        s.stimulate({"kind": "rect", "y0": 60, "x0": 10, "y1": 150, "x1": 14}, 1.0, 5)
    grp.step_all(steps)
    U = np.concatenate([s.read_owned(0)[0] for s in slabs])
    V = np.concatenate([s.read_owned(0)[1] for s in slabs])
    # the blocks ran split (SURVEY.md §8(e) overlap / push): an interior slab
    # launches interior + top band + bottom band per block, except the blocks
    # holding the stimuli (steps 0 and 5) and, with the push, the partial
    # last block (one plain launch each)
    blocks = -(-steps // halo)
    if G >= 3:
        assert slabs[1].stats()["step_launches"] >= 3 * (blocks - 3) + 3
    for s in slabs:
        s.close()

    ev = [(sh, 1.0, 0) for sh in shapes] + [({"kind": "rect", "y0": 60, "x0": 10, "y1": 150, "x1": 14}, 1.0, 5)]
    ref = oracle.run(u_fn(0, 0, H), v_fn(0, 0, H), phi_fn(0, 0, H).astype(dtype), steps, events=ev)
    assert_bitwise(U, ref.u, "u")
    assert_bitwise(V, ref.v, "v")
    sim = rd.Sim(phi_fn(0, 0, H).astype(dtype), dtype=dtype)
    sim.write(0, u_fn(0, 0, H), v_fn(0, 0, H))
    for (sh, val, at) in ev:
        sim.stimulate(sh, val, at)
    sim.step(steps)
    u1, v1 = sim.read(0)
    sim.close()
    assert_bitwise(U, u1, "u single")


@pytest.mark.parametrize("p2p", [False, True], ids=["nccl-style", "p2p-push"])
@pytest.mark.parametrize("G", [2, 3])
def test_virtual_slabs_fault_and_guard_replay(G, p2p):
    """Super-step protocol: an unmasked stimulus inside a phi=0.2 obstacle on
    noisy u,v diverges; the slabs detect it, restore, replay step by step and
    stop at the oracle's failing step, reporting the oracle's first cell (in
    global coordinates) with identical fields."""
    H, W, steps = 96, 128, 400
    dtype = np.float32

    def phi_fn(b, row0, rows):
        return np.full((rows, W), 0.2)

    def u_fn(b, row0, rows):
        return noise_plane(rows, W, 0, seed=7, dtype=dtype, row0=row0)

    def v_fn(b, row0, rows):
        return noise_plane(rows, W, 1, seed=7, dtype=dtype, row0=row0)

    shape = {"kind": "half_disc", "cy2": 2 * 47, "cx2": 128, "r": 8, "dir": 1}  # straddles the slab edge
    ref = oracle.run(u_fn(0, 0, H), v_fn(0, 0, H), phi_fn(0, 0, H).astype(dtype), steps, events=[(shape, 1.0, 0)])
    assert ref.status == -4
    grp = LoopbackGroup(G, p2p=p2p)
    slabs = [SlabSim(W, H, r, G, phi_fn, dtype=dtype, halo=4, transport=grp) for r in range(G)]
    for s in slabs:
        s.write(0, u_fn, v_fn)
        s.stimulate(shape, 1.0, 0)
    with pytest.raises(rd.RDError) as e:
        grp.step_all(steps)
    assert e.value.code == rd.RD_ENONFINITE
    faults = [rd.rd_get_fault(s.h) for s in slabs if rd.rd_get_fault(s.h)[0] > 0]
    assert faults and min((f[0], f[2], f[3]) for f in faults) == ref.fault
    U = np.concatenate([s.read_owned(0)[0] for s in slabs])
    assert_bitwise(U, ref.u, "u at fault")
    assert all(rd.rd_get_step(s.h) == ref.fault[0] for s in slabs)
    for s in slabs:
        s.close()


def test_p2p_push_blocks_run_and_stream_flags():
    """The peer-memory path takes push blocks (edge launches storing into the
    neighbours' ghost rows; no exchange copies) for every full block without
    a stimulus, and the stream-ordered flag calls work on one handle (a
    signal then a wait on its own word: nothing waits on another rank)."""
    H, W, steps, halo = 120, 96, 48, 4
    dtype = np.float32

    def phi_fn(b, row0, rows):
        return np.full((rows, W), 0.054)

    grp = LoopbackGroup(3, p2p=True)
    slabs = [SlabSim(W, H, r, 3, phi_fn, dtype=dtype, halo=halo, transport=grp) for r in range(3)]
    for s in slabs:
        s.fill_noise(seed=4)
        s.stimulate({"kind": "disc", "cy2": H, "cx2": W, "r": 6}, 1.0, 0)
    grp.step_all(steps)
    U = np.concatenate([s.read_owned(0)[0] for s in slabs])
    # block 1 holds the step-0 stimulus (plain); blocks 2..12 are push blocks:
    # the middle slab launches interior + 2 edge bands + the ghost mirror each
    st = slabs[1].stats()
    assert st["step_launches"] >= 3 * (steps // halo - 1) + 1
    ref = oracle.run(noise_plane(H, W, 0, seed=4, dtype=dtype), noise_plane(H, W, 1, seed=4, dtype=dtype),
                     np.full((H, W), 0.054, dtype), steps, events=[({"kind": "disc", "cy2": H, "cx2": W, "r": 6}, 1.0, 0)])
    assert_bitwise(U, ref.u, "u")
    f = rd.rd_flag_ptr(slabs[1].h, 0)
    rd.rd_stream_signal(slabs[1].h, f, 7)
    rd.rd_stream_wait(slabs[1].h, f, 7)
    import torch
    torch.cuda.synchronize()
    for s in slabs:
        s.close()
