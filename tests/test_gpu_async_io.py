"""Asynchronous host I/O (rd_write_fields_async / rd_commit_fields /
rd_read_fields_async / rd_io_wait, include/rd.h): a single handle driven as a
pipeline of jobs -- upload of job i+1 and download of job i-1 overlapped with
the steps of job i -- gives every job the oracle's fields bitwise."""
import numpy as np
import pytest
import torch

import oracle
import paper_1901_06535_b200 as rd
from gpu_util import assert_bitwise
from rdinputs import noise_plane

pytestmark = pytest.mark.gpu


def pinned(shape, dtype):
    t = torch.empty(shape, dtype=torch.float32 if np.dtype(dtype) == np.float32 else torch.float64, pin_memory=True)
    return t.numpy()


@pytest.mark.parametrize("dtype", [np.float32, np.float64], ids=["f32", "f64"])
def test_pipelined_jobs_equal_the_oracle(dtype, kernel):
    """Four jobs on one handle, one host thread: every job's inputs are staged
    while the job before it steps, its result is drained while the job after
    it steps. Ragged shape (several strips, W % V != 0)."""
    H, W, n, jobs = 97, 301, 37, 4
    phi = np.full((1, H, W), 0.054, dtype=dtype)
    phi[0, 20:40, 100:180] = 0.2
    sim = rd.Sim(phi, dtype=dtype)
    ins = []
    for j in range(jobs):
        u, v = pinned((H, W), dtype), pinned((H, W), dtype)
        u[...] = noise_plane(H, W, 0, seed=10 + j, dtype=dtype)
        v[...] = noise_plane(H, W, 1, seed=10 + j, dtype=dtype)
        u[30 + 5 * j:50 + 5 * j, 40:60] = 1.0  # a block that fires
        ins.append((u, v))
    outs = [(pinned((H, W), dtype), pinned((H, W), dtype)) for _ in range(jobs)]
    rd.rd_write_fields_async(sim.h, 0, *ins[0])
    rd.rd_commit_fields(sim.h)
    for j in range(jobs):
        if j + 1 < jobs:
            rd.rd_write_fields_async(sim.h, 0, *ins[j + 1])
        sim.step(n)
        rd.rd_read_fields_async(sim.h, 0, *outs[j])
        if j + 1 < jobs:
            rd.rd_commit_fields(sim.h)
    rd.rd_io_wait(sim.h)
    assert sim.step_count == jobs * n
    sim.close()
    for j in range(jobs):
        ref = oracle.run(ins[j][0].copy(), ins[j][1].copy(), phi[0], n)
        assert_bitwise(outs[j][0], ref.u, f"u job {j}")
        assert_bitwise(outs[j][1], ref.v, f"v job {j}")


def test_snapshot_is_not_disturbed_by_later_steps_or_commits():
    """rd_read_fields_async returns the fields as of the call, whatever the
    handle does before rd_io_wait; a plane that is not requested (NULL) is not
    touched; batch instances use their own staging slots."""
    dtype = np.float32
    B, H, W = 3, 64, 200
    phi = np.full((B, H, W), 0.054, dtype=dtype)
    sim = rd.Sim(phi, dtype=dtype)
    u0 = [noise_plane(H, W, 0, seed=30 + b, dtype=dtype) for b in range(B)]
    v0 = [noise_plane(H, W, 1, seed=30 + b, dtype=dtype) for b in range(B)]
    for b in range(B):
        sim.write(b, u0[b], v0[b])
    sim.step(20)
    want = [sim.read(b) for b in range(B)]
    got = [(pinned((H, W), dtype), pinned((H, W), dtype)) for _ in range(B)]
    for b in range(B):
        got[b][1][...] = -7.0
        rd.rd_read_fields_async(sim.h, b, got[b][0], None if b == 1 else got[b][1])
    # keep going: steps, an upload and a commit, a second snapshot of slot 0
    nu, nv = pinned((H, W), dtype), pinned((H, W), dtype)
    nu[...] = u0[2]
    nv[...] = v0[2]
    rd.rd_write_fields_async(sim.h, 0, nu, nv)
    sim.step(20)
    rd.rd_commit_fields(sim.h)
    later = (pinned((H, W), dtype), pinned((H, W), dtype))
    rd.rd_io_wait(sim.h)
    for b in range(B):
        assert_bitwise(got[b][0], want[b][0], f"u b={b}")
        if b == 1:
            assert np.all(got[b][1] == -7.0)
        else:
            assert_bitwise(got[b][1], want[b][1], f"v b={b}")
    rd.rd_read_fields_async(sim.h, 0, *later)
    rd.rd_io_wait(sim.h)
    assert_bitwise(later[0], u0[2], "committed u")
    assert_bitwise(later[1], v0[2], "committed v")
    # the committed fields step like any others (margins refreshed)
    sim.step(15)
    u, v = sim.read(0)
    ref = oracle.run(u0[2], v0[2], phi[0], 15)
    assert_bitwise(u, ref.u, "u after commit + steps")
    assert_bitwise(v, ref.v, "v after commit + steps")
    sim.close()


def test_rejected_commit_leaves_the_handle_untouched():
    dtype = np.float64
    H, W = 40, 50
    sim = rd.Sim(np.full((1, H, W), 0.054, dtype=dtype), dtype=dtype)
    u0 = noise_plane(H, W, 0, seed=3, dtype=dtype)
    v0 = noise_plane(H, W, 1, seed=3, dtype=dtype)
    sim.write(0, u0, v0)
    rd.rd_commit_fields(sim.h)  # nothing staged: a no-op
    bu, bv = pinned((H, W), dtype), pinned((H, W), dtype)
    bu[...] = 0.5
    bv[...] = 0.25
    bv[7, 9] = np.inf
    rd.rd_write_fields_async(sim.h, 0, bu, bv)
    with pytest.raises(rd.RDError) as e:
        rd.rd_commit_fields(sim.h)
    assert e.value.code == rd.RD_ENONFINITE
    u, v = sim.read(0)
    assert_bitwise(u, u0, "u kept")
    assert_bitwise(v, v0, "v kept")
    rd.rd_commit_fields(sim.h)  # the rejected set was dropped
    u, v = sim.read(0)
    assert_bitwise(u, u0, "u kept (2)")
    with pytest.raises(rd.RDError) as e:
        rd.rd_write_fields_async(sim.h, 1, bu, bv)
    assert e.value.code == rd.RD_ERANGE
    with pytest.raises(ValueError):
        rd.rd_read_fields_async(sim.h, 0, np.empty((H, W - 1), dtype=dtype), None)
    sim.close()
