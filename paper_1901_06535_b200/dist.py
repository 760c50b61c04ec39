"""Multi-GPU row slabs: marshalling only.

The decomposition runs inside librd (rd_create_dist, include/rd.h): rank r of
G owns global rows [r*H/G, (r+1)*H/G) (the first H % G ranks one more), and
its rd_step(n) does the whole super-step -- checkpoint, blocks of <= halo
steps with the halo exchange overlapped with the interior rows (copy-engine
copies into the neighbours' ghost rows over CUDA IPC / peer mappings, or NCCL
send/recv), the cross-rank fault flag OR (NCCL all-reduce) and the exact
replay. This module only computes the partition for building inputs,
broadcasts the 128-byte rendezvous id over torch.distributed (plumbing) and
forwards calls.
"""
from __future__ import annotations

import numpy as np

from . import (rd_create_dist, rd_destroy, rd_dist_local_id, rd_dist_shm_id, rd_dist_unique_id, rd_fill_noise, rd_get_geometry,
               rd_get_stats, rd_init_rest, rd_paint_phi, rd_probe, rd_probe_latch, rd_probe_result, rd_read_fields,
               rd_set_stream, rd_step, rd_stimulate, rd_timelapse, rd_write_fields, stream_handle)


def slab_rows(H: int, world: int, rank: int) -> tuple[int, int]:
    """(row0, rows) of rank's slab, the partition rd_create_dist uses: H need
    not divide evenly (the first H % G ranks get one extra row)."""
    base, extra = divmod(H, world)
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


def ghost_extent(H: int, row0: int, rows: int, halo: int) -> tuple[int, int]:
    """Global rows [lo, hi) a slab stores (owned + ghosts that exist)."""
    return max(0, row0 - halo), min(H, row0 + rows + halo)


def exchange_plan(world: int, rank: int, rows: int, halo: int):
    """The (peer, local send rows, local recv rows) pairs of one exchange.
    Local row x of a slab is global row row0 + x; ghosts are x < 0, x >= rows."""
    plan = []
    if rank > 0:
        plan.append((rank - 1, (0, halo), (-halo, 0)))
    if rank < world - 1:
        plan.append((rank + 1, (rows - halo, rows), (rows, rows + halo)))
    return plan


def unique_id(group=None) -> bytes:
    """rd_dist_unique_id on rank 0 of the torch.distributed group, broadcast
    to every rank (the only use of torch.distributed: the rendezvous)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return rd_dist_unique_id()  # a world of one process: nothing to broadcast
    obj = [rd_dist_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return obj[0]


def shm_id() -> bytes:
    """Rendezvous id for ranks that are processes of this box, without NCCL
    (rd_dist_shm_id): make it in one process and hand the 128 bytes to the
    others."""
    return rd_dist_shm_id()


def local_id() -> bytes:
    """Rendezvous id for ranks that are host threads of this process."""
    return rd_dist_local_id()


class DistSim:
    """One rank's slab, stepped by librd's distributed super-step.

    uid: the rendezvous id (rd_dist_unique_id broadcast to every rank, or one
    local_id() shared by threads); None = unique_id(group) over
    torch.distributed. phi_fn(b, row0, rows) -> host rows of global rows
    [row0, row0 + rows), or None for phi = 0 (paint on the device)."""

    def __init__(self, W: int, H: int, rank: int, world: int, phi_fn=None, *, uid: bytes | None = None,
                 group=None, dtype=np.float32, tb_depth: int = 0, batch: int = 1, params=None, flags: int = 0):
        self.W, self.H, self.rank, self.world, self.batch = W, H, rank, world, batch
        self.dtype = np.dtype(dtype)
        self.row0, self.rows = slab_rows(H, world, rank)
        if uid is None:
            uid = unique_id(group)
        phi = (None if phi_fn is None else
               np.stack([np.ascontiguousarray(phi_fn(b, self.row0, self.rows), dtype=self.dtype)
                         for b in range(batch)]))
        self.h = rd_create_dist(W, H, phi, rank, world, uid, batch=batch, dtype=dtype, tb_depth=tb_depth,
                                flags=flags, params=params)
        self.halo = rd_get_geometry(self.h)["halo"]

    def close(self):
        """Collective: every rank closes its slab."""
        if getattr(self, "h", None):
            rd_destroy(self.h)
            self.h = None

    def set_stream(self, stream):
        rd_set_stream(self.h, stream_handle(stream))

    def geometry(self) -> dict:
        return rd_get_geometry(self.h)

    def step(self, n: int):
        rd_step(self.h, n)

    def write(self, b: int, u_fn, v_fn=None):
        """Owned rows from global-row generators u_fn(b, row0, rows)."""
        u = np.ascontiguousarray(u_fn(b, self.row0, self.rows), dtype=self.dtype)
        v = None if v_fn is None else np.ascontiguousarray(v_fn(b, self.row0, self.rows), dtype=self.dtype)
        rd_write_fields(self.h, b, u, v)

    def read_owned(self, b: int = 0):
        u = np.empty((self.rows, self.W), dtype=self.dtype)
        v = np.empty((self.rows, self.W), dtype=self.dtype)
        rd_read_fields(self.h, b, u, v)
        return u, v

    def paint_phi(self, value: float, rect=None, b: int = -1):
        rd_paint_phi(self.h, b, rect, value)

    def fill_noise(self, b: int = -1, planes: int = 3, seed: int = 1, amplitude: float = 0.1):
        rd_fill_noise(self.h, b, planes, seed, amplitude)

    def init_rest(self, b: int = -1):
        rd_init_rest(self.h, b)

    def stimulate(self, shape: dict, value: float = 1.0, at_step: int = 0, b: int = -1):
        rd_stimulate(self.h, b, shape, value, at_step)  # collective; global coordinates

    def timelapse(self, stride: int):
        rd_timelapse(self.h, stride)  # collective

    def probe_latch(self, b, rect, threshold=0.1, stride=50):
        return rd_probe_latch(self.h, b, rect, threshold, stride)  # collective

    def probe_result(self, pid):
        return rd_probe_result(self.h, pid)  # collective: first firing over all ranks

    def probe(self, b, rect, threshold=0.1):
        return rd_probe(self.h, b, rect, threshold)  # collective: global maximum

    def stats(self):
        return rd_get_stats(self.h)
